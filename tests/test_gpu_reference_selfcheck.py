"""The reference's own verification suite (permkit.selfcheck, selfcheck.py:
51-256) run with its hot-path entry points replaced by this package's GPU
backend (SURVEY.md §8c parity protocol).

permkit resolves perm_nw / perm_spa / run_range through its module objects at
call time (selfcheck.py:8-10), so patching permkit.kernels, permkit.parallel
and permkit.preprocess routes every walk of the suite -- oracle agreement,
closed forms, exact binary counting, bit-identical partition invariance over
plans and hierarchies, matching filter, compressions, precision ordering,
resumable partial-file merge -- through the B200 kernels, while permkit's own
planners, reducers and oracles check the results. The reference comes from
its offline install under baseline/_ref; the test skips when
that install is absent.
"""

import os
import sys

import pytest

import paper_2502_16577_b200 as pk

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def permkit_ref(tmp_path_factory):
    if not os.path.isdir(os.path.join(REF, "permkit")):
        pytest.skip("reference install baseline/_ref absent")
    os.environ.setdefault("NUMBA_CACHE_DIR", str(tmp_path_factory.mktemp("numba")))
    sys.path.insert(0, REF)
    import permkit
    yield permkit
    sys.path.remove(REF)


def test_reference_selfcheck_passes_on_the_gpu_backend(permkit_ref, monkeypatch, capsys):
    import permkit.kernels as rk
    import permkit.parallel as rp
    import permkit.preprocess as rpp
    import permkit.selfcheck as sc
    from permkit.parallel import PartialResult as RefPartial
    from permkit.precision import DoubleDouble as RefDD

    calls = {"perm": 0, "range": 0}

    def gpu_perm_nw(m, policy=rk.AccumulatorPolicy.DD):
        calls["perm"] += 1
        return pk.perm_nw(pk.coerce_matrix(m), policy)

    def gpu_perm_spa(s, policy=rk.AccumulatorPolicy.DD):
        calls["perm"] += 1
        return pk.perm_spa(pk.coerce_matrix(s), policy)

    def gpu_run_range(m, start, end, policy=rk.AccumulatorPolicy.DD, worker_id=0):
        calls["range"] += 1
        p = pk.run_range(pk.coerce_matrix(m), start, end, policy, worker_id)
        v = p.value
        if isinstance(v, pk.DoubleDouble):
            v = RefDD(v.hi, v.lo)
        return RefPartial(p.worker_id, p.start, p.end, p.iterations_done, p.kind, v)

    for mod in (rk, rpp):
        monkeypatch.setattr(mod, "perm_nw", gpu_perm_nw)
        monkeypatch.setattr(mod, "perm_spa", gpu_perm_spa)
    monkeypatch.setattr(rp, "run_range", gpu_run_range)

    ok = sc.run_selfcheck(verbose=True)
    out = capsys.readouterr().out
    print(out)
    assert ok, out
    assert "FAIL" not in out
    assert calls["perm"] > 100 and calls["range"] > 10, calls


@pytest.mark.parametrize("kind", ["real64", "integer", "complex128"])
def test_reference_merges_our_gpu_partial_files(permkit_ref, tmp_path, kind):
    # each GPU (here: each process index of a hierarchy
    # plan) emits the reference's partial-file format; permkit's own
    # merge_partial_files reads them and reduces to our value
    import permkit.generate as rg
    import permkit.parallel as rp
    from permkit.matrix import DenseMatrix as RefDense
    n = 14
    if kind == "real64":
        ours = pk.random_real(n, 5, 0.0, 1.0)
    elif kind == "integer":
        ours = pk.random_binary(n, 5, 0.5)
    else:
        ours = pk.haar_unitary_block(n, 5)
    ref_m = RefDense.from_rows(ours.rows())
    hp = pk.plan_hierarchy(n, 4, 2)
    paths = []
    for pi in range(hp.processes):
        parts = pk.execute_hierarchy(ours, hp, "dd", process_index=pi)
        path = tmp_path / f"partial-{pi}.txt"
        pk.write_partials_file(path, ours, "dd", parts)
        paths.append(str(path))
    ref_val = rp.merge_partial_files(paths, ref_m, rp.AccumulatorPolicy.DD)
    our_val = pk.merge_partial_files(paths, ours, "dd")
    assert ref_val == our_val
    single = pk.reduce_partials(pk.execute_hierarchy(ours, hp, "dd"),
                                pk.initial_product(ours, "dd"), n)
    assert ref_val == single
