"""GPU parity of the sparse real path (SpaRyser, generated per-pattern kernels)
against the reference's golden vectors, the C oracle and the dense kernel K1.

* chunk partials of the generated kernel in exact mode are bit-identical to
  the oracle's chunk_sparse_f64 restatement (_loops.py:110-183) over the
  same chunk, for every policy
* whole walks are bit-identical to K1 on the densified pair with the sparse
  seed (same arithmetic, only the x + 0.0 updates are skipped), fast and
  exact mode, single and split devices
* whole permanents: <= 1e-10 relative to the reference's compensated result
"""

import numpy as np
import pytest

import golden_io as gio
import oracle
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200 import kernels as K
from paper_2502_16577_b200.precision import AccumulatorPolicy, dd_pairwise

pytestmark = pytest.mark.gpu

POLS = ["dd", "kahan", "dq", "qq"]


def _sparse(n, density, seed, lo=0.0):
    rng = np.random.default_rng(seed)
    a = rng.uniform(lo, 1.0, size=(n, n)) * (rng.uniform(size=(n, n)) < density)
    trip = [(i, j, float(a[i, j])) for i in range(n) for j in range(n) if a[i, j] != 0.0]
    return a, trip, pk.sparse_from_triplets(n, trip, "real64")


def _dense_twin(s):
    """K1 problem on the densified pair with the sparse seed."""
    prob = K.DenseF64Problem(pk.matrix.sparse_to_dense(s))
    prob.x0 = K.SparseF64Problem(s).x0.copy()
    return prob


@pytest.mark.parametrize("n,k,density", [(16, 6, 0.3), (22, 8, 0.5), (27, 10, 0.3),
                                         (33, 12, 0.2), (52, 20, 0.3)])
@pytest.mark.parametrize("policy", POLS)
def test_spa_chunks_bitwise_vs_oracle(n, k, density, policy):
    a, trip, s = _sparse(n, density, 500 + n)
    prob = K.SparseF64Problem(s)
    nchunks = 32 if n > 40 else min(1 << (n - 1 - k), 64)
    chunk_lo = (1 << (n - 1 - k)) - nchunks  # the last chunks: includes the clipped one
    pol = AccumulatorPolicy.parse(policy)
    parts, total = prob.chunks(k, chunk_lo, nchunks, pol, exact=True)
    T = K.total_iterates(n)
    size = 1 << k
    step = 7 if n <= 40 else 31
    for i in range(0, nchunks, step):
        c = chunk_lo + i
        st, e = 1 + c * size, min((c + 1) * size, T)
        want = oracle.sparse_f64_range(n, trip, st, e, policy)
        assert (parts[i][0].hex(), parts[i][1].hex()) == (want[0].hex(), want[1].hex()), (c, st, e)
    host = dd_pairwise([tuple(p) for p in parts])
    assert (host.hi, host.lo) == (total.hi, total.lo)
    # the dense kernel on the densified pair computes the same chunk bits
    dparts, dtotal = _dense_twin(s).chunks(k, chunk_lo, nchunks, pol, exact=True)
    assert np.array_equal(parts, dparts) and dtotal == total


@pytest.mark.parametrize("n,density", [(12, 0.5), (20, 0.3), (26, 0.3), (30, 0.15), (31, 0.6)])
@pytest.mark.parametrize("policy", ["kahan", "dd", "qq"])
def test_spa_walk_bitwise_vs_dense_kernel(n, density, policy):
    _, _, s = _sparse(n, density, 900 + n, lo=-1.0)
    pol = AccumulatorPolicy.parse(policy)
    T = K.total_iterates(n)
    sp, dn = K.SparseF64Problem(s), _dense_twin(s)
    for exact in (False, True):
        if exact and n > 28:
            continue
        a = sp.walk(1, T, pol, exact=exact)
        b = dn.walk(1, T, pol, exact=exact)
        assert (a.hi, a.lo) == (b.hi, b.lo), (exact, a, b)
    # arbitrary range: head / aligned middle / tail
    st, e = T // 7 + 3, T - T // 5
    assert sp.walk(st, e, pol) == dn.walk(st, e, pol)


def test_spa_device_split_reproduces_single_device_bits():
    _, _, s = _sparse(28, 0.3, 77)
    prob = K.SparseF64Problem(s)
    T = K.total_iterates(28)
    one = prob.walk(1, T, AccumulatorPolicy.KAHAN)
    assert one == prob.walk(1, T, AccumulatorPolicy.KAHAN, devices=[0, 0])
    assert one == prob.walk(1, T, AccumulatorPolicy.KAHAN, devices=[0, 0, 0, 0])


@pytest.mark.parametrize("name", ["sparse_real12", "sparse_real18"])
def test_perm_spa_vs_reference(golden, name):
    case = next(c for c in golden["cases"] if c["name"] == name)
    m = case["matrix"]
    s = pk.sparse_from_triplets(m["n"], gio.triplets(case), "real64")
    comp = [ch for ch in case["chunked"] if ch["policy"] in ("kahan", "dq", "qq")]
    ref = float.fromhex(max(comp, key=lambda ch: ch["tau"])["value"])
    for p in POLS:
        got = pk.perm_spa(s, p)
        assert abs(got - ref) <= 1e-10 * abs(ref), (name, p, got, ref)
    # run_range through the sparse path, bitwise against the golden partials
    for r in case["ranges"]:
        if r["end"] - r["start"] < (1 << 21):
            p = pk.run_range(s, r["start"], r["end"], r["policy"], exact=True)
            assert (p.value.hi.hex(), p.value.lo.hex()) == tuple(r["value"]), r


def test_perm_spa_large_matches_dense_and_oracle():
    # n = 34, density 0.3: the generated kernel over the whole walk vs K1 on
    # the dense matrix (same permanent to 1e-10; different seeds/rounding)
    n = 34
    a, trip, s = _sparse(n, 0.3, 4242)
    got = pk.perm_spa(s, "kahan")
    want = pk.perm_nw(pk.DenseMatrix.from_array(a), "kahan")
    assert abs(got - want) <= 1e-10 * abs(want), (got, want)


def test_spa_structure_errors():
    n = 12
    _, trip, s = _sparse(n, 0.4, 3)
    prob = K.SparseF64Problem(s)
    bad = prob.rids.copy()
    c0, c1 = int(prob.cptrs[0]), int(prob.cptrs[1])
    if c1 - c0 >= 2:
        bad[c0], bad[c0 + 1] = bad[c0 + 1], bad[c0]
        prob.rids = bad
        with pytest.raises(pk.StructureError):
            prob.walk(1, K.total_iterates(n), AccumulatorPolicy.DD)


@pytest.mark.parametrize("policy", ["kahan", "qq"])
def test_sparse_exact_equals_dense_exact_on_non_power_of_two_groups(policy):
    # the tail tree has a fixed leaf count (pk_reduce.cuh
    # kTreeLeaves), so the generated sparse kernel (one 384/256-thread block
    # per SM from n = 33) and the dense kernel (128-thread blocks in exact
    # mode) fold the same group partials identically even when the range's
    # group count is not a power of two
    from paper_2502_16577_b200.kernels import DenseF64Problem, SparseF64Problem
    n = 36
    s = pk.random_sparse_real(n, 0.35, 11, 0.0, 1.0)
    sp, dn = SparseF64Problem(s), DenseF64Problem(pk.sparse_to_dense(s))
    pol = AccumulatorPolicy.parse(policy)
    k = 12
    start = 1 + 5 * (1 << k) + 77          # unaligned head
    end = start + 37 * 32 * (1 << k) + 123  # 37 groups of 32 chunks + tail
    a = sp.walk(start, end, pol, exact=True, log2_chunk=k)
    b = dn.walk(start, end, pol, exact=True, log2_chunk=k)
    assert (a.hi, a.lo) == (b.hi, b.lo)
