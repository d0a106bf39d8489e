"""Structural preprocessing (matching filter, compressions, decomposition
worklist) against the reference's own outputs in tests/golden/preprocess.json
(tools/make_golden_preprocess.py ran permkit.preprocess to make them).

CPU tests: dm_filter, min_nnz_row_col, d1/d2/d34 compressions and the whole
decomposition task tree (every kernel leaf matrix and multiplier, in
permkit's evaluation order) are bit-identical to permkit's; cases whose tree
has no kernel leaf reproduce permkit's final value bit for bit. GPU tests:
decomp_run with batched leaf evaluation matches permkit's value (integers
exactly, floats within 1e-10) and every recorded leaf value.
"""

import json
import os

import numpy as np
import pytest

import paper_2502_16577_b200 as pk
from paper_2502_16577_b200 import preprocess as pp

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "preprocess.json")
GOLD = json.load(open(PATH))["cases"]
NAMES = [c["name"] for c in GOLD]


def dec(v, kind):
    if kind == "integer":
        return int(v)
    if kind == "complex128":
        return complex(float.fromhex(v[0]), float.fromhex(v[1]))
    return float.fromhex(v)


def trips(lst, kind):
    return [(i, j, dec(v, kind)) for (i, j, v) in lst]


def case(name):
    return next(c for c in GOLD if c["name"] == name)


def pair(c):
    return pk.sparse_from_triplets(c["n"], trips(c["triplets"], c["kind"]), c["kind"])


def same_trips(s, lst, kind):
    got = s.crs.triplets()
    want = trips(lst, kind)
    assert len(got) == len(want)
    for (i, j, v), (a, b, w) in zip(got, want):
        assert (i, j) == (a, b)
        if kind == "integer":
            assert v == w
        elif kind == "complex128":
            assert (v.real.hex(), v.imag.hex()) == (w.real.hex(), w.imag.hex())
        else:
            assert float(v).hex() == float(w).hex()


@pytest.mark.parametrize("name", NAMES)
def test_dm_filter_and_min_nnz_match_reference(name):
    c = case(name)
    s = pair(c)
    res = pp.dm_filter(s)
    if c["dm_filter"]["singular"]:
        assert isinstance(res, pp.SingularVerdict) and res.value == 0
    else:
        assert not isinstance(res, pp.SingularVerdict)
        assert res.crs.nnz == c["dm_filter"]["nnz_after"]
        same_trips(res, c["dm_filter"]["triplets"], c["kind"])
    pick = pp.min_nnz_row_col(s)
    assert [pick.axis, pick.index, pick.count] == c["min_nnz"]


@pytest.mark.parametrize("name", NAMES)
def test_compressions_match_reference(name):
    c = case(name)
    s = pair(c)
    kind = c["kind"]
    comp = c["compress"]
    if "d1" in comp:
        d = comp["d1"]
        alpha, minor = pp.d1compress(s, d["axis"], d["index"])
        assert dec(d["alpha"], kind) == alpha
        same_trips(minor, d["triplets"], kind)
    if "d2" in comp:
        d = comp["d2"]
        same_trips(pp.d2compress(s, d["axis"], d["index"]), d["triplets"], kind)
    for key in ("d34_row", "d34_col"):
        if key in comp:
            d = comp[key]
            z, f = pp.d34compress(s, d["axis"], d["index"])
            same_trips(z, d["zeroed"], kind)
            same_trips(f, d["folded"], kind)


@pytest.mark.parametrize("name", NAMES)
def test_decomposition_tree_matches_reference(name):
    c = case(name)
    s = pair(c)
    kind = c["kind"]
    leaves, contribs, st = pp.decomp_leaves(s)
    gold = c["decomp"]
    for k, v in gold["stats"].items():
        if k != "dense_kernel_leaves":
            assert getattr(st, k) == v, (k, getattr(st, k), v)
    assert len(leaves) == len(gold["leaves"]) == st.kernel_leaves
    for (tid, mult, m), g in zip(leaves, gold["leaves"]):
        assert m.n == g["n"]
        if "triplets" in g:
            same_trips(m, g["triplets"], kind)
    if not leaves:
        # no kernel leaf: the whole value is host arithmetic, bit for bit
        got = pp._combine_contributions(contribs, kind)
        want = dec(gold["value"], kind)
        if kind == "complex128":
            assert (got.real.hex(), got.imag.hex()) == (want.real.hex(), want.imag.hex())
        elif kind == "integer":
            assert got == want
        else:
            assert got.hex() == want.hex()


def test_max_matching_is_maximum_and_valid():
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import maximum_bipartite_matching
    rng = np.random.default_rng(3)
    for t in range(60):
        n = int(rng.integers(2, 40))
        d = float(rng.uniform(0.02, 0.3))
        a = rng.uniform(size=(n, n)) < d
        trip = [(i, j, 1) for i in range(n) for j in range(n) if a[i, j]]
        s = pk.sparse_from_triplets(n, trip, "integer")
        m = pp.max_matching(pp.BipartiteGraph.from_sparse(s))
        ref = maximum_bipartite_matching(csr_matrix(a.astype(np.int8)), perm_type="column")
        assert m.size == int((ref >= 0).sum()), (n, d)
        for r, cc in enumerate(m.row_to_col):
            if cc >= 0:
                assert a[r, cc] and m.col_to_row[cc] == r


def test_dm_filter_keeps_the_permanent_small_cases():
    # entries removed by the filter lie on no perfect matching: the exact
    # permanent (expansion over permutations, small n) is unchanged
    import itertools
    rng = np.random.default_rng(11)
    for _ in range(25):
        n = int(rng.integers(2, 7))
        a = (rng.uniform(size=(n, n)) < 0.45) * rng.integers(1, 5, size=(n, n))
        s = pk.dense_to_sparse(pk.DenseMatrix.from_rows(a.tolist()))
        if s.crs.nnz == 0:
            continue

        def perm(rows):
            return sum(int(np.prod([rows[i][p[i]] for i in range(n)]))
                       for p in itertools.permutations(range(n)))

        res = pp.dm_filter(s)
        want = perm(a.tolist())
        if isinstance(res, pp.SingularVerdict):
            assert want == 0
        else:
            assert perm(pk.sparse_to_dense(res).rows()) == want


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_decomp_run_matches_reference_value(name):
    c = case(name)
    s = pair(c)
    kind = c["kind"]
    gold = c["decomp"]
    got, st = pp.decomp_run(s, gold["policy"])
    want = dec(gold["value"], kind)
    # the native and the Python worklists build the same tree and the leaves
    # go through the same batched kernels: identical results
    got_py, st_py = pp.decomp_run(s, gold["policy"], native=False)
    assert got == got_py and st.tasks_created == st_py.tasks_created
    if kind == "integer":
        assert got == want
    else:
        assert abs(got - want) <= 1e-10 * abs(want) + 1e-300, (got, want)
    assert st.kernel_leaves == gold["stats"]["kernel_leaves"]
    if st.kernel_leaves:
        # one batched launch per leaf order (every kind)
        assert st.leaf_launches <= len(set(st.leaf_sizes))


@pytest.mark.gpu
def test_decomp_leaf_values_match_reference():
    # every recorded leaf value (permkit's perm_nw / perm_spa on that leaf)
    for name in ("real18_d33", "int20_d30", "cplx18_d30", "real28_d30"):
        c = case(name)
        kind = c["kind"]
        leaves, _, _ = pp.decomp_leaves(pair(c))
        pol = c["decomp"]["policy"]
        vals = pk.permanent_batch([pk.sparse_to_dense(m) for (_, _, m) in leaves], pol)
        for v, g in zip(vals, c["decomp"]["leaves"]):
            w = dec(g["value"], kind)
            if kind == "integer":
                assert v == w
            else:
                assert abs(v - w) <= 1e-10 * abs(w) + 1e-300, (name, v, w)


def native_leaves(s):
    """The native worklist's tree in the shape of decomp_leaves' output."""
    trivial, leaves, st = pp._native_tree(s, pp.DEFAULT_TASK_LIMIT, 1e9, 4, pp.DENSE_LEAF_DENSITY)
    out = []
    for n, (ids, mults, mats) in leaves.items():
        for tid, mult, mat in zip(ids, mults, mats):
            rows = [[mat[i][j] for j in range(n)] for i in range(n)]
            trip = [(i, j, rows[i][j]) for i in range(n) for j in range(n) if rows[i][j] != 0]
            out.append((tid, mult, pk.sparse_from_triplets(n, trip, s.kind)))
    return out, trivial, st


@pytest.mark.parametrize("name", NAMES)
def test_native_tree_equals_python_tree_and_reference(name):
    c = case(name)
    s = pair(c)
    kind = c["kind"]
    nat_leaves, nat_triv, nst = native_leaves(s)
    py_leaves, py_triv, pst = pp.decomp_leaves(s)
    for k in ("tasks_created", "d1_applied", "d2_applied", "d34_applied", "trivial_leaves",
              "kernel_leaves", "max_depth"):
        assert getattr(nst, k) == getattr(pst, k) == c["decomp"]["stats"][k], k
    assert sorted(nat_triv, key=lambda t: t[0]) == sorted(py_triv, key=lambda t: t[0])
    py = {tid: (mult, m) for tid, mult, m in py_leaves}
    assert len(nat_leaves) == len(py_leaves)
    for tid, mult, m in nat_leaves:
        pm, pmat = py[tid]
        assert mult == pm
        got = m.crs.triplets()
        want = pmat.crs.triplets()
        assert [(i, j) for i, j, _ in got] == [(i, j) for i, j, _ in want]
        for (_, _, v), (_, _, w) in zip(got, want):
            if kind == "real64":
                assert float(v).hex() == float(w).hex()
            else:
                assert v == w
    if not nat_leaves:
        got = pp._combine_contributions(list(nat_triv), kind)
        want = dec(c["decomp"]["value"], kind)
        assert got == want


def test_dense_states_match_scalar_state_builders():
    from paper_2502_16577_b200.batch import dense_states
    from paper_2502_16577_b200.kernels import dense_complex_state, dense_float_state
    rng = np.random.default_rng(5)
    for n in (2, 7, 20):
        A = rng.uniform(-1, 1, size=(4, n, n)) * (rng.uniform(size=(4, n, n)) < 0.6)
        cols, x0 = dense_states(A)
        for b in range(4):
            c1, x1 = dense_float_state(pk.DenseMatrix.from_array(A[b]))
            assert np.array_equal(cols[b], c1) and x0[b].tobytes() == x1.tobytes()
        C = A + 1j * rng.uniform(-1, 1, size=(4, n, n))
        cols, x0 = dense_states(C)
        for b in range(4):
            c1, x1 = dense_complex_state(pk.DenseMatrix.from_array(C[b]))
            assert np.array_equal(cols[b], c1) and x0[b].tobytes() == x1.tobytes()


def test_native_tree_budgets_and_integer_overflow_fallback():
    # task budget -> DecompTimeout from the native worklist (no device work)
    c = case("int20_d30")
    with pytest.raises(pk.DecompTimeout):
        pp.decomp_run(pair(c), task_limit=50)
    # integer folds beyond 128 bits: the native tree declines (None) and
    # decomp_run falls back to the arbitrary-precision Python worklist
    n = 8
    big = 1 << 61
    trip = [(i, i, big + i) for i in range(n)] + [(i, (i + 1) % n, big - 3 * i) for i in range(n)]
    trip += [(i, (i + 3) % n, big // 3 + i) for i in range(n)]
    s = pk.sparse_from_triplets(n, trip, "integer")
    assert pp._native_tree(s, pp.DEFAULT_TASK_LIMIT, 1e9, 4, pp.DENSE_LEAF_DENSITY) is None
    leaves, contribs, st = pp.decomp_leaves(s)
    assert st.tasks_created > 1 and not leaves
    # exact value by the permutation expansion
    import itertools
    rows = pk.sparse_to_dense(s).rows()
    want = sum(int(np.prod([rows[i][p[i]] for i in range(n)], dtype=object))
               for p in itertools.permutations(range(n)))
    assert pp._combine_contributions(contribs, "integer") == want
