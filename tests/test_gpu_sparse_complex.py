"""GPU parity of the sparse complex path (SpaRyser, generated per-pattern
kernels with K3's arithmetic) against the C oracle's chunk_sparse_c128
restatement (_loops.py:212-235), the reference's golden sparse case and the
dense complex kernel K3 on the densified pair."""

import numpy as np
import pytest

import golden_io as gio
import oracle
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200.complex_walk import DenseC128Problem
from paper_2502_16577_b200.precision import dd_pairwise

pytestmark = pytest.mark.gpu


def _sparse(n, density, seed):
    rng = np.random.default_rng(seed)
    a = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) / np.sqrt(2 * n)
    a = a * (rng.uniform(size=(n, n)) < density)
    trip = [(i, j, complex(a[i, j])) for i in range(n) for j in range(n) if a[i, j] != 0]
    return a, trip, pk.sparse_from_triplets(n, trip, "complex128")


def _dense_twin(s):
    d = DenseC128Problem(pk.sparse_to_dense(s))
    d.x0 = DenseC128Problem(s).x0.copy()
    return d


@pytest.mark.parametrize("n,k,density", [(14, 4, 0.4), (20, 6, 0.3), (26, 9, 0.3),
                                         (36, 16, 0.25)])
def test_spa_c128_chunks_bitwise_vs_oracle(n, k, density):
    a, trip, s = _sparse(n, density, 60 + n)
    prob = DenseC128Problem(s)
    nchunks = min(1 << (n - 1 - k), 64) if n <= 30 else 32
    chunk_lo = (1 << (n - 1 - k)) - nchunks
    parts, (tre, tim) = prob.chunks(k, chunk_lo, nchunks, exact=True)
    T = pk.total_iterates(n)
    for i in range(0, nchunks, 5 if n <= 30 else 31):
        c = chunk_lo + i
        st, e = 1 + (c << k), min((c + 1) << k, T)
        want = oracle.sparse_c128_range(n, trip, st, e)
        assert (parts[i][0].hex(), parts[i][1].hex()) == (want.real.hex(), want.imag.hex())
    assert dd_pairwise([(p[0], 0.0) for p in parts]) == tre
    assert dd_pairwise([(p[1], 0.0) for p in parts]) == tim
    dparts, dtot = _dense_twin(s).chunks(k, chunk_lo, nchunks, exact=True)
    assert np.array_equal(parts, dparts) and dtot == (tre, tim)


@pytest.mark.parametrize("n,density", [(12, 0.5), (20, 0.3), (27, 0.2), (34, 0.3)])
def test_spa_c128_walk_bitwise_vs_dense_kernel(n, density):
    _, _, s = _sparse(n, density, 300 + n)
    T = pk.total_iterates(n)
    sp, dn = DenseC128Problem(s), _dense_twin(s)
    for exact in ((False, True) if n <= 27 else (False,)):
        assert sp.walk(1, T, exact=exact) == dn.walk(1, T, exact=exact), exact
    st, e = T // 9 + 5, T - T // 3
    assert sp.walk(st, e) == dn.walk(st, e)
    assert sp.walk(1, T) == sp.walk(1, T, devices=[0, 0])


def test_perm_spa_complex_vs_reference(golden):
    case = next(c for c in golden["cases"] if c["name"] == "sparse_cplx10")
    s = pk.sparse_from_triplets(case["matrix"]["n"], gio.triplets(case), "complex128")
    ref = max(case["chunked"], key=lambda ch: ch["tau"])["value"]
    ref = complex(float.fromhex(ref[0]), float.fromhex(ref[1]))
    got = pk.perm_spa(s)
    assert abs(got - ref) <= 1e-10 * abs(ref), (got, ref)


def test_perm_spa_complex_large_matches_dense():
    n = 30
    a, _, s = _sparse(n, 0.35, 99)
    got = pk.perm_spa(s)
    want = pk.perm_nw(pk.DenseMatrix.from_array(a))
    assert abs(got - want) <= 1e-10 * abs(want), (got, want)
