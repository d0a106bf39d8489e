"""GPU parity of the complex path (K3) against the reference's golden
vectors (complex runs are plain-double only in the reference)."""

import numpy as np
import pytest

import golden_io as gio
import oracle
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200.complex_walk import DenseC128Problem
from paper_2502_16577_b200.precision import dd_pairwise

pytestmark = pytest.mark.gpu

CPLX = [c["name"] for c in gio.cases(gio.load(), kind="complex128")]
WALKER_LIMIT = 1 << 21


def _case(golden, name):
    return next(c for c in golden["cases"] if c["name"] == name)


def _matrix(case):
    m = case["matrix"]
    if m["container"] == "dense":
        return pk.DenseMatrix.from_array(gio.dense_array(case))
    return pk.sparse_from_triplets(m["n"], gio.triplets(case), "complex128")


def crel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("name", CPLX)
def test_complex_run_range_bitwise(golden, name):
    case = _case(golden, name)
    m = _matrix(case)
    for r in case["ranges"]:
        if r["end"] - r["start"] >= WALKER_LIMIT:
            continue
        p = pk.run_range(m, r["start"], r["end"], "dd", exact=True)
        assert [p.value.real.hex(), p.value.imag.hex()] == r["value"], (name, r)


@pytest.mark.parametrize("name", CPLX)
def test_complex_chunked_bitwise(golden, name):
    case = _case(golden, name)
    m = _matrix(case)
    for ch in case["chunked"]:
        plan = pk.plan_chunks(m.n, ch["tau"], ch["aligned"])
        if max(e - s for (_, s, e) in plan.jobs()) >= WALKER_LIMIT:
            continue
        got = pk.permanent_chunked(m, "dd", tau=ch["tau"], aligned=ch["aligned"], exact=True)
        assert [got.real.hex(), got.imag.hex()] == ch["value"], (name, ch)


@pytest.mark.parametrize("n,k", [(16, 4), (20, 6), (24, 5)])
def test_complex_register_chunks_bitwise_vs_oracle(n, k):
    m = pk.haar_unitary_block(n, 500 + n)
    a = np.array(m.data, dtype=np.complex128).reshape(n, n)
    prob = DenseC128Problem(m)
    nchunks = min(1 << (n - 1 - k), 64)
    chunk_lo = (1 << (n - 1 - k)) - nchunks
    parts, (tre, tim) = prob.chunks(k, chunk_lo, nchunks, exact=True)
    T = pk.total_iterates(n)
    for i in range(0, nchunks, 5):
        c = chunk_lo + i
        s, e = 1 + (c << k), min((c + 1) << k, T)
        want = oracle.dense_c128_range(a, s, e)
        assert (parts[i][0].hex(), parts[i][1].hex()) == (want.real.hex(), want.imag.hex())
    assert dd_pairwise([(p[0], 0.0) for p in parts]) == tre
    assert dd_pairwise([(p[1], 0.0) for p in parts]) == tim


@pytest.mark.parametrize("name", ["haar16", "haar24", "cplx_rand12"])
def test_complex_perm_within_tolerance(golden, name):
    case = _case(golden, name)
    m = _matrix(case)
    ref = max(case["chunked"], key=lambda ch: ch["tau"])["value"]
    ref = complex(float.fromhex(ref[0]), float.fromhex(ref[1]))
    got = pk.perm_nw(m)
    assert crel(got, ref) <= 1e-10, (name, got, ref)
    assert pk.permanent(m) == got


def test_complex_uniform_closed_form():
    import math
    for n in (12, 16, 20, 24):
        a = complex(0.6, 0.35)
        m = pk.DenseMatrix.from_rows([[a] * n for _ in range(n)])
        exact = math.factorial(n) * a ** n
        assert crel(pk.perm_nw(m), exact) <= 1e-10


def test_complex_policy_error():
    m = pk.DenseMatrix.from_rows([[1j, 2], [3, 4]])
    for p in ("kahan", "dq", "qq"):
        with pytest.raises(pk.PolicyError):
            pk.perm_nw(m, p)
        with pytest.raises(pk.PolicyError):
            pk.run_range(m, 1, 1, p)


def test_complex_sparse_equals_dense():
    m = pk.haar_unitary_block(14, 3)
    s = pk.dense_to_sparse(m)
    assert crel(pk.perm_spa(s), pk.perm_nw(m)) <= 1e-12


@pytest.mark.parametrize("n", [14, 20, 24])
def test_complex_precise_mode_uniform_closed_form(n):
    from fractions import Fraction
    import math
    a = complex(0.6, 0.7)
    m = pk.DenseMatrix.from_rows([[a] * n for _ in range(n)])
    got = pk.perm_nw(m, precise=True)
    # n! a^n exactly (a's binary value), compared in rationals
    ar, ai = Fraction(a.real), Fraction(a.imag)
    pr, pi = Fraction(1), Fraction(0)
    for _ in range(n):
        pr, pi = pr * ar - pi * ai, pr * ai + pi * ar
    f = math.factorial(n)
    er, ei = f * pr, f * pi
    err = math.hypot(float(Fraction(got.real) - er), float(Fraction(got.imag) - ei))
    assert err <= 1e-13 * math.hypot(float(er), float(ei)), (n, got, err)
