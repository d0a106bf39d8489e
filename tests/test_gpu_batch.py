"""Batched walks (pk_dense_f64_batch): one launch for many matrices must give
each matrix exactly what a single launch with the same chunking gives."""

import numpy as np
import pytest

import golden_io as gio
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200 import _native
from paper_2502_16577_b200.csrc_params import batch_log2_chunk, dense_logu
from paper_2502_16577_b200.kernels import DenseF64Problem, fast_p0, policy_product, _sign_factor
from paper_2502_16577_b200.precision import AccumulatorPolicy, DoubleDouble, dd_add

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [11, 16, 20, 24])
@pytest.mark.parametrize("policy", ["dd", "kahan", "qq"])
def test_batch_equals_single_launch_bitwise(n, policy):
    pol = AccumulatorPolicy.parse(policy)
    ms = [pk.random_real(n, 100 + s, 0.0, 1.0) for s in range(7)]
    got = pk.permanent_batch(ms, policy)
    k = batch_log2_chunk(n, dense_logu(n))
    for m, g in zip(ms, got):
        prob = DenseF64Problem(m)
        part = prob.walk(1, pk.total_iterates(n), pol, log2_chunk=k)
        acc = dd_add(fast_p0(prob.cols, prob.x0, n, pol), part)
        assert g == acc.hi * _sign_factor(n)


def test_small_orders_match_reference_bitwise(golden):
    # n < 11 walks one thread per matrix over [1, 2^(n-1)-1]: the reference's
    # run_range over that range reduced with its g = 0 term
    from paper_2502_16577_b200.parallel import PartialResult
    case = next(c for c in golden["cases"] if c["name"] == "real_rand8")
    m = pk.DenseMatrix.from_array(gio.dense_array(case))
    T = pk.total_iterates(8)
    for r in case["ranges"]:
        if (r["start"], r["end"]) != (1, T):
            continue
        pol = r["policy"]
        p0 = case["p0"][pol]
        p0 = DoubleDouble(*gio.dec_dd(p0)) if pol == "qq" else float.fromhex(p0)
        part = PartialResult(0, 1, T, T, "real64", DoubleDouble(*gio.dec_dd(r["value"])))
        want = pk.reduce_partials([part], p0, 8)
        assert pk.permanent_batch([m, m], pol)[1] == want


def test_mixed_batch_and_throughput_stats():
    ms = [pk.random_real(22, s, 0.0, 1.0) for s in range(300)]
    ms += [pk.uniform(16, 0.91), pk.DenseMatrix.from_rows([[1, 2], [3, 4]]),
           pk.haar_unitary_block(12, 1), pk.random_real(5, 1)]
    st = _native.RunStats()
    got = pk.permanent_batch(ms, "dd", stats=st)
    assert got[301] == 10 and isinstance(got[302], complex)
    import math
    assert abs(got[300] - math.factorial(16) * 0.91 ** 16) <= 1e-12 * got[300]
    for i in (0, 150, 299):
        assert abs(got[i] - pk.perm_nw(ms[i], "kahan")) <= 1e-11 * abs(got[i])
    with pytest.raises(pk.PolicyError):  # complex members keep the DD-only rule
        pk.permanent_batch([pk.haar_unitary_block(12, 1)], "kahan")
    assert st.launches == 1 and st.iterates > 0


@pytest.mark.parametrize("n", [11, 16, 22, 30])
@pytest.mark.parametrize("exact", [False, True])
def test_complex_batch_equals_single_launch_bitwise(n, exact):
    # one launch for many Haar submatrices (boson sampling) must give each
    # matrix exactly what pk_dense_c128 gives with the same chunk exponent
    from paper_2502_16577_b200.complex_walk import DenseC128Problem
    from paper_2502_16577_b200.csrc_params import c128_fast_logu, c128_logu
    ms = [pk.haar_unitary_block(n, 40 + s) for s in range(5)]
    got = pk.permanent_batch(ms, exact=exact)
    k = batch_log2_chunk(n, c128_logu(n) if exact else c128_fast_logu(n))
    for m, g in zip(ms, got):
        prob = DenseC128Problem(m)
        wr, wi = prob.walk(1, pk.total_iterates(n), exact=exact, log2_chunk=k)
        if exact:
            p0 = prob.p0()
            r0, i0 = DoubleDouble(p0.real, 0.0), DoubleDouble(p0.imag, 0.0)
        else:
            from paper_2502_16577_b200.complex_walk import fast_p0 as cfast_p0
            r0, i0 = cfast_p0(prob)
        re = dd_add(r0, wr)
        im = dd_add(i0, wi)
        s = _sign_factor(n)
        assert g == complex(re.hi * s, im.hi * s), (n, g)


def test_complex_batch_small_orders_and_tolerance(golden):
    # n < 11: one thread per matrix, the reference loop exactly
    case = next(c for c in golden["cases"] if c["name"] == "cplx_rand6")
    m = pk.DenseMatrix.from_array(gio.dense_array(case))
    serial = case["serial"]["dd"]
    want = complex(float.fromhex(serial[0]), float.fromhex(serial[1]))
    got = pk.permanent_batch([m, m, m])
    assert got[0] == got[2]
    assert abs(got[0] - want) <= 1e-13 * abs(want)
    ms = [pk.haar_unitary_block(24, s) for s in range(3)]
    for g, m in zip(pk.permanent_batch(ms), ms):
        ref = pk.perm_nw(m)
        assert abs(g - ref) <= 1e-10 * abs(ref)


@pytest.mark.parametrize("n", [6, 11, 18, 24])
def test_integer_batch_is_exact_and_one_launch(n):
    # one pk_int_batch launch for many integer matrices: every permanent
    # equals the single-matrix exact walk (and the reference's integer rule)
    from paper_2502_16577_b200.integer import int_batch_totals, int_walk_total
    rng = np.random.default_rng(n)
    ms = [pk.DenseMatrix.from_rows(rng.integers(-3, 4, size=(n, n)).tolist(), kind="integer")
          for _ in range(6)]
    ms.append(pk.random_binary(n, 5, 0.4))
    st = _native.RunStats()
    got = int_batch_totals(ms, 0, st)
    for m, g in zip(ms, got):
        assert g == int_walk_total(m, [0], sparse=False)
    assert st.launches == 1
    assert pk.permanent_batch(ms) == got
