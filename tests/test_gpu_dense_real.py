"""GPU parity of the dense real path (K1) against the reference's golden
vectors and the C oracle.

* range walkers: run_range partials bit-identical to permkit's
* register kernel, exact mode: every chunk partial bit-identical to the
  oracle's run_range over the same chunk; the device tree equals the host's
  pairwise fold of those partials
* whole permanents: <= 1e-10 relative to the reference's KAHAN/DQ/QQ results
  (never DD), closed forms n! a^n, TERNARY12 == 2 exactly
"""

import math
from fractions import Fraction

import numpy as np
import pytest

import golden_io as gio
import oracle
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200 import kernels as K
from paper_2502_16577_b200.precision import AccumulatorPolicy, DoubleDouble, dd_add, dd_pairwise

pytestmark = pytest.mark.gpu

REAL_DENSE = [c["name"] for c in gio.cases(gio.load(), "dense", "real64")]
POLS = ["dd", "kahan", "dq", "qq"]
WALKER_LIMIT = 1 << 21


def _case(golden, name):
    return next(c for c in golden["cases"] if c["name"] == name)


def _matrix(case):
    return pk.DenseMatrix.from_array(gio.dense_array(case))


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("name", REAL_DENSE)
def test_run_range_bitwise_vs_reference(golden, name):
    case = _case(golden, name)
    m = _matrix(case)
    for r in case["ranges"]:
        if r["end"] - r["start"] >= WALKER_LIMIT:
            continue  # one device thread per range: keep the suite fast
        p = pk.run_range(m, r["start"], r["end"], r["policy"], worker_id=3, exact=True)
        assert (p.value.hi.hex(), p.value.lo.hex()) == tuple(r["value"]), (name, r)
        assert p.worker_id == 3 and p.iterations_done == r["end"] - r["start"] + 1


@pytest.mark.parametrize("name", REAL_DENSE)
def test_permanent_chunked_bitwise_vs_reference(golden, name):
    case = _case(golden, name)
    m = _matrix(case)
    T = K.total_iterates(m.n)
    for ch in case["chunked"]:
        plan = pk.plan_chunks(m.n, ch["tau"], ch["aligned"])
        if max(e - s for (_, s, e) in plan.jobs()) >= WALKER_LIMIT or plan.worker_count > 4096:
            continue
        got = pk.permanent_chunked(m, ch["policy"], tau=ch["tau"], aligned=ch["aligned"],
                                   exact=True)
        assert got.hex() == ch["value"], (name, ch)


@pytest.mark.parametrize("n,k", [(20, 5), (20, 9), (24, 6), (31, 12)])
@pytest.mark.parametrize("policy", POLS)
def test_register_chunks_bitwise_vs_oracle(n, k, policy):
    a = np.random.default_rng(1000 + n).uniform(0.0, 1.0, size=(n, n))
    m = pk.DenseMatrix.from_array(a)
    prob = K.DenseF64Problem(m)
    nchunks = min(1 << (n - 1 - k), 64)
    chunk_lo = (1 << (n - 1 - k)) - nchunks  # the last chunks: includes the clipped one
    parts, total = prob.chunks(k, chunk_lo, nchunks, AccumulatorPolicy.parse(policy), exact=True)
    T = K.total_iterates(n)
    size = 1 << k
    for i in range(0, nchunks, 7):
        c = chunk_lo + i
        s, e = 1 + c * size, min((c + 1) * size, T)
        want = oracle.dense_f64_range(a, s, e, policy)
        assert (parts[i][0].hex(), parts[i][1].hex()) == (want[0].hex(), want[1].hex()), (c, s, e)
    host = dd_pairwise([tuple(p) for p in parts])
    assert (host.hi, host.lo) == (total.hi, total.lo)


@pytest.mark.parametrize("name,pols", [("config1_real20", ["kahan", "dq", "qq"]),
                                       ("real24", ["kahan", "dq", "qq"]),
                                       ("real28", ["kahan", "dq"]),
                                       ("real_unit12", ["kahan", "dq", "qq"])])
def test_perm_nw_within_1e10_of_reference(golden, name, pols):
    # anchor: the reference's compensated policy with the SHORTEST chunks it
    # was run with -- long reference chunks let the per-row state drift
    # (real28 at tau=64 is 3.6e-10 off its own tau=65536 value)
    case = _case(golden, name)
    m = _matrix(case)
    comp = [ch for ch in case["chunked"] if ch["policy"] in ("kahan", "dq", "qq")]
    ref = float.fromhex(max(comp, key=lambda ch: ch["tau"])["value"])
    for p in pols + ["dd"]:
        got = pk.perm_nw(m, p)
        assert rel(got, ref) <= 1e-10, (name, p, got, ref)


@pytest.mark.parametrize("n", [16, 20, 24, 28, 30])
def test_uniform_closed_form(n):
    exact = math.factorial(n) * Fraction(0.91) ** n
    m = pk.uniform(n, 0.91)
    for p in POLS:
        got = pk.perm_nw(m, p)
        err = float(abs(Fraction(got) - exact) / exact)
        assert err <= 1e-10, (n, p, err)


def test_ternary12_is_exactly_two_everywhere(golden):
    case = _case(golden, "ternary12_real")
    m = _matrix(case)
    for p in POLS:
        assert pk.perm_nw(m, p) == 2.0
        for tau in (1, 3, 16):
            assert pk.permanent_chunked(m, p, tau=tau) == 2.0
    assert pk.permanent(m) == 2.0


def test_device_split_reproduces_single_device_bits():
    # two logical devices (the same GPU twice) take half of the chunk groups
    # each; the host tree must reproduce the single-launch tree bit for bit
    m = pk.random_real(26, 7, 0.0, 1.0)
    prob = K.DenseF64Problem(m)
    T = K.total_iterates(26)
    for p in (AccumulatorPolicy.KAHAN, AccumulatorPolicy.DD):
        one = prob.walk(1, T, p)
        two = prob.walk(1, T, p, devices=[0, 0])
        four = prob.walk(1, T, p, devices=[0, 0, 0, 0])
        assert one == two == four


@pytest.mark.parametrize("n", [14, 22, 25])
def test_unaligned_ranges_fast_path(n):
    # head / middle / tail split of an arbitrary range vs the exact walker
    a = np.random.default_rng(n).uniform(-1.0, 1.0, size=(n, n))
    m = pk.DenseMatrix.from_array(a)
    prob = K.DenseF64Problem(m)
    rng = np.random.default_rng(99 + n)
    T = K.total_iterates(n)
    for _ in range(6):
        s = int(rng.integers(1, T // 3))
        e = int(rng.integers(2 * T // 3, T + 1))
        st = pk._native.RunStats()
        fast = prob.walk(s, e, AccumulatorPolicy.KAHAN, stats=st)
        ref = oracle.dense_f64_range(a, s, e, "dq")
        scale = float(np.prod(np.abs(a).sum(axis=1)))  # bound on |terms|
        assert abs((fast.hi + fast.lo) - (ref[0] + ref[1])) <= 1e-12 * scale
        assert st.iterates == e - s + 1


def test_large_range_run_range_uses_register_kernels():
    m = pk.random_real(30, 5, 0.0, 1.0)
    T = K.total_iterates(30)
    p = pk.run_range(m, 1, T, "kahan")
    q = pk.run_range(m, 1, T // 2, "kahan")
    r = pk.run_range(m, T // 2 + 1, T, "kahan")
    whole = p.value.hi + p.value.lo
    parts = (q.value.hi + q.value.lo) + (r.value.hi + r.value.lo)
    assert abs(whole - parts) <= 1e-12 * abs(whole) + 1e-300


def test_errors_are_the_reference_classes():
    m = pk.random_real(12, 3)
    with pytest.raises(ValueError):
        pk.run_range(m, 0, 5)
    with pytest.raises(ValueError):
        pk.run_range(m, 5, 1 << 11)
    prob = K.DenseF64Problem(m)
    with pytest.raises(ValueError):
        prob.chunks(3, 0, 32, AccumulatorPolicy.DD)  # k below the body length


def test_fast_states_are_exact_so_chunk_length_does_not_matter():
    # fast mode walks the input rounded onto per-row grids on which every
    # state is a double (pk_abi.cu quantize_walk): x never
    # drifts, so the chunk length only reorders the product sums. The
    # reference's incremental walk of 2^k-step chunks drifted by ~1e-9 here.
    n = 34
    g = np.random.default_rng(20261017).uniform(0.0, 1.0, size=(n, n))
    m = pk.DenseMatrix.from_array(g)
    prob = K.DenseF64Problem(m)
    p0 = K.policy_product(prob.x0, AccumulatorPolicy.KAHAN)
    T = K.total_iterates(n)
    vals = []
    for k in (8, 12, 16, 20):
        part = prob.walk(1, T, AccumulatorPolicy.KAHAN, log2_chunk=k)
        vals.append(dd_add(DoubleDouble(p0, 0.0), part).hi)
    for v in vals[1:]:
        assert abs(v - vals[0]) <= 1e-12 * abs(vals[0]), vals


@pytest.mark.parametrize("n", [24, 30, 34])
def test_fast_within_1e11_of_precise_mode(n):
    # precise mode: exact fixed-point row sums, double-double products and
    # sums (pk_precise.cuh) -- the reference-grade value
    g = np.random.default_rng(77 + n).uniform(0.0, 1.0, size=(n, n))
    m = pk.DenseMatrix.from_array(g)
    want = pk.perm_nw(m, precise=True)
    for p in POLS:
        got = pk.perm_nw(m, p)
        assert rel(got, want) <= 1e-11, (n, p, got, want, rel(got, want))


@pytest.mark.parametrize("n", [16, 24, 30])
def test_precise_mode_uniform_closed_form(n):
    exact = math.factorial(n) * Fraction(0.91) ** n
    got = pk.perm_nw(pk.uniform(n, 0.91), precise=True)
    assert float(abs(Fraction(got) - exact) / exact) <= 1e-14


@pytest.mark.parametrize("n", [36, 40])
def test_uniform_closed_form_large(n):
    # uniform(n, 0.91): every x_i is equal, so the double product x^n rounds
    # the same way for every subset of one size and product rounding does not
    # average out under KAHAN / DQ / DD (2.3e-10 at n = 40); QQ's double-double
    # product removes it (2.8e-13; the paper: 6.5e-11 at n = 40)
    exact = math.factorial(n) * Fraction(0.91) ** n
    m = pk.uniform(n, 0.91)
    err_qq = float(abs(Fraction(pk.perm_nw(m, "qq")) - exact) / exact)
    assert err_qq <= 1e-12, err_qq
    err_k = float(abs(Fraction(pk.perm_nw(m, "kahan")) - exact) / exact)
    assert err_k <= 5e-10, err_k
