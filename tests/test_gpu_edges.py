"""Edge cases of the GPU path: the smallest orders, the walker / register
kernel boundaries (n = 10 | 11, complex n = 40 | 41), the largest
instantiated order n = 63, zero rows / zero matrices, mixed-sign entries,
and the reference's error classes (ValueError for bad ranges,
ImpossibleError for n > 63)."""

import itertools
import math

import numpy as np
import pytest

import oracle
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200 import kernels as K
from paper_2502_16577_b200.complex_walk import DenseC128Problem
from paper_2502_16577_b200.integer import IntProblem, _signed
from paper_2502_16577_b200.precision import AccumulatorPolicy

pytestmark = pytest.mark.gpu


def expand(rows):
    """permanent by the permutation expansion (small n, exact for ints)"""
    n = len(rows)
    tot = 0
    for p in itertools.permutations(range(n)):
        t = 1
        for i in range(n):
            t = t * rows[i][p[i]]
        tot = tot + t
    return tot


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_smallest_orders_all_kinds(n):
    rng = np.random.default_rng(n)
    ints = rng.integers(-4, 5, size=(n, n)).tolist()
    reals = rng.uniform(-1, 1, size=(n, n))
    cplx = reals + 1j * rng.uniform(-1, 1, size=(n, n))
    assert pk.permanent(ints) == expand(ints)
    assert pk.perm_spa(pk.dense_to_sparse(pk.DenseMatrix.from_rows(ints))) == expand(ints)
    want = expand(reals.tolist())
    for pol in ("dd", "kahan", "dq", "qq"):
        got = pk.perm_nw(pk.DenseMatrix.from_array(reals), pol)
        assert abs(got - want) <= 1e-13 * max(1.0, abs(want))
    wc = expand(cplx.tolist())
    gc = pk.perm_nw(pk.DenseMatrix.from_array(cplx))
    assert abs(gc - wc) <= 1e-13 * max(1.0, abs(wc))


def test_zero_rows_and_zero_matrices():
    for n in (6, 12, 24):
        z = np.zeros((n, n))
        assert pk.perm_nw(pk.DenseMatrix.from_array(z), "kahan") == 0.0
        a = np.random.default_rng(n).uniform(size=(n, n))
        a[n // 2, :] = 0.0
        assert pk.perm_nw(pk.DenseMatrix.from_array(a), "kahan") == 0.0
        ia = np.random.default_rng(n).integers(0, 3, size=(n, n))
        ia[:, 1] = 0
        assert pk.permanent(ia.tolist()) == 0


@pytest.mark.parametrize("n", [10, 11, 12])
def test_walker_register_boundary_real(n):
    # n = 10 walks with one-thread walkers, n >= 11 with register kernels;
    # both must agree with the oracle's KAHAN over the whole walk
    a = np.random.default_rng(40 + n).uniform(-1, 1, size=(n, n))
    m = pk.DenseMatrix.from_array(a)
    want = oracle.dense_f64_permanent(a, "kahan", tau=1 << 4, threads=2)
    for pol in ("kahan", "dq", "qq", "dd"):
        got = pk.perm_nw(m, pol)
        assert abs(got - want) <= 1e-12 * abs(want), (n, pol)


@pytest.mark.parametrize("n", [39, 40, 41])
def test_complex_register_boundary(n):
    # K3 stops at n = 40; n = 41 takes the lane-pair kernel K3p.
    # A unaligned range walked both ways must equal the oracle's partial.
    h = pk.haar_unitary_block(n, 5)
    a = np.array(h.data, dtype=np.complex128).reshape(n, n)
    prob = DenseC128Problem(h)
    s, e = (1 << 20) + 3, (1 << 20) + 50000
    (wr, wi) = prob.walk(s, e, exact=True)
    want = oracle.dense_c128_range(a, s, e)
    got = complex(wr.hi + wr.lo, wi.hi + wi.lo)
    # head / middle / tail pieces are combined in double-double, the oracle
    # sums serially: the partial cancels heavily, so compare loosely here and
    # bit for bit through the range walkers below
    assert abs(got - want) <= 1e-9 * abs(want) + 1e-300
    [r] = prob.ranges([(s, e)])
    assert (r.real.hex(), r.imag.hex()) == (want.real.hex(), want.imag.hex())


@pytest.mark.parametrize("policy", ["kahan", "qq"])
def test_largest_order_63_register_chunks(policy):
    n = 63
    a = np.random.default_rng(63).uniform(0.0, 1.0, size=(n, n))
    prob = K.DenseF64Problem(pk.DenseMatrix.from_array(a))
    k = 6
    parts, _ = prob.chunks(k, 0, 32, AccumulatorPolicy.parse(policy), exact=True)
    for i in (0, 7, 31):
        s, e = 1 + (i << k), (i + 1) << k
        want = oracle.dense_f64_range(a, s, e, policy)
        assert (parts[i][0].hex(), parts[i][1].hex()) == (want[0].hex(), want[1].hex())


def test_largest_order_63_integer_ranges():
    n = 63
    rng = np.random.default_rng(630)
    rows = [[0] * n for _ in range(n)]
    for i in range(n):  # diagonal + 1-2 extra entries per row: terms stay < 2^127
        rows[i][i] = 1
        for j in rng.choice(n, size=int(rng.integers(1, 3)), replace=False):
            rows[i][int(j)] = int(rng.integers(1, 3))
    m = pk.DenseMatrix.from_rows(rows, kind="integer")
    prob = IntProblem(m)
    for (s, e) in [(1, 1 << 12), ((1 << 40) + 5, (1 << 40) + 3000)]:
        words, info = prob.walk(s, e)
        got = prob.z_to_y(_signed(words, 192), info)
        want = oracle.dense_int_range(rows, s, e)
        assert got == want, (s, e)


def test_mixed_sign_and_scaled_entries():
    # large dynamic range and signs: closed form perm(c * A) = c^n perm(A)
    n = 22
    a = np.random.default_rng(9).uniform(-1, 1, size=(n, n))
    base = pk.perm_nw(pk.DenseMatrix.from_array(a), "qq")
    for c in (1e-8, 3.0, -2.0, 1e6):
        got = pk.perm_nw(pk.DenseMatrix.from_array(a * c), "qq")
        want = base * c ** n
        assert abs(got - want) <= 1e-11 * abs(want), c


def test_reference_error_classes():
    m = pk.random_real(12, 3)
    with pytest.raises(ValueError):
        pk.run_range(m, 0, 10)
    with pytest.raises(ValueError):
        pk.run_range(m, 10, 5)
    with pytest.raises(ValueError):
        pk.run_range(m, 1, 1 << 11)
    with pytest.raises(pk.ImpossibleError):
        pk.DenseMatrix.from_array(np.ones((64, 64)))
    with pytest.raises(pk.PolicyError):
        pk.perm_nw(pk.DenseMatrix.from_rows([[1j, 1], [1, 1]]), "qq")
    # T = 2^(n-1) - 1 is the last iterate; one past it is refused
    T = pk.total_iterates(12)
    assert pk.run_range(m, T, T).iterations_done == 1
    assert math.isfinite(pk.run_range(m, 1, T).value.hi)


def test_concurrent_host_threads_share_a_device_safely():
    # the C ABI serialises per-device work behind a mutex; ctypes releases the
    # GIL, so permkit's thread pool can call in concurrently
    from concurrent.futures import ThreadPoolExecutor
    ms = [pk.random_real(24, s, 0.0, 1.0) for s in range(6)]
    want = [pk.perm_nw(m, "kahan") for m in ms]
    with ThreadPoolExecutor(max_workers=6) as ex:
        got = list(ex.map(lambda m: pk.perm_nw(m, "kahan"), ms))
    assert got == want
    bs = [pk.random_binary(22, s, 0.4) for s in range(4)]
    with ThreadPoolExecutor(max_workers=4) as ex:
        got = list(ex.map(pk.permanent, bs))
    assert got == [pk.permanent(b) for b in bs]


def test_missing_device_ordinal_is_a_device_error():
    m = pk.random_real(14, 2)
    with pytest.raises(pk.DeviceError):
        pk.perm_nw(m, "kahan", devices=[pk._native.device_count() + 3])
