"""The fast modes' input rounding (pk_quantize_walk, csrc/pk_abi.cu
quantize_walk; DESIGN.md §3 "Exact states"), checked on the host: after it,
every Gray-walk state -- every subset sum x0_i + sum_{j in S} a_ij -- is a
double, so the device walk's incremental DADDs are exact whatever the order,
and each entry moved by at most half an ulp of its row's largest reachable
state. Pure host code: runs without a GPU."""

import ctypes
from fractions import Fraction

import numpy as np
import pytest

from paper_2502_16577_b200 import _native
from paper_2502_16577_b200.kernels import dense_float_state
from paper_2502_16577_b200.matrix import DenseMatrix


def quantize(cols, x0, n, comps):
    lib = _native.load()
    qc = np.zeros_like(cols)
    qx = np.zeros_like(x0)
    rc = lib.pk_quantize_walk(_native.dptr(cols), _native.dptr(x0), n, comps, _native.dptr(qc),
                              _native.dptr(qx))
    assert rc == 0, _native.last_error()
    return qc, qx


@pytest.mark.parametrize("n,lo,hi,seed", [(12, 0.0, 1.0, 1), (20, -3.0, 5.0, 2), (40, 0.0, 1.0, 3),
                                          (63, -1e-3, 1e4, 4)])
def test_every_walk_state_is_a_double(n, lo, hi, seed):
    rng = np.random.default_rng(seed)
    a = rng.uniform(lo, hi, size=(n, n))
    cols, x0 = dense_float_state(DenseMatrix.from_array(a))
    cols = np.ascontiguousarray(cols, dtype=np.float64).reshape(-1)
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    qc, qx = quantize(cols, x0, n, 1)
    qc = qc.reshape(n - 1, n)
    c2 = cols.reshape(n - 1, n)
    for i in range(n):
        bound = abs(x0[i]) + float(np.abs(c2[:, i]).sum())
        half_ulp = 2.0 ** (np.frexp(bound)[1] - 53)
        assert abs(qx[i] - x0[i]) <= half_ulp
        assert np.all(np.abs(qc[:, i] - c2[:, i]) <= half_ulp)
        # a random walk of incremental double updates stays exact
        x = qx[i]
        exact = Fraction(qx[i])
        inside = np.zeros(n - 1, dtype=bool)
        for j in rng.integers(0, n - 1, size=400):
            v = qc[j, i]
            if inside[j]:
                x, exact = x - v, exact - Fraction(v)
            else:
                x, exact = x + v, exact + Fraction(v)
            inside[j] = not inside[j]
            assert Fraction(x) == exact


def test_complex_components_get_their_own_grid():
    n = 16
    rng = np.random.default_rng(9)
    # real parts ~1e3, imaginary parts ~1e-3: separate grids keep the small parts
    cols = np.empty(2 * (n - 1) * n)
    cols[0::2] = rng.uniform(0, 1e3, size=(n - 1) * n)
    cols[1::2] = rng.uniform(0, 1e-3, size=(n - 1) * n)
    x0 = rng.uniform(-1, 1, size=2 * n)
    qc, qx = quantize(cols, x0, n, 2)
    im = cols[1::2].reshape(n - 1, n)
    qim = qc[1::2].reshape(n - 1, n)
    for i in range(n):
        bound_im = abs(x0[2 * i + 1]) + float(im[:, i].sum())  # ~1, the real bound is ~1e4
        half_ulp = 2.0 ** (np.frexp(bound_im)[1] - 53)
        assert np.all(np.abs(qim[:, i] - im[:, i]) <= half_ulp)


def test_zero_rows_and_bad_arguments():
    n = 5
    cols = np.zeros((n - 1) * n)
    x0 = np.zeros(n)
    qc, qx = quantize(cols, x0, n, 1)
    assert not qc.any() and not qx.any()
    lib = _native.load()
    assert lib.pk_quantize_walk(_native.dptr(cols), _native.dptr(x0), n, 3, _native.dptr(cols),
                                _native.dptr(x0)) == _native.PK_ERR_ARG
    assert lib.pk_quantize_walk(_native.dptr(cols), _native.dptr(x0), 64, 1, _native.dptr(cols),
                                _native.dptr(x0)) == _native.PK_ERR_IMPOSSIBLE


def test_subnormal_rows_stay_on_a_representable_grid():
    n = 6
    rng = np.random.default_rng(3)
    cols = rng.uniform(0, 1, size=(n - 1) * n) * 1e-310  # subnormal entries
    x0 = rng.uniform(-1, 1, size=n) * 1e-310
    qc, qx = quantize(cols, x0, n, 1)
    # the walk's states of grid values are exact sums
    c2 = qc.reshape(n - 1, n)
    for i in range(n):
        x = qx[i]
        exact = Fraction(qx[i])
        for j in range(n - 1):
            x, exact = x + c2[j, i], exact + Fraction(c2[j, i])
            assert Fraction(x) == exact
