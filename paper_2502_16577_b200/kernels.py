"""Serial-engine entry points and the per-row state builders.

Same names and semantics as permkit.kernels (/root/reference/pkg/src/
permkit/kernels.py): ``perm_nw`` (dense Gray walk), ``perm_spa`` (sparse
walk), the ``*_state`` builders, ``policy_product``, ``total_iterates``. The
walk itself runs on the GPU through the C ABI (csrc/pk_abi.cu); what stays in
Python is O(n^2) marshalling, done with exactly the reference's rounding
order so the device sees bit-identical inputs:

  cols[j, i] = a_ij (j < n-1),  x0_i = a_{i,n-1} - rowsum_i / 2   (kernels.py:75-89)

Whole walks go through the register kernels, whose per-chunk arithmetic is
the reference's but whose chunking (2^k-iterate chunks reduced by a fixed
double-double tree) is the GPU's, so floating-point results agree with the
reference to rounding, not bit for bit; integer results are exact.
"""

from __future__ import annotations

from typing import List, Optional, Sequence, Tuple, Union

import ctypes

import numpy as np

from . import _native as nat
from .errors import PolicyError
from .matrix import (
    KIND_COMPLEX,
    KIND_INT,
    KIND_REAL,
    DenseMatrix,
    Scalar,
    SparsePair,
    row_sums,
    sparse_to_dense,
)
from .precision import AccumulatorPolicy, DoubleDouble, as_policy, dd_add, dd_mul_double


def _sign_factor(n: int) -> int:
    """Global factor of the half-space walk: +2 for odd n, -2 for even n."""
    return 2 if n % 2 else -2


def total_iterates(n: int) -> int:
    """Iterates beyond g = 0: 2^(n-1) - 1."""
    return (1 << (n - 1)) - 1


# ---------------------------------------------------------------------------
# state builders (host side of the C ABI)


def dense_float_state(a: DenseMatrix) -> Tuple[np.ndarray, np.ndarray]:
    n = a.n
    grid = np.array(a.data, dtype=np.float64).reshape(n, n)
    cols = np.ascontiguousarray(grid[:, : n - 1].T) if n > 1 else np.zeros((0, 1))
    rs = np.array(row_sums(a), dtype=np.float64)
    return cols, np.ascontiguousarray(grid[:, n - 1] - rs / 2.0)


def dense_complex_state(a: DenseMatrix) -> Tuple[np.ndarray, np.ndarray]:
    n = a.n
    grid = np.array(a.data, dtype=np.complex128).reshape(n, n)
    cols = (np.ascontiguousarray(grid[:, : n - 1].T) if n > 1
            else np.zeros((0, 1), dtype=np.complex128))
    rs = np.array(row_sums(a), dtype=np.complex128)
    return cols, np.ascontiguousarray(grid[:, n - 1] - rs / 2.0)


def dense_int_state(a: DenseMatrix) -> Tuple[List[Tuple[int, ...]], List[int]]:
    """Doubled columns and y0 = 2 x0 of the exact walk (kernels.py:104-110)."""
    n = a.n
    cols2 = [tuple(2 * a.entry(i, j) for i in range(n)) for j in range(n - 1)]
    sums = row_sums(a)
    return cols2, [2 * a.entry(i, n - 1) - sums[i] for i in range(n)]


def _sparse_seed(s: SparsePair, zero):
    n = s.n
    x0 = [zero] * n
    rows_last, vals_last = s.ccs.col_slice(n - 1)
    for r, v in zip(rows_last, vals_last):
        x0[r] = v
    return x0, row_sums(s)


def sparse_float_state(s: SparsePair):
    ccs = s.ccs
    x0, sums = _sparse_seed(s, 0.0)
    x = np.array(x0, dtype=np.float64)
    x = x - np.array(sums, dtype=np.float64) / 2.0
    return (np.array(ccs.cptrs, dtype=np.int64), np.array(ccs.rids, dtype=np.int64),
            np.array(ccs.vals, dtype=np.float64), x)


def sparse_complex_state(s: SparsePair):
    ccs = s.ccs
    x0, sums = _sparse_seed(s, 0j)
    x = np.array(x0, dtype=np.complex128)
    x = x - np.array(sums, dtype=np.complex128) / 2.0
    return (np.array(ccs.cptrs, dtype=np.int64), np.array(ccs.rids, dtype=np.int64),
            np.array(ccs.vals, dtype=np.complex128), x)


def sparse_int_state(s: SparsePair):
    ccs = s.ccs
    n = s.n
    colrows, colvals2 = [], []
    for j in range(n - 1):
        rows, vals = ccs.col_slice(j)
        colrows.append(tuple(rows))
        colvals2.append(tuple(2 * v for v in vals))
    y0, sums = _sparse_seed(s, 0)
    y0 = [2 * v for v in y0]
    return colrows, colvals2, [y0[i] - sums[i] for i in range(n)]


def policy_product(xs, policy: AccumulatorPolicy) -> Union[float, DoubleDouble]:
    """Product of the state in the policy's inner precision (kernels.py:166-180)."""
    if as_policy(policy) is AccumulatorPolicy.QQ:
        acc = DoubleDouble(1.0, 0.0)
        for v in xs:
            acc = dd_mul_double(acc, float(v))
        return acc
    p = 1.0
    for v in xs:
        p = p * float(v)
    return p


def quantized_seed(cols: np.ndarray, x0: np.ndarray, n: int, comps: int = 1) -> np.ndarray:
    """The seed x0 as the fast kernels walk it: rounded onto the same per-row
    (per component) grids as the columns (pk_quantize_walk; DESIGN.md §3
    "Exact states"). Host-only."""
    c = np.ascontiguousarray(cols, dtype=np.float64).reshape(-1)
    x = np.ascontiguousarray(x0, dtype=np.float64).reshape(-1)
    qc = np.zeros_like(c)
    qx = np.zeros_like(x)
    nat.check(nat.load().pk_quantize_walk(nat.dptr(c), nat.dptr(x), n, comps, nat.dptr(qc),
                                          nat.dptr(qx)), "pk_quantize_walk")
    return qx


def _dd_of(f) -> DoubleDouble:
    hi = float(f)
    from fractions import Fraction
    return DoubleDouble(hi, float(f - Fraction(hi)))


def fast_p0(cols: np.ndarray, x0: np.ndarray, n: int,
            policy: "AccumulatorPolicy | str" = AccumulatorPolicy.DD) -> DoubleDouble:
    """The g = 0 term of a fast walk: the exact product of the seed the device
    walks (grid-rounded from n = 11, where the register kernels start),
    rounded once to double-double. It is the largest single term of the
    cancelling sum, so it must belong to the same (rounded) matrix as the
    walk and carry no product rounding: 3.4e-12 of the n = 40 error under QQ
    and more under the double-product policies came from the seed being the
    unrounded one (tools/quantization_effect.py)."""
    from fractions import Fraction
    if n < 11:  # below the register kernels the walk is the reference's loop
        p0 = policy_product(x0, as_policy(policy))
        return p0 if isinstance(p0, DoubleDouble) else DoubleDouble(float(p0), 0.0)
    p = Fraction(1)
    for v in quantized_seed(cols, x0, n):
        p *= Fraction(float(v))
    return _dd_of(p)


def seed_accumulator(p0, policy: AccumulatorPolicy) -> Tuple[float, float]:
    if as_policy(policy) is AccumulatorPolicy.QQ:
        return p0.hi, p0.lo
    return float(p0), 0.0


def collapse_accumulator(acc_a: float, acc_b: float, policy: AccumulatorPolicy) -> float:
    return acc_a if as_policy(policy) is AccumulatorPolicy.DD else acc_a + acc_b


# ---------------------------------------------------------------------------
# device calls


class DenseF64Problem:
    """Marshalled dense real walk: C-contiguous cols / x0 for the C ABI."""

    def __init__(self, a: DenseMatrix):
        self.n = a.n
        cols, x0 = dense_float_state(a)
        self.cols = np.ascontiguousarray(cols, dtype=np.float64).reshape(-1)
        if self.cols.size == 0:
            self.cols = np.zeros(1)
        self.x0 = np.ascontiguousarray(x0, dtype=np.float64)

    def walk(self, start: int, end: int, policy: AccumulatorPolicy, *, exact: bool = False,
             devices: Optional[Sequence[int]] = None, log2_chunk: int = 0,
             stats: Optional[nat.RunStats] = None, precise: bool = False) -> DoubleDouble:
        """precise=True: exact fixed-point row sums, double-double products and
        sums (PK_FLAG_PRECISE; the policy is then irrelevant)."""
        lib = nat.load()
        out = np.zeros(2)
        dptr, nd, _keep = nat.devices_arg(devices)
        st = stats if stats is not None else nat.RunStats()
        flags = (nat.PK_FLAG_EXACT if exact else 0) | (nat.PK_FLAG_PRECISE if precise else 0)
        rc = lib.pk_dense_f64(nat.dptr(self.cols), nat.dptr(self.x0), self.n, start, end,
                              policy.code, flags, log2_chunk, dptr, nd, nat.dptr(out), st)
        nat.check(rc, "pk_dense_f64")
        return DoubleDouble(float(out[0]), float(out[1]))

    def ranges(self, spans: Sequence[Tuple[int, int]], policy: AccumulatorPolicy,
               device: int = 0) -> List[DoubleDouble]:
        """Bit-exact run_range partials, one device thread per range."""
        if not spans:
            return []
        lib = nat.load()
        s = np.ascontiguousarray(np.array([a for a, _ in spans], dtype=np.uint64))
        e = np.ascontiguousarray(np.array([b for _, b in spans], dtype=np.uint64))
        out = np.zeros(2 * len(spans))
        rc = lib.pk_dense_f64_ranges(nat.dptr(self.cols), nat.dptr(self.x0), self.n, nat.u64ptr(s),
                                     nat.u64ptr(e), len(spans), policy.code, device, nat.dptr(out))
        nat.check(rc, "pk_dense_f64_ranges")
        return [DoubleDouble(float(out[2 * i]), float(out[2 * i + 1])) for i in range(len(spans))]

    flags = 0  # PK_FLAG_SPARSE for the SpaRyser subclass

    def chunks(self, log2_chunk: int, chunk_lo: int, nchunks: int, policy: AccumulatorPolicy,
               exact: bool = True, device: int = 0, precise: bool = False):
        """Per-chunk partials of the register kernel (parity diagnostics)."""
        lib = nat.load()
        out = np.zeros(2 * nchunks)
        tot = np.zeros(2)
        flags = self.flags | (nat.PK_FLAG_EXACT if exact else 0) | \
            (nat.PK_FLAG_PRECISE if precise else 0)
        rc = lib.pk_dense_f64_chunks(nat.dptr(self.cols), nat.dptr(self.x0), self.n, log2_chunk,
                                     chunk_lo, nchunks, policy.code, flags, device,
                                     nat.dptr(out), nat.dptr(tot))
        nat.check(rc, "pk_dense_f64_chunks")
        return out.reshape(-1, 2), DoubleDouble(float(tot[0]), float(tot[1]))


class SparseF64Problem(DenseF64Problem):
    """Marshalled sparse real walk (SpaRyser): the reference's CCS state
    (sparse_float_state, kernels.py:113-127) for pk_sparse_f64, whose aligned
    middle runs a kernel generated for the nonzero pattern (each step adds
    only the flipped column's nonzeros, _loops.py:122-124). Range walkers and
    the bit-exact paths use the densified columns (x + 0.0 == x)."""

    flags = nat.PK_FLAG_SPARSE

    def __init__(self, s: SparsePair):
        super().__init__(sparse_to_dense(s))
        cptrs, rids, vals, x0 = sparse_float_state(s)
        self.cptrs = np.ascontiguousarray(cptrs, dtype=np.int64)
        self.rids = np.ascontiguousarray(rids if len(rids) else np.zeros(1), dtype=np.int64)
        self.vals = np.ascontiguousarray(vals if len(vals) else np.zeros(1), dtype=np.float64)
        self.x0 = np.ascontiguousarray(x0, dtype=np.float64)

    def walk(self, start: int, end: int, policy: AccumulatorPolicy, *, exact: bool = False,
             devices: Optional[Sequence[int]] = None, log2_chunk: int = 0,
             stats: Optional[nat.RunStats] = None) -> DoubleDouble:
        lib = nat.load()
        out = np.zeros(2)
        dptr, nd, _keep = nat.devices_arg(devices)
        st = stats if stats is not None else nat.RunStats()
        rc = lib.pk_sparse_f64(nat.i64ptr(self.cptrs), nat.i64ptr(self.rids), nat.dptr(self.vals),
                               self.n, nat.dptr(self.x0), start, end, policy.code,
                               nat.PK_FLAG_EXACT if exact else 0, log2_chunk, dptr, nd,
                               nat.dptr(out), st)
        nat.check(rc, "pk_sparse_f64")
        return DoubleDouble(float(out[0]), float(out[1]))

    def source(self, policy: AccumulatorPolicy, exact: bool = False) -> str:
        """CUDA source of the generated kernel for this pattern (diagnostics)."""
        lib = nat.load()
        ln = np.zeros(1, dtype=np.uint64)
        flags = nat.PK_FLAG_EXACT if exact else 0
        nat.check(lib.pk_spa_f64_source(nat.dptr(self.cols), self.n, policy.code, flags, None, 0,
                                        nat.u64ptr(ln)), "pk_spa_f64_source")
        buf = ctypes.create_string_buffer(int(ln[0]) + 1)
        nat.check(lib.pk_spa_f64_source(nat.dptr(self.cols), self.n, policy.code, flags, buf,
                                        len(buf), nat.u64ptr(ln)), "pk_spa_f64_source")
        return buf.value.decode()


def _real_walk_total(a: DenseMatrix, policy: AccumulatorPolicy, devices=None,
                     stats: Optional[nat.RunStats] = None, precise: bool = False) -> float:
    n = a.n
    prob = DenseF64Problem(a)
    # precise mode: the g = 0 product in double-double of the input's seed;
    # fast mode: the exact product of the grid-rounded seed the device walks
    acc = policy_product(prob.x0, AccumulatorPolicy.QQ) if precise else \
        fast_p0(prob.cols, prob.x0, n, policy)
    if n > 1:
        acc = dd_add(acc, prob.walk(1, total_iterates(n), policy, devices=devices, stats=stats,
                                    precise=precise))
    return acc.hi * _sign_factor(n)


def perm_nw(a: DenseMatrix, policy: "AccumulatorPolicy | str" = AccumulatorPolicy.DD,
            *, devices: Optional[Sequence[int]] = None, precise: bool = False) -> Scalar:
    """Permanent by the Gray walk over the 2^(n-1) half-space subsets,
    computed on the GPU (kernels.py:297-324). precise=True (dense real or
    complex, n >= 11): exact fixed-point row sums with double-double products
    and sums -- reference-grade, about 10x (real) / 15x (complex) slower
    (DESIGN.md §3)."""
    policy = as_policy(policy)
    if precise and a.kind == KIND_INT:
        raise PolicyError("precise mode serves real and complex matrices (integers are exact)")
    if a.kind == KIND_INT:
        from .integer import int_walk_total
        return int_walk_total(a, devices=devices)
    if a.kind == KIND_COMPLEX:
        if policy is not AccumulatorPolicy.DD:
            raise PolicyError("complex matrices support the plain-double policy only")
        from .complex_walk import complex_walk_total
        return complex_walk_total(a, devices=devices, precise=precise)
    return _real_walk_total(a, policy, devices, precise=precise)


def perm_spa(s: SparsePair, policy: "AccumulatorPolicy | str" = AccumulatorPolicy.DD,
             *, devices: Optional[Sequence[int]] = None) -> Scalar:
    """Permanent of a CRS/CCS pair (kernels.py:327-362). Structurally
    inconsistent pairs are rejected before any arithmetic."""
    policy = as_policy(policy)
    s.validate()
    if s.kind == KIND_INT:
        from .integer import int_walk_total
        return int_walk_total(s, devices=devices)
    if s.kind == KIND_COMPLEX:
        if policy is not AccumulatorPolicy.DD:
            raise PolicyError("complex matrices support the plain-double policy only")
        from .complex_walk import complex_walk_total
        return complex_walk_total(s, devices=devices)
    return _real_walk_total_sparse(s, policy, devices)


def _real_walk_total_sparse(s: SparsePair, policy, devices) -> float:
    n = s.n
    prob = SparseF64Problem(s)
    acc = fast_p0(prob.cols, prob.x0, n, policy)
    if n > 1:
        acc = dd_add(acc, prob.walk(1, total_iterates(n), policy, devices=devices))
    return acc.hi * _sign_factor(n)
