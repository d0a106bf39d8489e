"""Complex (boson-sampling) walks on the GPU: dense complex register kernels
(csrc/pk_dense_c128.cuh, 11 <= n <= 40) and complex range walkers.

Sparse complex pairs (SpaRyser, _loops.py:212-235) go through
pk_sparse_c128: the aligned middle of a walk runs a kernel generated for the
pair's nonzero pattern (each step updates only the flipped column's
nonzeros) with K3's arithmetic; range walkers and exact paths use the
densified columns with the sparse seed (x + 0 == x).
"""

from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as nat
from .kernels import _sign_factor, dense_complex_state, sparse_complex_state, total_iterates
from .matrix import DenseMatrix, SparsePair, sparse_to_dense
from .precision import DoubleDouble, dd_add


class DenseC128Problem:
    def __init__(self, m):
        self.sparse = isinstance(m, SparsePair)
        if self.sparse:
            dense = sparse_to_dense(m)
            cols, _ = dense_complex_state(dense)
            cptrs, rids, vals, x0 = sparse_complex_state(m)
            self.cptrs = np.ascontiguousarray(cptrs, dtype=np.int64)
            self.rids = np.ascontiguousarray(rids if len(rids) else np.zeros(1), dtype=np.int64)
            v = np.ascontiguousarray(vals if len(vals) else np.zeros(1), dtype=np.complex128)
            self.vals = np.ascontiguousarray(v.view(np.float64))
            self.n = m.n
        else:
            cols, x0 = dense_complex_state(m)
            self.n = m.n
        c = np.ascontiguousarray(cols, dtype=np.complex128).reshape(-1)
        self.cols = np.ascontiguousarray(c.view(np.float64)) if c.size else np.zeros(2)
        self.x0c = np.ascontiguousarray(x0, dtype=np.complex128)
        self.x0 = np.ascontiguousarray(self.x0c.view(np.float64))

    def walk(self, start: int, end: int, *, exact: bool = False,
             devices: Optional[Sequence[int]] = None, log2_chunk: int = 0,
             stats: Optional[nat.RunStats] = None,
             precise: bool = False) -> Tuple[DoubleDouble, DoubleDouble]:
        """precise=True (dense): exact fixed-point states per component,
        double-double complex products and sums (PK_FLAG_PRECISE)."""
        lib = nat.load()
        out = np.zeros(4)
        dptr, nd, _keep = nat.devices_arg(devices)
        st = stats if stats is not None else nat.RunStats()
        flags = (nat.PK_FLAG_EXACT if exact else 0) | (nat.PK_FLAG_PRECISE if precise else 0)
        if self.sparse:
            rc = lib.pk_sparse_c128(nat.i64ptr(self.cptrs), nat.i64ptr(self.rids),
                                    nat.dptr(self.vals), self.n, nat.dptr(self.x0), start, end,
                                    flags, log2_chunk, dptr, nd, nat.dptr(out), st)
            nat.check(rc, "pk_sparse_c128")
        else:
            rc = lib.pk_dense_c128(nat.dptr(self.cols), nat.dptr(self.x0), self.n, start, end,
                                   flags, log2_chunk, dptr, nd, nat.dptr(out), st)
            nat.check(rc, "pk_dense_c128")
        return DoubleDouble(out[0], out[1]), DoubleDouble(out[2], out[3])

    def ranges(self, spans: Sequence[Tuple[int, int]], device: int = 0) -> List[complex]:
        if not spans:
            return []
        lib = nat.load()
        s = np.ascontiguousarray(np.array([a for a, _ in spans], dtype=np.uint64))
        e = np.ascontiguousarray(np.array([b for _, b in spans], dtype=np.uint64))
        out = np.zeros(2 * len(spans))
        rc = lib.pk_dense_c128_ranges(nat.dptr(self.cols), nat.dptr(self.x0), self.n,
                                      nat.u64ptr(s), nat.u64ptr(e), len(spans), device,
                                      nat.dptr(out))
        nat.check(rc, "pk_dense_c128_ranges")
        return [complex(out[2 * i], out[2 * i + 1]) for i in range(len(spans))]

    def chunks(self, log2_chunk: int, chunk_lo: int, nchunks: int, exact: bool = True,
               device: int = 0):
        lib = nat.load()
        out = np.zeros(2 * nchunks)
        tot = np.zeros(4)
        flags = (nat.PK_FLAG_EXACT if exact else 0) | (nat.PK_FLAG_SPARSE if self.sparse else 0)
        rc = lib.pk_dense_c128_chunks(nat.dptr(self.cols), nat.dptr(self.x0), self.n, log2_chunk,
                                      chunk_lo, nchunks, flags, device, nat.dptr(out),
                                      nat.dptr(tot))
        nat.check(rc, "pk_dense_c128_chunks")
        return out.reshape(-1, 2), (DoubleDouble(tot[0], tot[1]), DoubleDouble(tot[2], tot[3]))

    def source(self, exact: bool = False) -> str:
        """CUDA source of the generated SpaRyser kernel for this pattern."""
        import ctypes
        lib = nat.load()
        ln = np.zeros(1, dtype=np.uint64)
        flags = nat.PK_FLAG_EXACT if exact else 0
        nat.check(lib.pk_spa_c128_source(nat.dptr(self.cols), self.n, flags, None, 0,
                                         nat.u64ptr(ln)), "pk_spa_c128_source")
        buf = ctypes.create_string_buffer(int(ln[0]) + 1)
        nat.check(lib.pk_spa_c128_source(nat.dptr(self.cols), self.n, flags, buf, len(buf),
                                         nat.u64ptr(ln)), "pk_spa_c128_source")
        return buf.value.decode()

    def p0(self) -> complex:
        p = complex(1.0)
        for v in self.x0c:
            p = p * complex(v)
        return p


def _exact_p0(x0c) -> Tuple[DoubleDouble, DoubleDouble]:
    """The g = 0 product of the (double) seed, exact in rationals, rounded to
    double-double per component (the precise mode's p0)."""
    from fractions import Fraction
    pr, pi = Fraction(1), Fraction(0)
    for v in x0c:
        a, b = Fraction(float(v.real)), Fraction(float(v.imag))
        pr, pi = pr * a - pi * b, pr * b + pi * a

    def dd(f):
        hi = float(f)
        return DoubleDouble(hi, float(f - Fraction(hi)))
    return dd(pr), dd(pi)


def fast_p0(prob: "DenseC128Problem") -> Tuple[DoubleDouble, DoubleDouble]:
    """g = 0 term of a fast complex walk: the exact product of the seed the
    device walks (grid-rounded per component from n = 11), per component in
    double-double (as kernels.fast_p0)."""
    from .kernels import quantized_seed
    n = prob.n
    if n < 11:  # below the register kernels the walk is the reference's loop
        p0 = prob.p0()
        return DoubleDouble(p0.real, 0.0), DoubleDouble(p0.imag, 0.0)
    q = quantized_seed(prob.cols, prob.x0, n, comps=2)
    return _exact_p0(q.view(np.complex128))


def complex_walk_total(m, devices=None, stats=None, precise: bool = False) -> complex:
    prob = DenseC128Problem(m)
    n = prob.n
    re, im = _exact_p0(prob.x0c) if precise else fast_p0(prob)
    if n > 1:
        wr, wi = prob.walk(1, total_iterates(n), devices=devices, stats=stats, precise=precise)
        re, im = dd_add(re, wr), dd_add(im, wi)
    sign = _sign_factor(n)
    return complex(re.hi * sign, im.hi * sign)


EXACT_RANGE_LIMIT = 1 << 22


def complex_ranges(m, spans, exact=None, devices=None) -> List[complex]:
    prob = DenseC128Problem(m)
    dev0 = devices[0] if devices else 0
    out: List[Optional[complex]] = [None] * len(spans)
    small = [i for i, (s, e) in enumerate(spans)
             if exact is True or (exact is None and e - s + 1 <= EXACT_RANGE_LIMIT)]
    if small:
        for i, v in zip(small, prob.ranges([spans[i] for i in small], device=dev0)):
            out[i] = v
    for i, (s, e) in enumerate(spans):
        if out[i] is None:
            wr, wi = prob.walk(s, e, devices=devices)
            out[i] = complex(wr.hi + wr.lo, wi.hi + wi.lo)
    return out
