"""Exact integer walks on the GPU (csrc/pk_int.cuh via pk_int / pk_int_ranges).

The device walks z_i = y_i / 2 (even row sum) or y_i (odd row sum), y = 2x
being the reference's doubled state (kernels.py:104-110); partials come back
in z-space and are rescaled here by 2^even_rows, which gives exactly the
y-space integers permkit's run_range returns (parallel.py:232-255) and
reduce_partials / _finalize_int consume (parallel.py:371-375,
kernels.py:290-294).

Exactness: every term is exact when the product of the per-row bounds is
below 2^127 (always true for the 40x40 density-0.3 binary configuration:
about 2^122); range partials are then exact 192-bit sums. Otherwise only the
whole-walk total is recoverable (mod 2^128 plus a permanent bound); partial
ranges raise OverflowError rather than return something inexact.
"""

from __future__ import annotations

import ctypes
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as nat
from .matrix import DenseMatrix, SparsePair, sparse_to_dense


class IntInfo(ctypes.Structure):
    _fields_ = [("zbits", ctypes.c_int32), ("even_rows", ctypes.c_int32),
                ("exact_terms", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("log2_term_bound", ctypes.c_double)]


def finalize_int(total_y: int, n: int) -> int:
    """Global sign, then the exact division by 2^(n-1) (kernels.py:290-294)."""
    signed = total_y if n % 2 else -total_y
    q, r = divmod(signed, 1 << (n - 1))
    if r:
        raise ArithmeticError("integer-exact walk produced a non-divisible total")
    return q


def _signed(words, bits: int) -> int:
    v = 0
    for i, w in enumerate(words):
        v |= (int(w) & ((1 << 64) - 1)) << (64 * i)
    v &= (1 << bits) - 1
    return v - (1 << bits) if v >> (bits - 1) else v


SPARSE_MIN_N = 36


def spa_source(m) -> str:
    """CUDA source of the generated SpaRyser kernel for an integer matrix."""
    prob = IntProblem(m)
    ln = ctypes.c_uint64(0)
    buf = ctypes.create_string_buffer(1 << 22)
    rc = nat.load().pk_int_spa_source(prob._a(), prob.n, buf, 1 << 22, ctypes.byref(ln))
    nat.check(rc, "pk_int_spa_source")
    return buf.value.decode()


class IntProblem:
    def __init__(self, m):
        dense = sparse_to_dense(m) if isinstance(m, SparsePair) else m
        self.n = dense.n
        a = [int(v) for v in dense.data]
        if any(abs(v) >= (1 << 62) for v in a):
            raise OverflowError("integer entries beyond 2^62 are not supported on the GPU path")
        self.a = np.ascontiguousarray(np.array(a, dtype=np.int64))
        self.rows = [a[i * self.n:(i + 1) * self.n] for i in range(self.n)]
        self.info = IntInfo()

    def _a(self):
        return self.a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))

    def walk(self, start: int, end: int, devices=None, log2_chunk: int = 0,
             stats: Optional[nat.RunStats] = None,
             sparse: Optional[bool] = None) -> Tuple[List[int], IntInfo]:
        """sparse=None picks the generated SpaRyser kernel for n >= SPARSE_MIN_N
        (its one-off NVRTC compile, ~1 s, then pays for itself)."""
        lib = nat.load()
        out = np.zeros(3, dtype=np.uint64)
        dptr, nd, _keep = nat.devices_arg(devices)
        st = stats if stats is not None else nat.RunStats()
        if sparse is None:
            sparse = self.n >= SPARSE_MIN_N
        flags = nat.PK_FLAG_SPARSE if sparse else 0
        rc = lib.pk_int(self._a(), self.n, start, end, flags, log2_chunk, dptr, nd,
                        nat.u64ptr(out), ctypes.byref(self.info), st)
        nat.check(rc, "pk_int")
        return [int(w) for w in out], self.info

    def ranges(self, spans, device: int = 0) -> Tuple[List[List[int]], IntInfo]:
        lib = nat.load()
        s = np.ascontiguousarray(np.array([a for a, _ in spans], dtype=np.uint64))
        e = np.ascontiguousarray(np.array([b for _, b in spans], dtype=np.uint64))
        out = np.zeros(3 * max(1, len(spans)), dtype=np.uint64)
        rc = lib.pk_int_ranges(self._a(), self.n, nat.u64ptr(s), nat.u64ptr(e), len(spans), device,
                               nat.u64ptr(out), ctypes.byref(self.info))
        nat.check(rc, "pk_int_ranges")
        return [[int(w) for w in out[3 * i:3 * i + 3]] for i in range(len(spans))], self.info

    # -- y-space helpers (Python ints are exact)

    def y0(self) -> List[int]:
        n = self.n
        return [2 * self.rows[i][n - 1] - sum(self.rows[i]) for i in range(n)]

    def p0_y(self) -> int:
        p = 1
        for v in self.y0():
            p *= v
        return p

    def z_to_y(self, z: int, info: IntInfo) -> int:
        return z << info.even_rows

    def perm_bound(self) -> int:
        """|perm| bound: product of row absolute sums (Bregman for 0/1 rows
        would be tighter; this one holds for every integer matrix)."""
        b = 1
        for r in self.rows:
            b *= sum(abs(v) for v in r)
        return b


def int_walk_total(m, devices=None, stats=None, sparse: Optional[bool] = None) -> int:
    """Exact permanent of an integer matrix (perm_nw / perm_spa integer branch,
    kernels.py:301-306, 339-344). sparse: see IntProblem.walk."""
    prob = IntProblem(m)
    n = prob.n
    p0 = prob.p0_y()
    if n == 1:
        from .integer import finalize_int as fin
        return fin(p0, n)
    words, info = prob.walk(1, (1 << (n - 1)) - 1, devices=devices, stats=stats, sparse=sparse)
    if info.exact_terms:
        part_y = prob.z_to_y(_signed(words, 192), info)
        return finalize_int(p0 + part_y, n)
    # modular route: total_z mod 2^128 is exact once |total_z| < 2^127
    odd_rows = n - info.even_rows
    bound = prob.perm_bound() << max(odd_rows - 1, 0)
    if bound >= (1 << 127):
        raise OverflowError("integer permanent exceeds the exact range of the GPU walk")
    p0_z = p0 >> info.even_rows  # exact: every even row contributes a factor 2
    total_z = _signed([(_signed(words, 192) + p0_z) & ((1 << 128) - 1), 0], 128)
    return finalize_int(total_z << info.even_rows, n)


def int_batch_totals(ms, device: int = 0, stats=None) -> List[int]:
    """Exact permanents of many integer matrices of one order in one launch
    (pk_int_batch); matrices whose terms may reach 2^127 are walked one by
    one (int_walk_total's modular route)."""
    if not ms:
        return []
    probs = [IntProblem(m) for m in ms]
    n = probs[0].n
    a = np.ascontiguousarray(np.concatenate([p.a for p in probs]))
    out = np.zeros(3 * len(probs), dtype=np.uint64)
    infos = (IntInfo * len(probs))()
    st = stats if stats is not None else nat.RunStats()
    lib = nat.load()
    rc = lib.pk_int_batch(a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n, len(probs), device,
                          nat.u64ptr(out), ctypes.cast(infos, ctypes.c_void_p), st)
    if rc == nat.PK_ERR_OVERFLOW:
        return [int_walk_total(m, [device], sparse=False) for m in ms]
    nat.check(rc, "pk_int_batch")
    res = []
    for b, p in enumerate(probs):
        z = _signed([int(w) for w in out[3 * b:3 * b + 3]], 192)
        res.append(finalize_int(p.p0_y() + p.z_to_y(z, infos[b]), n))
    return res


EXACT_WALKER_LIMIT = 1 << 20


def int_ranges(m, spans: Sequence[Tuple[int, int]], devices=None) -> List[int]:
    """Exact y-space partials (run_range semantics) for each range."""
    prob = IntProblem(m)
    out: List[Optional[int]] = [None] * len(spans)
    small = [i for i, (s, e) in enumerate(spans) if e - s + 1 <= EXACT_WALKER_LIMIT]
    dev0 = devices[0] if devices else 0
    if small:
        words, info = prob.ranges([spans[i] for i in small], device=dev0)
        if not info.exact_terms:
            raise OverflowError("integer terms may exceed 2^127: range partials are not exact")
        for i, w in zip(small, words):
            out[i] = prob.z_to_y(_signed(w, 192), info)
    for i, (s, e) in enumerate(spans):
        if out[i] is None:
            words, info = prob.walk(s, e, devices=devices)
            if not info.exact_terms:
                raise OverflowError("integer terms may exceed 2^127: range partials are not exact")
            out[i] = prob.z_to_y(_signed(words, 192), info)
    return out
