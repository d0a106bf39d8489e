"""CPU parity oracle for the Gray-walk permanent -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline
leg may import this package, and only as the checker. The product package
(``paper_2502_16577_b200``) never imports it and has no CPU fallback.

``liboracle.so`` (built from ``permref.c`` by ``oracle/build.sh`` or
``__graft_entry__.build()``) restates permkit's chunk loops operation for
operation; see the header of ``permref.c`` for the file:line map. The helpers
below build the same per-row states as permkit's state builders
(/root/reference/pkg/src/permkit/kernels.py:75-163) from plain numpy / Python
matrices, and reduce partials like reduce_partials (parallel.py:344-387).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction
from typing import List, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

POLICY_CODE = {"dd": 0, "kahan": 1, "dq": 2, "qq": 3}


def build() -> str:
    """Compile liboracle.so next to permref.c (gcc, no fp contraction)."""
    src = os.path.join(_HERE, "permref.c")
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-o", _LIB_PATH, src, "-lpthread"]
    subprocess.check_call(cmd)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        lp = ctypes.POINTER(ctypes.c_int64)
        up = ctypes.POINTER(ctypes.c_uint64)
        u64 = ctypes.c_uint64
        i = ctypes.c_int
        L.oracle_dense_f64_state.argtypes = [dp, i, dp, dp]
        L.oracle_dense_f64_range.argtypes = [dp, dp, i, u64, u64, i, dp]
        L.oracle_dense_f64_p0.argtypes = [dp, i, i, dp]
        L.oracle_sparse_f64_range.argtypes = [lp, lp, dp, dp, i, u64, u64, i, dp]
        L.oracle_dense_c128_range.argtypes = [dp, dp, i, u64, u64, dp]
        L.oracle_sparse_c128_range.argtypes = [lp, lp, dp, dp, i, u64, u64, dp]
        L.oracle_dense_int_range.argtypes = [lp, lp, i, u64, u64, lp]
        L.oracle_sparse_int_range.argtypes = [lp, lp, lp, lp, i, u64, u64, lp]
        L.oracle_dense_f64_ranges_mt.argtypes = [dp, dp, i, up, up, i, i, i, dp]
        for f in ("oracle_dense_f64_range", "oracle_sparse_f64_range", "oracle_dense_c128_range",
                  "oracle_sparse_c128_range", "oracle_dense_int_range", "oracle_sparse_int_range",
                  "oracle_dense_f64_ranges_mt"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _lp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _up(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def _check(rc, what):
    if rc == -2:
        raise OverflowError(f"{what}: exceeds the oracle's int128 range")
    if rc != 0:
        raise ValueError(f"{what}: bad arguments (rc={rc})")


def total_iterates(n: int) -> int:
    return (1 << (n - 1)) - 1


def sign_factor(n: int) -> int:
    return 4 * (n % 2) - 2


# ---------------------------------------------------------------------------
# states


def dense_f64_state(a: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.shape[0]
    cols = np.zeros(max(n - 1, 1) * n, dtype=np.float64)
    x0 = np.zeros(n, dtype=np.float64)
    lib().oracle_dense_f64_state(_dp(a), n, _dp(cols), _dp(x0))
    return cols, x0


def _row_sums_sparse(n, triplets):
    """Left-to-right sums of the nonzeros of each row, ascending column
    (matrix.py:344-355); an empty row sums to zero."""
    rows: List[list] = [[] for _ in range(n)]
    for (i, j, v) in sorted(triplets, key=lambda t: (t[0], t[1])):
        rows[i].append(v)
    out = []
    for r in rows:
        if not r:
            out.append(0)
            continue
        acc = r[0]
        for v in r[1:]:
            acc = acc + v
        out.append(acc)
    return out


def ccs_from_triplets(n, triplets):
    """CCS arrays, rows ascending within each column (matrix.py:293-300)."""
    trips = sorted(((i, j, v) for (i, j, v) in triplets if v != 0), key=lambda t: (t[1], t[0]))
    cptrs = np.zeros(n + 1, dtype=np.int64)
    for (_, j, _) in trips:
        cptrs[j + 1] += 1
    cptrs = np.cumsum(cptrs).astype(np.int64)
    rids = np.array([i for (i, _, _) in trips], dtype=np.int64)
    vals = [v for (_, _, v) in trips]
    return cptrs, rids, vals


def sparse_x0(n, triplets, zero):
    """x0 of sparse_float_state / sparse_complex_state (kernels.py:113-143)."""
    x0 = [zero] * n
    for (i, j, v) in triplets:
        if j == n - 1 and v != 0:
            x0[i] = v
    sums = _row_sums_sparse(n, [t for t in triplets if t[2] != 0])
    return [x0[i] - sums[i] / 2.0 for i in range(n)]


# ---------------------------------------------------------------------------
# range partials, run_range semantics (parallel.py:232-289)


def dense_f64_range(a: np.ndarray, start: int, end: int, policy: str) -> Tuple[float, float]:
    cols, x0 = dense_f64_state(a)
    out = np.zeros(2)
    _check(lib().oracle_dense_f64_range(_dp(cols), _dp(x0), a.shape[0], start, end,
                                        POLICY_CODE[policy], _dp(out)), "dense_f64_range")
    return float(out[0]), float(out[1])


def dense_f64_p0(a: np.ndarray, policy: str) -> Tuple[float, float]:
    cols, x0 = dense_f64_state(a)
    out = np.zeros(2)
    lib().oracle_dense_f64_p0(_dp(x0), a.shape[0], POLICY_CODE[policy], _dp(out))
    return float(out[0]), float(out[1])


def sparse_f64_range(n, triplets, start, end, policy):
    cptrs, rids, vals = ccs_from_triplets(n, triplets)
    v = np.array(vals, dtype=np.float64)
    x0 = np.array(sparse_x0(n, triplets, 0.0), dtype=np.float64)
    out = np.zeros(2)
    _check(lib().oracle_sparse_f64_range(_lp(cptrs), _lp(rids), _dp(v), _dp(x0), n, start, end,
                                         POLICY_CODE[policy], _dp(out)), "sparse_f64_range")
    return float(out[0]), float(out[1])


def dense_c128_state(a: np.ndarray):
    a = np.asarray(a, dtype=np.complex128)
    n = a.shape[0]
    cols = np.ascontiguousarray(a[:, : n - 1].T) if n > 1 else np.zeros((1, 1), np.complex128)
    x0 = np.empty(n, dtype=np.complex128)
    for i in range(n):
        acc = complex(a[i, 0])
        for j in range(1, n):
            acc = acc + complex(a[i, j])
        x0[i] = complex(a[i, n - 1]) - acc / 2.0
    return cols, x0


def dense_c128_range(a, start, end):
    cols, x0 = dense_c128_state(a)
    c = np.ascontiguousarray(cols).view(np.float64)
    x = np.ascontiguousarray(x0).view(np.float64)
    out = np.zeros(2)
    _check(lib().oracle_dense_c128_range(_dp(c), _dp(x), a.shape[0], start, end, _dp(out)),
           "dense_c128_range")
    return complex(out[0], out[1])


def sparse_c128_range(n, triplets, start, end):
    cptrs, rids, vals = ccs_from_triplets(n, triplets)
    v = np.array(vals, dtype=np.complex128).view(np.float64)
    x0 = np.array(sparse_x0(n, triplets, 0j), dtype=np.complex128).view(np.float64)
    out = np.zeros(2)
    _check(lib().oracle_sparse_c128_range(_lp(cptrs), _lp(rids), _dp(v), _dp(x0), n, start, end,
                                          _dp(out)), "sparse_c128_range")
    return complex(out[0], out[1])


def _i128(words) -> int:
    lo = int(words[0]) & ((1 << 64) - 1)
    hi = int(words[1])
    return (hi << 64) | lo


def dense_int_state(rows):
    n = len(rows)
    cols2 = np.zeros(max(n - 1, 1) * n, dtype=np.int64)
    for j in range(n - 1):
        for i in range(n):
            cols2[j * n + i] = 2 * int(rows[i][j])
    y0 = np.array([2 * int(rows[i][n - 1]) - sum(int(v) for v in rows[i]) for i in range(n)],
                  dtype=np.int64)
    return cols2, y0


def dense_int_range(rows, start, end) -> int:
    cols2, y0 = dense_int_state(rows)
    out = np.zeros(2, dtype=np.int64)
    _check(lib().oracle_dense_int_range(_lp(cols2), _lp(y0), len(rows), start, end, _lp(out)),
           "dense_int_range")
    return _i128(out)


def sparse_int_range(n, triplets, start, end) -> int:
    cptrs, rids, vals = ccs_from_triplets(n, triplets)
    vals2 = np.array([2 * int(v) for v in vals], dtype=np.int64)
    # the last column's entries are not doubled-and-toggled; they seed y0
    y0 = [0] * n
    for (i, j, v) in triplets:
        if j == n - 1 and v != 0:
            y0[i] = 2 * int(v)
    sums = _row_sums_sparse(n, [t for t in triplets if t[2] != 0])
    y0 = np.array([y0[i] - int(sums[i]) for i in range(n)], dtype=np.int64)
    out = np.zeros(2, dtype=np.int64)
    _check(lib().oracle_sparse_int_range(_lp(cptrs), _lp(rids), _lp(vals2), _lp(y0), n, start,
                                         end, _lp(out)), "sparse_int_range")
    return _i128(out)


# ---------------------------------------------------------------------------
# reduction (parallel.py:344-387, precision.py:52-96) and whole permanents


def two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def quick_two_sum(a, b):
    s = a + b
    return s, b - (s - a)


def dd_add(a, b):
    s1, s2 = two_sum(a[0], b[0])
    t1, t2 = two_sum(a[1], b[1])
    s2 += t1
    s1, s2 = quick_two_sum(s1, s2)
    s2 += t2
    s1, s2 = quick_two_sum(s1, s2)
    return (s1, s2)


def aligned_plan(n: int, tau: int) -> List[Tuple[int, int]]:
    """plan_chunks(n, tau, aligned=True) ranges incl. residual (parallel.py:95-122)."""
    total = total_iterates(n)
    if total == 0:
        return []
    tau = min(tau, total)
    size = -(-total // tau)
    size = 1 << (size.bit_length() - 1)
    out = []
    for t in range(tau):
        s = 1 + t * size
        if s > total:
            break
        out.append((s, min(total, s + size - 1)))
    if out[-1][1] < total:
        out.append((out[-1][1] + 1, total))
    return out


def dense_f64_permanent(a: np.ndarray, policy: str = "kahan", tau: int = 64, threads: int = 0) -> float:
    """permanent_chunked(m, policy, tau) restated: threaded ranges, dd reduce."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.shape[0]
    cols, x0 = dense_f64_state(a)
    p0 = dense_f64_p0(a, policy)
    plan = aligned_plan(n, tau)
    if not plan:
        return p0[0] * sign_factor(n)
    starts = np.array([s for s, _ in plan], dtype=np.uint64)
    ends = np.array([e for _, e in plan], dtype=np.uint64)
    out = np.zeros(2 * len(plan))
    threads = threads or (os.cpu_count() or 1)
    _check(lib().oracle_dense_f64_ranges_mt(_dp(cols), _dp(x0), n, _up(starts), _up(ends),
                                            len(plan), POLICY_CODE[policy], threads, _dp(out)),
           "dense_f64_ranges_mt")
    acc = (p0[0], p0[1])
    for r in range(len(plan)):
        acc = dd_add(acc, (float(out[2 * r]), float(out[2 * r + 1])))
    return acc[0] * sign_factor(n)


def dense_f64_ranges_mt(a: np.ndarray, ranges: Sequence[Tuple[int, int]], policy: str,
                        threads: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    cols, x0 = dense_f64_state(a)
    starts = np.array([s for s, _ in ranges], dtype=np.uint64)
    ends = np.array([e for _, e in ranges], dtype=np.uint64)
    out = np.zeros(2 * len(ranges))
    _check(lib().oracle_dense_f64_ranges_mt(_dp(cols), _dp(x0), a.shape[0], _up(starts), _up(ends),
                                            len(ranges), POLICY_CODE[policy], threads, _dp(out)),
           "dense_f64_ranges_mt")
    return out.reshape(-1, 2)


def exact_uniform(n: int, a: float) -> Fraction:
    """n! * a^n exactly (precision.py:200-213)."""
    import math
    return math.factorial(n) * Fraction(a) ** n
