"""Many permanents per launch: the caller side of SURVEY.md §8f-2.

permkit evaluates decomposition leaves one by one (preprocess.py:495-504),
and boson-sampling workloads need the permanents of many n ~ 20-30
submatrices. ``permanent_batch`` groups the matrices by kind and order and
walks every real group in ONE launch of ``pk_dense_f64_batch`` and every
complex group of order <= 63 in ONE launch of ``pk_dense_c128_batch`` and
every integer group in ONE launch of ``pk_int_batch`` (one block per matrix
at a time, each matrix's aligned chunks reduced exactly like a single
launch). Complex orders above 40 take one device call per matrix (still on
the GPU).
"""

from __future__ import annotations

from collections import defaultdict
from typing import List, Optional, Sequence

import numpy as np

from . import _native as nat
from .kernels import (DenseF64Problem, _sign_factor, perm_nw, perm_spa, policy_product,
                      sparse_float_state, total_iterates)
from .matrix import (KIND_COMPLEX, KIND_INT, KIND_REAL, DenseMatrix, SparsePair, coerce_matrix,
                     sparse_to_dense)
from .precision import AccumulatorPolicy, DoubleDouble, as_policy, dd_add


def dense_states(A: np.ndarray):
    """Vectorised dense_float_state / dense_complex_state of a stack of
    matrices A[b, n, n] (kernels.py:75-101): columns cols[b, j, i] = a_ij for
    j < n-1 and the seed x0 = a[:, n-1] - rowsum / 2 with the row sums taken
    left to right (np.add.accumulate is sequential: the reference's rounding
    order, matrix.py:333-355)."""
    b, n, _ = A.shape
    sums = np.add.accumulate(A, axis=2)[:, :, n - 1]
    x0 = np.ascontiguousarray(A[:, :, n - 1] - sums / 2.0)
    cols = np.ascontiguousarray(np.transpose(A[:, :, : n - 1], (0, 2, 1)))
    return cols, x0


def _stack(ms: Sequence, dtype) -> np.ndarray:
    n = ms[0].n
    rows = []
    for m in ms:
        d = sparse_to_dense(m) if isinstance(m, SparsePair) else m
        rows.append(np.array(d.data, dtype=dtype).reshape(n, n))
    return np.stack(rows)


def real_batch_arrays(A: np.ndarray, policy: AccumulatorPolicy, device: int = 0,
                      exact: bool = False, stats: Optional[nat.RunStats] = None) -> List[float]:
    """Permanents of the real matrices A[b, n, n] in one pk_dense_f64_batch launch."""
    b, n, _ = A.shape
    cols, x0 = dense_states(np.asarray(A, dtype=np.float64))
    cflat = np.ascontiguousarray(cols.reshape(-1)) if n > 1 else np.zeros(1)
    xflat = np.ascontiguousarray(x0.reshape(-1))
    out = np.zeros(2 * b)
    st = stats if stats is not None else nat.RunStats()
    rc = nat.load().pk_dense_f64_batch(nat.dptr(cflat), nat.dptr(xflat), n, b, policy.code,
                                       nat.PK_FLAG_EXACT if exact else 0, device, nat.dptr(out), st)
    nat.check(rc, "pk_dense_f64_batch")
    res = []
    from .kernels import fast_p0
    for i in range(b):
        if exact:
            p0 = policy_product(x0[i], policy)
            acc = p0 if isinstance(p0, DoubleDouble) else DoubleDouble(float(p0), 0.0)
        else:  # the rounded seed the device walks, exact product (kernels.fast_p0)
            acc = fast_p0(cols[i].reshape(-1) if n > 1 else np.zeros(1), x0[i], n, policy)
        if n > 1:
            acc = dd_add(acc, DoubleDouble(float(out[2 * i]), float(out[2 * i + 1])))
        res.append(acc.hi * _sign_factor(n))
    return res


def complex_batch_arrays(A: np.ndarray, device: int = 0, exact: bool = False,
                         stats: Optional[nat.RunStats] = None) -> List[complex]:
    """Permanents of the complex matrices A[b, n, n] (n <= 63) in one
    pk_dense_c128_batch launch."""
    b, n, _ = A.shape
    cols, x0 = dense_states(np.asarray(A, dtype=np.complex128))
    cflat = np.ascontiguousarray(cols.reshape(-1).view(np.float64)) if n > 1 else np.zeros(2)
    xflat = np.ascontiguousarray(x0.reshape(-1).view(np.float64))
    out = np.zeros(4 * b)
    st = stats if stats is not None else nat.RunStats()
    rc = nat.load().pk_dense_c128_batch(nat.dptr(cflat), nat.dptr(xflat), n, b,
                                        nat.PK_FLAG_EXACT if exact else 0, device, nat.dptr(out),
                                        st)
    nat.check(rc, "pk_dense_c128_batch")
    res = []
    sign = _sign_factor(n)
    from .complex_walk import _exact_p0
    from .kernels import quantized_seed
    for i in range(b):
        if exact:
            p = complex(1.0)
            for v in x0[i]:
                p = p * complex(v)
            re, im = DoubleDouble(p.real, 0.0), DoubleDouble(p.imag, 0.0)
        elif n < 11:  # the reference loop's walk and product
            p = complex(1.0)
            for v in x0[i]:
                p = p * complex(v)
            re, im = DoubleDouble(p.real, 0.0), DoubleDouble(p.imag, 0.0)
        else:  # the rounded seed the device walks (complex_walk.fast_p0)
            xs = quantized_seed(np.ascontiguousarray(cols[i]).reshape(-1).view(np.float64),
                                np.ascontiguousarray(x0[i]).view(np.float64), n,
                                comps=2).view(np.complex128)
            re, im = _exact_p0(xs)
        if n > 1:
            re = dd_add(re, DoubleDouble(float(out[4 * i]), float(out[4 * i + 1])))
            im = dd_add(im, DoubleDouble(float(out[4 * i + 2]), float(out[4 * i + 3])))
        res.append(complex(re.hi * sign, im.hi * sign))
    return res


def _real_batch(ms: Sequence, policy: AccumulatorPolicy, device: int, exact: bool,
                stats: Optional[nat.RunStats]) -> List[float]:
    return real_batch_arrays(_stack(ms, np.float64), policy, device, exact, stats)


def _complex_batch(ms: Sequence, device: int, exact: bool,
                   stats: Optional[nat.RunStats]) -> List[complex]:
    return complex_batch_arrays(_stack(ms, np.complex128), device, exact, stats)


def permanent_batch(matrices, policy="dd", *, device: int = 0, exact: bool = False,
                    stats: Optional[nat.RunStats] = None) -> list:
    """Permanents of many matrices; results in input order."""
    policy = as_policy(policy)
    ms = [coerce_matrix(m) for m in matrices]
    out: list = [None] * len(ms)
    groups = defaultdict(list)
    for i, m in enumerate(ms):
        groups[(m.kind, m.n)].append(i)
    for (kind, n), idx in groups.items():
        if kind == KIND_REAL:
            vals = _real_batch([ms[i] for i in idx], policy, device, exact, stats)
            for i, v in zip(idx, vals):
                out[i] = v
        elif kind == KIND_INT:
            from .integer import int_batch_totals
            ds = [sparse_to_dense(ms[i]) if isinstance(ms[i], SparsePair) else ms[i] for i in idx]
            for i, v in zip(idx, int_batch_totals(ds, device, stats)):
                out[i] = v
        elif kind == KIND_COMPLEX and n <= 63:
            if policy is not AccumulatorPolicy.DD:
                from .errors import PolicyError
                raise PolicyError("complex matrices support the plain-double policy only")
            vals = _complex_batch([ms[i] for i in idx], device, exact, stats)
            for i, v in zip(idx, vals):
                out[i] = v
        else:
            for i in idx:
                m = ms[i]
                out[i] = (perm_spa(m, policy, devices=[device]) if isinstance(m, SparsePair)
                          else perm_nw(m, policy, devices=[device]))
    return out
