"""Accumulator policies and the double-double arithmetic of the host-side
reduction.

Policy names and codes follow permkit (precision.py:139-165 and
_loops.py:27-30): two letters, inner-product precision then partial-sum
precision -- DD plain/plain, KAHAN plain products with compensated partials,
DQ plain products with double-double partials, QQ double-double both. The
device kernels implement all four (csrc/pk_common.cuh); this module carries
the host side: the DoubleDouble value type partials travel in, the robust
double-double add used to combine them, and the error measures used by tests.
"""

from __future__ import annotations

import math
from enum import Enum
from fractions import Fraction
from typing import NamedTuple, Tuple, Union

EPS_DOUBLE = 2.0 ** -53
_SPLIT = 134217729.0  # 2^27 + 1


class AccumulatorPolicy(Enum):
    DD = "dd"
    KAHAN = "kahan"
    DQ = "dq"
    QQ = "qq"

    @classmethod
    def parse(cls, name: str) -> "AccumulatorPolicy":
        key = str(name).strip().lower()
        for p in cls:
            if p.value == key:
                return p
        raise ValueError(f"unknown policy {name!r}; expected one of dd, kahan, dq, qq")

    @property
    def code(self) -> int:
        """Integer code of the C ABI (PK_POLICY_*)."""
        return _CODES[self]

    @property
    def inner_precision(self) -> str:
        return "double-double" if self is AccumulatorPolicy.QQ else "double"

    @property
    def partial_precision(self) -> str:
        if self is AccumulatorPolicy.KAHAN:
            return "double (compensated)"
        return "double-double" if self in (AccumulatorPolicy.DQ, AccumulatorPolicy.QQ) else "double"


_CODES = {AccumulatorPolicy.DD: 0, AccumulatorPolicy.KAHAN: 1, AccumulatorPolicy.DQ: 2,
          AccumulatorPolicy.QQ: 3}


def as_policy(p: "AccumulatorPolicy | str") -> AccumulatorPolicy:
    """This package's policy, its name, or permkit's own enum member (duck
    typed on its string .value) -> AccumulatorPolicy."""
    if isinstance(p, AccumulatorPolicy):
        return p
    v = getattr(p, "value", None)
    return AccumulatorPolicy.parse(v if isinstance(v, str) else p)


class DoubleDouble(NamedTuple):
    """hi + lo, unevaluated; the payload of every real-kind partial."""

    hi: float
    lo: float

    @classmethod
    def from_float(cls, v: float) -> "DoubleDouble":
        return cls(float(v), 0.0)

    def to_float(self) -> float:
        return self.hi

    def to_fraction(self) -> Fraction:
        return Fraction(self.hi) + Fraction(self.lo)


class KahanAccumulator(NamedTuple):
    sum: float
    compensation: float

    def to_double_double(self) -> DoubleDouble:
        return DoubleDouble(*two_sum(self.sum, self.compensation))


def two_sum(a: float, b: float) -> Tuple[float, float]:
    """Knuth's error-free sum: s = fl(a + b), e = (a + b) - s exactly."""
    s = a + b
    v = s - a
    return s, (a - (s - v)) + (b - v)


def quick_two_sum(a: float, b: float) -> Tuple[float, float]:
    """Dekker's fast two-sum; requires |a| >= |b| or a == 0."""
    s = a + b
    return s, b - (s - a)


def split(a: float) -> Tuple[float, float]:
    t = _SPLIT * a
    hi = t - (t - a)
    return hi, a - hi


def two_prod(a: float, b: float) -> Tuple[float, float]:
    """Error-free product via Dekker splitting (no fma in CPython)."""
    p = a * b
    ah, al = split(a)
    bh, bl = split(b)
    return p, ((ah * bh - p) + ah * bl + al * bh) + al * bl


def dd_add(a: DoubleDouble, b: DoubleDouble) -> DoubleDouble:
    """Accurate double-double sum: both limb pairs go through two_sum. Same
    operation sequence as the device/host reducers (csrc/pk_common.cuh)."""
    hi, e = two_sum(a[0], b[0])
    lo, f = two_sum(a[1], b[1])
    e += lo
    hi, e = quick_two_sum(hi, e)
    e += f
    hi, e = quick_two_sum(hi, e)
    return DoubleDouble(hi, e)


def dd_add_double(a: DoubleDouble, b: float) -> DoubleDouble:
    s, e = two_sum(a[0], b)
    e += a[1]
    return DoubleDouble(*quick_two_sum(s, e))


def dd_mul(a: DoubleDouble, b: DoubleDouble) -> DoubleDouble:
    p, e = two_prod(a[0], b[0])
    e += a[0] * b[1] + a[1] * b[0]
    return DoubleDouble(*quick_two_sum(p, e))


def dd_mul_double(a: DoubleDouble, b: float) -> DoubleDouble:
    p, e = two_prod(a[0], b)
    e += a[1] * b
    return DoubleDouble(*quick_two_sum(p, e))


def dd_neg(a: DoubleDouble) -> DoubleDouble:
    return DoubleDouble(-a[0], -a[1])


def kahan_add(acc: KahanAccumulator, term: float) -> KahanAccumulator:
    y = term + acc.compensation
    t = acc.sum + y
    return KahanAccumulator(t, (acc.sum - t) + y)


def dd_pairwise(values) -> DoubleDouble:
    """Pairwise (binary-counter) double-double fold in index order -- the
    same tree the device reducer and the C-ABI host combiner use."""
    stack = []
    for idx, v in enumerate(values):
        cur = DoubleDouble(*v)
        t = idx
        while t & 1:
            cur = dd_add(stack.pop(), cur)
            t >>= 1
        stack.append(cur)
    if not stack:
        return DoubleDouble(0.0, 0.0)
    acc = stack.pop()
    while stack:
        acc = dd_add(stack.pop(), acc)
    return acc


class ErrorMeasure(NamedTuple):
    value: float
    absolute_fallback: bool


ExactLike = Union[int, float, complex, Fraction]


def relative_error(computed: ExactLike, exact: ExactLike) -> ErrorMeasure:
    """|computed - exact| / |exact|; rational arithmetic for real values,
    absolute error (flagged) when exact == 0."""
    if isinstance(computed, complex) or isinstance(exact, complex):
        d = abs(complex(computed) - complex(exact))
        m = abs(complex(exact))
        return ErrorMeasure(d, True) if m == 0 else ErrorMeasure(d / m, False)
    c, e = Fraction(computed), Fraction(exact)
    if e == 0:
        return ErrorMeasure(float(abs(c)), True)
    return ErrorMeasure(float(abs(c - e) / abs(e)), False)


def reference_permanent(n: int, a: ExactLike) -> ExactLike:
    """perm of the constant n x n matrix: n! a^n, exact for int/float fills."""
    if n < 1:
        raise ValueError("n must be >= 1")
    f = math.factorial(n)
    if isinstance(a, (int, complex)):
        return f * a ** n
    return f * Fraction(a) ** n
