"""Gray-code bookkeeping of the walk (permkit graycode.py:21-73).

Iterate g >= 1 turns Gray code gray(g-1) into gray(g) = g ^ (g >> 1) by
flipping bit j = ctz(g); the bit is switched on iff bit j+1 of g is 0. The
device kernels inline exactly this arithmetic (csrc/pk_common.cuh).
"""

from __future__ import annotations

from typing import List, NamedTuple, Set


class GrayStep(NamedTuple):
    j: int
    s: int


def gray_of(g: int) -> int:
    return g ^ (g >> 1)


def changed_bit(g: int) -> GrayStep:
    if g <= 0:
        raise ValueError("changed_bit is defined for g >= 1")
    j = (g & -g).bit_length() - 1
    return GrayStep(j, -1 if (g >> (j + 1)) & 1 else 1)


def subset_columns(g: int, n: int) -> Set[int]:
    if n < 1:
        raise ValueError("n must be >= 1")
    if not 0 <= g < (1 << (n - 1)):
        raise ValueError(f"iterate {g} out of range for n={n}")
    code = gray_of(g)
    return {j for j in range(n - 1) if (code >> j) & 1}


def cbl_sequence(k: int) -> List[int]:
    """Changed-bit locations of the k-bit walk: seq(k) = seq(k-1), k-1, seq(k-1)."""
    if not 1 <= k <= 20:
        raise ValueError("cbl_sequence supports 1 <= k <= 20")
    return [(g & -g).bit_length() - 1 for g in range(1, 1 << k)]
