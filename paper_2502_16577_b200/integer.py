"""Exact integer walk (placeholder until the int128 kernels land)."""

from __future__ import annotations


def finalize_int(total_y: int, n: int) -> int:
    """Global sign, then divide the y-space total by 2^(n-1) (kernels.py:290-294)."""
    signed = total_y if n % 2 else -total_y
    q, r = divmod(signed, 1 << (n - 1))
    if r:
        raise ArithmeticError("integer walk produced a non-divisible total")
    return q


def int_walk_total(m, devices=None):
    raise NotImplementedError("integer kernels not built yet")


def int_ranges(m, spans, devices=None):
    raise NotImplementedError("integer kernels not built yet")
