"""Mirror of the compile-time tuning in csrc/pk_launch.h (kept in sync by
tests/test_host.py::test_csrc_params_mirror)."""


def dense_logu(n: int) -> int:
    return 4 if n <= 50 else 3


def dense_minb(n: int) -> int:
    return 3 if n <= 36 else 2


def batch_log2_chunk(n: int, logu: int) -> int:
    return max(n - 1 - 10, logu + 1)


def c128_logu(n: int) -> int:
    return 2 if n <= 32 else 1


def c128_fast_logu(n: int) -> int:
    """K3's fast (row-major) body length: 8 steps at every order."""
    return 3


def auto_log2_chunk(bit_len: int, logu: int, chunks_log2: int) -> int:
    """pk_abi.cu plan_dense's automatic chunk exponent for a range whose
    length has `bit_len` bits (a whole walk: n - 1)."""
    k = max(bit_len - chunks_log2, min(12, bit_len - 17))
    return max(k, logu + 1)


# largest order of the one-thread-per-chunk complex kernel K3 (pk_launch.h
# kC128NMax); orders above it run the lane-pair kernel K3p up to 63
C128_N_MAX = 40
C128_PAIR_N_MAX = 63


def c128_pair_logu(n: int) -> int:
    """K3p exact-mode body length (log2)."""
    return 2 if n <= 48 else 1


def c128_pair_fast_logu(n: int) -> int:
    return 4 if n <= 42 else 3


def c128_register_logu(n: int) -> int:
    """Body length exponent of the fast complex register kernel at order n."""
    return c128_fast_logu(n) if n <= C128_N_MAX else c128_pair_fast_logu(n)
