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


def auto_log2_chunk(bit_len: int, logu: int, chunks_log2: int) -> int:
    """pk_abi.cu plan_dense's automatic chunk exponent for a range whose
    length has `bit_len` bits (a whole walk: n - 1)."""
    k = max(bit_len - chunks_log2, min(12, bit_len - 17))
    return max(k, logu + 1)


# largest order with complex register kernels (pk_launch.h kC128NMax)
C128_N_MAX = 40
