// Instantiates the precise dense real walk (pk_precise.cuh) for every order
// with register kernels, and its run-time dispatch.
#include "pk_launch.h"
#include "pk_precise.cuh"

namespace pk {

template <int N>
static int launch_precise_n(const PreciseLaunch& a) {
  auto kern = dense_f64_precise<N>;
  static std::atomic<int> slots[kMaxDevices];  // per device ordinal
  int occ = 1;
  if (int rc = prep_kernel(kern, kPreciseBlock, 0, slots, &occ)) return rc;
  PreciseParams p;
  p.fix = a.fix;
  p.group_part = a.group_part;
  p.chunk_part = a.chunk_part;
  p.out = a.out;
  p.counter = a.counter;
  p.chunk_lo = a.chunk_lo;
  p.num_groups = a.num_groups;
  p.g_end = a.g_end;
  p.k = a.k;
  const uint64_t blocks_needed = (a.num_groups * 32 + kPreciseBlock - 1) / kPreciseBlock;
  uint64_t grid = (uint64_t)a.sms * (uint64_t)occ;
  if (blocks_needed < grid) grid = blocks_needed;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kPreciseBlock, 0, a.stream>>>(p);
  return (int)cudaGetLastError();
}

template <int N>
static int launch_c128_precise_n(const PreciseLaunch& a) {
  auto kern = dense_c128_precise<N>;
  constexpr size_t smem = 2 * sizeof(long long) * fix_words<N>();
  static std::atomic<int> slots[kMaxDevices];  // per device ordinal
  int occ = 1;
  if (int rc = prep_kernel(kern, kPreciseBlock, smem, slots, &occ)) return rc;
  PreciseParams p;
  p.fix = a.fix;
  p.group_part = a.group_part;
  p.chunk_part = a.chunk_part;
  p.out = a.out;
  p.counter = a.counter;
  p.chunk_lo = a.chunk_lo;
  p.num_groups = a.num_groups;
  p.g_end = a.g_end;
  p.k = a.k;
  const uint64_t blocks_needed = (a.num_groups * 32 + kPreciseBlock - 1) / kPreciseBlock;
  uint64_t grid = (uint64_t)a.sms * (uint64_t)occ;
  if (blocks_needed < grid) grid = blocks_needed;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kPreciseBlock, smem, a.stream>>>(p);
  return (int)cudaGetLastError();
}

int launch_dense_c128_precise(int n, const PreciseLaunch& a) {
  switch (n) {
#define PK_P(N) \
  case N:       \
    return launch_c128_precise_n<N>(a);
    PK_P(11) PK_P(12) PK_P(13) PK_P(14) PK_P(15) PK_P(16) PK_P(17) PK_P(18) PK_P(19)
    PK_P(20) PK_P(21) PK_P(22) PK_P(23) PK_P(24) PK_P(25) PK_P(26) PK_P(27) PK_P(28)
    PK_P(29) PK_P(30) PK_P(31) PK_P(32) PK_P(33) PK_P(34) PK_P(35) PK_P(36) PK_P(37)
    PK_P(38) PK_P(39) PK_P(40) PK_P(41) PK_P(42) PK_P(43) PK_P(44) PK_P(45) PK_P(46)
    PK_P(47) PK_P(48) PK_P(49) PK_P(50) PK_P(51) PK_P(52) PK_P(53) PK_P(54) PK_P(55)
    PK_P(56) PK_P(57) PK_P(58) PK_P(59) PK_P(60) PK_P(61) PK_P(62) PK_P(63)
#undef PK_P
    default:
      return (int)cudaErrorInvalidValue;
  }
}

int launch_dense_f64_precise(int n, const PreciseLaunch& a) {
  switch (n) {
#define PK_P(N) \
  case N:       \
    return launch_precise_n<N>(a);
    PK_P(11) PK_P(12) PK_P(13) PK_P(14) PK_P(15) PK_P(16) PK_P(17) PK_P(18) PK_P(19)
    PK_P(20) PK_P(21) PK_P(22) PK_P(23) PK_P(24) PK_P(25) PK_P(26) PK_P(27) PK_P(28)
    PK_P(29) PK_P(30) PK_P(31) PK_P(32) PK_P(33) PK_P(34) PK_P(35) PK_P(36) PK_P(37)
    PK_P(38) PK_P(39) PK_P(40) PK_P(41) PK_P(42) PK_P(43) PK_P(44) PK_P(45) PK_P(46)
    PK_P(47) PK_P(48) PK_P(49) PK_P(50) PK_P(51) PK_P(52) PK_P(53) PK_P(54) PK_P(55)
    PK_P(56) PK_P(57) PK_P(58) PK_P(59) PK_P(60) PK_P(61) PK_P(62) PK_P(63)
#undef PK_P
    default:
      return (int)cudaErrorInvalidValue;
  }
}

}  // namespace pk
