// Host-side launcher template for the lane-pair complex kernel (K3p).
#pragma once
#include <cstring>

#include "pk_c128_pair.cuh"
#include "pk_launch.h"

namespace pk {

template <int N, class C>
static int launch_c128_pair_cfg(const C128Launch& a) {
  auto kern = dense_c128_pair<N, C>;
  constexpr size_t smem = pair_smem_bytes<N>();
  static std::atomic<int> slots[kMaxDevices];  // per device ordinal
  int occ = 1;
  if (int rc = prep_kernel(kern, C::BLOCK, smem, slots, &occ)) return rc;
  C128PairParams<N> p;
  std::memcpy(p.x0, a.x0, sizeof(double) * 2 * N);
  p.cols = a.d_cols;
  p.group_part = a.group_part;
  p.chunk_part = a.chunk_part;
  p.out = a.out;
  p.counter = a.counter;
  p.chunk_lo = a.chunk_lo;
  p.num_groups = a.num_groups;
  p.g_end = a.g_end;
  p.k = a.k;
  // one warp per group of 32 chunks
  const uint64_t blocks_needed = (a.num_groups * 32 + C::BLOCK - 1) / C::BLOCK;
  uint64_t grid = (uint64_t)a.sms * (uint64_t)occ;
  if (blocks_needed < grid) grid = blocks_needed;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, C::BLOCK, smem, a.stream>>>(p);
  return (int)cudaGetLastError();
}

template <int N>
int launch_c128_pair(const C128Launch& a) {
  static_assert(N >= kC128NMin && N <= kDenseNMax, "order out of range");
  constexpr int LOGU = c128_pair_logu(N);
  constexpr int BLK = c128_pair_block(N), MB = c128_pair_minb(N);
  if (a.exact) return launch_c128_pair_cfg<N, C128Cfg<LOGU, true, MB, false, BLK>>(a);
  // row-major bodies (C128Cfg::RM, +1..4 %, profiles/r02_c128_variants_rm.txt);
  // PK_C128_VARIANT=2 selects the step-major body, as for K3
  return a.variant == 2
             ? launch_c128_pair_cfg<N, C128Cfg<LOGU, false, MB, false, BLK>>(a)
             : launch_c128_pair_cfg<N, C128Cfg<c128_pair_fast_logu(N), false, MB, false, BLK,
                                               false, true>>(a);
}

template <int N, class C>
static int launch_c128_pair_batch_cfg(const C128BatchLaunch& a) {
  auto kern = dense_c128_pair_batch<N, C>;
  constexpr size_t smem = pair_smem_bytes<N>();
  static std::atomic<int> slots[kMaxDevices];  // per device ordinal
  int occ = 1;
  if (int rc = prep_kernel(kern, C::BLOCK, smem, slots, &occ)) return rc;
  C128BatchParams<N> p;
  p.cols = a.d_cols;
  p.x0 = a.d_x0;
  p.group_part = a.group_part;
  p.out = a.out;
  p.batch = a.batch;
  p.k = a.k;
  uint64_t grid = (uint64_t)a.sms * (uint64_t)occ;
  if ((uint64_t)a.batch < grid) grid = a.batch;
  kern<<<(unsigned)grid, C::BLOCK, smem, a.stream>>>(p);
  return (int)cudaGetLastError();
}

template <int N>
int launch_c128_pair_batch(const C128BatchLaunch& a) {
  constexpr int LOGU = c128_pair_logu(N);
  constexpr int BLK = c128_pair_block(N), MB = c128_pair_minb(N);
  if (a.exact) return launch_c128_pair_batch_cfg<N, C128Cfg<LOGU, true, MB, false, BLK>>(a);
  return launch_c128_pair_batch_cfg<N, C128Cfg<c128_pair_fast_logu(N), false, MB, false, BLK,
                                                false, true>>(a);
}

}  // namespace pk

#define PK_INSTANTIATE_C128_PAIR(N)                                    \
  template int pk::launch_c128_pair<N>(const pk::C128Launch&); \
  template int pk::launch_c128_pair_batch<N>(const pk::C128BatchLaunch&);
