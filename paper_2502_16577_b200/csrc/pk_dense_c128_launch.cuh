// Host-side launcher template for the N-specialised dense complex kernel.
#pragma once
#include <cstring>

#include "pk_dense_c128.cuh"
#include "pk_launch.h"

namespace pk {

template <int N, class C>
static int launch_c128_cfg(const C128Launch& a, const DenseC128Params<N>& p) {
  auto kern = dense_c128_chunks<N, C>;
  constexpr size_t smem = c128_smem_bytes<N>();
  static std::atomic<int> slots[kMaxDevices];  // per device ordinal
  int occ = 1;
  if (int rc = prep_kernel(kern, C::BLOCK, smem, slots, &occ)) return rc;
  const uint64_t blocks_needed = (a.num_groups * 32 + C::BLOCK - 1) / C::BLOCK;
  uint64_t grid = (uint64_t)a.sms * (uint64_t)occ;
  if (blocks_needed < grid) grid = blocks_needed;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, C::BLOCK, smem, a.stream>>>(p);
  return (int)cudaGetLastError();
}

template <int N>
int launch_dense_c128(const C128Launch& a) {
  static_assert(N >= kC128NMin && N <= kC128NMax, "order out of range");
  constexpr int LOGU = c128_logu(N);
  constexpr int MB = c128_minb(N);
  DenseC128Params<N> p;
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
  // fast mode: one 256-thread block per SM to n = 32 (+5 %,
  // profiles/r01_c128_sweep5_blocks.txt); the tail tree has a fixed leaf
  // count (pk_reduce.cuh kTreeLeaves), so results do not depend on it.
  // a.variant (pk_abi.cu c128_variant): 4 row-major bodies of 2^(LOGU+1)
  // steps (default), 2 the round-1 step-major bodies of 2^LOGU (A/B runs;
  // two product chains, the fused last multiply and other body lengths were
  // measured slower, profiles/r02_c128_variants*.txt)
  constexpr int FB = N <= 32 ? 256 : kC128Block;
  constexpr int FM = N <= 32 ? 1 : MB;
  if (a.exact) return launch_c128_cfg<N, C128Cfg<LOGU, true, MB>>(a, p);
  if (a.variant == 2) return launch_c128_cfg<N, C128Cfg<LOGU, false, FM, false, FB>>(a, p);
  return launch_c128_cfg<N, C128Cfg<c128_fast_logu(N), false, FM, false, FB, false, true>>(a, p);
}

template <int N, class C>
static int launch_c128_batch_cfg(const C128BatchLaunch& a) {
  auto kern = dense_c128_batch<N, C>;
  constexpr size_t smem = c128_smem_bytes<N>() + sizeof(double) * 2 * N;
  static std::atomic<int> slots[kMaxDevices];  // per device ordinal
  int occ = 1;
  if (int rc = prep_kernel(kern, kC128Block, smem, slots, &occ)) return rc;
  C128BatchParams<N> p;
  p.cols = a.d_cols;
  p.x0 = a.d_x0;
  p.group_part = a.group_part;
  p.out = a.out;
  p.batch = a.batch;
  p.k = a.k;
  uint64_t grid = (uint64_t)a.sms * (uint64_t)occ;
  if ((uint64_t)a.batch < grid) grid = a.batch;
  kern<<<(unsigned)grid, kC128Block, smem, a.stream>>>(p);
  return (int)cudaGetLastError();
}

template <int N>
int launch_dense_c128_batch(const C128BatchLaunch& a) {
  constexpr int LOGU = c128_logu(N);
  constexpr int MB = c128_minb(N);
  // fast: the single launch's default body (row-major, 2^(LOGU+1) steps),
  // so a batch entry and a single walk of the same matrix agree bit for bit
  return a.exact ? launch_c128_batch_cfg<N, C128Cfg<LOGU, true, MB>>(a)
                 : launch_c128_batch_cfg<N, C128Cfg<c128_fast_logu(N), false, MB, false,
                                                    kC128Block, false, true>>(a);
}

}  // namespace pk

#define PK_INSTANTIATE_DENSE_C128(N)                                  \
  template int pk::launch_dense_c128<N>(const pk::C128Launch&); \
  template int pk::launch_dense_c128_batch<N>(const pk::C128BatchLaunch&);
