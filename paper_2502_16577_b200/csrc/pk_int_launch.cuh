// Host-side launcher template for the N-specialised exact integer kernel.
#pragma once
#include <cstring>

#include "pk_int.cuh"
#include "pk_launch.h"

namespace pk {

template <int N, class C>
static int launch_int_cfg(const IntLaunch& a, const IntParams<N>& p) {
  auto kern = int_chunks<N, C>;
  static std::atomic<int> slots[kMaxDevices];  // per device ordinal
  int occ = 1;
  if (int rc = prep_kernel(kern, kIntBlock, 0, slots, &occ)) return rc;
  const uint64_t blocks_needed = (a.num_groups * 32 + kIntBlock - 1) / kIntBlock;
  uint64_t grid = (uint64_t)a.sms * (uint64_t)occ;
  if (blocks_needed < grid) grid = blocks_needed;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kIntBlock, 0, a.stream>>>(p);
  return (int)cudaGetLastError();
}

template <int N>
int launch_int(const IntLaunch& a) {
  static_assert(N >= kIntNMin && N <= kIntNMax, "order out of range");
  constexpr int L = int_logu(N);
  constexpr int MB = int_minb(N);
  IntParams<N> p;
  std::memcpy(p.z0, a.z0, sizeof(int) * N);
  p.cols = a.d_cols;
  p.group_part = (i192*)a.group_part;
  p.chunk_part = (i192*)a.chunk_part;
  p.out = (i192*)a.out;
  p.counter = a.counter;
  p.chunk_lo = a.chunk_lo;
  p.num_groups = a.num_groups;
  p.g_end = a.g_end;
  p.k = a.k;
  switch (a.zb) {
    case 5: return launch_int_cfg<N, IntCfg<5, L, MB>>(a, p);
    case 7: return launch_int_cfg<N, IntCfg<7, L, MB>>(a, p);
    case 15: return launch_int_cfg<N, IntCfg<15, L, MB>>(a, p);
    case 31: return launch_int_cfg<N, IntCfg<31, L, MB>>(a, p);
    default: return (int)cudaErrorInvalidValue;
  }
}

template <int N, class C>
static int launch_int_batch_cfg(const IntBatchLaunch& a) {
  auto kern = int_batch<N, C>;
  static std::atomic<int> slots[kMaxDevices];  // per device ordinal
  int occ = 1;
  if (int rc = prep_kernel(kern, kIntBlock, 0, slots, &occ)) return rc;
  IntBatchParams<N> p;
  p.cols = a.d_cols;
  p.z0 = a.d_z0;
  p.group_part = (i192*)a.group_part;
  p.out = (i192*)a.out;
  p.batch = a.batch;
  p.k = a.k;
  uint64_t grid = (uint64_t)a.sms * (uint64_t)occ;
  if ((uint64_t)a.batch < grid) grid = a.batch;
  kern<<<(unsigned)grid, kIntBlock, 0, a.stream>>>(p);
  return (int)cudaGetLastError();
}

template <int N>
int launch_int_batch(const IntBatchLaunch& a) {
  constexpr int L = int_logu(N);
  constexpr int MB = int_minb(N);
  switch (a.zb) {
    case 5: return launch_int_batch_cfg<N, IntCfg<5, L, MB>>(a);
    case 7: return launch_int_batch_cfg<N, IntCfg<7, L, MB>>(a);
    case 15: return launch_int_batch_cfg<N, IntCfg<15, L, MB>>(a);
    case 31: return launch_int_batch_cfg<N, IntCfg<31, L, MB>>(a);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace pk

#define PK_INSTANTIATE_INT(N)                                \
  template int pk::launch_int<N>(const pk::IntLaunch&); \
  template int pk::launch_int_batch<N>(const pk::IntBatchLaunch&);
