// Host-side launcher template for the N-specialised dense real kernel.
// Included by the pk_dense_f64_n*.cu units, each instantiating a range of N.
#pragma once
#include <cstring>

#include "pk_dense_f64.cuh"
#include "pk_launch.h"

namespace pk {

template <int N, class C>
static int launch_cfg(const DenseLaunch& a, const DenseF64Params<N>& p) {
  auto kern = dense_f64_chunks<N, C>;
  constexpr size_t smem = dense_smem_bytes<N>();
  static std::atomic<int> slots[kMaxDevices];  // per device ordinal
  int occ = 1;
  if (int rc = prep_kernel(kern, C::BLOCK, smem, slots, &occ)) return rc;
  const uint64_t warps_needed = a.num_groups;
  const uint64_t blocks_needed = (warps_needed * 32 + C::BLOCK - 1) / C::BLOCK;
  uint64_t grid = (uint64_t)a.sms * (uint64_t)occ;
  if (blocks_needed < grid) grid = blocks_needed;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, C::BLOCK, smem, a.stream>>>(p);
  return (int)cudaGetLastError();
}

template <int N>
int launch_dense_f64(const DenseLaunch& a) {
  static_assert(N >= kDenseNMin && N <= kDenseNMax, "order out of range");
  constexpr int LOGU = dense_logu(N);
  constexpr int MB = dense_minb(N);
  constexpr int BLK = dense_block(N), BMB = dense_block_minb(N);
  DenseF64Params<N> p;
  std::memcpy(p.cols, a.cols, sizeof(double) * (N - 1) * N);
  std::memcpy(p.x0, a.x0, sizeof(double) * N);
  p.group_part = a.group_part;
  p.chunk_part = a.chunk_part;
  p.out = a.out;
  p.counter = a.counter;
  p.chunk_lo = a.chunk_lo;
  p.num_groups = a.num_groups;
  p.g_end = a.g_end;
  p.k = a.k;
  switch (a.policy) {
    case POL_DD:
      if (a.exact) return launch_cfg<N, DenseCfg<POL_DD, 1, LOGU, false, MB, 128, false, false, true>>(a, p);
      // row-major above n = 36, as KAHAN (same bits)
      if ((N > 36 && a.variant != 2) || a.variant == 1)
        return launch_cfg<N, DenseCfg<POL_DD, 1, LOGU, true, BMB, BLK, true, false, true>>(a, p);
      return launch_cfg<N, DenseCfg<POL_DD, 1, LOGU, true, BMB, BLK, true>>(a, p);
    case POL_KAHAN:
      if (a.exact) return launch_cfg<N, DenseCfg<POL_KAHAN, 1, LOGU, false, MB, 128, false, false, true>>(a, p);
      // row-major body above n = 36 (same bits; +0.2 % at n = 40, +1 % at
      // n = 48), step-major below (-0.3 % at n = 36) -- profiles/r02_k1_variants.txt;
      // PK_DENSE_VARIANT=1 forces row-major, 2 step-major (A/B runs)
      if ((N > 36 && a.variant != 2) || a.variant == 1)
        return launch_cfg<N, DenseCfg<POL_KAHAN, 1, LOGU, true, BMB, BLK, true, false, true>>(a, p);
      return launch_cfg<N, DenseCfg<POL_KAHAN, 1, LOGU, true, BMB, BLK, true>>(a, p);
    case POL_DQ:
      if (a.exact) return launch_cfg<N, DenseCfg<POL_DQ, 1, LOGU, false, MB, 128, false, false, true>>(a, p);
      if ((N > 36 && a.variant != 2) || a.variant == 1)
        return launch_cfg<N, DenseCfg<POL_DQ, 1, LOGU, true, BMB, BLK, true, false, true>>(a, p);
      return launch_cfg<N, DenseCfg<POL_DQ, 1, LOGU, true, BMB, BLK, true>>(a, p);
    case POL_QQ:
      if (a.exact) return launch_cfg<N, DenseCfg<POL_QQ, 1, LOGU, false, MB, 128, false, false, true>>(a, p);
      // row-major fast QQ (same bits) above n = 36, where the step-major body
      // spills: +12 % at n = 40, -3..5 % at n = 32..36
      // (profiles/r02_qq_variants.txt); PK_DENSE_VARIANT=1 forces it
      if (N > 36 || a.variant == 1)
        return launch_cfg<N, DenseCfg<POL_QQ, 1, qf_logu(N), false, MB, 128, false, true, true>>(a, p);
      return launch_cfg<N, DenseCfg<POL_QQ, 1, qf_logu(N), false, MB, 128, false, true>>(a, p);
    default:
      return (int)cudaErrorInvalidValue;
  }
}

template <int N, class C>
static int launch_batch_cfg(const DenseBatchLaunch& a) {
  auto kern = dense_f64_batch<N, C>;
  constexpr size_t smem = dense_smem_bytes<N>() + sizeof(double) * N;  // + x0
  static std::atomic<int> slots[kMaxDevices];  // per device ordinal
  int occ = 1;
  if (int rc = prep_kernel(kern, C::BLOCK, smem, slots, &occ)) return rc;
  DenseBatchParams<N> p;
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
int launch_dense_f64_batch(const DenseBatchLaunch& a) {
  constexpr int LOGU = dense_logu(N);
  constexpr int MB = dense_minb(N);
  switch (a.policy) {
    case POL_DD:
      return a.exact ? launch_batch_cfg<N, DenseCfg<POL_DD, 1, LOGU, false, MB>>(a)
                     : launch_batch_cfg<N, DenseCfg<POL_DD, 1, LOGU, true, MB, 128, true>>(a);
    case POL_KAHAN:
      return a.exact ? launch_batch_cfg<N, DenseCfg<POL_KAHAN, 1, LOGU, false, MB>>(a)
                     : launch_batch_cfg<N, DenseCfg<POL_KAHAN, 1, LOGU, true, MB, 128, true>>(a);
    case POL_DQ:
      return a.exact ? launch_batch_cfg<N, DenseCfg<POL_DQ, 1, LOGU, false, MB>>(a)
                     : launch_batch_cfg<N, DenseCfg<POL_DQ, 1, LOGU, true, MB, 128, true>>(a);
    case POL_QQ:
      return a.exact ? launch_batch_cfg<N, DenseCfg<POL_QQ, 1, LOGU, false, MB>>(a)
                     : launch_batch_cfg<N, DenseCfg<POL_QQ, 1, qf_logu(N), false, MB, 128, false, true>>(a);
    default:
      return (int)cudaErrorInvalidValue;
  }
}

}  // namespace pk

#define PK_INSTANTIATE_DENSE_F64(N)                                 \
  template int pk::launch_dense_f64<N>(const pk::DenseLaunch&); \
  template int pk::launch_dense_f64_batch<N>(const pk::DenseBatchLaunch&);
