// Range walkers: one thread walks one arbitrary inclusive iterate range
// [start, end] exactly as permkit's run_range does (parallel.py:232-289):
// jump in at start-1 (init_x_at / _y_init_at, parallel.py:162-229), then the
// chunk loop (_loops.py:35-284) with a run-time changed column per step.
//
// These serve (a) the unaligned head/tail pieces of a range around the
// aligned chunk region of the fast kernels, (b) small matrices (n < 11), and
// (c) the bit-exact per-range partials behind run_range / execute_plan.
// n is a run-time value, so the per-row state lives in local memory (L1);
// that is acceptable here because walkers never carry the bulk of a walk.
#pragma once
#include "pk_common.cuh"
#include "pk_int.cuh"

namespace pk {

constexpr int kWalkBlock = 128;

template <int POL>
__device__ __forceinline__ void walk_fold_real(Acc<POL>& acc, const double* x, int n, bool odd) {
  if constexpr (POL == POL_QQ) {
    double ph = 1.0, pl = 0.0;
    for (int i = 0; i < n; ++i) qq_mul_step(ph, pl, x[i]);
    if (odd) acc.sub2(ph, pl); else acc.add2(ph, pl);
  } else {
    double p = 1.0;
    for (int i = 0; i < n; ++i) p = __dmul_rn(p, x[i]);
    if (odd) acc.sub(p); else acc.add(p);
  }
}

// dense real: cols[j*n + i] (global), x0[n]
template <int POL>
__global__ void __launch_bounds__(kWalkBlock)
    walk_dense_f64(const double* __restrict__ cols, const double* __restrict__ x0, int n,
                   const unsigned long long* __restrict__ starts,
                   const unsigned long long* __restrict__ ends, int nranges, dd_t* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nranges) return;
  const uint64_t start = starts[r], end = ends[r];
  double x[64];
  for (int i = 0; i < n; ++i) x[i] = x0[i];
  uint64_t code = (start - 1) ^ ((start - 1) >> 1);
  for (int j = 0; code; ++j, code >>= 1)
    if (code & 1ull)
      for (int i = 0; i < n; ++i) x[i] = __dadd_rn(x[i], cols[j * n + i]);
  Acc<POL> acc;
  for (uint64_t g = start;; ++g) {
    const int j = changed_col(g);
    const double s = flip_on(g, j) ? 1.0 : -1.0;
    const double* c = cols + (size_t)j * n;
    for (int i = 0; i < n; ++i) x[i] = __fma_rn(s, c[i], x[i]);
    walk_fold_real<POL>(acc, x, n, (g & 1ull) != 0);
    if (g == end) break;
  }
  out[r] = acc.partial();
}

// whole walks of `batch` small matrices, one thread per matrix: matrix r has
// columns cols + r*(n-1)*n and seed x0 + r*n (batched API for n < 11)
template <int POL>
__global__ void __launch_bounds__(kWalkBlock)
    walk_dense_f64_multi(const double* __restrict__ cols, const double* __restrict__ x0, int n,
                         int batch, dd_t* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= batch) return;
  const double* cr = cols + (size_t)r * (n - 1) * n;
  double x[64];
  for (int i = 0; i < n; ++i) x[i] = x0[(size_t)r * n + i];
  Acc<POL> acc;
  const uint64_t end = (1ull << (n - 1)) - 1;
  for (uint64_t g = 1; g <= end; ++g) {
    const int j = changed_col(g);
    const double s = flip_on(g, j) ? 1.0 : -1.0;
    for (int i = 0; i < n; ++i) x[i] = __fma_rn(s, cr[j * n + i], x[i]);
    walk_fold_real<POL>(acc, x, n, (g & 1ull) != 0);
  }
  out[r] = end ? acc.partial() : dd_t{0.0, 0.0};
}

// sparse real, CCS: cptrs[n+1], rids[nnz], vals[nnz]
template <int POL>
__global__ void __launch_bounds__(kWalkBlock)
    walk_sparse_f64(const int* __restrict__ cptrs, const int* __restrict__ rids,
                    const double* __restrict__ vals, const double* __restrict__ x0, int n,
                    const unsigned long long* __restrict__ starts,
                    const unsigned long long* __restrict__ ends, int nranges, dd_t* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nranges) return;
  const uint64_t start = starts[r], end = ends[r];
  double x[64];
  for (int i = 0; i < n; ++i) x[i] = x0[i];
  uint64_t code = (start - 1) ^ ((start - 1) >> 1);
  for (int j = 0; code; ++j, code >>= 1)
    if (code & 1ull)
      for (int p = cptrs[j]; p < cptrs[j + 1]; ++p) x[rids[p]] = __dadd_rn(x[rids[p]], vals[p]);
  Acc<POL> acc;
  for (uint64_t g = start;; ++g) {
    const int j = changed_col(g);
    const double s = flip_on(g, j) ? 1.0 : -1.0;
    for (int p = cptrs[j]; p < cptrs[j + 1]; ++p) x[rids[p]] = __fma_rn(s, vals[p], x[rids[p]]);
    walk_fold_real<POL>(acc, x, n, (g & 1ull) != 0);
    if (g == end) break;
  }
  out[r] = acc.partial();
}

// ---------------------------------------------------------------------------
// complex walkers (helpers in pk_common.cuh)

// out[r] = (re, im) of the plain complex partial
__global__ void __launch_bounds__(kWalkBlock)
    walk_dense_c128(const double* __restrict__ cols, const double* __restrict__ x0, int n,
                    const unsigned long long* __restrict__ starts,
                    const unsigned long long* __restrict__ ends, int nranges, dd_t* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nranges) return;
  const uint64_t start = starts[r], end = ends[r];
  double x[128];
  for (int i = 0; i < 2 * n; ++i) x[i] = x0[i];
  uint64_t code = (start - 1) ^ ((start - 1) >> 1);
  for (int j = 0; code; ++j, code >>= 1)
    if (code & 1ull)
      for (int i = 0; i < n; ++i) {
        x[2 * i] = __dadd_rn(x[2 * i], cols[2 * (j * n + i)]);
        x[2 * i + 1] = __dadd_rn(x[2 * i + 1], cols[2 * (j * n + i) + 1]);
      }
  double accr = 0.0, acci = 0.0;
  for (uint64_t g = start;; ++g) {
    const int j = changed_col(g);
    const double s = flip_on(g, j) ? 1.0 : -1.0;
    const double* c = cols + 2 * (size_t)j * n;
    for (int i = 0; i < n; ++i) c_update_ref(x[2 * i], x[2 * i + 1], s, c[2 * i], c[2 * i + 1]);
    c_fold_ref(accr, acci, x, n, (g & 1ull) != 0);
    if (g == end) break;
  }
  out[r] = dd_t{accr, acci};
}

// whole complex walks of `batch` small matrices, one thread per matrix
// (batched API for n < 11): out[r] = (re, im) plain partial
__global__ void __launch_bounds__(kWalkBlock)
    walk_dense_c128_multi(const double* __restrict__ cols, const double* __restrict__ x0, int n,
                          int batch, dd_t* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= batch) return;
  const double* cr = cols + (size_t)r * 2 * (n - 1) * n;
  double x[128];
  for (int i = 0; i < 2 * n; ++i) x[i] = x0[(size_t)r * 2 * n + i];
  double accr = 0.0, acci = 0.0;
  const uint64_t end = (1ull << (n - 1)) - 1;
  for (uint64_t g = 1; g <= end; ++g) {
    const int j = changed_col(g);
    const double s = flip_on(g, j) ? 1.0 : -1.0;
    const double* c = cr + 2 * (size_t)j * n;
    for (int i = 0; i < n; ++i) c_update_ref(x[2 * i], x[2 * i + 1], s, c[2 * i], c[2 * i + 1]);
    c_fold_ref(accr, acci, x, n, (g & 1ull) != 0);
  }
  out[r] = dd_t{accr, acci};
}

__global__ void __launch_bounds__(kWalkBlock)
    walk_sparse_c128(const int* __restrict__ cptrs, const int* __restrict__ rids,
                     const double* __restrict__ vals, const double* __restrict__ x0, int n,
                     const unsigned long long* __restrict__ starts,
                     const unsigned long long* __restrict__ ends, int nranges, dd_t* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nranges) return;
  const uint64_t start = starts[r], end = ends[r];
  double x[128];
  for (int i = 0; i < 2 * n; ++i) x[i] = x0[i];
  uint64_t code = (start - 1) ^ ((start - 1) >> 1);
  for (int j = 0; code; ++j, code >>= 1)
    if (code & 1ull)
      for (int p = cptrs[j]; p < cptrs[j + 1]; ++p) {
        const int q = rids[p];
        x[2 * q] = __dadd_rn(x[2 * q], vals[2 * p]);
        x[2 * q + 1] = __dadd_rn(x[2 * q + 1], vals[2 * p + 1]);
      }
  double accr = 0.0, acci = 0.0;
  for (uint64_t g = start;; ++g) {
    const int j = changed_col(g);
    const double s = flip_on(g, j) ? 1.0 : -1.0;
    for (int p = cptrs[j]; p < cptrs[j + 1]; ++p) {
      const int q = rids[p];
      c_update_ref(x[2 * q], x[2 * q + 1], s, vals[2 * p], vals[2 * p + 1]);
    }
    c_fold_ref(accr, acci, x, n, (g & 1ull) != 0);
    if (g == end) break;
  }
  out[r] = dd_t{accr, acci};
}

// ---------------------------------------------------------------------------
// range walker: run-time n, exact product by repeated 128-bit wrapping
// multiply (exact under the same host bound), one thread per range

// whole exact walks of `batch` small integer matrices, one thread each
// (batched API for n < 11): out[r] = z-space partial over [1, 2^(n-1)-1]
__global__ void __launch_bounds__(128)
    walk_int_multi(const int* __restrict__ cols, const int* __restrict__ z0, int n, int batch,
                   i192* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= batch) return;
  const int* cr = cols + (size_t)r * (n - 1) * n;
  int z[64];
  for (int i = 0; i < n; ++i) z[i] = z0[(size_t)r * n + i];
  i192 acc{0ull, 0ull, 0ull};
  const uint64_t end = (1ull << (n - 1)) - 1;
  for (uint64_t g = 1; g <= end; ++g) {
    const int j = changed_col(g);
    const int s = flip_on(g, j) ? 1 : -1;
    for (int i = 0; i < n; ++i) z[i] += s * cr[j * n + i];
    unsigned __int128 p = 1;
    for (int i = 0; i < n; ++i) p *= (unsigned __int128)(__int128)z[i];
    const unsigned long long lo = (unsigned long long)p, hi = (unsigned long long)(p >> 64);
    if (g & 1ull) i192_sub128(acc, lo, hi); else i192_add128(acc, lo, hi);
  }
  out[r] = acc;
}

__global__ void __launch_bounds__(128)
    walk_int(const int* __restrict__ cols, const int* __restrict__ z0, int n,
             const unsigned long long* __restrict__ starts,
             const unsigned long long* __restrict__ ends, int nranges, i192* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nranges) return;
  const uint64_t start = starts[r], end = ends[r];
  int z[64];
  for (int i = 0; i < n; ++i) z[i] = z0[i];
  uint64_t code = (start - 1) ^ ((start - 1) >> 1);
  for (int j = 0; code; ++j, code >>= 1)
    if (code & 1ull)
      for (int i = 0; i < n; ++i) z[i] += cols[j * n + i];
  i192 acc{0ull, 0ull, 0ull};
  for (uint64_t g = start;; ++g) {
    const int j = changed_col(g);
    const int s = flip_on(g, j) ? 1 : -1;
    const int* c = cols + (size_t)j * n;
    for (int i = 0; i < n; ++i) z[i] += s * c[i];
    unsigned __int128 p = 1;
    for (int i = 0; i < n; ++i) p *= (unsigned __int128)(__int128)z[i];
    const unsigned long long lo = (unsigned long long)p, hi = (unsigned long long)(p >> 64);
    if (g & 1ull) i192_sub128(acc, lo, hi); else i192_add128(acc, lo, hi);
    if (g == end) break;
  }
  out[r] = acc;
}

}  // namespace pk
