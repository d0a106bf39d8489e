// Precise mode of the dense real walk (PK_FLAG_PRECISE): reference-grade
// values for the accuracy gates at orders where no reference run is feasible.
//
// The reference's loop (_loops.py:35-107, /root/reference/pkg/src/permkit)
// keeps the row sums x in doubles and updates them incrementally, so x drifts
// by the rounding of every update; its most accurate policy (QQ) only
// hardens the product and the partial. Here the row sums are exact: X_i is a
// fixed-point int64 (row scale 2^F_i, fixed_image in pk_abi.cu) updated with
// integer adds, converted every step to the exact double-double value
// (hi, lo) = X_i 2^-F_i, multiplied in double-double and summed with dd_add.
// The only approximation left is the one-off rounding of the entries to the
// row grid (|error| <= 2^-(F_i+1), about 2^-63 of the row's absolute sum).
// Cost: about 12x the fast walk (three conversions, a double-double product
// and a double-double sum per row and step).
#pragma once
#include "pk_common.cuh"
#include "pk_dense_f64.cuh"
#include "pk_reduce.cuh"

namespace pk {

constexpr int kPreciseBlock = 128;

struct PreciseParams {
  const long long* fix;  // fixed-point image, layout of fixed_image (device)
  dd_t* group_part;
  dd_t* chunk_part;      // optional per-chunk partials
  dd_t* out;
  unsigned int* counter;
  unsigned long long chunk_lo;
  unsigned long long num_groups;
  unsigned long long g_end;
  int k;
};

// (ph, pl) *= (xh, xl), double-double (relative error ~2^-104)
__device__ __forceinline__ void dd_mul_dd(double& ph, double& pl, double xh, double xl) {
  const double p = __dmul_rn(ph, xh);
  double e = __fma_rn(ph, xh, -p);
  e = __fma_rn(ph, xl, e);
  e = __fma_rn(pl, xh, e);
  ph = __dadd_rn(p, e);
  pl = __dsub_rn(e, __dsub_rn(ph, p));
}

template <int N>
__device__ __forceinline__ dd_t precise_chunk(const long long* sfix, int k, uint64_t g_end,
                                              uint64_t c) {
  constexpr int NP = smem_stride<N>();
  const long long* sX0 = sfix + (N - 1) * NP;
  const double* ssc = reinterpret_cast<const double*>(sX0 + N);
  long long X[N];
  const uint64_t base = c << k;
  const uint64_t code = base ^ (base >> 1);
#pragma unroll
  for (int i = 0; i < N; ++i) X[i] = sX0[i];
  for (uint64_t m = code; m; m &= m - 1) {
    const long long* col = sfix + (__ffsll((long long)m) - 1) * NP;
#pragma unroll
    for (int i = 0; i < N; ++i) X[i] += col[i];
  }
  dd_t acc{0.0, 0.0};
  const uint64_t steps = 1ull << k;
  for (uint64_t r = 1; r <= steps; ++r) {
    const uint64_t g = base + r;
    if (g > g_end) break;
    const int j = changed_col(g);
    const long long msk = flip_on(g, j) ? 0ll : -1ll;  // add the column or subtract it
    const long long* col = sfix + j * NP;
    double ph = 1.0, pl = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      X[i] += (col[i] ^ msk) - msk;
      const double h = __ll2double_rn(X[i]);                        // RN(X)
      const double l = __ll2double_rn(X[i] - __double2ll_rn(h));    // exact remainder
      dd_mul_dd(ph, pl, __dmul_rn(h, ssc[i]), __dmul_rn(l, ssc[i]));
    }
    if (g & 1ull) {
      ph = -ph;
      pl = -pl;
    }
    acc = dd_add(acc, dd_t{ph, pl});
  }
  return acc;
}

template <int N>
__global__ void __launch_bounds__(kPreciseBlock)
    dense_f64_precise(const __grid_constant__ PreciseParams p) {
  __shared__ __align__(16) long long sfix[fix_words<N>()];
  stage_fix<N>(sfix, p.fix);
  __syncthreads();
  const unsigned int lane = threadIdx.x & 31u;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t grp = warp; grp < p.num_groups; grp += nwarps) {
    const uint64_t c = p.chunk_lo + grp * 32 + lane;
    dd_t part = precise_chunk<N>(sfix, p.k, p.g_end, c);
    if (p.chunk_part) p.chunk_part[grp * 32 + lane] = part;
    part = warp_tree_dd(part);
    if (lane == 0) p.group_part[grp] = part;
  }
  grid_tail_reduce<kPreciseBlock>(p.group_part, p.num_groups, p.out, p.counter);
}

// ---------------------------------------------------------------------------
// complex precise mode: X = (X_re, X_im) per row, each component its own
// fixed-point grid (two real images back to back); the product and the sums
// are double-double per component.

__device__ __forceinline__ dd_t dd_mul(dd_t a, dd_t b) {
  double ph = a.hi, pl = a.lo;
  dd_mul_dd(ph, pl, b.hi, b.lo);
  return dd_t{ph, pl};
}

__device__ __forceinline__ dd_t dd_neg(dd_t a) { return dd_t{-a.hi, -a.lo}; }

template <int N>
__device__ __forceinline__ dd_t fx_dd(long long X, double sc) {
  const double h = __ll2double_rn(X);
  const double l = __ll2double_rn(X - __double2ll_rn(h));
  return dd_t{__dmul_rn(h, sc), __dmul_rn(l, sc)};
}

template <int N>
__device__ __forceinline__ void precise_c128_chunk(const long long* sre, const long long* sim,
                                                   int k, uint64_t g_end, uint64_t c, dd_t& ar,
                                                   dd_t& ai) {
  constexpr int NP = smem_stride<N>();
  const double* scr = reinterpret_cast<const double*>(sre + (N - 1) * NP + N);
  const double* sci = reinterpret_cast<const double*>(sim + (N - 1) * NP + N);
  long long Xr[N], Xi[N];
  const uint64_t base = c << k;
  const uint64_t code = base ^ (base >> 1);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    Xr[i] = sre[(N - 1) * NP + i];
    Xi[i] = sim[(N - 1) * NP + i];
  }
  for (uint64_t m = code; m; m &= m - 1) {
    const int j = __ffsll((long long)m) - 1;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      Xr[i] += sre[j * NP + i];
      Xi[i] += sim[j * NP + i];
    }
  }
  ar = dd_t{0.0, 0.0};
  ai = dd_t{0.0, 0.0};
  const uint64_t steps = 1ull << k;
  for (uint64_t r = 1; r <= steps; ++r) {
    const uint64_t g = base + r;
    if (g > g_end) break;
    const int j = changed_col(g);
    const long long msk = flip_on(g, j) ? 0ll : -1ll;
    dd_t pr{1.0, 0.0}, pi{0.0, 0.0};
#pragma unroll
    for (int i = 0; i < N; ++i) {
      Xr[i] += (sre[j * NP + i] ^ msk) - msk;
      Xi[i] += (sim[j * NP + i] ^ msk) - msk;
      const dd_t xr = fx_dd<N>(Xr[i], scr[i]), xi = fx_dd<N>(Xi[i], sci[i]);
      if (i == 0) {
        pr = xr;
        pi = xi;
      } else {
        const dd_t nr = dd_add(dd_mul(pr, xr), dd_neg(dd_mul(pi, xi)));
        const dd_t ni = dd_add(dd_mul(pr, xi), dd_mul(pi, xr));
        pr = nr;
        pi = ni;
      }
    }
    if (g & 1ull) {
      pr = dd_neg(pr);
      pi = dd_neg(pi);
    }
    ar = dd_add(ar, pr);
    ai = dd_add(ai, pi);
  }
}

template <int N>
__global__ void __launch_bounds__(kPreciseBlock)
    dense_c128_precise(const __grid_constant__ PreciseParams p) {
  extern __shared__ __align__(16) long long sfix[];  // 2 * fix_words<N>() (dynamic: > 48 KB at large N)
  stage_fix<N>(sfix, p.fix);
  stage_fix<N>(sfix + fix_words<N>(), p.fix + (N - 1) * N + 2 * N);
  __syncthreads();
  const unsigned int lane = threadIdx.x & 31u;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t grp = warp; grp < p.num_groups; grp += nwarps) {
    const uint64_t c = p.chunk_lo + grp * 32 + lane;
    dd_t re, im;
    precise_c128_chunk<N>(sfix, sfix + fix_words<N>(), p.k, p.g_end, c, re, im);
    if (p.chunk_part)
      p.chunk_part[grp * 32 + lane] = dd_t{__dadd_rn(re.hi, re.lo), __dadd_rn(im.hi, im.lo)};
    re = warp_tree_dd(re);
    im = warp_tree_dd(im);
    if (lane == 0) {
      p.group_part[2 * grp] = re;
      p.group_part[2 * grp + 1] = im;
    }
  }
  grid_tail_reduce_pairs<kPreciseBlock>(p.group_part, p.num_groups, p.out, p.counter);
}

}  // namespace pk
