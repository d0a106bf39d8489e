// K3: dense complex fp64 Gray walk (boson-sampling permanents), same chunk
// geometry as K1 (pk_dense_f64.cuh): aligned 2^k chunks, register-resident
// state, compile-time column indices inside each unrolled body, columns
// staged once per block in shared memory (one LDS.128 per complex entry).
//
// Replaces chunk_dense_c128 (/root/reference/pkg/src/permkit/_loops.py:186-209)
// under run_range (parallel.py:232-289). The reference accumulates complex
// partials in plain double only (kernels.py:309-310).
//
// Two arithmetic modes (template EXACT):
//   EXACT  -- the reference's operation sequence: s promoted to complex(s,0)
//             for the column update, products as (ac - bd) + (ad + bc)i with
//             one rounding each, plain per-term partial sums; chunk partials
//             are bit-identical to run_range over the same chunk.
//   fast   -- x += s*c per component (exact anyway), products with two fmas
//             (4 FP64 ops instead of 6, one rounding fewer per component),
//             body sums folded with compensation per component.
#pragma once
#include "pk_common.cuh"
#include "pk_reduce.cuh"

namespace pk {

constexpr int kC128Block = 128;

template <int N>
struct DenseC128Params {
  double x0[2 * N];          // interleaved (re, im)
  const double* cols;        // device, cols[(j*N + i)*2 + {0,1}], j < N-1
  dd_t* group_part;          // [num_groups] (re, im) per warp group
  dd_t* chunk_part;          // optional [num_groups*32]
  dd_t* out;                 // launch total (re, im)
  unsigned int* counter;
  unsigned long long chunk_lo;
  unsigned long long num_groups;
  unsigned long long g_end;
  int k;
};

// FA (fast mode): the last complex multiply of each product and the body sum
// fold into four DFMAs, b += (+-p) * x[N-1] per component (two FP64
// instructions fewer per update)
// TC (fast mode): the product runs as two interleaved chains over the even
// and the odd rows, and four DFMAs multiply them into the body sum -- the
// same FP64 instruction count as FA, twice the independent work per term
// (the single chain is latency bound at 2 warps per scheduler)
// RM (fast mode): the body is walked row-major -- for each row i the U
// states of the body are formed one after the other (x_i +- c_{j_q,i}, the
// same roundings as the step-major walk) and each multiplies its term's
// running product. The U product chains are independent, the state needs no
// copies, and each distinct column entry is loaded once per row: same
// arithmetic, same bits as the step-major schedule, U-fold product ILP.
template <int LOGU_, bool EXACT_, int MINB_, bool FA_ = false, int BLOCK_ = kC128Block,
          bool TC_ = false, bool RM_ = false>
struct C128Cfg {
  static constexpr int LOGU = LOGU_, MINB = MINB_, BLOCK = BLOCK_;
  static constexpr bool EXACT = EXACT_;
  static constexpr bool TC = TC_ && !EXACT_;
  static constexpr bool RM = RM_ && !EXACT_;
  static constexpr bool FA = FA_ && !EXACT_ && !TC && !RM;
};

// complex partial sum: plain (reference) or compensated per component
template <bool EXACT>
struct CAcc;

template <>
struct CAcc<true> {
  double r = 0.0, i = 0.0;
  __device__ __forceinline__ void add(double pr, double pi) {
    r = __dadd_rn(r, pr);
    i = __dadd_rn(i, pi);
  }
  __device__ __forceinline__ void sub(double pr, double pi) {
    r = __dsub_rn(r, pr);
    i = __dsub_rn(i, pi);
  }
  __device__ __forceinline__ dd_t partial() const { return dd_t{r, i}; }
};

template <>
struct CAcc<false> {
  Acc<POL_KAHAN> r, i;
  __device__ __forceinline__ void add(double pr, double pi) {
    r.add(pr);
    i.add(pi);
  }
  __device__ __forceinline__ void sub(double pr, double pi) {
    r.sub(pr);
    i.sub(pi);
  }
  // collapse the compensation: the partial type of complex runs is one
  // complex double per range (parallel.py:265-267)
  __device__ __forceinline__ dd_t partial() const {
    return dd_t{__dadd_rn(r.a, r.b), __dadd_rn(i.a, i.b)};
  }
};

template <int N, class C>
struct C128Walk {
  const double* scols;  // shared, (N-1) x N complex
  double xr[N], xi[N];
  CAcc<C::EXACT> acc;
  double br, bi;  // body sums (fast mode)

  __device__ __forceinline__ void update(const double* col, double s) {
    const double2* c2 = reinterpret_cast<const double2*>(col);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double2 v = c2[i];
      if constexpr (C::EXACT) {
        c_update_ref(xr[i], xi[i], s, v.x, v.y);
      } else {
        xr[i] = __fma_rn(s, v.x, xr[i]);
        xi[i] = __fma_rn(s, v.y, xi[i]);
      }
    }
  }

  template <int SIGN>
  __device__ __forceinline__ void update_static(const double* col) {
    if constexpr (C::EXACT) {
      update(col, SIGN > 0 ? 1.0 : -1.0);
    } else {
      const double2* c2 = reinterpret_cast<const double2*>(col);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double2 v = c2[i];
        xr[i] = SIGN > 0 ? __dadd_rn(xr[i], v.x) : __dsub_rn(xr[i], v.x);
        xi[i] = SIGN > 0 ? __dadd_rn(xi[i], v.y) : __dsub_rn(xi[i], v.y);
      }
    }
  }

  __device__ __forceinline__ void product(double& pr, double& pi) const {
    if constexpr (C::EXACT) {
      // prod = complex(1, 0); prod *= x[i]  (_loops.py:199-201)
      pr = 1.0;
      pi = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double r, m;
        cmul_ref(pr, pi, xr[i], xi[i], r, m);
        pr = r;
        pi = m;
      }
    } else {
      pr = xr[0];
      pi = xi[0];
#pragma unroll
      for (int i = 1; i < N; ++i) {
        const double r = __fma_rn(pr, xr[i], -__dmul_rn(pi, xi[i]));
        const double m = __fma_rn(pr, xi[i], __dmul_rn(pi, xr[i]));
        pr = r;
        pi = m;
      }
    }
  }

  __device__ __forceinline__ void fold(bool odd, bool first_in_body) {
    if constexpr (C::TC) {
      double er = xr[0], ei = xi[0], orr = xr[1], oi = xi[1];
#pragma unroll
      for (int i = 2; i < N; ++i) {
        double& pr = (i & 1) ? orr : er;
        double& pi = (i & 1) ? oi : ei;
        const double r = __fma_rn(pr, xr[i], -__dmul_rn(pi, xi[i]));
        const double m = __fma_rn(pr, xi[i], __dmul_rn(pi, xr[i]));
        pr = r;
        pi = m;
      }
      if (odd) {
        er = -er;
        ei = -ei;
      }
      const double r0 = first_in_body ? 0.0 : br, i0 = first_in_body ? 0.0 : bi;
      br = __fma_rn(er, orr, __fma_rn(-ei, oi, r0));
      bi = __fma_rn(er, oi, __fma_rn(ei, orr, i0));
      return;
    }
    if constexpr (C::FA) {
      double pr = xr[0], pi = xi[0];
#pragma unroll
      for (int i = 1; i < N - 1; ++i) {
        const double r = __fma_rn(pr, xr[i], -__dmul_rn(pi, xi[i]));
        const double m = __fma_rn(pr, xi[i], __dmul_rn(pi, xr[i]));
        pr = r;
        pi = m;
      }
      if (odd) {
        pr = -pr;
        pi = -pi;
      }
      if (first_in_body) {
        br = __fma_rn(pr, xr[N - 1], -__dmul_rn(pi, xi[N - 1]));
        bi = __fma_rn(pr, xi[N - 1], __dmul_rn(pi, xr[N - 1]));
      } else {
        br = __fma_rn(-pi, xi[N - 1], __fma_rn(pr, xr[N - 1], br));
        bi = __fma_rn(pi, xr[N - 1], __fma_rn(pr, xi[N - 1], bi));
      }
      return;
    }
    double pr, pi;
    product(pr, pi);
    if constexpr (C::EXACT) {
      if (odd) acc.sub(pr, pi); else acc.add(pr, pi);
    } else {
      if (first_in_body) {
        br = odd ? -pr : pr;
        bi = odd ? -pi : pi;
      } else {
        br = odd ? __dsub_rn(br, pr) : __dadd_rn(br, pr);
        bi = odd ? __dsub_rn(bi, pi) : __dadd_rn(bi, pi);
      }
    }
  }

  __device__ __forceinline__ void end_body() {
    if constexpr (!C::EXACT) acc.add(br, bi);
  }
};

template <int N, class C, int Q>
__device__ __forceinline__ void c128_static_step(C128Walk<N, C>& w, double s_mid, int jz) {
  constexpr int J = ctz_c(Q);
  const double* col = w.scols + 2 * (J + jz) * N;
  if constexpr (J + 1 < C::LOGU) {
    w.template update_static<(((Q >> (J + 1)) & 1) == 0) ? 1 : -1>(col);
  } else {
    w.update(col, s_mid);
  }
  w.fold((Q & 1) != 0, Q == 1);
}

template <int N, class C, int Q, int U>
struct C128Steps {
  __device__ __forceinline__ static void run(C128Walk<N, C>& w, double s_mid, int jz) {
    c128_static_step<N, C, Q>(w, s_mid, jz);
    C128Steps<N, C, Q + 1, U>::run(w, s_mid, jz);
  }
};
template <int N, class C, int U>
struct C128Steps<N, C, U, U> {
  __device__ __forceinline__ static void run(C128Walk<N, C>&, double, int) {}
};

// one body of U steps, row-major (C::RM): steps 1..U-1 static (column ctz(q),
// direction from q or s_mid), step U the run-time column jd with direction sd
// (sd = 0 and no fold when the walk's last step is clipped)
template <int N, class C>
__device__ __forceinline__ void c128_body_rm(C128Walk<N, C>& w, double s_mid, int jz, int jd,
                                             double sd, bool okd) {
  constexpr int LOGU = C::LOGU;
  constexpr int U = 1 << LOGU;
  const double2* cb = reinterpret_cast<const double2*>(w.scols);
  double pr[U], pi[U];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double vr = w.xr[i], vi = w.xi[i];
#pragma unroll
    for (int q = 1; q <= U; ++q) {
      if (q < U) {
        const int J = ctz_c(q);
        const double2 v = cb[(J + jz) * N + i];
        if (J + 1 < LOGU) {
          if (((q >> (J + 1)) & 1) == 0) {
            vr = __dadd_rn(vr, v.x);
            vi = __dadd_rn(vi, v.y);
          } else {
            vr = __dsub_rn(vr, v.x);
            vi = __dsub_rn(vi, v.y);
          }
        } else {
          vr = __fma_rn(s_mid, v.x, vr);
          vi = __fma_rn(s_mid, v.y, vi);
        }
      } else {
        const double2 v = cb[jd * N + i];
        vr = __fma_rn(sd, v.x, vr);
        vi = __fma_rn(sd, v.y, vi);
      }
      if (i == 0) {
        pr[q - 1] = vr;
        pi[q - 1] = vi;
      } else {
        const double r = __fma_rn(pr[q - 1], vr, -__dmul_rn(pi[q - 1], vi));
        const double m = __fma_rn(pr[q - 1], vi, __dmul_rn(pi[q - 1], vr));
        pr[q - 1] = r;
        pi[q - 1] = m;
      }
    }
    w.xr[i] = vr;
    w.xi[i] = vi;
  }
  // fold the terms in step order, exactly as the step-major fold()
#pragma unroll
  for (int q = 1; q <= U; ++q) {
    if (q == U && !okd) break;
    const bool odd = (q & 1) != 0;
    if (q == 1) {
      w.br = odd ? -pr[0] : pr[0];
      w.bi = odd ? -pi[0] : pi[0];
    } else {
      w.br = odd ? __dsub_rn(w.br, pr[q - 1]) : __dadd_rn(w.br, pr[q - 1]);
      w.bi = odd ? __dsub_rn(w.bi, pi[q - 1]) : __dadd_rn(w.bi, pi[q - 1]);
    }
  }
  w.end_body();
}

template <int N, class C>
__device__ __forceinline__ dd_t c128_walk_chunk(const double* x0, int k, uint64_t g_end,
                                                const double* scols, uint64_t c) {
  constexpr int LOGU = C::LOGU;
  constexpr int U = 1 << LOGU;
  C128Walk<N, C> w;
  w.scols = scols;
  const uint64_t base = c << k;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    w.xr[i] = x0[2 * i];
    w.xi[i] = x0[2 * i + 1];
  }
  // jump-in: x0 + columns of gray(base), ascending (parallel.py:162-188)
  const uint64_t code = base ^ (base >> 1);
  for (int j = 0; j < N - 1; ++j) {
    if ((code >> j) & 1ull) {
      const double2* c2 = reinterpret_cast<const double2*>(scols + 2 * j * N);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double2 v = c2[i];
        w.xr[i] = __dadd_rn(w.xr[i], v.x);
        w.xi[i] = __dadd_rn(w.xi[i], v.y);
      }
    }
  }
  const uint64_t nbody = 1ull << (k - LOGU);
  for (uint64_t m = 0; m < nbody; ++m) {
    const uint64_t gb = base + (m << LOGU);
    const double s_mid = flip_on(gb + (U >> 1), LOGU - 1) ? 1.0 : -1.0;
    const int jz = (int)(m >> 62);
    const uint64_t g = gb + U;
    if constexpr (C::RM) {
      const bool ok = (m + 1 < nbody) || g <= g_end;
      const int j = ok ? changed_col(g) : 0;
      c128_body_rm<N, C>(w, s_mid, jz, j, ok ? (flip_on(g, j) ? 1.0 : -1.0) : 0.0, ok);
      continue;
    }
    C128Steps<N, C, 1, U>::run(w, s_mid, jz);
    if (m + 1 < nbody || g <= g_end) {
      const int j = changed_col(g);
      w.update(scols + 2 * j * N, flip_on(g, j) ? 1.0 : -1.0);
      w.fold(false, false);
    }
    w.end_body();
  }
  return w.acc.partial();
}

// (re, im) pairs are reduced as two independent double-double trees: each
// lane's partial (re, im) becomes two dd values; the warp / grid trees keep
// them side by side in group_part[2*g], group_part[2*g+1].
__device__ __forceinline__ void warp_tree_cdd(dd_t& re, dd_t& im) {
  re = warp_tree_dd(re);
  im = warp_tree_dd(im);
}

template <int N, class C>
__global__ void __launch_bounds__(C::BLOCK, C::MINB)
    dense_c128_chunks(const __grid_constant__ DenseC128Params<N> p) {
  extern __shared__ __align__(16) double scols[];
  for (int t = threadIdx.x; t < 2 * (N - 1) * N; t += blockDim.x) scols[t] = p.cols[t];
  __syncthreads();
  const unsigned int lane = threadIdx.x & 31u;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t grp = warp; grp < p.num_groups; grp += nwarps) {
    const uint64_t c = p.chunk_lo + grp * 32 + lane;
    const dd_t part = c128_walk_chunk<N, C>(p.x0, p.k, p.g_end, scols, c);
    if (p.chunk_part) p.chunk_part[grp * 32 + lane] = part;
    dd_t re{part.hi, 0.0}, im{part.lo, 0.0};
    warp_tree_cdd(re, im);
    if (lane == 0) {
      p.group_part[2 * grp] = re;
      p.group_part[2 * grp + 1] = im;
    }
  }
  grid_tail_reduce_pairs<C::BLOCK>(p.group_part, p.num_groups, p.out, p.counter);
}

template <int N>
__host__ __device__ constexpr size_t c128_smem_bytes() {
  return sizeof(double) * 2 * (N - 1) * N;
}

// ---------------------------------------------------------------------------
// batched walks (boson-sampling submatrices, decomposition leaves; SURVEY.md
// §8f-2): one block per matrix at a time, its 2^(N-1-k) aligned chunks walked
// by the block's warps and reduced exactly like a single launch of the same k
// (per-component pairwise fold over the group partials).

template <int N>
struct C128BatchParams {
  const double* cols;  // [batch][2*(N-1)*N] interleaved
  const double* x0;    // [batch][2*N]
  dd_t* group_part;    // [batch][2*groups] scratch
  dd_t* out;           // [batch][2]: (re, im) partials over [1, 2^(N-1)-1]
  int batch;
  int k;
};

template <int N, class C>
__global__ void __launch_bounds__(kC128Block, C::MINB)
    dense_c128_batch(const __grid_constant__ C128BatchParams<N> p) {
  extern __shared__ __align__(16) double smem[];
  double* scols = smem;
  double* sx0 = smem + 2 * (N - 1) * N;
  const uint64_t total = (1ull << (N - 1)) - 1;
  const int groups = (int)((1ull << (N - 1 - p.k)) / 32);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  for (int b = blockIdx.x; b < p.batch; b += gridDim.x) {
    __syncthreads();
    const double* cb = p.cols + (size_t)b * 2 * (N - 1) * N;
    for (int t = threadIdx.x; t < 2 * (N - 1) * N; t += blockDim.x) scols[t] = cb[t];
    for (int t = threadIdx.x; t < 2 * N; t += blockDim.x) sx0[t] = p.x0[(size_t)b * 2 * N + t];
    __syncthreads();
    dd_t* gp = p.group_part + (size_t)b * 2 * groups;
    for (int grp = wib; grp < groups; grp += wpb) {
      const dd_t part = c128_walk_chunk<N, C>(sx0, p.k, total, scols, (uint64_t)grp * 32 + lane);
      dd_t re{part.hi, 0.0}, im{part.lo, 0.0};
      warp_tree_cdd(re, im);
      if (lane == 0) {
        gp[2 * grp] = re;
        gp[2 * grp + 1] = im;
      }
    }
    __syncthreads();
    if (threadIdx.x < 2) p.out[2 * b + threadIdx.x] = pairwise_fold(gp, 0, groups, 2, threadIdx.x);
  }
}

}  // namespace pk
