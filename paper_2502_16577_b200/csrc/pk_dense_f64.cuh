// K1: dense real fp64 Gray walk over power-of-two aligned chunks.
//
// Replaces permkit's hot loop chunk_dense_f64 (/root/reference/pkg/src/permkit/
// _loops.py:35-107) driven by run_range/init_x_at (parallel.py:162-188,
// :232-289) over an aligned plan (parallel.py:95-122).
//
// Work unit: chunk c covers iterates [1 + c*2^k, (c+1)*2^k] -- the reference's
// aligned chunk layout. Its state is jumped in at g_prev = c*2^k. Within the
// chunk the changed column j = ctz(r) of local step r < 2^k is the same for
// every chunk (the CEG property), so the walk is unrolled in
// bodies of U = 2^LOGU steps whose U-1 inner steps have compile-time column
// indices: their column entries are read straight out of the kernel-parameter
// constant bank (DADD R, R, c[0x0][imm]) -- no load instruction at all. The
// U-th step of each body flips a column >= LOGU chosen at run time (uniform
// across the grid, read with LDC); the final step of the chunk flips a
// chunk-specific column.
//
// x[N] is register resident (N is a template parameter). The product is a
// sequential chain by default (PS = 1), which reproduces the reference's
// rounding exactly; PS > 1 splits it into PS interleaved chains.
#pragma once
#include "pk_common.cuh"
#include "pk_reduce.cuh"

namespace pk {

constexpr int kDenseBlock = 128;

template <int N>
struct DenseF64Params {
  double cols[(N - 1) * N];  // cols[j*N + i] = a_ij for the n-1 toggled columns
  double x0[N];              // a_{i,n-1} - rowsum_i / 2 (kernels.py:75-89)
  dd_t* group_part;          // [num_groups] warp-tree partials
  dd_t* chunk_part;          // optional [num_groups*32] per-chunk partials
  dd_t* out;                 // launch total (tree over groups)
  unsigned int* counter;     // last-block detector, zero on entry
  unsigned long long chunk_lo;    // first chunk index of this launch
  unsigned long long num_groups;  // groups of 32 consecutive chunks
  unsigned long long g_end;       // inclusive last iterate of the walk
  int k;                          // log2 chunk size, k > LOGU
};

template <int N, int PS>
__device__ __forceinline__ double row_product(const double (&x)[N]) {
  if constexpr (PS == 1) {
    // prod = 1.0; prod *= x[i] (_loops.py:85-87); 1.0 * x[0] == x[0] exactly
    double p = x[0];
#pragma unroll
    for (int i = 1; i < N; ++i) p = __dmul_rn(p, x[i]);
    return p;
  } else {
    double q[PS];
#pragma unroll
    for (int s = 0; s < PS; ++s) q[s] = (s < N) ? x[s] : 1.0;
#pragma unroll
    for (int i = PS; i < N; ++i) q[i % PS] = __dmul_rn(q[i % PS], x[i]);
#pragma unroll
    for (int w = 1; w < PS; w <<= 1)
#pragma unroll
      for (int s = 0; s + w < PS; s += 2 * w) q[s] = __dmul_rn(q[s], q[s + w]);
    return q[0];
  }
}

// Compile-time knobs of the walk:
//   POL  accumulator policy of the per-chunk partial (pk_common.cuh)
//   PS   product chains (1 = the reference's sequential product, bit exact)
//   LOGU log2 of the unrolled body length U
//   (the column operands always come from a shared-memory copy of the
//    columns read with warp-uniform LDS.128; parameter-bank and hoisted
//    variants were slower, profiles/r01_k1_variants.md)
//   BA   block accumulation: sum the U terms of a body in plain double and
//        fold the body sum once (1 policy fold per U terms instead of per
//        term). Not bit-identical to the reference's per-term fold.
//   MINB minimum resident blocks per SM requested from ptxas (register cap)
//   BLOCK threads per block (small blocks pack more warps per SM when the
//        register count is not a divisor-friendly number)
//   FA   fused accumulate (with BA): the last product multiply and the body
//        sum become one DFMA, bsum = fma(+-p', x[n-1], bsum)
//   QF   fast QQ (POL_QQ, not bit-identical): the double-double product
//        keeps (hi, lo) unnormalised -- hi' = hi*x, lo' = fma(lo, x,
//        fma(hi, x, -hi')) -- 3 FP64 ops per row instead of qq_mul_step's 7;
//        the body's terms are summed with a two_sum on the hi parts plus a
//        plain sum of the lo parts and folded once per body into the
//        double-double partial
//   RM   row-major body (with FA): for each row the U states of the body are
//        formed one after the other -- the same additions in the same order
//        as the step-major walk -- and multiply the U independent running
//        products; the last row's multiply folds into the body sum in step
//        order. Same bits as the step-major body, U independent chains, no
//        state copies, each distinct column entry loaded once per row
template <int POL_, int PS_, int LOGU_, bool BA_, int MINB_ = 1, int BLOCK_ = 128,
          bool FA_ = false, bool QF_ = false, bool RM_ = false>
struct DenseCfg {
  static constexpr int POL = POL_, PS = PS_, LOGU = LOGU_, MINB = MINB_;
  static constexpr int BLOCK = BLOCK_;
  static constexpr bool BA = BA_ && POL_ != POL_QQ;
  static constexpr bool FA = FA_ && BA;
  static constexpr bool QF = QF_ && POL_ == POL_QQ;
  static constexpr bool RM = RM_ && (FA || QF || !BA);
};

template <int N>
__host__ __device__ constexpr int smem_stride() { return (N + 1) & ~1; }

template <int N, class C>
struct DenseWalk {
  const double* scols;  // shared-memory columns, stride smem_stride<N>()
  double x[N];
  Acc<C::POL> acc;
  double bsum;
  double qs, qc, ql;  // fast-QQ body sums: hi parts (two_sum s + c), lo parts

  __device__ __forceinline__ explicit DenseWalk(const double* s_) : scols(s_) {}

  template <int SIGN>
  __device__ __forceinline__ static double apply(double xi, double c, double s) {
    if constexpr (SIGN > 0) return __dadd_rn(xi, c);
    else if constexpr (SIGN < 0) return __dsub_rn(xi, c);
    else return __fma_rn(s, c, xi);  // s = +-1: x + s*c exactly as _loops.py:48
  }

  // x[i] += sign * column entry, for a compile-time column J (SIGN 0: run-time s)
  template <int J, int SIGN>
  __device__ __forceinline__ void update_static(int jz, double s) {
    constexpr int NP = smem_stride<N>();
    const double2* c2 = reinterpret_cast<const double2*>(scols + (J + jz) * NP);
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const double2 v = c2[i / 2];
      x[i] = apply<SIGN>(x[i], v.x, s);
      if (i + 1 < N) x[i + 1] = apply<SIGN>(x[i + 1], v.y, s);
    }
  }

  // run-time column j (uniform in the body's last step, per-chunk at the end)
  __device__ __forceinline__ void update_dynamic(int j, double s) {
    constexpr int NP = smem_stride<N>();
    const double2* c2 = reinterpret_cast<const double2*>(scols + j * NP);
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const double2 v = c2[i / 2];
      x[i] = __fma_rn(s, v.x, x[i]);
      if (i + 1 < N) x[i + 1] = __fma_rn(s, v.y, x[i + 1]);
    }
  }

  // jump-in (init_x_at, parallel.py:162-188): x0 + columns of gray(g_prev), ascending
  __device__ __forceinline__ void jump_in(const double* x0, uint64_t g_prev) {
    constexpr int NP = smem_stride<N>();
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = x0[i];
    const uint64_t code = g_prev ^ (g_prev >> 1);
    for (int j = 0; j < N - 1; ++j) {
      if ((code >> j) & 1ull) {
        const double2* c2 = reinterpret_cast<const double2*>(scols + j * NP);
#pragma unroll
        for (int i = 0; i < N; i += 2) {
          const double2 v = c2[i / 2];
          x[i] = __dadd_rn(x[i], v.x);
          if (i + 1 < N) x[i + 1] = __dadd_rn(x[i + 1], v.y);
        }
      }
    }
  }

  // fold the current state's signed product (term sign = iterate parity)
  __device__ __forceinline__ void fold(bool odd, bool first_in_body) {
    if constexpr (C::QF) {
      double hi = __dmul_rn(x[0], x[1]);
      double lo = __fma_rn(x[0], x[1], -hi);
#pragma unroll
      for (int i = 2; i < N; ++i) {
        const double h2 = __dmul_rn(hi, x[i]);
        lo = __fma_rn(lo, x[i], __fma_rn(hi, x[i], -h2));
        hi = h2;
      }
      if (odd) {
        hi = -hi;
        lo = -lo;
      }
      if (first_in_body) {
        qs = hi;
        qc = 0.0;
        ql = lo;
      } else {
        double e;
        two_sum(qs, hi, qs, e);
        qc = __dadd_rn(qc, e);
        ql = __dadd_rn(ql, lo);
      }
    } else if constexpr (C::POL == POL_QQ) {
      double ph = 1.0, pl = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) qq_mul_step(ph, pl, x[i]);
      if (odd) acc.sub2(ph, pl); else acc.add2(ph, pl);
    } else if constexpr (C::FA) {
      // product of rows 0..N-2, then one DFMA folds the last row and the sum
      double pr = x[0];
#pragma unroll
      for (int i = 1; i < N - 1; ++i) pr = __dmul_rn(pr, x[i]);
      const double sp = odd ? -pr : pr;
      if (first_in_body) bsum = __dmul_rn(sp, x[N - 1]);
      else bsum = __fma_rn(sp, x[N - 1], bsum);
    } else {
      const double pr = row_product<N, C::PS>(x);
      if constexpr (C::BA) {
        if (first_in_body) bsum = odd ? -pr : pr;
        else bsum = odd ? __dsub_rn(bsum, pr) : __dadd_rn(bsum, pr);
      } else {
        if (odd) acc.sub(pr); else acc.add(pr);
      }
    }
  }

  __device__ __forceinline__ void end_body() {
    if constexpr (C::BA) acc.add(bsum);
    if constexpr (C::QF) acc.add2(qs, __dadd_rn(qc, ql));
  }
};

// One compile-time step q (1 <= q < U) of a body: column J = ctz(q).
template <int N, class C, int Q>
__device__ __forceinline__ void static_step(DenseWalk<N, C>& w, double s_mid, int jz) {
  constexpr int J = ctz_c(Q);
  if constexpr (J + 1 < C::LOGU) {
    // direction from bit J+1 of the local index: compile time
    w.template update_static<J, (((Q >> (J + 1)) & 1) == 0) ? 1 : -1>(jz, 0.0);
  } else {
    // J == LOGU-1: direction from bit LOGU of g, fixed per body
    w.template update_static<J, 0>(jz, s_mid);
  }
  // iterate parity == local parity (chunk bases are even): odd -> subtract
  w.fold((Q & 1) != 0, Q == 1);
}

template <int N, class C, int Q, int U>
struct StaticSteps {
  __device__ __forceinline__ static void run(DenseWalk<N, C>& w, double s_mid, int jz) {
    static_step<N, C, Q>(w, s_mid, jz);
    StaticSteps<N, C, Q + 1, U>::run(w, s_mid, jz);
  }
};
template <int N, class C, int U>
struct StaticSteps<N, C, U, U> {
  __device__ __forceinline__ static void run(DenseWalk<N, C>&, double, int) {}
};

// One body, row-major (C::RM): static steps q < U (column ctz(q), direction
// from q or s_mid), step U the run-time column jd with direction sd (sd = 0
// and no fold when the walk's last step is clipped).
template <int N, class C>
__device__ __forceinline__ void body_rm(DenseWalk<N, C>& w, double s_mid, int jz, int jd,
                                        double sd, bool okd) {
  constexpr int LOGU = C::LOGU;
  constexpr int U = 1 << LOGU;
  constexpr int NP = smem_stride<N>();
  const double* cb = w.scols;
  double p[U];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double v = w.x[i];
#pragma unroll
    for (int q = 1; q <= U; ++q) {
      if (q < U) {
        const int J = ctz_c(q);
        const double c = cb[(J + jz) * NP + i];
        if (J + 1 < LOGU) v = (((q >> (J + 1)) & 1) == 0) ? __dadd_rn(v, c) : __dsub_rn(v, c);
        else v = __fma_rn(s_mid, c, v);
      } else {
        v = __fma_rn(sd, cb[jd * NP + i], v);
      }
      if (i == 0) {
        p[q - 1] = v;
      } else if (i < N - 1) {
        p[q - 1] = __dmul_rn(p[q - 1], v);
      } else if (q < U || okd) {
        // FA: the last multiply fused with the body sum, in step order
        const double sp = (q & 1) ? -p[q - 1] : p[q - 1];
        w.bsum = q == 1 ? __dmul_rn(sp, v) : __fma_rn(sp, v, w.bsum);
      }
    }
    w.x[i] = v;
  }
  w.end_body();
}

// Fast QQ body, row-major (C::RM with C::QF): the U double-double products
// advance row by row, then fold in step order exactly as DenseWalk::fold.
template <int N, class C>
__device__ __forceinline__ void body_rm_qf(DenseWalk<N, C>& w, double s_mid, int jz, int jd,
                                           double sd, bool okd) {
  constexpr int LOGU = C::LOGU;
  constexpr int U = 1 << LOGU;
  constexpr int NP = smem_stride<N>();
  const double* cb = w.scols;
  double hi[U], lo[U];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double v = w.x[i];
#pragma unroll
    for (int q = 1; q <= U; ++q) {
      if (q < U) {
        const int J = ctz_c(q);
        const double c = cb[(J + jz) * NP + i];
        if (J + 1 < LOGU) v = (((q >> (J + 1)) & 1) == 0) ? __dadd_rn(v, c) : __dsub_rn(v, c);
        else v = __fma_rn(s_mid, c, v);
      } else {
        v = __fma_rn(sd, cb[jd * NP + i], v);
      }
      if (i == 0) {
        hi[q - 1] = v;  // x_0, multiplied at row 1
      } else if (i == 1) {
        const double h = __dmul_rn(hi[q - 1], v);
        lo[q - 1] = __fma_rn(hi[q - 1], v, -h);
        hi[q - 1] = h;
      } else {
        const double h2 = __dmul_rn(hi[q - 1], v);
        lo[q - 1] = __fma_rn(lo[q - 1], v, __fma_rn(hi[q - 1], v, -h2));
        hi[q - 1] = h2;
      }
    }
    w.x[i] = v;
  }
#pragma unroll
  for (int q = 1; q <= U; ++q) {
    if (q == U && !okd) break;
    double h = hi[q - 1], l = lo[q - 1];
    if (q & 1) {
      h = -h;
      l = -l;
    }
    if (q == 1) {
      w.qs = h;
      w.qc = 0.0;
      w.ql = l;
    } else {
      double e;
      two_sum(w.qs, h, w.qs, e);
      w.qc = __dadd_rn(w.qc, e);
      w.ql = __dadd_rn(w.ql, l);
    }
  }
  w.end_body();
}

// Per-term policy fold (exact modes: no body sums), row-major: the U
// products are the reference's sequential chains (prod = x_0 * x_1 ...; QQ
// from (1, 0) with qq_mul_step, _loops.py:50-87), folded term by term in step
// order -- bit-identical to the step-major walk and to run_range per chunk.
template <int N, class C>
__device__ __forceinline__ void body_rm_exact(DenseWalk<N, C>& w, double s_mid, int jz, int jd,
                                              double sd, bool okd) {
  constexpr int LOGU = C::LOGU;
  constexpr int U = 1 << LOGU;
  constexpr int NP = smem_stride<N>();
  constexpr bool QQ = C::POL == POL_QQ;
  const double* cb = w.scols;
  double ph[U], pl[U];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double v = w.x[i];
#pragma unroll
    for (int q = 1; q <= U; ++q) {
      if (q < U) {
        const int J = ctz_c(q);
        const double c = cb[(J + jz) * NP + i];
        if (J + 1 < LOGU) v = (((q >> (J + 1)) & 1) == 0) ? __dadd_rn(v, c) : __dsub_rn(v, c);
        else v = __fma_rn(s_mid, c, v);
      } else {
        v = __fma_rn(sd, cb[jd * NP + i], v);
      }
      if constexpr (QQ) {
        if (i == 0) {
          ph[q - 1] = 1.0;
          pl[q - 1] = 0.0;
        }
        qq_mul_step(ph[q - 1], pl[q - 1], v);
      } else {
        ph[q - 1] = i == 0 ? v : __dmul_rn(ph[q - 1], v);
      }
    }
    w.x[i] = v;
  }
#pragma unroll
  for (int q = 1; q <= U; ++q) {
    if (q == U && !okd) break;
    if constexpr (QQ) {
      if (q & 1) w.acc.sub2(ph[q - 1], pl[q - 1]); else w.acc.add2(ph[q - 1], pl[q - 1]);
    } else {
      if (q & 1) w.acc.sub(ph[q - 1]); else w.acc.add(ph[q - 1]);
    }
  }
}

// Walk one aligned chunk c (iterates [1 + c*2^k, (c+1)*2^k], clipped at
// g_end) incrementally from its jump-in state, like run_range; returns its
// normalised partial (parallel.py:282-289). In the fast modes the host has
// rounded the inputs onto per-row fixed-point grids (quantize_walk in
// pk_abi.cu), which makes every state of the walk -- and so every DADD of
// the jump-in and of the updates -- exact: x never drifts.
template <int N, class C>
__device__ __forceinline__ dd_t walk_chunk(const double* scols, const double* x0, int k,
                                           uint64_t g_end, uint64_t c) {
  constexpr int LOGU = C::LOGU;
  constexpr int U = 1 << LOGU;
  DenseWalk<N, C> w(scols);
  const uint64_t base = c << k;
  w.jump_in(x0, base);
  const uint64_t nbody = 1ull << (k - LOGU);
  for (uint64_t m = 0; m < nbody; ++m) {
    const uint64_t gb = base + (m << LOGU);
    const double s_mid = flip_on(gb + (U >> 1), LOGU - 1) ? 1.0 : -1.0;
    const int jz = (int)(m >> 62);  // always 0 (m < 2^62) but opaque to ptxas
    // step U of the body: iterate gb + U flips column ctz(gb + U) >= LOGU
    const uint64_t g = gb + U;
    if constexpr (C::RM) {
      const bool ok = (m + 1 < nbody) || g <= g_end;
      const int j = ok ? changed_col(g) : 0;
      const double sd = ok ? (flip_on(g, j) ? 1.0 : -1.0) : 0.0;
      if constexpr (C::QF) body_rm_qf<N, C>(w, s_mid, jz, j, sd, ok);
      else if constexpr (C::FA) body_rm<N, C>(w, s_mid, jz, j, sd, ok);
      else body_rm_exact<N, C>(w, s_mid, jz, j, sd, ok);
      continue;
    }
    StaticSteps<N, C, 1, U>::run(w, s_mid, jz);
    if (m + 1 < nbody || g <= g_end) {
      const int j = changed_col(g);
      w.update_dynamic(j, flip_on(g, j) ? 1.0 : -1.0);
      w.fold(false, false);
    }
    w.end_body();
  }
  return w.acc.partial();
}

// stage the (N-1) x N columns into shared memory with a stride of
// smem_stride<N>() doubles (16-byte aligned rows for LDS.128)
template <int N>
__device__ __forceinline__ void stage_columns(double* scols, const double* cols) {
  constexpr int NP = smem_stride<N>();
  for (int t = threadIdx.x; t < (N - 1) * NP; t += blockDim.x) {
    const int j = t / NP, i = t % NP;
    scols[t] = (i < N) ? cols[j * N + i] : 0.0;
  }
}

template <int N>
__host__ __device__ constexpr size_t dense_cols_doubles() {
  return (size_t)(N - 1) * smem_stride<N>();
}

// fixed-point image of the precise mode (pk_precise.cuh): (N-1) columns at the
// smem stride, X0[N], 2^-F[N]
template <int N>
__host__ __device__ constexpr size_t fix_words() {
  return (size_t)(N - 1) * smem_stride<N>() + 2 * N;
}

// stage the host image (dense [j*N + i] columns, X0, scales) at the smem stride
template <int N>
__device__ __forceinline__ void stage_fix(long long* sfix, const long long* fix) {
  constexpr int NP = smem_stride<N>();
  for (int t = threadIdx.x; t < (N - 1) * NP; t += blockDim.x) {
    const int j = t / NP, i = t % NP;
    sfix[t] = (i < N) ? fix[j * N + i] : 0ll;
  }
  for (int t = threadIdx.x; t < 2 * N; t += blockDim.x)
    sfix[(N - 1) * NP + t] = fix[(N - 1) * N + t];
}

template <int N, class C>
__global__ void __launch_bounds__(C::BLOCK, C::MINB)
    dense_f64_chunks(const __grid_constant__ DenseF64Params<N> p) {
  extern __shared__ __align__(16) double scols[];
  stage_columns<N>(scols, p.cols);
  __syncthreads();
  const unsigned int lane = threadIdx.x & 31u;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t grp = warp; grp < p.num_groups; grp += nwarps) {
    const uint64_t c = p.chunk_lo + grp * 32 + lane;
    dd_t part = walk_chunk<N, C>(scols, p.x0, p.k, p.g_end, c);
    if (p.chunk_part) p.chunk_part[grp * 32 + lane] = part;
    part = warp_tree_dd(part);
    if (lane == 0) p.group_part[grp] = part;
  }
  grid_tail_reduce<C::BLOCK>(p.group_part, p.num_groups, p.out, p.counter);
}

template <int N>
__host__ __device__ constexpr size_t dense_smem_bytes() {
  return sizeof(double) * dense_cols_doubles<N>();
}

// ---------------------------------------------------------------------------
// batched walks: many matrices of one order, one block per matrix at a time
// (decomposition leaves, boson-sampling submatrices). Each
// matrix is split into 2^(n-1-k) aligned chunks walked by the block's warps;
// its partial is the same fixed tree over its groups as a single launch.

template <int N>
struct DenseBatchParams {
  const double* cols;   // [batch][(N-1)*N]
  const double* x0;     // [batch][N]
  dd_t* group_part;     // [batch][groups] scratch
  dd_t* out;            // [batch] partial over [1, 2^(N-1)-1]
  int batch;
  int k;
};

template <int N, class C>
__global__ void __launch_bounds__(C::BLOCK, C::MINB)
    dense_f64_batch(const __grid_constant__ DenseBatchParams<N> p) {
  extern __shared__ __align__(16) double smem[];
  double* scols = smem;
  double* sx0 = smem + dense_cols_doubles<N>();
  const uint64_t total = (1ull << (N - 1)) - 1;
  const int groups = (int)((1ull << (N - 1 - p.k)) / 32);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  for (int b = blockIdx.x; b < p.batch; b += gridDim.x) {
    __syncthreads();
    stage_columns<N>(scols, p.cols + (size_t)b * (N - 1) * N);
    for (int i = threadIdx.x; i < N; i += blockDim.x) sx0[i] = p.x0[(size_t)b * N + i];
    __syncthreads();
    dd_t* gp = p.group_part + (size_t)b * groups;
    for (int grp = wib; grp < groups; grp += wpb) {
      dd_t part = walk_chunk<N, C>(scols, sx0, p.k, total, (uint64_t)grp * 32 + lane);
      part = warp_tree_dd(part);
      if (lane == 0) gp[grp] = part;
    }
    __syncthreads();
    if (threadIdx.x == 0) p.out[b] = pairwise_fold(gp, 0, groups);
  }
}

}  // namespace pk
