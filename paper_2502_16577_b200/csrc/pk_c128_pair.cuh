// K3p: dense complex fp64 Gray walk with each chunk's rows split over a lane
// pair -- the complex kernel for every order up to 63.
//
// Replaces chunk_dense_c128 (/root/reference/pkg/src/permkit/_loops.py:186-209)
// under run_range (parallel.py:232-289), like K3 (pk_dense_c128.cuh), whose
// one-thread-per-chunk state (4N registers) stops fitting the register file
// above N = 40. Here lane A (even lane) holds rows 0..H-1 and lane B (odd
// lane) rows H..N-1 of the same chunk, H = ceil(N/2): 4H registers of state.
//
// Two product schedules (template EXACT):
//   fast  -- both lanes walk the same step; A multiplies the product of its
//            rows, B of its rows (fma form, 4 FP64 ops per complex multiply),
//            and B combines the halves with one shuffle and four DFMAs that
//            also add the term to the body sum. The halves of consecutive
//            steps are independent, so their chains overlap. The inputs are
//            grid-rounded on the host (pk_abi.cu quantize_walk): every state
//            is exact. Terms are summed per body of U and folded with
//            compensation (CAcc<false>).
//   EXACT -- the reference's sequential product: lane A multiplies the prefix
//            prod = ((1 * x_0) * x_1) ... * x_{H-1} of step t and hands it to
//            lane B, which continues the same chain over its rows one step
//            later (B's rows run one Gray step behind A's). Both lanes execute
//            the same instruction stream on different rows: at step t A applies
//            update t and multiplies the prefix of term t while B applies update
//            t-1 and finishes term t-1, which it folds with the reference's
//            per-term sums (CAcc<true>). Chunk partials are bit-identical to
//            run_range over the chunk; a chunk of 2^k steps takes 2^k + 1 pair
//            steps (one drain step for B).
// With odd N, lane B's last row is a dummy (1 + 0i, zero column entries).
#pragma once
#include "pk_common.cuh"
#include "pk_dense_c128.cuh"
#include "pk_reduce.cuh"

namespace pk {

template <int N>
__host__ __device__ constexpr int pair_rows() { return (N + 1) / 2; }
// complex entries per staged column: A's rows, then B's rows (dummy padded)
template <int N>
__host__ __device__ constexpr int pair_col_stride() { return 2 * pair_rows<N>(); }

// staged columns, then x0 at the pair stride (dummy row 1 + 0i)
template <int N>
__host__ __device__ constexpr size_t pair_smem_bytes() {
  return sizeof(double) * 2 * (size_t)N * pair_col_stride<N>();
}

template <int N>
struct C128PairParams {
  double x0[2 * N];      // interleaved (re, im)
  const double* cols;    // device, cols[(j*N + i)*2 + {0,1}], j < N-1
  dd_t* group_part;
  dd_t* chunk_part;
  dd_t* out;
  unsigned int* counter;
  unsigned long long chunk_lo;
  unsigned long long num_groups;
  unsigned long long g_end;
  int k;
};

template <int N, class C>
struct C128Pair {
  static constexpr int H = pair_rows<N>();
  static constexpr int CS = pair_col_stride<N>();
  const double* scols;
  int half;  // 0: lane A (rows 0..H-1), 1: lane B (rows H..2H-1)
  double xr[H], xi[H];
  CAcc<C::EXACT> acc;
  double br = 0.0, bi = 0.0;  // fast mode: running sum of the current body (B)
  double rr = 0.0, ri = 0.0;  // B: prefix received from A for its next term

  // x += s * column j over this lane's rows (j < 0: no update)
  __device__ __forceinline__ void update(int j, double s) {
    if (j < 0) return;
    const double2* c2 = reinterpret_cast<const double2*>(scols) + j * CS + half * H;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const double2 v = c2[i];
      if constexpr (C::EXACT) {
        c_update_ref(xr[i], xi[i], s, v.x, v.y);
      } else {
        xr[i] = __fma_rn(s, v.x, xr[i]);
        xi[i] = __fma_rn(s, v.y, xi[i]);
      }
    }
  }

  // A: prefix of the current term from (1, 0); B: the received prefix times
  // its rows = the whole product of its (one step older) term
  __device__ __forceinline__ void chain(double& pr, double& pi) const {
    pr = half ? rr : 1.0;
    pi = half ? ri : 0.0;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      double r, m;
      if constexpr (C::EXACT) {
        cmul_ref(pr, pi, xr[i], xi[i], r, m);
      } else {
        r = __fma_rn(pr, xr[i], -__dmul_rn(pi, xi[i]));
        m = __fma_rn(pr, xi[i], __dmul_rn(pi, xr[i]));
      }
      pr = r;
      pi = m;
    }
  }

  // one lane-pair step: A does (jA, sA), B does (jB, sB) one step behind; B
  // folds its finished term when `valid` (odd iterate: subtract)
  // jz is always 0 but opaque to ptxas (K1's trick): it keeps the static
  // columns' loads inside the body loop instead of hoisting them to registers
  __device__ __forceinline__ void step(int jA, double sA, int jB, double sB, bool valid,
                                       bool odd, bool first, int jz) {
    const int j = half ? jB : jA;
    update(j < 0 ? j : j + jz, half ? sB : sA);
    double pr, pi;
    chain(pr, pi);
    if (half && valid) {
      if constexpr (C::EXACT) {
        if (odd) acc.sub(pr, pi); else acc.add(pr, pi);
      } else {
        if (odd) {
          pr = -pr;
          pi = -pi;
        }
        if (first) {
          br = pr;
          bi = pi;
        } else {
          br = __dadd_rn(br, pr);
          bi = __dadd_rn(bi, pi);
        }
      }
    }
    rr = __shfl_xor_sync(0xffffffffu, pr, 1);
    ri = __shfl_xor_sync(0xffffffffu, pi, 1);
  }

  __device__ __forceinline__ void flush() {
    if constexpr (!C::EXACT) {
      if (half) acc.add(br, bi);
      br = 0.0;
      bi = 0.0;
    }
  }
};

// static sign of step q (1 <= q < U) whose column J = ctz(q) has J + 1 < LOGU
template <int Q>
__host__ __device__ constexpr double pair_static_sign() {
  return (((Q >> (ctz_c(Q) + 1)) & 1) == 0) ? 1.0 : -1.0;
}

// column / sign of local step q (1 <= q < U) of a body with body-uniform s_mid
template <int Q, int LOGU>
__device__ __forceinline__ double pair_sign(double s_mid) {
  if constexpr (ctz_c(Q) + 1 < LOGU) return pair_static_sign<Q>();
  else return s_mid;
}

template <int N, class C, int Q, int U>
struct PairSteps {
  // steps 2..U-1 of a body: both lanes static (A: q, B: q - 1)
  __device__ __forceinline__ static void run(C128Pair<N, C>& w, double s_mid, bool first_body,
                                             int jz) {
    w.step(ctz_c(Q), pair_sign<Q, C::LOGU>(s_mid), ctz_c(Q - 1),
           pair_sign<Q - 1, C::LOGU>(s_mid), true, ((Q - 1) & 1) != 0,
           first_body && Q == 2, jz);
    PairSteps<N, C, Q + 1, U>::run(w, s_mid, first_body, jz);
  }
};
template <int N, class C, int U>
struct PairSteps<N, C, U, U> {
  __device__ __forceinline__ static void run(C128Pair<N, C>&, double, bool, int) {}
};

// one aligned chunk c (iterates [1 + c*2^k, (c+1)*2^k], clipped at g_end);
// the partial is on lane B (lane A returns zero)
template <int N, class C>
__device__ __forceinline__ dd_t pair_walk_chunk(const double* x0, int k, uint64_t g_end,
                                                const double* scols, uint64_t c, int half) {
  constexpr int LOGU = C::LOGU;
  constexpr int U = 1 << LOGU;
  constexpr int H = pair_rows<N>();
  C128Pair<N, C> w;
  w.scols = scols;
  w.half = half;
  const uint64_t base = c << k;
#pragma unroll
  for (int i = 0; i < H; ++i) {  // x0 staged at the pair stride (dummy row 1 + 0i)
    w.xr[i] = x0[2 * (half * H + i)];
    w.xi[i] = x0[2 * (half * H + i) + 1];
  }
  // jump-in: x0 + columns of gray(base), ascending (parallel.py:162-188)
  const uint64_t code = base ^ (base >> 1);
  for (int j = 0; j < N - 1; ++j) {
    if ((code >> j) & 1ull) {
      const double2* c2 = reinterpret_cast<const double2*>(scols) + j * (2 * H) + half * H;
#pragma unroll
      for (int i = 0; i < H; ++i) {
        const double2 v = c2[i];
        w.xr[i] = __dadd_rn(w.xr[i], v.x);
        w.xi[i] = __dadd_rn(w.xi[i], v.y);
      }
    }
  }
  const uint64_t nbody = 1ull << (k - LOGU);
  int jprev = -1;        // A's last (dynamic) column: B applies it one step later
  double sprev = 1.0;
  bool last_ok = false;  // A's last step was within the walk
  for (uint64_t m = 0; m < nbody; ++m) {
    const uint64_t gb = base + (m << LOGU);
    const double s_mid = flip_on(gb + (U >> 1), LOGU - 1) ? 1.0 : -1.0;
    const bool first_body = (m == 0);
    const int jz = (int)(m >> 62);
    // q = 1: A static column 0, B the previous body's dynamic step (iterate gb)
    w.step(0, pair_sign<1, LOGU>(s_mid), jprev, sprev, !first_body, false, true, jz);
    PairSteps<N, C, 2, U>::run(w, s_mid, first_body, jz);
    // q = U: A the dynamic column of iterate gb + U, B static column 0 (iterate gb + U - 1)
    const uint64_t g = gb + U;
    last_ok = (m + 1 < nbody) || g <= g_end;
    jprev = last_ok ? changed_col(g) : -1;
    sprev = last_ok && flip_on(g, jprev) ? 1.0 : -1.0;
    w.step(jprev, sprev, 0, pair_sign<U - 1, LOGU>(s_mid), true, true,
           first_body && U == 2, jz);
    // body boundary: B has folded the terms of iterates gb .. gb + U - 1
    // (gb + 1 .. gb + U - 1 in the first body)
    w.flush();
  }
  // drain: B finishes the chunk's last term (iterate base + 2^k)
  w.step(-1, 1.0, jprev, sprev, last_ok, false, true, 0);
  w.flush();
  if (!half) return dd_t{0.0, 0.0};
  return w.acc.partial();
}

// fast schedule: both lanes at the same step, independent half products
template <int N, class C>
struct C128PairFast {
  static constexpr int H = pair_rows<N>();
  static constexpr int CS = pair_col_stride<N>();
  const double* scols;
  int half;
  double xr[H], xi[H];
  CAcc<false> acc;
  double br = 0.0, bi = 0.0;

  template <int SIGN>
  __device__ __forceinline__ void update_static(int j) {
    const double2* c2 = reinterpret_cast<const double2*>(scols) + j * CS + half * H;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const double2 v = c2[i];
      xr[i] = SIGN > 0 ? __dadd_rn(xr[i], v.x) : __dsub_rn(xr[i], v.x);
      xi[i] = SIGN > 0 ? __dadd_rn(xi[i], v.y) : __dsub_rn(xi[i], v.y);
    }
  }

  __device__ __forceinline__ void update(int j, double s) {
    const double2* c2 = reinterpret_cast<const double2*>(scols) + j * CS + half * H;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const double2 v = c2[i];
      xr[i] = __fma_rn(s, v.x, xr[i]);
      xi[i] = __fma_rn(s, v.y, xi[i]);
    }
  }

  // this lane's half product; B adds (+-)(A's half) * (its half) to the body
  // sum. Every lane of the warp must call it (shuffle); `valid` false leaves
  // the sum unchanged (the clipped last step of the walk).
  __device__ __forceinline__ void fold(bool odd, bool first, bool valid = true) {
    double pr = xr[0], pi = xi[0];
#pragma unroll
    for (int i = 1; i < H; ++i) {
      const double r = __fma_rn(pr, xr[i], -__dmul_rn(pi, xi[i]));
      const double m = __fma_rn(pr, xi[i], __dmul_rn(pi, xr[i]));
      pr = r;
      pi = m;
    }
    double ar = __shfl_xor_sync(0xffffffffu, pr, 1);
    double ai = __shfl_xor_sync(0xffffffffu, pi, 1);
    if (odd) {
      ar = -ar;
      ai = -ai;
    }
    const double r0 = first ? 0.0 : br, i0 = first ? 0.0 : bi;
    const double nr = __fma_rn(ar, pr, __fma_rn(-ai, pi, r0));
    const double ni = __fma_rn(ar, pi, __fma_rn(ai, pr, i0));
    br = valid ? nr : br;
    bi = valid ? ni : bi;
  }
};

template <int N, class C, int Q>
__device__ __forceinline__ void pair_fast_step(C128PairFast<N, C>& w, double s_mid, int jz) {
  constexpr int J = ctz_c(Q);
  if constexpr (J + 1 < C::LOGU) {
    w.template update_static<(((Q >> (J + 1)) & 1) == 0) ? 1 : -1>(J + jz);
  } else {
    w.update(J + jz, s_mid);
  }
  w.fold((Q & 1) != 0, Q == 1);
}

template <int N, class C, int Q, int U>
struct PairFastSteps {
  __device__ __forceinline__ static void run(C128PairFast<N, C>& w, double s_mid, int jz) {
    pair_fast_step<N, C, Q>(w, s_mid, jz);
    PairFastSteps<N, C, Q + 1, U>::run(w, s_mid, jz);
  }
};
template <int N, class C, int U>
struct PairFastSteps<N, C, U, U> {
  __device__ __forceinline__ static void run(C128PairFast<N, C>&, double, int) {}
};

// one body of the fast schedule, row-major (C::RM, as K3's c128_body_rm):
// each lane forms the U states of its rows one after the other and advances
// U independent half products; then per step, in order, the shuffle and the
// combine-and-sum. Same arithmetic and order as the step-major body.
template <int N, class C>
__device__ __forceinline__ void pair_body_rm(C128PairFast<N, C>& w, double s_mid, int jz, int jd,
                                             double sd, bool okd) {
  constexpr int LOGU = C::LOGU;
  constexpr int U = 1 << LOGU;
  constexpr int H = pair_rows<N>();
  constexpr int CS = pair_col_stride<N>();
  const double2* cb = reinterpret_cast<const double2*>(w.scols) + w.half * H;
  double pr[U], pi[U];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    double vr = w.xr[i], vi = w.xi[i];
#pragma unroll
    for (int q = 1; q <= U; ++q) {
      if (q < U) {
        const int J = ctz_c(q);
        const double2 v = cb[(J + jz) * CS + i];
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
        const double2 v = cb[jd * CS + i];
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
  // combine the halves term by term (independent), then sum the body's U
  // terms as a pairwise tree: dependency depth 2 + log2(U) instead of 2U
  double tr[U], ti[U];
#pragma unroll
  for (int q = 1; q <= U; ++q) {
    double ar = __shfl_xor_sync(0xffffffffu, pr[q - 1], 1);
    double ai = __shfl_xor_sync(0xffffffffu, pi[q - 1], 1);
    if (q & 1) {
      ar = -ar;
      ai = -ai;
    }
    const bool valid = q < U || okd;
    tr[q - 1] = valid ? __fma_rn(ar, pr[q - 1], -__dmul_rn(ai, pi[q - 1])) : 0.0;
    ti[q - 1] = valid ? __fma_rn(ar, pi[q - 1], __dmul_rn(ai, pr[q - 1])) : 0.0;
  }
#pragma unroll
  for (int w2 = 1; w2 < U; w2 <<= 1)
#pragma unroll
    for (int q = 0; q + w2 < U; q += 2 * w2) {
      tr[q] = __dadd_rn(tr[q], tr[q + w2]);
      ti[q] = __dadd_rn(ti[q], ti[q + w2]);
    }
  w.br = tr[0];
  w.bi = ti[0];
}

template <int N, class C>
__device__ __forceinline__ dd_t pair_walk_chunk_fast(const double* x0, int k, uint64_t g_end,
                                                     const double* scols, uint64_t c,
                                                     int half) {
  constexpr int LOGU = C::LOGU;
  constexpr int U = 1 << LOGU;
  constexpr int H = pair_rows<N>();
  C128PairFast<N, C> w;
  w.scols = scols;
  w.half = half;
  const uint64_t base = c << k;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    w.xr[i] = x0[2 * (half * H + i)];
    w.xi[i] = x0[2 * (half * H + i) + 1];
  }
  const uint64_t code = base ^ (base >> 1);
  for (int j = 0; j < N - 1; ++j) {
    if ((code >> j) & 1ull) {
      const double2* c2 = reinterpret_cast<const double2*>(scols) + j * (2 * H) + half * H;
#pragma unroll
      for (int i = 0; i < H; ++i) {
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
    // step U: iterate gb + U flips column ctz(gb + U); the lanes of a warp
    // walk different chunks, so the walk's clipped last step is predicated
    // (s = 0 leaves x unchanged) rather than branched around the shuffle
    const uint64_t g = gb + U;
    const bool ok = (m + 1 < nbody) || g <= g_end;
    const int j = ok ? changed_col(g) : 0;
    if constexpr (C::RM) {
      pair_body_rm<N, C>(w, s_mid, jz, j, ok ? (flip_on(g, j) ? 1.0 : -1.0) : 0.0, ok);
    } else {
      PairFastSteps<N, C, 1, U>::run(w, s_mid, jz);
      w.update(j, ok ? (flip_on(g, j) ? 1.0 : -1.0) : 0.0);
      w.fold(false, false, ok);
    }
    if (half) w.acc.add(w.br, w.bi);
  }
  if (!half) return dd_t{0.0, 0.0};
  return w.acc.partial();
}

// stage the columns at the pair stride (dummy rows zero) and x0 after them
// (dummy row 1 + 0i)
template <int N>
__device__ __forceinline__ void pair_stage(double* scols, const double* cols, const double* x0) {
  constexpr int CS = pair_col_stride<N>();
  for (int t = threadIdx.x; t < (N - 1) * CS; t += blockDim.x) {
    const int j = t / CS, r = t % CS;
    scols[2 * t] = r < N ? cols[2 * (j * N + r)] : 0.0;
    scols[2 * t + 1] = r < N ? cols[2 * (j * N + r) + 1] : 0.0;
  }
  double* sx0 = scols + 2 * (N - 1) * CS;
  for (int r = threadIdx.x; r < CS; r += blockDim.x) {
    sx0[2 * r] = r < N ? x0[2 * r] : 1.0;
    sx0[2 * r + 1] = r < N ? x0[2 * r + 1] : 0.0;
  }
}

// Each warp walks a group of 32 chunks in two passes of 16 lane pairs; the
// chunk partials are then moved so lane l holds chunk l's partial and reduced
// by the same warp tree as K3 -- both kernels give the same group partials.
template <int N, class C>
__global__ void __launch_bounds__(C::BLOCK, C::MINB)
    dense_c128_pair(const __grid_constant__ C128PairParams<N> p) {
  extern __shared__ __align__(16) double scols[];
  pair_stage<N>(scols, p.cols, p.x0);
  __syncthreads();
  const double* sx0 = scols + 2 * (N - 1) * pair_col_stride<N>();
  const unsigned int lane = threadIdx.x & 31u;
  const int half = (int)(lane & 1u);
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t grp = warp; grp < p.num_groups; grp += nwarps) {
    dd_t part[2];
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      const uint64_t c = p.chunk_lo + grp * 32 + pass * 16 + (lane >> 1);
      if constexpr (C::EXACT)
        part[pass] = pair_walk_chunk<N, C>(sx0, p.k, p.g_end, scols, c, half);
      else
        part[pass] = pair_walk_chunk_fast<N, C>(sx0, p.k, p.g_end, scols, c, half);
    }
    // lane l <- chunk l's partial (held by lane 2(l mod 16) + 1 of pass l / 16)
    const int src = 2 * (int)(lane & 15u) + 1;
    const double r0 = __shfl_sync(0xffffffffu, part[0].hi, src);
    const double i0 = __shfl_sync(0xffffffffu, part[0].lo, src);
    const double r1 = __shfl_sync(0xffffffffu, part[1].hi, src);
    const double i1 = __shfl_sync(0xffffffffu, part[1].lo, src);
    const dd_t mine = lane < 16 ? dd_t{r0, i0} : dd_t{r1, i1};
    if (p.chunk_part) p.chunk_part[grp * 32 + lane] = mine;
    dd_t re{mine.hi, 0.0}, im{mine.lo, 0.0};
    warp_tree_cdd(re, im);
    if (lane == 0) {
      p.group_part[2 * grp] = re;
      p.group_part[2 * grp + 1] = im;
    }
  }
  grid_tail_reduce_pairs<C::BLOCK>(p.group_part, p.num_groups, p.out, p.counter);
}

// batched whole walks (boson-sampling submatrices, decomposition leaves) of
// order 41..63: one block per matrix at a time, its 2^(N-1-k) aligned chunks
// walked by the block's warps in the single launch's lane-pair layout and
// folded with the same trees, so a batch entry equals the single walk of the
// same chunk exponent bit for bit (as dense_c128_batch does for K3)
template <int N, class C>
__global__ void __launch_bounds__(C::BLOCK, C::MINB)
    dense_c128_pair_batch(const __grid_constant__ C128BatchParams<N> p) {
  extern __shared__ __align__(16) double scols[];
  const double* sx0 = scols + 2 * (N - 1) * pair_col_stride<N>();
  const uint64_t total = (1ull << (N - 1)) - 1;
  const int groups = (int)((1ull << (N - 1 - p.k)) / 32);
  const unsigned int lane = threadIdx.x & 31u;
  const int half = (int)(lane & 1u);
  const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  for (int b = blockIdx.x; b < p.batch; b += gridDim.x) {
    __syncthreads();
    pair_stage<N>(scols, p.cols + (size_t)b * 2 * (N - 1) * N, p.x0 + (size_t)b * 2 * N);
    __syncthreads();
    dd_t* gp = p.group_part + (size_t)b * 2 * groups;
    for (int grp = wib; grp < groups; grp += wpb) {
      dd_t part[2];
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        const uint64_t c = (uint64_t)grp * 32 + pass * 16 + (lane >> 1);
        if constexpr (C::EXACT)
          part[pass] = pair_walk_chunk<N, C>(sx0, p.k, total, scols, c, half);
        else
          part[pass] = pair_walk_chunk_fast<N, C>(sx0, p.k, total, scols, c, half);
      }
      const int src = 2 * (int)(lane & 15u) + 1;
      const double r0 = __shfl_sync(0xffffffffu, part[0].hi, src);
      const double i0 = __shfl_sync(0xffffffffu, part[0].lo, src);
      const double r1 = __shfl_sync(0xffffffffu, part[1].hi, src);
      const double i1 = __shfl_sync(0xffffffffu, part[1].lo, src);
      const dd_t mine = lane < 16 ? dd_t{r0, i0} : dd_t{r1, i1};
      dd_t re{mine.hi, 0.0}, im{mine.lo, 0.0};
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
