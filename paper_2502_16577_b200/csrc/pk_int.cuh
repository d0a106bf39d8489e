// K5/K6: exact integer Gray walk (0/1 matching counts, SpaRyser binary).
//
// Replaces chunk_dense_int / chunk_sparse_int (/root/reference/pkg/src/
// permkit/_loops.py:238-284), which walk the doubled state y = 2x in Python
// big ints (kernels.py:104-163). Here the state is rescaled per row to
//     z_i = y_i / 2  if row sum r_i is even,   z_i = y_i  if r_i is odd,
// which is an integer either way and saves one bit per even row; the host
// multiplies the range total by 2^(#even rows) to return the reference's
// y-space partial. z lives in int32 registers; the product of the n row
// values is formed exactly in a widening tree -- groups of G values in
// int32 (G = 31 / ZB, |z| < 2^ZB), pairs of groups in int64 (IMAD.WIDE),
// pairs of those in int128, the rest multiplied mod 2^128 -- and folded into
// a 192-bit accumulator. The host guarantees exactness: every term is below
// 2^127 in magnitude (product of the per-row bounds) and no partial can pass
// 2^191; otherwise it takes the modular full-walk route or refuses.
//
// Integer arithmetic is associative, so chunk partials, trees and device
// splits all give the same exact value as the reference's sequential walk.
#pragma once
#include "pk_common.cuh"

namespace pk {

constexpr int kIntBlock = 128;

struct i192 {
  unsigned long long w0, w1, w2;
};

__device__ __forceinline__ void i192_add128(i192& a, unsigned long long lo, unsigned long long hi) {
  const unsigned long long ext = (unsigned long long)((long long)hi >> 63);
  asm("add.cc.u64 %0, %0, %3;\n\t"
      "addc.cc.u64 %1, %1, %4;\n\t"
      "addc.u64 %2, %2, %5;"
      : "+l"(a.w0), "+l"(a.w1), "+l"(a.w2)
      : "l"(lo), "l"(hi), "l"(ext));
}

__device__ __forceinline__ void i192_sub128(i192& a, unsigned long long lo, unsigned long long hi) {
  const unsigned long long ext = (unsigned long long)((long long)hi >> 63);
  asm("sub.cc.u64 %0, %0, %3;\n\t"
      "subc.cc.u64 %1, %1, %4;\n\t"
      "subc.u64 %2, %2, %5;"
      : "+l"(a.w0), "+l"(a.w1), "+l"(a.w2)
      : "l"(lo), "l"(hi), "l"(ext));
}

__device__ __forceinline__ void i192_add(i192& a, const i192& b) {
  asm("add.cc.u64 %0, %0, %3;\n\t"
      "addc.cc.u64 %1, %1, %4;\n\t"
      "addc.u64 %2, %2, %5;"
      : "+l"(a.w0), "+l"(a.w1), "+l"(a.w2)
      : "l"(b.w0), "l"(b.w1), "l"(b.w2));
}

__device__ __forceinline__ i192 shfl_down_i192(const i192& v, int off) {
  i192 r;
  r.w0 = __shfl_down_sync(0xffffffffu, v.w0, off);
  r.w1 = __shfl_down_sync(0xffffffffu, v.w1, off);
  r.w2 = __shfl_down_sync(0xffffffffu, v.w2, off);
  return r;
}

__device__ __forceinline__ i192 warp_sum_i192(i192 v) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const i192 o = shfl_down_i192(v, off);
    if (((threadIdx.x & 31) & (2 * off - 1)) == 0) i192_add(v, o);
  }
  return v;
}

// exact product of the N row values (mod 2^128; exact when |product| < 2^127)
template <int N, int ZB>
__device__ __forceinline__ unsigned __int128 z_product(const int (&z)[N]) {
  constexpr int G = 31 / ZB;            // values per int32 group
  constexpr int NG = (N + G - 1) / G;   // int32 groups
  constexpr int NH = (NG + 1) / 2;      // int64 pairs
  constexpr int NQ = (NH + 1) / 2;      // int128 pairs
  int g[NG];
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    g[k] = z[k * G];
#pragma unroll
    for (int t = 1; t < G; ++t)
      if (k * G + t < N) g[k] *= z[k * G + t];
  }
  long long h[NH];
#pragma unroll
  for (int k = 0; k < NH; ++k)
    h[k] = (2 * k + 1 < NG) ? (long long)g[2 * k] * (long long)g[2 * k + 1] : (long long)g[2 * k];
  __int128 q[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k)
    q[k] = (2 * k + 1 < NH) ? (__int128)h[2 * k] * (__int128)h[2 * k + 1] : (__int128)h[2 * k];
  unsigned __int128 p = (unsigned __int128)q[0];
#pragma unroll
  for (int k = 1; k < NQ; ++k) p *= (unsigned __int128)q[k];
  return p;
}

template <int N>
struct IntParams {
  int z0[N];                 // z-space seed
  const int* cols;           // device, z-space column steps cols[j*N + i], j < N-1
  i192* group_part;          // [num_groups]
  i192* chunk_part;          // optional [num_groups*32]
  i192* out;                 // launch total
  unsigned int* counter;
  unsigned long long chunk_lo;
  unsigned long long num_groups;
  unsigned long long g_end;
  int k;
};

template <int ZB_, int LOGU_, int MINB_>
struct IntCfg {
  static constexpr int ZB = ZB_, LOGU = LOGU_, MINB = MINB_;
};

template <int N>
__host__ __device__ constexpr int int_stride() { return (N + 3) & ~3; }

template <int N, class C>
struct IntWalk {
  const int* scols;  // shared, stride int_stride<N>()
  int z[N];
  i192 acc{0ull, 0ull, 0ull};

  template <int SIGN>
  __device__ __forceinline__ void update_static(const int* col) {
    const int4* c4 = reinterpret_cast<const int4*>(col);
#pragma unroll
    for (int i = 0; i < N; i += 4) {
      const int4 v = c4[i / 4];
      const int vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (i + t < N) z[i + t] = SIGN > 0 ? z[i + t] + vv[t] : z[i + t] - vv[t];
    }
  }

  __device__ __forceinline__ void update(const int* col, int s) {
    const int4* c4 = reinterpret_cast<const int4*>(col);
#pragma unroll
    for (int i = 0; i < N; i += 4) {
      const int4 v = c4[i / 4];
      const int vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (i + t < N) z[i + t] += s * vv[t];
    }
  }

  __device__ __forceinline__ void fold(bool odd) {
    const unsigned __int128 p = z_product<N, C::ZB>(z);
    const unsigned long long lo = (unsigned long long)p, hi = (unsigned long long)(p >> 64);
    if (odd) i192_sub128(acc, lo, hi); else i192_add128(acc, lo, hi);
  }
};

template <int N, class C, int Q>
__device__ __forceinline__ void int_static_step(IntWalk<N, C>& w, int s_mid, int jz) {
  constexpr int J = ctz_c(Q);
  const int* col = w.scols + (J + jz) * int_stride<N>();
  if constexpr (J + 1 < C::LOGU) {
    w.template update_static<(((Q >> (J + 1)) & 1) == 0) ? 1 : -1>(col);
  } else {
    w.update(col, s_mid);
  }
  w.fold((Q & 1) != 0);
}

template <int N, class C, int Q, int U>
struct IntSteps {
  __device__ __forceinline__ static void run(IntWalk<N, C>& w, int s_mid, int jz) {
    int_static_step<N, C, Q>(w, s_mid, jz);
    IntSteps<N, C, Q + 1, U>::run(w, s_mid, jz);
  }
};
template <int N, class C, int U>
struct IntSteps<N, C, U, U> {
  __device__ __forceinline__ static void run(IntWalk<N, C>&, int, int) {}
};

template <int N, class C>
__device__ __forceinline__ i192 int_walk_chunk(const int* z0, int k, uint64_t g_end,
                                               const int* scols, uint64_t c) {
  constexpr int LOGU = C::LOGU;
  constexpr int U = 1 << LOGU;
  constexpr int NP = int_stride<N>();
  IntWalk<N, C> w;
  w.scols = scols;
  const uint64_t base = c << k;
#pragma unroll
  for (int i = 0; i < N; ++i) w.z[i] = z0[i];
  const uint64_t code = base ^ (base >> 1);
  for (int j = 0; j < N - 1; ++j)
    if ((code >> j) & 1ull) w.template update_static<1>(scols + j * NP);
  const uint64_t nbody = 1ull << (k - LOGU);
  for (uint64_t m = 0; m < nbody; ++m) {
    const uint64_t gb = base + (m << LOGU);
    const int s_mid = flip_on(gb + (U >> 1), LOGU - 1) ? 1 : -1;
    const int jz = (int)(m >> 62);
    IntSteps<N, C, 1, U>::run(w, s_mid, jz);
    const uint64_t g = gb + U;
    if (m + 1 < nbody || g <= g_end) {
      const int j = changed_col(g);
      w.update(scols + j * NP, flip_on(g, j) ? 1 : -1);
      w.fold(false);
    }
  }
  return w.acc;
}

// last block sums the group partials (any order gives the same integer;
// the fixed order keeps it reproducible anyway)
template <int BLOCK>
__device__ inline void grid_tail_sum_i192(const i192* parts, uint64_t count, i192* out,
                                          unsigned int* counter) {
  __shared__ bool is_last;
  __shared__ i192 tree[BLOCK];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const unsigned t = threadIdx.x;
  i192 s{0ull, 0ull, 0ull};
  for (uint64_t i = t; i < count; i += BLOCK) {
    i192 v;
    v.w0 = __ldcg(&parts[i].w0);
    v.w1 = __ldcg(&parts[i].w1);
    v.w2 = __ldcg(&parts[i].w2);
    i192_add(s, v);
  }
  tree[t] = s;
  __syncthreads();
  for (unsigned w = BLOCK / 2; w > 0; w >>= 1) {
    if (t < w) i192_add(tree[t], tree[t + w]);
    __syncthreads();
  }
  if (t == 0) {
    *out = tree[0];
    *counter = 0u;
  }
}

template <int N, class C>
__global__ void __launch_bounds__(kIntBlock, C::MINB) int_chunks(const __grid_constant__ IntParams<N> p) {
  constexpr int NP = int_stride<N>();
  __shared__ __align__(16) int scols[(N - 1) * NP];
  for (int t = threadIdx.x; t < (N - 1) * NP; t += blockDim.x) {
    const int j = t / NP, i = t % NP;
    scols[t] = (i < N) ? p.cols[j * N + i] : 0;
  }
  __syncthreads();
  const unsigned int lane = threadIdx.x & 31u;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t grp = warp; grp < p.num_groups; grp += nwarps) {
    const uint64_t c = p.chunk_lo + grp * 32 + lane;
    i192 part = int_walk_chunk<N, C>(p.z0, p.k, p.g_end, scols, c);
    if (p.chunk_part) p.chunk_part[grp * 32 + lane] = part;
    part = warp_sum_i192(part);
    if (lane == 0) p.group_part[grp] = part;
  }
  grid_tail_sum_i192<kIntBlock>(p.group_part, p.num_groups, p.out, p.counter);
}

// batched whole walks of `batch` integer matrices of order N (decomposition
// leaves): one block per matrix at a time, 2^(N-1-k) aligned chunks per
// matrix; the matrix total is an exact sum, so any order gives its value
template <int N>
struct IntBatchParams {
  const int* cols;  // [batch][(N-1)*N] z-space column steps
  const int* z0;    // [batch][N]
  i192* group_part; // [batch][groups] scratch
  i192* out;        // [batch] z-space partial over [1, 2^(N-1)-1]
  int batch;
  int k;
};

template <int N, class C>
__global__ void __launch_bounds__(kIntBlock, C::MINB) int_batch(const __grid_constant__ IntBatchParams<N> p) {
  constexpr int NP = int_stride<N>();
  __shared__ __align__(16) int scols[(N - 1) * NP];
  __shared__ int sz0[N];
  const uint64_t total = (1ull << (N - 1)) - 1;
  const int groups = (int)((1ull << (N - 1 - p.k)) / 32);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  for (int b = blockIdx.x; b < p.batch; b += gridDim.x) {
    __syncthreads();
    const int* cb = p.cols + (size_t)b * (N - 1) * N;
    for (int t = threadIdx.x; t < (N - 1) * NP; t += blockDim.x) {
      const int j = t / NP, i = t % NP;
      scols[t] = (i < N) ? cb[j * N + i] : 0;
    }
    for (int t = threadIdx.x; t < N; t += blockDim.x) sz0[t] = p.z0[(size_t)b * N + t];
    __syncthreads();
    i192* gp = p.group_part + (size_t)b * groups;
    for (int grp = wib; grp < groups; grp += wpb) {
      i192 part = int_walk_chunk<N, C>(sz0, p.k, total, scols, (uint64_t)grp * 32 + lane);
      part = warp_sum_i192(part);
      if (lane == 0) gp[grp] = part;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      i192 s{0ull, 0ull, 0ull};
      for (int g = 0; g < groups; ++g) i192_add(s, gp[g]);
      p.out[b] = s;
    }
  }
}

}  // namespace pk
