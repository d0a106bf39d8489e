// Deterministic grid-level reduction of per-group double-double partials.
//
// The reduction order is a pure function of the partial count: a pairwise
// (binary-counter) fold over each thread's contiguous segment, then a
// balanced shared-memory tree over the segments. For power-of-two counts this
// is exactly the balanced binary tree over the partial index, so a launch that
// owns an aligned power-of-two slice of the chunks computes a subtree of the
// single-launch tree; combining per-device results with the same tree on the
// host reproduces the single-device bits (SURVEY.md §8e determinism).
//
// Replaces the fixed-order dd_add loop of reduce_partials
// (/root/reference/pkg/src/permkit/parallel.py:384-387).
#pragma once
#include "pk_common.cuh"

namespace pk {

// Pairwise fold of parts[i*S + s] for i in [lo, hi), in index order.
__device__ inline dd_t pairwise_fold(const dd_t* parts, uint64_t lo, uint64_t hi, int S = 1,
                                     int s = 0) {
  dd_t stack[64];
  int depth = 0;
  uint64_t idx = 0;
  for (uint64_t i = lo; i < hi; ++i, ++idx) {
    dd_t v;
    v.hi = __ldcg(&parts[i * S + s].hi);
    v.lo = __ldcg(&parts[i * S + s].lo);
    // merge once per trailing one of the running index
    uint64_t t = idx;
    while (t & 1ull) {
      v = dd_add(stack[--depth], v);
      t >>= 1;
    }
    stack[depth++] = v;
  }
  dd_t acc = stack[--depth];
  while (depth > 0) acc = dd_add(stack[--depth], acc);
  return acc;
}

// Leaf count of the tail tree. It is a constant of the library, not of the
// launching kernel: every kernel -- dense or sparse, fast or exact, whatever
// its block size -- folds the same group partials in the same order, so the
// sparse and dense walks of one matrix agree bit for bit for any group count.
constexpr unsigned int kTreeLeaves = 128;

// Called by every block at the end of a chunk kernel. The last block to
// arrive folds the S interleaved streams of group partials (parts[i*S + s])
// into out[s] and re-arms the counter.
template <int BLOCK, int S>
__device__ inline void grid_tail_reduce_streams(const dd_t* parts, uint64_t count, dd_t* out,
                                                unsigned int* counter) {
  static_assert(BLOCK >= (int)kTreeLeaves, "the tail tree needs kTreeLeaves threads");
  __shared__ bool is_last;
  __shared__ dd_t tree[kTreeLeaves];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  unsigned int b = 1;
  while (2ull * b <= (uint64_t)kTreeLeaves && 2ull * b <= count) b *= 2;
  const unsigned int t = threadIdx.x;
  for (int s = 0; s < S; ++s) {
    if (t < b && count > 0) {
      const uint64_t lo = count * t / b;
      const uint64_t hi = count * (t + 1) / b;
      tree[t] = pairwise_fold(parts, lo, hi, S, s);
    }
    __syncthreads();
    for (unsigned int w = 1; w < b; w <<= 1) {
      if (t < b && (t & (2 * w - 1)) == 0) tree[t] = dd_add(tree[t], tree[t + w]);
      __syncthreads();
    }
    if (t == 0) out[s] = count > 0 ? tree[0] : dd_t{0.0, 0.0};
    __syncthreads();
  }
  if (t == 0) *counter = 0u;
}

template <int BLOCK>
__device__ inline void grid_tail_reduce(const dd_t* parts, uint64_t count, dd_t* out,
                                        unsigned int* counter) {
  grid_tail_reduce_streams<BLOCK, 1>(parts, count, out, counter);
}

template <int BLOCK>
__device__ inline void grid_tail_reduce_pairs(const dd_t* parts, uint64_t count, dd_t* out,
                                              unsigned int* counter) {
  grid_tail_reduce_streams<BLOCK, 2>(parts, count, out, counter);
}

}  // namespace pk
