// Internal launch descriptors shared by the C-ABI layer (pk_abi.cu) and the
// per-N kernel instantiation units (pk_dense_f64_n*.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "pk_common.cuh"

namespace pk {

constexpr int kDenseNMin = 11;  // below this the range walkers take the whole walk
constexpr int kDenseNMax = 63;

// Tuning of the dense register kernel per order N, from the sweep in
// profiles/r01_k1_variants.md: 16-step bodies (LOGU 4) while x[N] plus the
// body's product chains fit the register file, 8-step bodies above; three
// resident 128-thread blocks per SM up to N = 36, two above.
constexpr int dense_logu(int N) { return N <= 50 ? 4 : 3; }
constexpr int dense_minb(int N) { return N <= 36 ? 3 : 2; }

struct DenseLaunch {
  const double* cols;   // host, (n-1)*n
  const double* x0;     // host, n
  int policy;
  bool exact;
  int k;                // log2 chunk size, k > dense_logu(n)
  uint64_t chunk_lo;
  uint64_t num_groups;  // groups of 32 chunks
  uint64_t g_end;
  dd_t* group_part;     // device [num_groups]
  dd_t* chunk_part;     // device [num_groups*32] or null
  dd_t* out;            // device [1]
  unsigned int* counter;
  cudaStream_t stream;
  int sms;
};

// Launches the N-specialised register kernel; returns cudaError_t.
template <int N>
int launch_dense_f64(const DenseLaunch& a);

}  // namespace pk
