// Internal launch descriptors shared by the C-ABI layer (pk_abi.cu) and the
// per-N kernel instantiation units (pk_dense_f64_n*.cu).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>

#include "pk_common.cuh"

namespace pk {

constexpr int kMaxDevices = 64;

// Per-device launch preparation of one kernel instantiation: function
// attributes (the dynamic shared-memory opt-in above 48 KB) are per device,
// so they are set -- and the occupancy measured -- once for every device
// ordinal the kernel is launched on. `slots` is the instantiation's own
// table (a function-local static of the caller); concurrent host threads of
// different devices touch different slots, and a race on one slot only
// repeats the idempotent attribute call.
template <class K>
inline int prep_kernel(K kern, int block, size_t smem, std::atomic<int>* slots, int* occ) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  if (dev < 0 || dev >= kMaxDevices) return (int)cudaErrorInvalidDevice;
  int o = slots[dev].load(std::memory_order_acquire);
  if (o <= 0) {
    // opt in whenever there is dynamic shared memory: the 48 KB default
    // covers static + dynamic together
    if (smem > 0) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return (int)e;
    }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, block, smem);
    if (e != cudaSuccess) return (int)e;
    if (o < 1) o = 1;
    slots[dev].store(o, std::memory_order_release);
  }
  *occ = o;
  return 0;
}

constexpr int kDenseNMin = 11;  // below this the range walkers take the whole walk
constexpr int kDenseNMax = 63;

// Tuning of the dense register kernel per order N, from the sweep in
// profiles/r01_k1_variants.md: 16-step bodies (LOGU 4) while x[N] plus the
// body's product chains fit the register file, 8-step bodies above; three
// resident 128-thread blocks per SM up to N = 36, two above.
constexpr int dense_logu(int N) { return N <= 50 ? 4 : 3; }
constexpr int dense_minb(int N) { return N <= 36 ? 3 : 2; }
// fast-mode block shape of the chunk kernel: one large block per SM beats
// several 128-thread blocks with the same warp count by 4-6 % from n = 33
// (profiles/r01_k1_variants_sweep10_blocks.txt); n <= 32 keeps 3 x 128
constexpr int dense_block(int N) { return N <= 32 ? 128 : (N <= 36 ? 384 : 256); }
constexpr int dense_block_minb(int N) { return N <= 32 ? 3 : 1; }
// fast QQ (DenseCfg::QF) carries two registers per product chain: shorter
// bodies (profiles/r01_qf_sweep.txt)
constexpr int qf_logu(int N) { return N <= 36 ? 2 : 3; }


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
  int variant;          // fast-mode body schedule (pk_dense_f64_launch.cuh)
};

// Launches the N-specialised register kernel; returns cudaError_t.
template <int N>
int launch_dense_f64(const DenseLaunch& a);

// precise mode (pk_precise.cuh): exact fixed-point row sums, double-double
// products and sums; any order in [kDenseNMin, kDenseNMax]
struct PreciseLaunch {
  const long long* fix;  // device fixed-point image (fixed_image in pk_abi.cu)
  int k;
  uint64_t chunk_lo;
  uint64_t num_groups;
  uint64_t g_end;
  dd_t* group_part;
  dd_t* chunk_part;
  dd_t* out;
  unsigned int* counter;
  cudaStream_t stream;
  int sms;
};

int launch_dense_f64_precise(int n, const PreciseLaunch& a);
// complex: fix = the re image then the im image (two fixed_image layouts)
int launch_dense_c128_precise(int n, const PreciseLaunch& a);

// batched whole walks of `batch` matrices of order N (device inputs)
struct DenseBatchLaunch {
  const double* d_cols;  // [batch][(N-1)*N]
  const double* d_x0;    // [batch][N]
  int policy;
  bool exact;
  int batch;
  int k;
  dd_t* group_part;      // [batch][2^(N-1-k)/32]
  dd_t* out;             // [batch]
  cudaStream_t stream;
  int sms;
};

// chunk exponent of a batched walk: at most 2^10 chunks per matrix
constexpr int batch_log2_chunk(int N, int logu) {
  return (N - 1 - 10) > (logu + 1) ? (N - 1 - 10) : (logu + 1);
}

template <int N>
int launch_dense_f64_batch(const DenseBatchLaunch& a);

// complex: register kernels for N in [kC128NMin, kC128NMax]; cols/x0 are
// interleaved (re, im); cols must already be on the device (d_cols)
constexpr int kC128NMin = 11;
constexpr int kC128NMax = 40;
// complex state is 4N registers; longer bodies make ptxas interleave more
// product chains than the register file holds, so bodies stay short
constexpr int c128_logu(int N) { return N <= 32 ? 2 : 1; }
// fast mode walks row-major 8-step bodies (C128Cfg::RM) at every order:
// +3..8 % over the step-major bodies at n = 28..40
// (profiles/r02_c128_variants_rm.txt, r02_c128_fast_logu.txt)
constexpr int c128_fast_logu(int N) { return 3; }
constexpr int c128_minb(int N) { return N <= 32 ? 2 : 1; }

struct C128Launch {
  const double* d_cols;  // device, (n-1)*n*2
  const double* x0;      // host, 2n
  bool exact;
  int k;
  uint64_t chunk_lo;
  uint64_t num_groups;
  uint64_t g_end;
  dd_t* group_part;      // device [2*num_groups]
  dd_t* chunk_part;      // device [num_groups*32] or null
  dd_t* out;             // device [2]
  unsigned int* counter;
  cudaStream_t stream;
  int sms;
  int variant;           // fast-mode product schedule of K3 (pk_dense_c128_launch.cuh)
};

template <int N>
int launch_dense_c128(const C128Launch& a);

// lane-pair complex kernel (pk_c128_pair.cuh): every order up to kDenseNMax;
// 4*ceil(N/2) registers of state per lane
constexpr int c128_pair_logu(int N) { return N <= 48 ? 2 : 1; }
// the fast (row-major) pair bodies are twice as long (A/B in
// profiles/r02_c128_pair_logu.txt)
constexpr int c128_pair_fast_logu(int N) { return N <= 42 ? 4 : 3; }
constexpr int c128_pair_block(int N) { return 256; }
constexpr int c128_pair_minb(int N) { return N <= 32 ? 2 : 1; }

template <int N>
int launch_c128_pair(const C128Launch& a);

// batched whole complex walks of `batch` matrices of order N (device inputs)
struct C128BatchLaunch {
  const double* d_cols;  // [batch][2*(N-1)*N]
  const double* d_x0;    // [batch][2*N]
  bool exact;
  int batch;
  int k;
  dd_t* group_part;      // [batch][2 * 2^(N-1-k)/32]
  dd_t* out;             // [batch][2]
  cudaStream_t stream;
  int sms;
};

template <int N>
int launch_dense_c128_batch(const C128BatchLaunch& a);

// batched lane-pair walks, orders above kC128NMax (pk_c128_pair.cuh)
template <int N>
int launch_c128_pair_batch(const C128BatchLaunch& a);

// exact integers (pk_int.cuh): z-space state, |z_i| < 2^zb
constexpr int kIntNMin = 11;
constexpr int kIntNMax = 63;
constexpr int int_logu(int N) { return 2; }
constexpr int int_minb(int N) { return N <= 40 ? 4 : (N <= 52 ? 3 : 2); }

struct IntLaunch {
  const int* d_cols;     // device, z-space column steps, (n-1)*n
  const int* z0;         // host, n
  int zb;                // 5, 7, 15 or 31
  int k;
  uint64_t chunk_lo;
  uint64_t num_groups;
  uint64_t g_end;
  void* group_part;      // device i192 [num_groups]
  void* chunk_part;      // device i192 [num_groups*32] or null
  void* out;             // device i192 [1]
  unsigned int* counter;
  cudaStream_t stream;
  int sms;
};

template <int N>
int launch_int(const IntLaunch& a);

// batched whole integer walks of `batch` matrices of order N (device inputs)
struct IntBatchLaunch {
  const int* d_cols;   // [batch][(N-1)*N]
  const int* d_z0;     // [batch][N]
  int zb;              // max over the batch
  int batch;
  int k;
  void* group_part;    // i192 [batch][2^(N-1-k)/32]
  void* out;           // i192 [batch]
  cudaStream_t stream;
  int sms;
};

template <int N>
int launch_int_batch(const IntBatchLaunch& a);

}  // namespace pk
