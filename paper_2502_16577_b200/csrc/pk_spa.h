// Interface of the per-matrix SpaRyser code generator (pk_spa_codegen.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace pk {

struct SpaIntSpec {
  int n = 0;
  std::vector<int> zcols;      // (n-1)*n z-space column steps, cols[j*n + i]
  std::vector<int64_t> zmax;   // per-row bound on |z_i| over the whole walk
};

struct SpaIntLaunch {
  const int* d_cols;  // device copy of zcols (jump-in)
  const int* d_z0;    // device z seed
  void* group_part;   // device i192 [num_groups]
  void* out;          // device i192 [1]
  unsigned int* counter;
  uint64_t chunk_lo;
  uint64_t num_groups;
  uint64_t g_end;
  int k;
  cudaStream_t stream;
  int sms;
};

// compiles (once per matrix and device) and launches; returns cudaError_t,
// err holds a message on failure
int spa_int_launch(const SpaIntSpec& sp, const SpaIntLaunch& a, std::string& err);
// the generated CUDA source (diagnostics / tests)
std::string spa_int_source(const SpaIntSpec& sp);

// ------------------------------------------------------------- sparse real
// Per-pattern generated kernel for the sparse fp64 walk (chunk_sparse_f64,
// _loops.py:110-183): x[n] in registers, each step adds only the flipped
// column's nonzeros (values staged in shared memory, positions literal).
// Arithmetic, chunking and reduction are K1's (pk_dense_f64.cuh), so the
// result is bit-identical to K1 on the densified matrix.
struct SpaF64Spec {
  int n = 0;
  std::vector<std::vector<int>> rows;  // rows[j]: nonzero rows of column j < n-1, ascending
  int policy = 0;                      // pk::Policy
  bool exact = false;                  // per-term fold (PK_FLAG_EXACT)
};

// packed value layout: column j's nonzeros at [off[j], off[j] + rows[j].size()),
// every column starting at an even offset (LDS.128 pairs)
std::vector<int> spa_f64_offsets(const SpaF64Spec& sp, int* total);

struct SpaF64Launch {
  const double* d_cols;  // device dense (n-1)*n columns (jump-in)
  const double* d_x0;    // device seed x0[n]
  const double* d_vals;  // device packed nonzeros (spa_f64_offsets layout)
  void* group_part;      // device dd_t [num_groups]
  void* chunk_part;      // device dd_t [num_groups*32] or null
  void* out;             // device dd_t [1]
  unsigned int* counter;
  uint64_t chunk_lo;
  uint64_t num_groups;
  uint64_t g_end;
  int k;
  cudaStream_t stream;
  int sms;
};

int spa_f64_launch(const SpaF64Spec& sp, const SpaF64Launch& a, std::string& err);
std::string spa_f64_source(const SpaF64Spec& sp);
// body length (log2) of the generated sparse real kernel for order n: K1's
// (dense_logu), or qf_logu for fast QQ, so the two stay bit-identical
constexpr int spa_f64_logu(int n, bool fast_qq = false) {
  return fast_qq ? (n <= 36 ? 2 : 3) : (n <= 50 ? 4 : 3);
}

// ---------------------------------------------------------- sparse complex
// Per-pattern generated kernel for the sparse complex walk (chunk_sparse_c128,
// _loops.py:212-235) with K3's arithmetic, body length and reduction
// (pk_dense_c128.cuh): bit-identical to K3 on the densified pair.
struct SpaC128Spec {
  int n = 0;
  std::vector<std::vector<int>> rows;  // nonzero rows of column j < n-1
  bool exact = false;
  int variant = 0;  // fast-mode product schedule, as K3's C128Launch::variant
  int logu = 0;     // body length (log2); 0: spa_c128_logu(n)
};

struct SpaC128Launch {
  const double* d_cols;  // device dense interleaved (n-1)*n complex columns (jump-in)
  const double* d_x0;    // device interleaved seed
  const double* d_vals;  // device packed interleaved nonzeros, column by column
  void* group_part;      // device dd_t [2*num_groups]
  void* chunk_part;      // device dd_t [num_groups*32] or null
  void* out;             // device dd_t [2]
  unsigned int* counter;
  uint64_t chunk_lo;
  uint64_t num_groups;
  uint64_t g_end;
  int k;
  cudaStream_t stream;
  int sms;
};

int spa_c128_launch(const SpaC128Spec& sp, const SpaC128Launch& a, std::string& err);
std::string spa_c128_source(const SpaC128Spec& sp);

// body length of the generated kernels (8 steps)
constexpr int kSpaLogU = 3;

}  // namespace pk
