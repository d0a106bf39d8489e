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

// body length of the generated kernels (8 steps)
constexpr int kSpaLogU = 3;

}  // namespace pk
