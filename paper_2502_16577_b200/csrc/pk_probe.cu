// FP64 roofline probe: the measured DFMA throughput of this device, used as
// the peak of the FP64-bound Gray-walk kernels (MEASURED_PEAKS.json carries
// only HBM and bf16 figures). Eight independent fma chains per thread keep
// the FP64 pipe saturated; the reported rate counts 2 flops per DFMA.
#include <cuda_runtime.h>

#include <string>

#include "permkit_b200.h"

namespace {

// The multiplier and addend are literals: ptxas keeps one in a uniform
// register (DFMA R, R, UR, R), the operand form that reaches the pipe peak
// (passing them as kernel arguments puts both in vector registers and reads
// ~7 % lower on a B200).
__global__ void __launch_bounds__(256) dfma_chains(double* sink, int iters) {
  const double m = 1.0000001, c = 1e-9;
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1234.5678) sink[0] = s;  // never true; keeps the chains alive
}

}  // namespace

extern "C" int pk_fp64_peak(int device, int iters, double* tflops, double* ms_out) {
  if (!tflops || iters <= 0) return PK_ERR_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return PK_ERR_CUDA;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return PK_ERR_CUDA;
  double* sink = nullptr;
  if (cudaMalloc(&sink, sizeof(double)) != cudaSuccess) return PK_ERR_CUDA;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  dfma_chains<<<blocks, threads, 0, s>>>(sink, 64);  // warm up clocks
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, s);
    dfma_chains<<<blocks, threads, 0, s>>>(sink, iters);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    if (t < best) best = t;
  }
  const cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(s);
  cudaFree(sink);
  if (err != cudaSuccess) return PK_ERR_CUDA;
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  *tflops = flops / (best * 1e-3) * 1e-12;
  if (ms_out) *ms_out = best;
  return PK_OK;
}
