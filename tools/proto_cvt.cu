// Throughput probe: int64 -> double conversions vs DADD on one B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/proto_cvt tools/proto_cvt.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 8;

template <int MODE>
__global__ void probe(long long* io, double* out, int iters) {
  long long v[CH];
  double acc[CH];
  for (int c = 0; c < CH; ++c) {
    v[c] = io[threadIdx.x + c] + c;
    acc[c] = 0.0;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (MODE == 0) {  // I2F.F64.S64 + DADD
        acc[c] = __dadd_rn(acc[c], __ll2double_rn(v[c]));
        v[c] += 0x10001;
      } else if (MODE == 1) {  // two I2F.F64.{S32,U32} + DFMA + DADD
        const double h = (double)(int)(v[c] >> 32);
        const double l = (double)(unsigned)(v[c]);
        acc[c] = __dadd_rn(acc[c], __fma_rn(h, 4294967296.0, l));
        v[c] += 0x10001;
      } else if (MODE == 2) {  // DADD only (+ the same int add)
        acc[c] = __dadd_rn(acc[c], __longlong_as_double(v[c]));
        v[c] += 0x10001;
      } else {  // I2F.F64.S32 + DADD
        acc[c] = __dadd_rn(acc[c], (double)(int)v[c]);
        v[c] += 0x10001;
      }
    }
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  long long* io;
  double* out;
  cudaMalloc(&io, 4096 * sizeof(long long));
  cudaMemset(io, 0, 4096 * sizeof(long long));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 256, iters = 20000;
  cudaMalloc(&out, (size_t)blocks * threads * sizeof(double));
  const char* names[] = {"I2F.F64.S64+DADD", "2xI2F.F64.32+DFMA+DADD", "DADD", "I2F.F64.S32+DADD"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      if (mode == 0) probe<0><<<blocks, threads>>>(io, out, iters);
      if (mode == 1) probe<1><<<blocks, threads>>>(io, out, iters);
      if (mode == 2) probe<2><<<blocks, threads>>>(io, out, iters);
      if (mode == 3) probe<3><<<blocks, threads>>>(io, out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)blocks * threads * iters * CH;
      if (rep) printf("%-26s %.3f ms  %.1f Gop/s (per op-group)  %.2f per SM per clk @1.965GHz\n",
                      names[mode], ms, ops / ms * 1e-6, ops / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  return 0;
}
