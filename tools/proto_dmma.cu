// Probe: do FP64 tensor-core MMAs (DMMA, mma.sync m8n8k4 f64) run concurrently
// with the FP64 vector pipe (DFMA) on sm_100a? Times DFMA-only, DMMA-only and
// mixed instruction streams with independent dependency chains.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a proto_dmma.cu
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// NF DFMA chains and NM DMMA accumulators per thread, interleaved R times per iteration
template <int NF, int NM, int RF, int RM>
__global__ void mix(double* out, int iters) {
  double f[NF > 0 ? NF : 1];
  double m0[NM > 0 ? NM : 1], m1[NM > 0 ? NM : 1];
  const double a = 1.0000001 + threadIdx.x * 1e-9, b = 0.9999999, c = 1e-9;
  for (int k = 0; k < NF; ++k) f[k] = threadIdx.x * 1e-3 + k;
  for (int k = 0; k < NM; ++k) { m0[k] = k; m1[k] = -k; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < (RF > RM ? RF : RM); ++r) {
      if (r < RF) {
#pragma unroll
        for (int k = 0; k < NF; ++k) f[k] = fma(f[k], a, c);
      }
      if (r < RM) {
#pragma unroll
        for (int k = 0; k < NM; ++k) dmma(m0[k], m1[k], a, b);
      }
    }
  }
  double s = 0;
  for (int k = 0; k < NF; ++k) s += f[k];
  for (int k = 0; k < NM; ++k) s += m0[k] + m1[k];
  if (s == 12345.678) out[0] = s;
}

// operand-count probe: 8 chains, distinct second/third operands per chain
template <int MODE>
__global__ void ops(double* out, int iters) {
  double f[8], g[8], h[8];
  for (int k = 0; k < 8; ++k) {
    f[k] = threadIdx.x * 1e-3 + k;
    g[k] = 1.0000001 + k * 1e-9 + threadIdx.x * 1e-12;
    h[k] = 1e-9 * (k + 1);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (MODE == 0) f[k] = fma(f[k], g[k], h[k]);          // 3 distinct operands
        else if (MODE == 1) f[k] = f[k] * g[k];               // DMUL, 2 operands
        else if (MODE == 2) f[k] = f[k] + g[k];               // DADD, 2 operands
        else f[k] = fma(f[k], g[0], h[0]);                    // shared operands (reuse)
      }
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += f[k];
  if (s == 12345.678) out[0] = s;
}

template <int MODE>
void run_ops(const char* name, int sms, int iters) {
  double* o;
  CK(cudaMalloc(&o, 8));
  const int blocks = sms * 8, threads = 256;
  ops<MODE><<<blocks, threads>>>(o, 10);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    ops<MODE><<<blocks, threads>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double inst = 8.0 * 16 * (double)iters * blocks * threads;
  printf("%-22s ms=%8.3f  %.3f T FP64-instr/s (lane ops)\n", name, best, inst / (best * 1e-3) * 1e-12);
  cudaFree(o);
}

template <int NF, int NM, int RF, int RM>
void run(const char* name, int sms, int blocks_per_sm, int threads, int iters) {
  double* o;
  CK(cudaMalloc(&o, 8));
  const int blocks = sms * blocks_per_sm;
  mix<NF, NM, RF, RM><<<blocks, threads>>>(o, 10);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    mix<NF, NM, RF, RM><<<blocks, threads>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  const double nthreads = (double)blocks * threads;
  const double dfma_flops = 2.0 * NF * RF * (double)iters * nthreads;          // per-thread DFMAs
  const double dmma_flops = 2.0 * 256 * NM * RM * (double)iters * nthreads / 32;  // per-warp MMA
  printf("%-22s ms=%8.3f dfma=%6.2f TF dmma=%6.2f TF total=%6.2f TF\n", name, best,
         dfma_flops / (best * 1e-3) * 1e-12, dmma_flops / (best * 1e-3) * 1e-12,
         (dfma_flops + dmma_flops) / (best * 1e-3) * 1e-12);
  cudaFree(o);
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int it = 4000;
  run<8, 0, 16, 0>("dfma_only", sms, 8, 256, it);
  run<0, 4, 0, 16>("dmma_only_4acc", sms, 8, 256, it);
  run<0, 8, 0, 16>("dmma_only_8acc", sms, 8, 256, it);
  run<8, 4, 16, 1>("mix_16f:1m", sms, 8, 256, it);
  run<8, 4, 16, 2>("mix_16f:2m", sms, 8, 256, it);
  run<8, 4, 16, 4>("mix_16f:4m", sms, 8, 256, it);
  run<8, 4, 16, 8>("mix_16f:8m", sms, 8, 256, it);
  run<8, 4, 8, 16>("mix_8f:16m", sms, 8, 256, it);
  run_ops<0>("dfma_3_distinct", sms, it);
  run_ops<1>("dmul_2_distinct", sms, it);
  run_ops<2>("dadd_2_distinct", sms, it);
  run_ops<3>("dfma_shared_ops", sms, it);
  return 0;
}
