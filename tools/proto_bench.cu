// Design-space probe for K1 (dense real fp64): FP64 DFMA peak and Gray-walk
// throughput for several kernel variants. Standalone, no Python.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I../paper_2502_16577_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cmath>
#include "pk_dense_f64.cuh"

using namespace pk;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__global__ void dfma_peak(double* out, int iters) {
  double a[8];
  const double m = 1.0000001, c = 1e-9;
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;
}

static uint64_t lcg_state = 20261017ull;
static double urand() {
  lcg_state = lcg_state * 6364136223846793005ull + 1442695040888963407ull;
  return (double)(lcg_state >> 11) * (1.0 / 9007199254740992.0);
}

template <int N>
struct Host {
  DenseF64Params<N> p;
  std::vector<double> a;
  Host() {
    a.resize(N * N);
    for (auto& v : a) v = urand();
    for (int j = 0; j < N - 1; ++j)
      for (int i = 0; i < N; ++i) p.cols[j * N + i] = a[i * N + j];
    for (int i = 0; i < N; ++i) {
      double rs = a[i * N];
      for (int j = 1; j < N; ++j) rs += a[i * N + j];
      p.x0[i] = a[i * N + N - 1] - rs / 2.0;
    }
  }
};

template <int N, class C, bool SPLIT = false>
void run_variant(const char* name, Host<N>& h, int k, unsigned long long groups_limit, int reps) {
  static_assert(!SPLIT, "the lane-pair split variant was retired (profiles/r01_k1_variants.md)");
  auto kern = dense_f64_chunks<N, C>;
  const size_t smem = dense_smem_bytes<N>();
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  int dev = 0, sms = 0, occ = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::BLOCK, smem));
  const int n = N;
  const unsigned long long total = (1ull << (n - 1)) - 1;
  unsigned long long chunks = 1ull << (n - 1 - k);
  unsigned long long groups = chunks / 32;
  if (groups_limit && groups > groups_limit) groups = groups_limit;
  DenseF64Params<N> p = h.p;
  dd_t *gp, *out; unsigned int* ctr;
  CK(cudaMalloc(&gp, 2 * groups * sizeof(dd_t)));
  CK(cudaMalloc(&out, sizeof(dd_t)));
  CK(cudaMalloc(&ctr, sizeof(unsigned)));
  CK(cudaMemset(ctr, 0, sizeof(unsigned)));
  p.group_part = gp; p.chunk_part = nullptr; p.out = out; p.counter = ctr;
  p.chunk_lo = 0; p.num_groups = groups; p.g_end = total; p.k = k;
  const int grid = sms * occ;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  kern<<<grid, C::BLOCK, smem>>>(p);  // warm
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<grid, C::BLOCK, smem>>>(p);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  dd_t res; CK(cudaMemcpy(&res, out, sizeof(dd_t), cudaMemcpyDeviceToHost));
  const double updates = (double)groups * 32.0 * (double)(1ull << k);
  const double ups = updates / (best * 1e-3);
  printf("%-28s n=%d k=%d regs=%d occ=%d grid=%d groups=%llu ms=%.3f upd/s=%.4e flop/s(3n)=%.3f TF val=%.17g\n",
         name, n, k, fa.numRegs, occ, grid, groups, best, ups, ups * 3 * n * 1e-12, res.hi + res.lo);
  fflush(stdout);
  cudaFree(gp); cudaFree(out); cudaFree(ctr);
}

int main(int argc, char** argv) {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  if (argc < 2 || strcmp(argv[1], "peak") == 0) {
    double* o; CK(cudaMalloc(&o, 8));
    const int iters = 20000;
    const int blocks = sms * 8, threads = 256;
    dfma_peak<<<blocks, threads>>>(o, 100);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      dfma_peak<<<blocks, threads>>>(o, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("dfma_peak: %.3f TFLOP/s (%.3f ms)\n", flops / (best * 1e-3) * 1e-12, best);
  }
  static Host<36> h36;
  static Host<40> h40;
  static Host<48> h48;
  static Host<56> h56;
  static Host<63> h63;
  static Host<20> h20;
  static Host<24> h24;
  struct V { const char* name; void (*fn)(); };
#define VAR(NM, NN, UX, MB, BL, FA, KK, GL, R) \
  V{NM, [] { run_variant<NN, DenseCfg<POL_KAHAN, 1, UX, true, MB, BL, FA>>(NM, h##NN, KK, GL, R); }}
#define SVAR(NM, NN, UX, MB, KK, GL, R) \
  V{NM, [] { run_variant<NN, DenseCfg<POL_KAHAN, 1, UX, true, MB, 128, true>, true>(NM, h##NN, KK, GL, R); }}
#define QVAR(NM, NN, UX, MB, KK, GL, R) \
  V{NM, [] { run_variant<NN, DenseCfg<POL_QQ, 1, UX, false, MB, 128, false, true>>(NM, h##NN, KK, GL, R); }}
  std::vector<V> vs = {
    VAR("36_kahan_fa", 36, 4, 3, 128, true, 14, 0, 2),
    QVAR("36_qf_u4_mb3", 36, 4, 3, 14, 0, 2),
    QVAR("36_qf_u4_mb2", 36, 4, 2, 14, 0, 2),
    QVAR("36_qf_u3_mb3", 36, 3, 3, 14, 0, 2),
    QVAR("36_qf_u3_mb2", 36, 3, 2, 14, 0, 2),
    QVAR("36_qf_u2_mb3", 36, 2, 3, 14, 0, 2),
    QVAR("40_qf_u4_mb2", 40, 4, 2, 17, 0, 1),
    QVAR("40_qf_u3_mb2", 40, 3, 2, 17, 0, 1),
    QVAR("48_qf_u3_mb2", 48, 3, 2, 20, 4736, 1),
    QVAR("48_qf_u4_mb2", 48, 4, 2, 20, 4736, 1),
  };
  for (auto& v : vs) {
    bool sel = argc < 2;
    for (int a = 1; a < argc; ++a) if (strstr(v.name, argv[a])) sel = true;
    if (sel) v.fn();
  }
  return 0;
}
