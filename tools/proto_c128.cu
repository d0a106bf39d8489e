// Design-space probe for K3 (dense complex fp64): body length, register
// budget and fused accumulation. Standalone:
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I../paper_2502_16577_b200/csrc
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pk_dense_c128.cuh"

using namespace pk;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

static uint64_t lcg = 20261017ull;
static double urand() {
  lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
  return (double)(lcg >> 11) * (1.0 / 9007199254740992.0);
}

template <int N>
struct Host {
  std::vector<double> cols, x0;
  double* d_cols = nullptr;
  Host() {
    std::vector<double> a(2 * N * N);
    for (auto& v : a) v = (urand() - 0.5) / std::sqrt((double)N);
    cols.assign(2 * (N - 1) * N, 0.0);
    x0.assign(2 * N, 0.0);
    for (int j = 0; j < N - 1; ++j)
      for (int i = 0; i < N; ++i) {
        cols[2 * (j * N + i)] = a[2 * (i * N + j)];
        cols[2 * (j * N + i) + 1] = a[2 * (i * N + j) + 1];
      }
    for (int i = 0; i < N; ++i) {
      double rr = 0, ri = 0;
      for (int j = 0; j < N; ++j) { rr += a[2 * (i * N + j)]; ri += a[2 * (i * N + j) + 1]; }
      x0[2 * i] = a[2 * (i * N + N - 1)] - rr / 2;
      x0[2 * i + 1] = a[2 * (i * N + N - 1) + 1] - ri / 2;
    }
    CK(cudaMalloc(&d_cols, cols.size() * 8));
    CK(cudaMemcpy(d_cols, cols.data(), cols.size() * 8, cudaMemcpyHostToDevice));
  }
};

template <int N, class C>
void run(const char* name, Host<N>& h, int k, int reps) {
  auto kern = dense_c128_chunks<N, C>;
  const size_t smem = c128_smem_bytes<N>();
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  int sms = 0, occ = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kC128Block, smem));
  const unsigned long long total = (1ull << (N - 1)) - 1;
  const unsigned long long groups = (1ull << (N - 1 - k)) / 32;
  DenseC128Params<N> p;
  std::memcpy(p.x0, h.x0.data(), 16 * N);
  p.cols = h.d_cols;
  dd_t *gp, *out;
  unsigned* ctr;
  CK(cudaMalloc(&gp, 2 * groups * sizeof(dd_t)));
  CK(cudaMalloc(&out, 2 * sizeof(dd_t)));
  CK(cudaMalloc(&ctr, 4));
  CK(cudaMemset(ctr, 0, 4));
  p.group_part = gp; p.chunk_part = nullptr; p.out = out; p.counter = ctr;
  p.chunk_lo = 0; p.num_groups = groups; p.g_end = total; p.k = k;
  unsigned long long grid = (unsigned long long)sms * occ;
  if ((groups * 32 + kC128Block - 1) / kC128Block < grid) grid = (groups * 32 + kC128Block - 1) / kC128Block;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  kern<<<(unsigned)grid, kC128Block, smem>>>(p);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<(unsigned)grid, kC128Block, smem>>>(p);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  dd_t res[2];
  CK(cudaMemcpy(res, out, sizeof(res), cudaMemcpyDeviceToHost));
  const double ups = (double)total / (best * 1e-3);
  printf("%-24s n=%d k=%d regs=%d occ=%d grid=%llu ms=%.3f upd/s=%.4e TF(10n)=%.3f val=(%.17g, %.17g)\n",
         name, N, k, fa.numRegs, occ, grid, best, ups, ups * 10 * N * 1e-12, res[0].hi + res[0].lo,
         res[1].hi + res[1].lo);
  fflush(stdout);
  cudaFree(gp); cudaFree(out); cudaFree(ctr);
}

int main(int argc, char** argv) {
  static Host<32> h32;
  static Host<28> h28;
  static Host<36> h36;
  struct V { const char* name; void (*fn)(); };
#define CV(NM, NN, UX, MB, FA, KK) V{NM, [] { run<NN, C128Cfg<UX, false, MB, FA>>(NM, h##NN, KK, 3); }}
  std::vector<V> vs = {
    CV("32_u2_k9", 32, 2, 2, false, 9),
    CV("32_u2_k10", 32, 2, 2, false, 10),
    CV("32_u2_k11", 32, 2, 2, false, 11),
    CV("32_u2_k12", 32, 2, 2, false, 12),
    CV("32_u2_k13", 32, 2, 2, false, 13),
    CV("32_u2_k14", 32, 2, 2, false, 14),
    CV("32_u2_k16", 32, 2, 2, false, 16),
    CV("36_u1_k12", 36, 1, 1, false, 12),
    CV("36_u1_k14", 36, 1, 1, false, 14),
    CV("36_u1_k16", 36, 1, 1, false, 16),
    CV("28_u2_k7", 28, 2, 2, false, 7),
    CV("28_u2_k9", 28, 2, 2, false, 9),
    CV("28_u2_k11", 28, 2, 2, false, 11),
  };
  for (auto& v : vs) {
    bool sel = argc < 2;
    for (int a = 1; a < argc; ++a) if (strstr(v.name, argv[a])) sel = true;
    if (sel) v.fn();
  }
  return 0;
}
