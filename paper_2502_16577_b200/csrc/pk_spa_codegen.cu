// SpaRyser on the GPU: per-matrix code generation for sparse exact walks.
//
// The reference's sparse integer loop touches only the nonzeros of the
// flipped column (chunk_sparse_int, /root/reference/pkg/src/permkit/
// _loops.py:263-284). With the row state in registers, a nonzero-only update
// needs the sparsity pattern at compile time -- the SUperman paper generates
// a kernel per matrix for the same reason. This unit writes
// that kernel as CUDA source (each column's update as literal register
// increments, the row product as a widening tree planned from the per-row
// bounds), compiles it with NVRTC for sm_100a, loads it with the runtime
// library API and caches it per (matrix, device).
//
// The arithmetic is pk_int.cuh's (z-space state, exact 192-bit partials);
// only the update is sparse and the product grouping per-matrix. NVRTC is
// dlopen'ed so the library loads where it is absent; requesting a sparse
// walk without it is a loud PK_ERR_CUDA.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "pk_spa.h"

namespace pk {
namespace {

// ---------------------------------------------------------------- NVRTC shim
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
  bool ok = false;
  std::string why;
  nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*,
                          const char* const*);
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*);
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*log)(nvrtcProgram_t, char*);
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char*);
  nvrtcResult_t (*destroy)(nvrtcProgram_t*);
};

Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12",
                           "libnvrtc.so"};
    void* h = nullptr;
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) {
      n.why = "libnvrtc.so.12 not found (needed for the sparse SpaRyser kernels)";
      return;
    }
    n.create = (decltype(n.create))dlsym(h, "nvrtcCreateProgram");
    n.compile = (decltype(n.compile))dlsym(h, "nvrtcCompileProgram");
    n.log_size = (decltype(n.log_size))dlsym(h, "nvrtcGetProgramLogSize");
    n.log = (decltype(n.log))dlsym(h, "nvrtcGetProgramLog");
    n.cubin_size = (decltype(n.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
    n.cubin = (decltype(n.cubin))dlsym(h, "nvrtcGetCUBIN");
    n.destroy = (decltype(n.destroy))dlsym(h, "nvrtcDestroyProgram");
    n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy;
    if (!n.ok) n.why = "libnvrtc is missing symbols";
  });
  return n;
}

// ------------------------------------------------------------ code generation

// Runtime helpers of the generated kernel (self-contained: NVRTC gets no
// system headers). Same arithmetic as pk_int.cuh.
const char* kPrelude = R"(
typedef unsigned long long u64;
struct i192 { u64 w0, w1, w2; };
__device__ __forceinline__ void add128(i192& a, u64 lo, u64 hi) {
  const u64 ext = (u64)((long long)hi >> 63);
  asm("add.cc.u64 %0, %0, %3;\n\taddc.cc.u64 %1, %1, %4;\n\taddc.u64 %2, %2, %5;"
      : "+l"(a.w0), "+l"(a.w1), "+l"(a.w2) : "l"(lo), "l"(hi), "l"(ext));
}
__device__ __forceinline__ void sub128(i192& a, u64 lo, u64 hi) {
  const u64 ext = (u64)((long long)hi >> 63);
  asm("sub.cc.u64 %0, %0, %3;\n\tsubc.cc.u64 %1, %1, %4;\n\tsubc.u64 %2, %2, %5;"
      : "+l"(a.w0), "+l"(a.w1), "+l"(a.w2) : "l"(lo), "l"(hi), "l"(ext));
}
__device__ __forceinline__ void add192(i192& a, const i192& b) {
  asm("add.cc.u64 %0, %0, %3;\n\taddc.cc.u64 %1, %1, %4;\n\taddc.u64 %2, %2, %5;"
      : "+l"(a.w0), "+l"(a.w1), "+l"(a.w2) : "l"(b.w0), "l"(b.w1), "l"(b.w2));
}
__device__ __forceinline__ i192 warp_sum(i192 v) {
  for (int off = 1; off < 32; off <<= 1) {
    i192 o;
    o.w0 = __shfl_down_sync(0xffffffffu, v.w0, off);
    o.w1 = __shfl_down_sync(0xffffffffu, v.w1, off);
    o.w2 = __shfl_down_sync(0xffffffffu, v.w2, off);
    if (((threadIdx.x & 31) & (2 * off - 1)) == 0) add192(v, o);
  }
  return v;
}
__device__ __forceinline__ int ctz64(u64 g) { return __ffsll((long long)g) - 1; }
__device__ __forceinline__ bool flip_on(u64 g, int j) { return ((g >> (j + 1)) & 1ull) == 0; }
)";

struct Plan {
  std::vector<std::vector<int>> groups;  // row indices per int32 group
};

// greedy grouping: each group's product of row bounds stays below 2^31
Plan plan_groups(const std::vector<int64_t>& zmax) {
  const int n = (int)zmax.size();
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return zmax[a] > zmax[b]; });
  Plan p;
  std::vector<char> used(n, 0);
  // first-fit decreasing on log bounds
  for (int idx = 0; idx < n; ++idx) {
    const int r = order[idx];
    bool placed = false;
    for (auto& g : p.groups) {
      __int128 prod = 1;
      for (int q : g) prod *= (zmax[q] > 0 ? zmax[q] : 1);
      prod *= (zmax[r] > 0 ? zmax[r] : 1);
      if (prod < ((__int128)1 << 31)) {
        g.push_back(r);
        placed = true;
        break;
      }
    }
    if (!placed) p.groups.push_back({r});
  }
  return p;
}

void emit_product(std::ostringstream& o, const Plan& pl) {
  const int ng = (int)pl.groups.size();
  for (int k = 0; k < ng; ++k) {
    o << "  int g" << k << " = z" << pl.groups[k][0];
    for (size_t t = 1; t < pl.groups[k].size(); ++t) o << " * z" << pl.groups[k][t];
    o << ";\n";
  }
  const int nh = (ng + 1) / 2;
  for (int k = 0; k < nh; ++k) {
    if (2 * k + 1 < ng)
      o << "  long long h" << k << " = (long long)g" << 2 * k << " * (long long)g" << 2 * k + 1
        << ";\n";
    else
      o << "  long long h" << k << " = (long long)g" << 2 * k << ";\n";
  }
  const int nq = (nh + 1) / 2;
  for (int k = 0; k < nq; ++k) {
    if (2 * k + 1 < nh)
      o << "  __int128 q" << k << " = (__int128)h" << 2 * k << " * (__int128)h" << 2 * k + 1
        << ";\n";
    else
      o << "  __int128 q" << k << " = (__int128)h" << 2 * k << ";\n";
  }
  o << "  unsigned __int128 P = (unsigned __int128)q0;\n";
  for (int k = 1; k < nq; ++k) o << "  P *= (unsigned __int128)q" << k << ";\n";
}

// z += sign * column j (nonzeros only); sign_expr is a literal (+1/-1) or a variable
void emit_update(std::ostringstream& o, const std::vector<int>& zcols, int n, int j,
                 const char* sign_expr, bool literal, int lit_sign) {
  for (int i = 0; i < n; ++i) {
    const int v = zcols[(size_t)j * n + i];
    if (v == 0) continue;
    if (literal) {
      const long long d = (long long)lit_sign * v;
      o << "    z" << i << (d >= 0 ? " += " : " -= ") << (d >= 0 ? d : -d) << ";\n";
    } else if (v == 1) {
      o << "    z" << i << " += " << sign_expr << ";\n";
    } else if (v == -1) {
      o << "    z" << i << " -= " << sign_expr << ";\n";
    } else {
      o << "    z" << i << " += " << sign_expr << " * " << v << ";\n";
    }
  }
}

std::string generate(const SpaIntSpec& sp, int logu, int minb) {
  const int n = sp.n;
  const int U = 1 << logu;
  Plan pl = plan_groups(sp.zmax);
  std::ostringstream o;
  o << kPrelude;
  o << "extern \"C\" __global__ void __launch_bounds__(128, " << minb << ")\n"
    << "spa_int(const int* __restrict__ cols, const int* __restrict__ zseed, i192* group_part, "
       "i192* out, unsigned int* counter, u64 chunk_lo, u64 num_groups, u64 g_end, int k) {\n";
  o << "  const int lane = threadIdx.x & 31;\n"
    << "  const u64 warp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;\n"
    << "  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;\n"
    << "  for (u64 grp = warp; grp < num_groups; grp += nwarps) {\n"
    << "    const u64 c = chunk_lo + grp * 32 + lane;\n"
    << "    const u64 base = c << k;\n";
  for (int i = 0; i < n; ++i) o << "    int z" << i << " = zseed[" << i << "];\n";
  // jump-in: columns of gray(base) (exact ints: order immaterial)
  o << "    {\n      const u64 code = base ^ (base >> 1);\n"
    << "      for (int j = 0; j < " << n - 1 << "; ++j) if ((code >> j) & 1ull) {\n"
    << "        const int* cj = cols + j * " << n << ";\n";
  for (int i = 0; i < n; ++i) o << "        z" << i << " += cj[" << i << "];\n";
  o << "      }\n    }\n";
  o << "    i192 acc = {0ull, 0ull, 0ull};\n"
    << "    const u64 nbody = 1ull << (k - " << logu << ");\n"
    << "    for (u64 m = 0; m < nbody; ++m) {\n"
    << "      const u64 gb = base + (m << " << logu << ");\n"
    << "      const int smid = flip_on(gb + " << (U >> 1) << ", " << logu - 1 << ") ? 1 : -1;\n";
  for (int q = 1; q < U; ++q) {
    int j = 0;
    while (((q >> j) & 1) == 0) ++j;
    o << "      {\n";
    if (j + 1 < logu) {
      const int sgn = ((q >> (j + 1)) & 1) == 0 ? 1 : -1;
      emit_update(o, sp.zcols, n, j, "", true, sgn);
    } else {
      emit_update(o, sp.zcols, n, j, "smid", false, 0);
    }
    emit_product(o, pl);
    o << "      " << ((q & 1) ? "sub128" : "add128")
      << "(acc, (u64)P, (u64)(P >> 64));\n      }\n";
  }
  // body step U: run-time column (uniform), then the chunk's last step
  o << "      const u64 g = gb + " << U << ";\n"
    << "      if (m + 1 < nbody || g <= g_end) {\n"
    << "        const int j = ctz64(g);\n"
    << "        const int s = flip_on(g, j) ? 1 : -1;\n"
    << "        switch (j) {\n";
  for (int j = logu; j < n - 1; ++j) {
    o << "        case " << j << ":\n";
    emit_update(o, sp.zcols, n, j, "s", false, 0);
    o << "          break;\n";
  }
  o << "        default: break;\n        }\n";
  emit_product(o, pl);
  o << "        add128(acc, (u64)P, (u64)(P >> 64));\n      }\n    }\n";
  o << "    acc = warp_sum(acc);\n"
    << "    if (lane == 0) group_part[grp] = acc;\n  }\n";
  // last block sums the group partials
  o << R"(  __shared__ bool is_last;
  __shared__ i192 tree[128];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  i192 s = {0ull, 0ull, 0ull};
  for (u64 i = threadIdx.x; i < num_groups; i += 128) {
    i192 v;
    v.w0 = __ldcg(&group_part[i].w0);
    v.w1 = __ldcg(&group_part[i].w1);
    v.w2 = __ldcg(&group_part[i].w2);
    add192(s, v);
  }
  tree[threadIdx.x] = s;
  __syncthreads();
  for (int w = 64; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) add192(tree[threadIdx.x], tree[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) { *out = tree[0]; *counter = 0u; }
}
)";
  return o.str();
}

struct Compiled {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  int occ = 1;
};

std::mutex g_mu;
std::map<std::string, Compiled> g_cache;

std::string cache_key(const SpaIntSpec& sp, int dev, int logu) {
  std::ostringstream o;
  o << dev << ":" << sp.n << ":" << logu << ":";
  for (int v : sp.zcols) o << v << ",";
  o << "|";
  for (auto v : sp.zmax) o << v << ",";
  return o.str();
}

}  // namespace

int spa_int_launch(const SpaIntSpec& sp, const SpaIntLaunch& a, std::string& err) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int logu = 3;
  const int minb = sp.n <= 40 ? 4 : 3;
  const std::string key = cache_key(sp, dev, logu);
  Compiled cm;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) {
      cm = it->second;
    } else {
      Nvrtc& nv = nvrtc();
      if (!nv.ok) {
        err = nv.why;
        return (int)cudaErrorNotSupported;
      }
      const std::string src = generate(sp, logu, minb);
      nvrtcProgram_t prog = nullptr;
      if (nv.create(&prog, src.c_str(), "spa_int.cu", 0, nullptr, nullptr) != 0) {
        err = "nvrtcCreateProgram failed";
        return (int)cudaErrorInvalidSource;
      }
      const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-default-device",
                            "--device-int128", "-lineinfo"};
      const int rc = nv.compile(prog, 5, opts);
      if (rc != 0) {
        size_t ls = 0;
        nv.log_size(prog, &ls);
        std::string log(ls, '\0');
        nv.log(prog, &log[0]);
        nv.destroy(&prog);
        err = "NVRTC compile of the SpaRyser kernel failed: " + log.substr(0, 2000);
        return (int)cudaErrorInvalidSource;
      }
      size_t cs = 0;
      nv.cubin_size(prog, &cs);
      std::vector<char> cubin(cs);
      nv.cubin(prog, cubin.data());
      nv.destroy(&prog);
      cudaError_t e = cudaLibraryLoadData(&cm.lib, cubin.data(), nullptr, nullptr, 0, nullptr,
                                          nullptr, 0);
      if (e != cudaSuccess) {
        err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e);
        return (int)e;
      }
      e = cudaLibraryGetKernel(&cm.kern, cm.lib, "spa_int");
      if (e != cudaSuccess) {
        err = std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e);
        return (int)e;
      }
      int occ = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)cm.kern, 128, 0);
      cm.occ = (e == cudaSuccess && occ > 0) ? occ : 1;
      g_cache[key] = cm;
    }
  }
  const uint64_t blocks_needed = (a.num_groups * 32 + 127) / 128;
  uint64_t grid = (uint64_t)a.sms * (uint64_t)cm.occ;
  if (blocks_needed < grid) grid = blocks_needed;
  if (grid < 1) grid = 1;
  const int* cols = a.d_cols;
  const int* z0 = a.d_z0;
  void* gp = a.group_part;
  void* out = a.out;
  unsigned int* counter = a.counter;
  unsigned long long chunk_lo = a.chunk_lo, num_groups = a.num_groups, g_end = a.g_end;
  int k = a.k;
  void* args[] = {&cols, &z0, &gp, &out, &counter, &chunk_lo, &num_groups, &g_end, &k};
  cudaError_t e = cudaLaunchKernel((const void*)cm.kern, dim3((unsigned)grid), dim3(128), args, 0,
                                   a.stream);
  if (e != cudaSuccess) err = std::string("spa_int launch: ") + cudaGetErrorString(e);
  return (int)e;
}

std::string spa_int_source(const SpaIntSpec& sp) { return generate(sp, 3, sp.n <= 40 ? 4 : 3); }

}  // namespace pk
