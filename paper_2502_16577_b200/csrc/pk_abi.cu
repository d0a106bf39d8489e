// C-ABI layer: argument checking, range planning, per-device workspace,
// multi-device fan-out and the fixed-order host reduction.
//
// The reference executes a plan of ranges on a thread pool and reduces the
// partials in worker order (parallel.py:318-387). Here one call covers a
// whole range: its aligned middle goes to the N-specialised register kernels
// (one tree-reduced double-double per device), the unaligned head and tail
// to the range walkers; the host combines the pieces in a fixed order.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "permkit_b200.h"
#include "pk_launch.h"
#include "pk_walker.cuh"

namespace {

using pk::dd_t;

thread_local std::string g_err;

struct PkError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw PkError{code, msg}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(PK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return PK_OK;
  } catch (const PkError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PK_ERR_CUDA;
  }
}

// ---------------------------------------------------------------------------
// host double-double, identical operation sequence to pk_common.cuh

inline void h_two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
inline void h_quick_two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  e = b - (s - a);
}
inline dd_t h_dd_add(dd_t a, dd_t b) {
  double s1, s2, t1, t2;
  h_two_sum(a.hi, b.hi, s1, s2);
  h_two_sum(a.lo, b.lo, t1, t2);
  s2 += t1;
  h_quick_two_sum(s1, s2, s1, s2);
  s2 += t2;
  h_quick_two_sum(s1, s2, s1, s2);
  return dd_t{s1, s2};
}

// pairwise (binary-counter) fold in index order; same shape as pk::pairwise_fold
dd_t h_pairwise(const std::vector<dd_t>& v) {
  if (v.empty()) return dd_t{0.0, 0.0};
  std::vector<dd_t> stack;
  uint64_t idx = 0;
  for (const dd_t& x : v) {
    dd_t c = x;
    for (uint64_t t = idx; t & 1ull; t >>= 1) {
      c = h_dd_add(stack.back(), c);
      stack.pop_back();
    }
    stack.push_back(c);
    ++idx;
  }
  dd_t acc = stack.back();
  stack.pop_back();
  while (!stack.empty()) {
    acc = h_dd_add(stack.back(), acc);
    stack.pop_back();
  }
  return acc;
}

// ---------------------------------------------------------------------------
// per-device workspace

struct DevCtx {
  std::mutex mu;
  bool ready = false;
  int dev = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  unsigned int* counter = nullptr;
  dd_t* out = nullptr;
  dd_t* groups = nullptr;
  size_t groups_cap = 0;
  dd_t* chunks = nullptr;
  size_t chunks_cap = 0;
  char* scratch = nullptr;
  size_t scratch_cap = 0;
};

constexpr int kMaxDev = 64;
DevCtx g_dev[kMaxDev];
std::mutex g_init_mu;

DevCtx& dev_ctx(int d) {
  std::lock_guard<std::mutex> init_lock(g_init_mu);
  int count = 0;
  ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  if (d < 0 || d >= count || d >= kMaxDev)
    fail(PK_ERR_CUDA, "device " + std::to_string(d) + " not available (" +
                          std::to_string(count) + " visible)");
  DevCtx& c = g_dev[d];
  if (!c.ready) {
    c.dev = d;
    ck(cudaSetDevice(d), "cudaSetDevice");
    ck(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, d), "sm count");
    ck(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreate(&c.e0), "event");
    ck(cudaEventCreate(&c.e1), "event");
    ck(cudaMalloc(&c.counter, sizeof(unsigned int)), "cudaMalloc counter");
    ck(cudaMemset(c.counter, 0, sizeof(unsigned int)), "memset counter");
    ck(cudaMalloc(&c.out, 4 * sizeof(dd_t)), "cudaMalloc out");
    c.ready = true;
  }
  return c;
}

template <class T>
void ensure(T*& p, size_t& cap, size_t need) {
  if (need <= cap) return;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  size_t want = need < 1024 ? 1024 : need + need / 4;
  ck(cudaMalloc((void**)&p, want * sizeof(T)), "cudaMalloc workspace");
  cap = want;
}

// ---------------------------------------------------------------------------
// planning

using Range = std::pair<uint64_t, uint64_t>;

uint64_t total_iterates(int n) { return n <= 1 ? 0ull : ((1ull << (n - 1)) - 1ull); }

int bit_length(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; }

void check_n(int n) {
  if (n > 63) fail(PK_ERR_IMPOSSIBLE, "matrix order " + std::to_string(n) + " exceeds 63");
  if (n < 1) fail(PK_ERR_ARG, "matrix order must be >= 1");
}

void check_range(int n, uint64_t s, uint64_t e) {
  const uint64_t T = total_iterates(n);
  if (!(1 <= s && s <= e && e <= T))
    fail(PK_ERR_ARG, "range [" + std::to_string(s) + ", " + std::to_string(e) +
                         "] invalid for n=" + std::to_string(n));
}

void check_policy(int p) {
  if (p < PK_POLICY_DD || p > PK_POLICY_QQ) fail(PK_ERR_POLICY, "unknown policy code");
}

// split [s, e] into walker pieces of at most `piece` iterates
void split_pieces(uint64_t s, uint64_t e, uint64_t piece, std::vector<Range>& out) {
  if (s > e) return;
  for (uint64_t a = s;; a += piece) {
    const uint64_t b = (e - a >= piece - 1) ? a + piece - 1 : e;
    out.emplace_back(a, b);
    if (b == e) break;
  }
}

uint64_t piece_size(uint64_t len) {
  uint64_t p = (len + 8191) / 8192;
  return p < 256 ? 256 : p;
}

struct DensePlan {
  int k = 0;
  uint64_t chunk_lo = 0;
  uint64_t num_groups = 0;  // total over devices
  std::vector<Range> head, tail;
};

DensePlan plan_dense(int n, uint64_t start, uint64_t end, int log2_chunk, int ndev) {
  DensePlan pl;
  const uint64_t len = end - start + 1;
  if (n >= pk::kDenseNMin) {
    const int logu = pk::dense_logu(n);
    int k = log2_chunk;
    if (k <= 0) {
      k = bit_length(len) - 22;
      if (k < logu + 1) k = logu + 1;
    }
    if (k < logu + 1 || k > n - 1 - 5)
      fail(PK_ERR_ARG, "log2_chunk " + std::to_string(k) + " outside [" +
                           std::to_string(logu + 1) + ", " + std::to_string(n - 6) + "]");
    // chunk c covers [1 + c*2^k, (c+1)*2^k]
    const uint64_t c_first = ((start - 1) + ((1ull << k) - 1)) >> k;
    const uint64_t c_lo = (c_first + 31) & ~31ull;
    const uint64_t c_end = (end + 1) >> k;  // chunks c < c_end fit (last step may clip)
    if (c_end > c_lo) {
      uint64_t groups = (c_end - c_lo) / 32;
      if (groups >= (uint64_t)ndev) {
        pl.k = k;
        pl.chunk_lo = c_lo;
        pl.num_groups = groups;
      }
    }
  }
  if (pl.num_groups == 0) {
    split_pieces(start, end, piece_size(len), pl.head);
    return pl;
  }
  const uint64_t first = 1 + (pl.chunk_lo << pl.k);
  uint64_t covered = (pl.chunk_lo + 32 * pl.num_groups) << pl.k;
  if (covered > end) covered = end;
  if (first > start) split_pieces(start, first - 1, piece_size(first - start), pl.head);
  if (covered < end) split_pieces(covered + 1, end, piece_size(end - covered), pl.tail);
  return pl;
}

// ---------------------------------------------------------------------------
// dense real

int dispatch_dense(int n, const pk::DenseLaunch& a) {
  switch (n) {
#define PK_CASE(N) \
  case N:          \
    return pk::launch_dense_f64<N>(a);
    PK_CASE(11) PK_CASE(12) PK_CASE(13) PK_CASE(14) PK_CASE(15) PK_CASE(16) PK_CASE(17)
    PK_CASE(18) PK_CASE(19) PK_CASE(20) PK_CASE(21) PK_CASE(22) PK_CASE(23) PK_CASE(24)
    PK_CASE(25) PK_CASE(26) PK_CASE(27) PK_CASE(28) PK_CASE(29) PK_CASE(30) PK_CASE(31)
    PK_CASE(32) PK_CASE(33) PK_CASE(34) PK_CASE(35) PK_CASE(36) PK_CASE(37) PK_CASE(38)
    PK_CASE(39) PK_CASE(40) PK_CASE(41) PK_CASE(42) PK_CASE(43) PK_CASE(44) PK_CASE(45)
    PK_CASE(46) PK_CASE(47) PK_CASE(48) PK_CASE(49) PK_CASE(50) PK_CASE(51) PK_CASE(52)
    PK_CASE(53) PK_CASE(54) PK_CASE(55) PK_CASE(56) PK_CASE(57) PK_CASE(58) PK_CASE(59)
    PK_CASE(60) PK_CASE(61) PK_CASE(62) PK_CASE(63)
#undef PK_CASE
    default:
      return (int)cudaErrorInvalidValue;
  }
}

struct DenseInputs {
  const double* cols;
  const double* x0;
  int n;
  int policy;
  bool exact;
};

// walker launch for a list of ranges on ctx (workspace laid out in scratch)
void launch_walk_dense(DevCtx& c, const DenseInputs& in, const std::vector<Range>& ranges,
                       dd_t* d_out) {
  const int n = in.n;
  const size_t ncol = (size_t)(n > 1 ? n - 1 : 1) * n;
  const size_t nr = ranges.size();
  const size_t bytes = ncol * 8 + (size_t)n * 8 + nr * 16;
  ensure(c.scratch, c.scratch_cap, bytes + 64);
  char* base = c.scratch;
  double* d_cols = (double*)base;
  double* d_x0 = d_cols + ncol;
  unsigned long long* d_s = (unsigned long long*)(d_x0 + n);
  unsigned long long* d_e = d_s + nr;
  std::vector<unsigned long long> hs(nr), he(nr);
  for (size_t i = 0; i < nr; ++i) {
    hs[i] = ranges[i].first;
    he[i] = ranges[i].second;
  }
  if (n > 1) ck(cudaMemcpyAsync(d_cols, in.cols, (size_t)(n - 1) * n * 8, cudaMemcpyHostToDevice, c.stream), "H2D cols");
  ck(cudaMemcpyAsync(d_x0, in.x0, (size_t)n * 8, cudaMemcpyHostToDevice, c.stream), "H2D x0");
  ck(cudaMemcpyAsync(d_s, hs.data(), nr * 8, cudaMemcpyHostToDevice, c.stream), "H2D starts");
  ck(cudaMemcpyAsync(d_e, he.data(), nr * 8, cudaMemcpyHostToDevice, c.stream), "H2D ends");
  const unsigned grid = (unsigned)((nr + pk::kWalkBlock - 1) / pk::kWalkBlock);
  switch (in.policy) {
    case PK_POLICY_DD:
      pk::walk_dense_f64<pk::POL_DD><<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, d_s, d_e, (int)nr, d_out);
      break;
    case PK_POLICY_KAHAN:
      pk::walk_dense_f64<pk::POL_KAHAN><<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, d_s, d_e, (int)nr, d_out);
      break;
    case PK_POLICY_DQ:
      pk::walk_dense_f64<pk::POL_DQ><<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, d_s, d_e, (int)nr, d_out);
      break;
    default:
      pk::walk_dense_f64<pk::POL_QQ><<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, d_s, d_e, (int)nr, d_out);
      break;
  }
  ck(cudaGetLastError(), "walk_dense_f64 launch");
}

struct DevResult {
  dd_t fast{0.0, 0.0};
  std::vector<dd_t> head, tail;
  float ms = 0.f;
  int launches = 0;
  int code = PK_OK;
  std::string err;
};

void run_dense_on_device(int dev, const DenseInputs& in, const DensePlan& pl, uint64_t g_lo,
                         uint64_t g_cnt, bool walkers, uint64_t g_end, DevResult& r) {
  try {
    DevCtx& c = dev_ctx(dev);
    std::lock_guard<std::mutex> lock(c.mu);
    ck(cudaSetDevice(dev), "cudaSetDevice");
    ck(cudaEventRecord(c.e0, c.stream), "event record");
    if (g_cnt > 0) {
      ensure(c.groups, c.groups_cap, g_cnt);
      pk::DenseLaunch a{};
      a.cols = in.cols;
      a.x0 = in.x0;
      a.policy = in.policy;
      a.exact = in.exact;
      a.k = pl.k;
      a.chunk_lo = pl.chunk_lo + 32 * g_lo;
      a.num_groups = g_cnt;
      a.g_end = g_end;
      a.group_part = c.groups;
      a.chunk_part = nullptr;
      a.out = c.out;
      a.counter = c.counter;
      a.stream = c.stream;
      a.sms = c.sms;
      ck((cudaError_t)dispatch_dense(in.n, a), "dense_f64 register kernel launch");
      ++r.launches;
    }
    std::vector<Range> pieces;
    if (walkers) {
      pieces = pl.head;
      pieces.insert(pieces.end(), pl.tail.begin(), pl.tail.end());
    }
    dd_t* d_walk = nullptr;
    if (!pieces.empty()) {
      ensure(c.chunks, c.chunks_cap, pieces.size());
      d_walk = c.chunks;
      launch_walk_dense(c, in, pieces, d_walk);
      ++r.launches;
    }
    ck(cudaEventRecord(c.e1, c.stream), "event record");
    ck(cudaStreamSynchronize(c.stream), "kernel execution");
    ck(cudaEventElapsedTime(&r.ms, c.e0, c.e1), "event time");
    if (g_cnt > 0) ck(cudaMemcpy(&r.fast, c.out, sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H total");
    if (!pieces.empty()) {
      std::vector<dd_t> w(pieces.size());
      ck(cudaMemcpy(w.data(), d_walk, w.size() * sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H walkers");
      r.head.assign(w.begin(), w.begin() + pl.head.size());
      r.tail.assign(w.begin() + pl.head.size(), w.end());
    }
  } catch (const PkError& e) {
    r.code = e.code;
    r.err = e.msg;
  }
}

}  // namespace

// ===========================================================================
// exported C ABI

extern "C" {

int pk_abi_version(void) { return PK_ABI_VERSION; }

int pk_device_count(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) return -1;
  return count;
}

const char* pk_last_error(void) { return g_err.c_str(); }

int pk_dense_f64(const double* cols, const double* x0, int n, uint64_t start, uint64_t end,
                 int policy, uint32_t flags, int log2_chunk, const int* devices, int ndev,
                 double out_dd[2], pk_run_stats* stats) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    check_n(n);
    check_policy(policy);
    if (!x0 || !out_dd || (n > 1 && !cols)) fail(PK_ERR_ARG, "null pointer argument");
    check_range(n, start, end);
    std::vector<int> devs;
    if (!devices || ndev <= 0) devs.push_back(0);
    else devs.assign(devices, devices + ndev);
    DenseInputs in{cols, x0, n, policy, (flags & PK_FLAG_EXACT) != 0};
    DensePlan pl = plan_dense(n, start, end, log2_chunk, (int)devs.size());
    const int nd = pl.num_groups ? (int)devs.size() : 1;
    std::vector<DevResult> res(nd);
    auto work = [&](int i) {
      const uint64_t lo = pl.num_groups * i / nd, hi = pl.num_groups * (i + 1) / nd;
      run_dense_on_device(devs[i], in, pl, lo, hi - lo, i == 0, end, res[i]);
    };
    if (nd == 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (int i = 0; i < nd; ++i) th.emplace_back(work, i);
      for (auto& t : th) t.join();
    }
    for (auto& r : res)
      if (r.code != PK_OK) fail(r.code, r.err);
    // fixed combination order: head pieces, device trees (pairwise over
    // devices), tail pieces
    std::vector<dd_t> parts;
    dd_t total{0.0, 0.0};
    bool have = false;
    auto add = [&](dd_t v) {
      total = have ? h_dd_add(total, v) : v;
      have = true;
    };
    if (!res[0].head.empty()) add(h_pairwise(res[0].head));
    if (pl.num_groups) {
      std::vector<dd_t> trees;
      for (auto& r : res) trees.push_back(r.fast);
      add(h_pairwise(trees));
    }
    if (!res[0].tail.empty()) add(h_pairwise(res[0].tail));
    out_dd[0] = total.hi;
    out_dd[1] = total.lo;
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      float mx = 0.f;
      int launches = 0;
      for (auto& r : res) {
        if (r.ms > mx) mx = r.ms;
        launches += r.launches;
      }
      stats->kernel_ms = mx;
      stats->iterates = end - start + 1;
      stats->chunks = pl.num_groups * 32;
      stats->walker_ranges = pl.head.size() + pl.tail.size();
      stats->log2_chunk = pl.k;
      stats->devices = nd;
      stats->launches = launches;
      stats->wall_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

int pk_dense_f64_ranges(const double* cols, const double* x0, int n, const uint64_t* starts,
                        const uint64_t* ends, int nranges, int policy, int device,
                        double* out_dd) {
  return guarded([&] {
    check_n(n);
    check_policy(policy);
    if (nranges < 0) fail(PK_ERR_ARG, "negative range count");
    if (nranges == 0) return;
    if (!x0 || !out_dd || !starts || !ends || (n > 1 && !cols)) fail(PK_ERR_ARG, "null pointer argument");
    std::vector<Range> rs(nranges);
    for (int i = 0; i < nranges; ++i) {
      check_range(n, starts[i], ends[i]);
      rs[i] = Range(starts[i], ends[i]);
    }
    DevCtx& c = dev_ctx(device);
    std::lock_guard<std::mutex> lock(c.mu);
    ck(cudaSetDevice(device), "cudaSetDevice");
    ensure(c.chunks, c.chunks_cap, rs.size());
    DenseInputs in{cols, x0, n, policy, true};
    launch_walk_dense(c, in, rs, c.chunks);
    ck(cudaStreamSynchronize(c.stream), "walker execution");
    ck(cudaMemcpy(out_dd, c.chunks, rs.size() * sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H");
  });
}

int pk_dense_f64_chunks(const double* cols, const double* x0, int n, int log2_chunk,
                        uint64_t chunk_lo, uint64_t nchunks, int policy, uint32_t flags,
                        int device, double* out_chunks, double out_total[2]) {
  return guarded([&] {
    check_n(n);
    check_policy(policy);
    if (n < pk::kDenseNMin) fail(PK_ERR_ARG, "register kernels need n >= 11");
    if (!x0 || !cols || !out_total) fail(PK_ERR_ARG, "null pointer argument");
    const int logu = pk::dense_logu(n);
    const int k = log2_chunk;
    if (k < logu + 1 || k > n - 6) fail(PK_ERR_ARG, "log2_chunk out of range");
    if (nchunks == 0 || nchunks % 32) fail(PK_ERR_ARG, "nchunks must be a positive multiple of 32");
    const uint64_t T = total_iterates(n);
    if (((chunk_lo + nchunks - 1) << k) + 1 > T || chunk_lo + nchunks > (1ull << (n - 1 - k)))
      fail(PK_ERR_ARG, "chunks exceed the walk");
    DevCtx& c = dev_ctx(device);
    std::lock_guard<std::mutex> lock(c.mu);
    ck(cudaSetDevice(device), "cudaSetDevice");
    const uint64_t groups = nchunks / 32;
    ensure(c.groups, c.groups_cap, groups);
    ensure(c.chunks, c.chunks_cap, nchunks);
    pk::DenseLaunch a{};
    a.cols = cols;
    a.x0 = x0;
    a.policy = policy;
    a.exact = (flags & PK_FLAG_EXACT) != 0;
    a.k = k;
    a.chunk_lo = chunk_lo;
    a.num_groups = groups;
    a.g_end = T;
    a.group_part = c.groups;
    a.chunk_part = c.chunks;
    a.out = c.out;
    a.counter = c.counter;
    a.stream = c.stream;
    a.sms = c.sms;
    ck((cudaError_t)dispatch_dense(n, a), "dense_f64 register kernel launch");
    ck(cudaStreamSynchronize(c.stream), "kernel execution");
    dd_t tot;
    ck(cudaMemcpy(&tot, c.out, sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H total");
    out_total[0] = tot.hi;
    out_total[1] = tot.lo;
    if (out_chunks)
      ck(cudaMemcpy(out_chunks, c.chunks, nchunks * sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H chunks");
  });
}

}  // extern "C"
