// C-ABI layer: argument checking, range planning, per-device workspace,
// multi-device fan-out and the fixed-order host reduction.
//
// The reference executes a plan of ranges on a thread pool and reduces the
// partials in worker order (parallel.py:318-387). Here one call covers a
// whole range: its aligned middle goes to the N-specialised register kernels
// (one tree-reduced double-double per device), the unaligned head and tail
// to the range walkers; the host combines the pieces in a fixed order.
#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "permkit_b200.h"
#include "pk_launch.h"
#include "pk_walker.cuh"
#include "pk_int.cuh"
#include "pk_spa.h"
#include <cmath>
#include <functional>
#include <memory>

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

// dd_t workspace slots that hold `count` i192 values (24 B each)
size_t i192_slots(size_t count) { return (count * 3 + 1) / 2; }

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

// chunks_log2: automatic chunk size aims at ~2^chunks_log2 chunks per walk
// (real: 2^22; complex: 2^19, profiles/r01_c128_sweep2.txt)
DensePlan plan_dense(int n, int logu, uint64_t start, uint64_t end, int log2_chunk, int ndev,
                     int chunks_log2 = 22) {
  DensePlan pl;
  const uint64_t len = end - start + 1;
  if (logu > 0) {
    int k = log2_chunk;
    if (k <= 0) {
      // ~2^chunks_log2 chunks for long walks; mid-size walks keep chunks of
      // up to 2^12 steps (while 2^17 chunks remain) so the per-chunk jump-in
      // and reduction stay small against the walk
      // (profiles/r01_k1_variants_sweep8_n32.txt, r01_k1_sweep_n.md)
      const int bl = bit_length(len);
      k = bl - chunks_log2;
      const int k_floor = std::min(12, bl - 17);
      if (k < k_floor) k = k_floor;
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
// kinds: each bundles its device inputs, its register-kernel launcher and
// its walker launcher; the driver below is shared.

struct Kind {
  int n = 0;
  int streams = 1;            // double-double streams per partial: 1 real, 2 complex
  int logu = 0;               // body length of the register kernel; 0 = walkers only
  int chunks_log2 = 22;       // automatic chunking target (plan_dense)
  std::vector<double> input;  // uploaded once per device call: cols then x0
  // register kernel over groups [chunk_lo, chunk_lo + 32*groups); returns cudaError_t
  std::function<int(DevCtx&, const double* d_in, uint64_t chunk_lo, uint64_t groups,
                    uint64_t g_end, int k, dd_t* gparts, dd_t* cparts, dd_t* out)>
      fast;
  // walkers: one thread per range, out[r] = range partial
  std::function<void(DevCtx&, const double* d_in, const unsigned long long* d_s,
                     const unsigned long long* d_e, int nr, dd_t* out)>
      walk;
  // walker partial -> per-stream double-double
  dd_t stream_of(const dd_t& w, int s) const {
    if (streams == 1) return w;
    return dd_t{s == 0 ? w.hi : w.lo, 0.0};
  }
};

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

int dispatch_dense_batch(int n, const pk::DenseBatchLaunch& a) {
  switch (n) {
#define PK_CASE(N) \
  case N:          \
    return pk::launch_dense_f64_batch<N>(a);
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

int dispatch_c128(int n, const pk::C128Launch& a) {
  switch (n) {
#define PK_CASE(N) \
  case N:          \
    return pk::launch_dense_c128<N>(a);
    PK_CASE(11) PK_CASE(12) PK_CASE(13) PK_CASE(14) PK_CASE(15) PK_CASE(16) PK_CASE(17)
    PK_CASE(18) PK_CASE(19) PK_CASE(20) PK_CASE(21) PK_CASE(22) PK_CASE(23) PK_CASE(24)
    PK_CASE(25) PK_CASE(26) PK_CASE(27) PK_CASE(28) PK_CASE(29) PK_CASE(30) PK_CASE(31)
    PK_CASE(32) PK_CASE(33) PK_CASE(34) PK_CASE(35) PK_CASE(36) PK_CASE(37) PK_CASE(38)
    PK_CASE(39) PK_CASE(40)
#undef PK_CASE
    default:
      return (int)cudaErrorInvalidValue;
  }
}

int dispatch_int_batch(int n, const pk::IntBatchLaunch& a) {
  switch (n) {
#define PK_CASE(N) \
  case N:          \
    return pk::launch_int_batch<N>(a);
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

int dispatch_c128_pair(int n, const pk::C128Launch& a) {
  switch (n) {
#define PK_CASE(N) \
  case N:          \
    return pk::launch_c128_pair<N>(a);
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

int dispatch_c128_pair_batch(int n, const pk::C128BatchLaunch& a) {
  switch (n) {
#define PK_CASE(N) \
  case N:          \
    return pk::launch_c128_pair_batch<N>(a);
    PK_CASE(11) PK_CASE(12) PK_CASE(13) PK_CASE(14) PK_CASE(15) PK_CASE(16) PK_CASE(17)
    PK_CASE(18) PK_CASE(19) PK_CASE(20) PK_CASE(21) PK_CASE(22) PK_CASE(23) PK_CASE(24)
    PK_CASE(25) PK_CASE(26) PK_CASE(27) PK_CASE(28) PK_CASE(29) PK_CASE(30) PK_CASE(31)
    PK_CASE(32) PK_CASE(33) PK_CASE(34) PK_CASE(35) PK_CASE(36) PK_CASE(37) PK_CASE(38)
    PK_CASE(39) PK_CASE(40) PK_CASE(41) PK_CASE(42) PK_CASE(43) PK_CASE(44) PK_CASE(45) PK_CASE(46) PK_CASE(47)
    PK_CASE(48) PK_CASE(49) PK_CASE(50) PK_CASE(51) PK_CASE(52) PK_CASE(53) PK_CASE(54)
    PK_CASE(55) PK_CASE(56) PK_CASE(57) PK_CASE(58) PK_CASE(59) PK_CASE(60) PK_CASE(61)
    PK_CASE(62) PK_CASE(63)
#undef PK_CASE
    default:
      return (int)cudaErrorInvalidValue;
  }
}

// Complex register kernel for order n: K3 (one thread per chunk) up to
// kC128NMax, the lane-pair kernel K3p above (PK_C128_PAIR=1 selects K3p for
// every order, for A/B runs).
// K1's fast body schedule (PK_DENSE_VARIANT, A/B runs): 0 the default
// (row-major above n = 36), 1 row-major, 2 step-major (pk_dense_f64_launch.cuh)
int dense_variant() {
  static const int v = [] {
    const char* e = getenv("PK_DENSE_VARIANT");
    const int r = e ? atoi(e) : 0;
    return (r == 1 || r == 2) ? r : 0;
  }();
  return v;
}

// K3's fast body schedule (PK_C128_VARIANT, A/B runs): 4 row-major bodies
// of twice the exact mode's length (default), 2 the step-major bodies of
// round 1 (profiles/r02_c128_variants*.txt)
int c128_variant() {
  static const int v = [] {
    const char* e = getenv("PK_C128_VARIANT");
    return (e && atoi(e) == 2) ? 2 : 4;
  }();
  return v;
}

// body length (log2) of K3's launch for order n, exact or fast
int c128_kernel_logu(int n, bool exact) {
  return exact || c128_variant() == 2 ? pk::c128_logu(n) : pk::c128_fast_logu(n);
}

bool c128_use_pair(int n) {
  static const bool all = [] {
    const char* e = getenv("PK_C128_PAIR");
    return e && atoi(e) == 1;
  }();
  return n >= pk::kC128NMin && n <= pk::kDenseNMax && (all || n > pk::kC128NMax);
}

int dispatch_c128_batch(int n, const pk::C128BatchLaunch& a) {
  switch (n) {
#define PK_CASE(N) \
  case N:          \
    return pk::launch_dense_c128_batch<N>(a);
    PK_CASE(11) PK_CASE(12) PK_CASE(13) PK_CASE(14) PK_CASE(15) PK_CASE(16) PK_CASE(17)
    PK_CASE(18) PK_CASE(19) PK_CASE(20) PK_CASE(21) PK_CASE(22) PK_CASE(23) PK_CASE(24)
    PK_CASE(25) PK_CASE(26) PK_CASE(27) PK_CASE(28) PK_CASE(29) PK_CASE(30) PK_CASE(31)
    PK_CASE(32) PK_CASE(33) PK_CASE(34) PK_CASE(35) PK_CASE(36) PK_CASE(37) PK_CASE(38)
    PK_CASE(39) PK_CASE(40)
#undef PK_CASE
    default:
      return (int)cudaErrorInvalidValue;
  }
}

size_t ncols_of(int n) { return (size_t)(n > 1 ? n - 1 : 1) * n; }

// Exact walk states for the fast modes (DESIGN.md §5 "x state"). The
// reference updates the row sums x_i incrementally in double, and every
// update rounds; the drift is what limits its accuracy (1.2e-9 at n = 36
// with 2^19-step chunks, tests/test_gpu_configs.py). Here the fast kernels
// walk the input rounded once onto a per-row (and per component) fixed-point
// grid 2^-F: with B = |x0_i| + sum_j |a_ij| < 2^e and F = 52 - e, every
// subset sum x0_i + sum_{j in S} a_ij of grid values is a multiple of 2^-F
// below 2^(e+1) in magnitude, i.e. a double -- so the jump-in sums and every
// update are exact and the states never drift. The rounding moves each entry
// by at most 2^-(F+1) <= B 2^-53 (half an ulp of the row's largest possible
// state), once, instead of a rounding of that size at every step.
// comps = 1 (real) or 2 (complex, interleaved re/im: independent grids).
void quantize_walk(const double* cols, const double* x0, int n, int comps, double* qcols,
                   double* qx0) {
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < comps; ++c) {
      double bound = std::fabs(x0[(size_t)comps * i + c]);
      for (int j = 0; j < n - 1; ++j) bound += std::fabs(cols[(size_t)comps * (j * n + i) + c]);
      int F = 0;
      const bool grid = bound > 0.0 && std::isfinite(bound);
      if (grid) {
        int e = 0;
        std::frexp(bound, &e);  // bound < 2^e
        F = 52 - e;
        if (F > 1074) F = 1074;  // subnormal rows: 2^-1074 is the finest grid there is
      }
      auto q = [&](double v) { return grid ? std::ldexp(std::nearbyint(std::ldexp(v, F)), -F) : v; };
      qx0[(size_t)comps * i + c] = q(x0[(size_t)comps * i + c]);
      for (int j = 0; j < n - 1; ++j)
        qcols[(size_t)comps * (j * n + i) + c] = q(cols[(size_t)comps * (j * n + i) + c]);
    }
}

// Fixed-point image of a dense real walk for the precise mode (pk_precise.cuh).
// Row i gets a scale 2^F_i with (|x0_i| + sum_j |a_ij|) 2^F_i < 2^62, so
// X_i = x0_i 2^F_i + sum_{j in S} a_ij 2^F_i is an exact int64 for every
// column subset S; every entry is rounded to the row's grid once (RN,
// |error| <= 2^-(F_i+1), 2^-63 of the row's absolute sum). Layout (int64
// words): A[j*n + i] for the n-1 walked columns, X0[n], then the bit
// patterns of the doubles 2^-F_i[n].
size_t fix_words_of(int n) { return (size_t)(n > 1 ? n - 1 : 0) * n + 2 * (size_t)n; }

void fixed_image(const double* cols, const double* x0, int n, long long* out) {
  long long* A = out;
  long long* X0 = out + (size_t)(n - 1) * n;
  long long* sc = X0 + n;
  for (int i = 0; i < n; ++i) {
    double bound = std::fabs(x0[i]);
    for (int j = 0; j < n - 1; ++j) bound += std::fabs(cols[(size_t)j * n + i]);
    int F = 0;
    if (bound > 0.0 && std::isfinite(bound)) {
      int e = 0;
      std::frexp(bound * (1.0 + 0x1p-40), &e);  // bound (with slack) < 2^e
      F = 62 - e;
      // 2^-F must be a double: at most 2^-1074, where subnormal entries are
      // integers on the grid (bound < 2^-1022 keeps X below 2^52); F >= -962
      // holds for every finite bound
      if (F > 1074) F = 1074;
    }
    for (int j = 0; j < n - 1; ++j)
      A[(size_t)j * n + i] = std::llrint(std::ldexp(cols[(size_t)j * n + i], F));
    X0[i] = std::llrint(std::ldexp(x0[i], F));
    const double s = std::ldexp(1.0, -F);
    std::memcpy(&sc[i], &s, 8);
  }
}

Kind dense_f64_kind(const double* cols, const double* x0, int n, int policy, bool exact,
                    bool sparse = false, bool precise = false) {
  Kind kd;
  kd.n = n;
  kd.streams = 1;
  kd.logu = n >= pk::kDenseNMin ? pk::dense_logu(n) : 0;
  const size_t nc = ncols_of(n);
  // fast modes walk the input rounded onto the per-row grids (exact states)
  std::shared_ptr<std::vector<double>> qbuf;
  if (!exact && !precise && n >= pk::kDenseNMin) {
    qbuf = std::make_shared<std::vector<double>>(nc + n);
    quantize_walk(cols, x0, n, 1, qbuf->data(), qbuf->data() + nc);
    cols = qbuf->data();
    x0 = qbuf->data() + nc;
  }
  kd.input.assign(nc + n, 0.0);
  if (n > 1) std::memcpy(kd.input.data(), cols, (size_t)(n - 1) * n * 8);
  std::memcpy(kd.input.data() + nc, x0, (size_t)n * 8);
  const double* h_cols = cols;
  const double* h_x0 = x0;
  if (sparse && n >= pk::kDenseNMin) {
    // SpaRyser: generated kernel over the nonzero pattern of the columns;
    // packed nonzero values appended to the inputs (16-byte aligned)
    auto sp = std::make_shared<pk::SpaF64Spec>();
    sp->n = n;
    sp->policy = policy;
    sp->exact = exact;
    sp->rows.resize(n - 1);
    for (int j = 0; j < n - 1; ++j)
      for (int i = 0; i < n; ++i)
        if (cols[(size_t)j * n + i] != 0.0) sp->rows[j].push_back(i);
    int nv = 0;
    const std::vector<int> off = pk::spa_f64_offsets(*sp, &nv);
    const size_t voff = (kd.input.size() + 1) & ~size_t(1);
    kd.input.resize(voff + nv, 0.0);
    for (int j = 0; j < n - 1; ++j)
      for (size_t t = 0; t < sp->rows[j].size(); ++t)
        kd.input[voff + off[j] + t] = cols[(size_t)j * n + sp->rows[j][t]];
    kd.logu = pk::spa_f64_logu(n);  // planning as K1 (the kernel needs k > its own body length)
    kd.fast = [=](DevCtx& c, const double* d_in, uint64_t chunk_lo, uint64_t groups,
                  uint64_t g_end, int k, dd_t* gparts, dd_t* cparts, dd_t* out) {
      pk::SpaF64Launch a{};
      a.d_cols = d_in;
      a.d_x0 = d_in + nc;
      a.d_vals = d_in + voff;
      a.group_part = gparts;
      a.chunk_part = cparts;
      a.out = out;
      a.counter = c.counter;
      a.chunk_lo = chunk_lo;
      a.num_groups = groups;
      a.g_end = g_end;
      a.k = k;
      a.stream = c.stream;
      a.sms = c.sms;
      std::string err;
      const int rc = pk::spa_f64_launch(*sp, a, err);
      if (rc != 0) fail(PK_ERR_CUDA, err);
      return 0;
    };
  } else if (precise && n >= pk::kDenseNMin) {
    // precise mode: exact fixed-point state, double-double products and sums
    const size_t fo = kd.input.size();
    kd.input.resize(fo + fix_words_of(n), 0.0);
    fixed_image(cols, x0, n, reinterpret_cast<long long*>(kd.input.data() + fo));
    kd.fast = [=](DevCtx& c, const double* d_in, uint64_t chunk_lo, uint64_t groups,
                  uint64_t g_end, int k, dd_t* gparts, dd_t* cparts, dd_t* out) {
      pk::PreciseLaunch a{};
      a.fix = reinterpret_cast<const long long*>(d_in + fo);
      a.k = k;
      a.chunk_lo = chunk_lo;
      a.num_groups = groups;
      a.g_end = g_end;
      a.group_part = gparts;
      a.chunk_part = cparts;
      a.out = out;
      a.counter = c.counter;
      a.stream = c.stream;
      a.sms = c.sms;
      return pk::launch_dense_f64_precise(n, a);
    };
  } else {
  kd.fast = [=](DevCtx& c, const double*, uint64_t chunk_lo, uint64_t groups, uint64_t g_end,
                int k, dd_t* gparts, dd_t* cparts, dd_t* out) {
    (void)qbuf;  // keeps the quantized inputs alive with the lambda
    pk::DenseLaunch a{};
    a.cols = h_cols;
    a.x0 = h_x0;
    a.variant = dense_variant();
    a.policy = policy;
    a.exact = exact;
    a.k = k;
    a.chunk_lo = chunk_lo;
    a.num_groups = groups;
    a.g_end = g_end;
    a.group_part = gparts;
    a.chunk_part = cparts;
    a.out = out;
    a.counter = c.counter;
    a.stream = c.stream;
    a.sms = c.sms;
    return dispatch_dense(n, a);
  };
  }
  kd.walk = [=](DevCtx& c, const double* d_in, const unsigned long long* d_s,
                const unsigned long long* d_e, int nr, dd_t* out) {
    const double* d_cols = d_in;
    const double* d_x0 = d_in + nc;
    const unsigned grid = (unsigned)((nr + pk::kWalkBlock - 1) / pk::kWalkBlock);
    switch (policy) {
      case PK_POLICY_DD:
        pk::walk_dense_f64<pk::POL_DD><<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, d_s, d_e, nr, out);
        break;
      case PK_POLICY_KAHAN:
        pk::walk_dense_f64<pk::POL_KAHAN><<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, d_s, d_e, nr, out);
        break;
      case PK_POLICY_DQ:
        pk::walk_dense_f64<pk::POL_DQ><<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, d_s, d_e, nr, out);
        break;
      default:
        pk::walk_dense_f64<pk::POL_QQ><<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, d_s, d_e, nr, out);
        break;
    }
    ck(cudaGetLastError(), "walk_dense_f64 launch");
  };
  return kd;
}

pk::SpaC128Spec spa_c128_spec(const double* cols, int n, bool exact) {
  pk::SpaC128Spec sp;
  sp.n = n;
  sp.exact = exact;
  sp.rows.resize(n - 1);
  for (int j = 0; j < n - 1; ++j)
    for (int i = 0; i < n; ++i) {
      const double* v = cols + 2 * ((size_t)j * n + i);
      if (v[0] != 0.0 || v[1] != 0.0) sp.rows[j].push_back(i);
    }
  return sp;
}

Kind dense_c128_kind(const double* cols, const double* x0, int n, bool exact,
                     bool sparse = false, bool precise = false) {
  Kind kd;
  kd.n = n;
  kd.streams = 2;
  const bool pair = c128_use_pair(n);
  kd.logu = pair ? ((exact || c128_variant() == 2) ? pk::c128_pair_logu(n)
                                                   : pk::c128_pair_fast_logu(n))
                 : (n >= pk::kC128NMin && n <= pk::kC128NMax) ? c128_kernel_logu(n, exact) : 0;
  kd.chunks_log2 = 19;
  const size_t nc = 2 * ncols_of(n);
  // fast modes walk the input rounded onto per-row, per-component grids
  std::shared_ptr<std::vector<double>> qbuf;
  if (!exact && !precise && kd.logu > 0) {
    qbuf = std::make_shared<std::vector<double>>(nc + 2 * n);
    quantize_walk(cols, x0, n, 2, qbuf->data(), qbuf->data() + nc);
    cols = qbuf->data();
    x0 = qbuf->data() + nc;
  }
  kd.input.assign(nc + 2 * n, 0.0);
  if (n > 1) std::memcpy(kd.input.data(), cols, (size_t)(n - 1) * n * 16);
  std::memcpy(kd.input.data() + nc, x0, (size_t)n * 16);
  const double* h_x0 = x0;
  if (precise && n >= pk::kC128NMin) {
    // precise mode: exact fixed-point states per component, double-double
    // complex products and sums (pk_precise.cuh); images of the (unrounded)
    // re and im parts back to back
    if (kd.logu <= 0) kd.logu = 1;
    const size_t fo = kd.input.size();
    const size_t fw = fix_words_of(n);
    kd.input.resize(fo + 2 * fw, 0.0);
    std::vector<double> cr(ncols_of(n)), ci(ncols_of(n)), xr(n), xi(n);
    for (size_t t = 0; t < (size_t)(n - 1) * n; ++t) {
      cr[t] = cols[2 * t];
      ci[t] = cols[2 * t + 1];
    }
    for (int i = 0; i < n; ++i) {
      xr[i] = x0[2 * i];
      xi[i] = x0[2 * i + 1];
    }
    fixed_image(cr.data(), xr.data(), n, reinterpret_cast<long long*>(kd.input.data() + fo));
    fixed_image(ci.data(), xi.data(), n, reinterpret_cast<long long*>(kd.input.data() + fo + fw));
    kd.fast = [=](DevCtx& c, const double* d_in, uint64_t chunk_lo, uint64_t groups,
                  uint64_t g_end, int k, dd_t* gparts, dd_t* cparts, dd_t* out) {
      pk::PreciseLaunch a{};
      a.fix = reinterpret_cast<const long long*>(d_in + fo);
      a.k = k;
      a.chunk_lo = chunk_lo;
      a.num_groups = groups;
      a.g_end = g_end;
      a.group_part = gparts;
      a.chunk_part = cparts;
      a.out = out;
      a.counter = c.counter;
      a.stream = c.stream;
      a.sms = c.sms;
      return pk::launch_dense_c128_precise(n, a);
    };
  } else if (sparse && kd.logu > 0 && !pair) {
    // SpaRyser: generated kernel over the nonzero pattern; packed nonzeros
    // (interleaved re, im) appended to the inputs
    auto sp = std::make_shared<pk::SpaC128Spec>(spa_c128_spec(cols, n, exact));
    sp->variant = c128_variant();
    sp->logu = kd.logu;  // the dense kernel's body length: same fold grouping, same bits
    const size_t voff = kd.input.size();
    for (int j = 0; j < n - 1; ++j)
      for (int r : sp->rows[j]) {
        kd.input.push_back(cols[2 * ((size_t)j * n + r)]);
        kd.input.push_back(cols[2 * ((size_t)j * n + r) + 1]);
      }
    kd.fast = [=](DevCtx& c, const double* d_in, uint64_t chunk_lo, uint64_t groups,
                  uint64_t g_end, int k, dd_t* gparts, dd_t* cparts, dd_t* out) {
      pk::SpaC128Launch a{};
      a.d_cols = d_in;
      a.d_x0 = d_in + nc;
      a.d_vals = d_in + voff;
      a.group_part = gparts;
      a.chunk_part = cparts;
      a.out = out;
      a.counter = c.counter;
      a.chunk_lo = chunk_lo;
      a.num_groups = groups;
      a.g_end = g_end;
      a.k = k;
      a.stream = c.stream;
      a.sms = c.sms;
      std::string err;
      const int rc = pk::spa_c128_launch(*sp, a, err);
      if (rc != 0) fail(PK_ERR_CUDA, err);
      return 0;
    };
  } else {
  kd.fast = [=](DevCtx& c, const double* d_in, uint64_t chunk_lo, uint64_t groups,
                uint64_t g_end, int k, dd_t* gparts, dd_t* cparts, dd_t* out) {
    (void)qbuf;  // keeps the rounded inputs alive with the lambda
    pk::C128Launch a{};
    a.variant = c128_variant();
    a.d_cols = d_in;
    a.x0 = h_x0;
    a.exact = exact;
    a.k = k;
    a.chunk_lo = chunk_lo;
    a.num_groups = groups;
    a.g_end = g_end;
    a.group_part = gparts;
    a.chunk_part = cparts;
    a.out = out;
    a.counter = c.counter;
    a.stream = c.stream;
    a.sms = c.sms;
    return pair ? dispatch_c128_pair(n, a) : dispatch_c128(n, a);
  };
  }
  kd.walk = [=](DevCtx& c, const double* d_in, const unsigned long long* d_s,
                const unsigned long long* d_e, int nr, dd_t* out) {
    const unsigned grid = (unsigned)((nr + pk::kWalkBlock - 1) / pk::kWalkBlock);
    pk::walk_dense_c128<<<grid, pk::kWalkBlock, 0, c.stream>>>(d_in, d_in + nc, n, d_s, d_e, nr, out);
    ck(cudaGetLastError(), "walk_dense_c128 launch");
  };
  return kd;
}

// ---------------------------------------------------------------------------
// shared driver

struct DevResult {
  dd_t fast[2] = {{0.0, 0.0}, {0.0, 0.0}};
  std::vector<dd_t> head, tail;  // walker partials
  float ms = 0.f;
  int launches = 0;
  int code = PK_OK;
  std::string err;
};

// inputs + range bounds in the device scratch area; returns d_in
const double* upload(DevCtx& c, const Kind& kd, const std::vector<Range>& ranges,
                     const unsigned long long** d_s, const unsigned long long** d_e) {
  const size_t nin = kd.input.size();
  const size_t nr = ranges.size();
  ensure(c.scratch, c.scratch_cap, nin * 8 + nr * 16 + 64);
  double* d_in = (double*)c.scratch;
  unsigned long long* s = (unsigned long long*)(d_in + nin);
  unsigned long long* e = s + nr;
  ck(cudaMemcpyAsync(d_in, kd.input.data(), nin * 8, cudaMemcpyHostToDevice, c.stream), "H2D inputs");
  if (nr) {
    std::vector<unsigned long long> hb(2 * nr);
    for (size_t i = 0; i < nr; ++i) {
      hb[i] = ranges[i].first;
      hb[nr + i] = ranges[i].second;
    }
    ck(cudaMemcpyAsync(s, hb.data(), 2 * nr * 8, cudaMemcpyHostToDevice, c.stream), "H2D ranges");
    ck(cudaStreamSynchronize(c.stream), "H2D ranges");  // hb is stack memory
  }
  *d_s = s;
  *d_e = e;
  return d_in;
}

void run_on_device(int dev, const Kind& kd, const DensePlan& pl, uint64_t g_lo, uint64_t g_cnt,
                   bool walkers, uint64_t g_end, DevResult& r) {
  try {
    DevCtx& c = dev_ctx(dev);
    std::lock_guard<std::mutex> lock(c.mu);
    ck(cudaSetDevice(dev), "cudaSetDevice");
    std::vector<Range> pieces;
    if (walkers) {
      pieces = pl.head;
      pieces.insert(pieces.end(), pl.tail.begin(), pl.tail.end());
    }
    const unsigned long long *d_s, *d_e;
    const double* d_in = upload(c, kd, pieces, &d_s, &d_e);
    ck(cudaEventRecord(c.e0, c.stream), "event record");
    if (g_cnt > 0) {
      ensure(c.groups, c.groups_cap, kd.streams * g_cnt);
      ck((cudaError_t)kd.fast(c, d_in, pl.chunk_lo + 32 * g_lo, g_cnt, g_end, pl.k, c.groups,
                              nullptr, c.out),
         "register kernel launch");
      ++r.launches;
    }
    if (!pieces.empty()) {
      ensure(c.chunks, c.chunks_cap, pieces.size());
      kd.walk(c, d_in, d_s, d_e, (int)pieces.size(), c.chunks);
      ++r.launches;
    }
    ck(cudaEventRecord(c.e1, c.stream), "event record");
    ck(cudaStreamSynchronize(c.stream), "kernel execution");
    ck(cudaEventElapsedTime(&r.ms, c.e0, c.e1), "event time");
    if (g_cnt > 0)
      ck(cudaMemcpy(r.fast, c.out, kd.streams * sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H total");
    if (!pieces.empty()) {
      std::vector<dd_t> w(pieces.size());
      ck(cudaMemcpy(w.data(), c.chunks, w.size() * sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H walkers");
      r.head.assign(w.begin(), w.begin() + pl.head.size());
      r.tail.assign(w.begin() + pl.head.size(), w.end());
    }
  } catch (const PkError& e) {
    r.code = e.code;
    r.err = e.msg;
  }
}

std::vector<int> device_list(const int* devices, int ndev) {
  std::vector<int> devs;
  if (!devices || ndev <= 0) devs.push_back(0);
  else devs.assign(devices, devices + ndev);
  return devs;
}

// whole-range walk; out[s] = stream s partial as a double-double
void drive(const Kind& kd, uint64_t start, uint64_t end, int log2_chunk,
           const std::vector<int>& devs, dd_t out[2], pk_run_stats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  DensePlan pl = plan_dense(kd.n, kd.logu, start, end, log2_chunk, (int)devs.size(),
                            kd.chunks_log2);
  const int nd = pl.num_groups ? (int)devs.size() : 1;
  std::vector<DevResult> res(nd);
  auto work = [&](int i) {
    const uint64_t lo = pl.num_groups * i / nd, hi = pl.num_groups * (i + 1) / nd;
    run_on_device(devs[i], kd, pl, lo, hi - lo, i == 0, end, res[i]);
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
  // fixed combination order per stream: head pieces, device trees (pairwise
  // over devices), tail pieces
  for (int s = 0; s < kd.streams; ++s) {
    dd_t total{0.0, 0.0};
    bool have = false;
    auto add = [&](dd_t v) {
      total = have ? h_dd_add(total, v) : v;
      have = true;
    };
    auto fold = [&](const std::vector<dd_t>& w) {
      std::vector<dd_t> v;
      for (auto& x : w) v.push_back(kd.stream_of(x, s));
      return h_pairwise(v);
    };
    if (!res[0].head.empty()) add(fold(res[0].head));
    if (pl.num_groups) {
      std::vector<dd_t> trees;
      for (auto& r : res) trees.push_back(r.fast[s]);
      add(h_pairwise(trees));
    }
    if (!res[0].tail.empty()) add(fold(res[0].tail));
    out[s] = total;
  }
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
}

// per-range walker partials on one device
void drive_ranges(const Kind& kd, const uint64_t* starts, const uint64_t* ends, int nranges,
                  int device, dd_t* out) {
  std::vector<Range> rs(nranges);
  for (int i = 0; i < nranges; ++i) {
    check_range(kd.n, starts[i], ends[i]);
    rs[i] = Range(starts[i], ends[i]);
  }
  DevCtx& c = dev_ctx(device);
  std::lock_guard<std::mutex> lock(c.mu);
  ck(cudaSetDevice(device), "cudaSetDevice");
  const unsigned long long *d_s, *d_e;
  const double* d_in = upload(c, kd, rs, &d_s, &d_e);
  ensure(c.chunks, c.chunks_cap, rs.size());
  kd.walk(c, d_in, d_s, d_e, nranges, c.chunks);
  ck(cudaStreamSynchronize(c.stream), "walker execution");
  ck(cudaMemcpy(out, c.chunks, rs.size() * sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H");
}

// register-kernel chunk partials on one device (parity diagnostics)
void drive_chunks(const Kind& kd, int log2_chunk, uint64_t chunk_lo, uint64_t nchunks,
                  int device, dd_t* out_chunks, dd_t* out_total) {
  const int n = kd.n;
  if (kd.logu <= 0) fail(PK_ERR_ARG, "no register kernel for this order");
  const int k = log2_chunk;
  if (k < kd.logu + 1 || k > n - 6) fail(PK_ERR_ARG, "log2_chunk out of range");
  if (nchunks == 0 || nchunks % 32) fail(PK_ERR_ARG, "nchunks must be a positive multiple of 32");
  const uint64_t T = total_iterates(n);
  if (((chunk_lo + nchunks - 1) << k) + 1 > T || chunk_lo + nchunks > (1ull << (n - 1 - k)))
    fail(PK_ERR_ARG, "chunks exceed the walk");
  DevCtx& c = dev_ctx(device);
  std::lock_guard<std::mutex> lock(c.mu);
  ck(cudaSetDevice(device), "cudaSetDevice");
  const unsigned long long *d_s, *d_e;
  const double* d_in = upload(c, kd, {}, &d_s, &d_e);
  const uint64_t groups = nchunks / 32;
  ensure(c.groups, c.groups_cap, kd.streams * groups);
  ensure(c.chunks, c.chunks_cap, nchunks);
  ck((cudaError_t)kd.fast(c, d_in, chunk_lo, groups, T, k, c.groups, c.chunks, c.out),
     "register kernel launch");
  ck(cudaStreamSynchronize(c.stream), "kernel execution");
  ck(cudaMemcpy(out_total, c.out, kd.streams * sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H total");
  if (out_chunks)
    ck(cudaMemcpy(out_chunks, c.chunks, nchunks * sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H chunks");
}

// ---------------------------------------------------------------------------
// exact integers

struct IntPrep {
  int n = 0;
  int zb = 31;
  int even_rows = 0;
  bool exact_terms = true;
  double log2_bound = 0.0;
  std::vector<int> zcols;  // (n-1)*n, z-space column steps
  std::vector<int> z0;
  std::vector<int64_t> zmax;  // per-row bound on |z_i|
  bool sparse = false;        // walk with the generated SpaRyser kernel
};

// y = 2x state of kernels.py:104-110, rescaled per row (pk_int.cuh header)
IntPrep prep_int(const int64_t* a, int n) {
  IntPrep ip;
  ip.n = n;
  ip.zcols.assign((size_t)(n > 1 ? n - 1 : 1) * n, 0);
  ip.z0.assign(n, 0);
  ip.zmax.assign(n, 0);
  const __int128 lim = ((__int128)1 << 31) - 1;
  int64_t zmax_all = 0;
  double lb = 0.0;
  bool zero_row = false;
  for (int i = 0; i < n; ++i) {
    __int128 r = 0, R = 0;
    for (int j = 0; j < n; ++j) {
      const __int128 v = a[(size_t)i * n + j];
      r += v;
      R += v < 0 ? -v : v;
    }
    const bool even = (r % 2) == 0;
    if (even) ++ip.even_rows;
    const __int128 y0 = 2 * (__int128)a[(size_t)i * n + n - 1] - r;
    const __int128 z0 = even ? y0 / 2 : y0;
    const __int128 zmax = even ? R / 2 : R;  // |y_i| <= R_i along the whole walk
    if (zmax > lim) fail(PK_ERR_OVERFLOW, "integer row sums exceed 2^31; exact GPU walk unavailable");
    ip.z0[i] = (int)z0;
    for (int j = 0; j < n - 1; ++j) {
      const __int128 v = a[(size_t)i * n + j];
      ip.zcols[(size_t)j * n + i] = (int)(even ? v : 2 * v);
    }
    ip.zmax[i] = (int64_t)zmax;
    if (zmax > zmax_all) zmax_all = (int64_t)zmax;
    if (zmax == 0) zero_row = true;
    else lb += std::log2((double)zmax);
  }
  ip.zb = zmax_all <= 31 ? 5 : zmax_all <= 127 ? 7 : zmax_all <= 32767 ? 15 : 31;
  ip.log2_bound = zero_row ? -INFINITY : lb;
  ip.exact_terms = zero_row || lb < 126.9;
  return ip;
}

int dispatch_int(int n, const pk::IntLaunch& a) {
  switch (n) {
#define PK_CASE(N) \
  case N:          \
    return pk::launch_int<N>(a);
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

inline void h_i192_add(pk::i192& a, const pk::i192& b) {
  unsigned __int128 lo = (unsigned __int128)a.w0 + b.w0;
  a.w0 = (uint64_t)lo;
  lo = (lo >> 64) + a.w1 + b.w1;
  a.w1 = (uint64_t)lo;
  a.w2 = a.w2 + b.w2 + (uint64_t)(lo >> 64);
}

struct IntDevResult {
  pk::i192 sum{0, 0, 0};
  float ms = 0.f;
  int launches = 0;
  int code = PK_OK;
  std::string err;
};

// upload z-space inputs and range bounds; returns device pointers
const int* upload_int(DevCtx& c, const IntPrep& ip, const std::vector<Range>& ranges,
                      const unsigned long long** d_s, const unsigned long long** d_e,
                      const int** d_z0) {
  const size_t ncol = ip.zcols.size(), nz = ip.z0.size(), nr = ranges.size();
  const size_t ints = ((ncol + nz) + 1) & ~size_t(1);  // keep the u64 arrays 8-byte aligned
  ensure(c.scratch, c.scratch_cap, ints * 4 + nr * 16 + 64);
  int* d_cols = (int*)c.scratch;
  int* z0 = d_cols + ncol;
  unsigned long long* s = (unsigned long long*)(d_cols + ints);
  std::vector<int> hin(ints, 0);
  std::memcpy(hin.data(), ip.zcols.data(), ncol * 4);
  std::memcpy(hin.data() + ncol, ip.z0.data(), nz * 4);
  std::vector<unsigned long long> hb(2 * nr);
  for (size_t i = 0; i < nr; ++i) {
    hb[i] = ranges[i].first;
    hb[nr + i] = ranges[i].second;
  }
  ck(cudaMemcpyAsync(d_cols, hin.data(), ints * 4, cudaMemcpyHostToDevice, c.stream), "H2D int inputs");
  if (nr) ck(cudaMemcpyAsync(s, hb.data(), 2 * nr * 8, cudaMemcpyHostToDevice, c.stream), "H2D ranges");
  ck(cudaStreamSynchronize(c.stream), "H2D int inputs");
  *d_s = s;
  *d_e = s + nr;
  *d_z0 = z0;
  return d_cols;
}

void launch_walk_int(DevCtx& c, const IntPrep& ip, const int* d_cols, const int* d_z0,
                     const unsigned long long* d_s, const unsigned long long* d_e, int nr,
                     pk::i192* out) {
  const unsigned grid = (unsigned)((nr + 127) / 128);
  pk::walk_int<<<grid, 128, 0, c.stream>>>(d_cols, d_z0, ip.n, d_s, d_e, nr, out);
  ck(cudaGetLastError(), "walk_int launch");
}

void run_int_on_device(int dev, const IntPrep& ip, const DensePlan& pl, uint64_t g_lo,
                       uint64_t g_cnt, bool walkers, uint64_t g_end, IntDevResult& r) {
  try {
    DevCtx& c = dev_ctx(dev);
    std::lock_guard<std::mutex> lock(c.mu);
    ck(cudaSetDevice(dev), "cudaSetDevice");
    std::vector<Range> pieces;
    if (walkers) {
      pieces = pl.head;
      pieces.insert(pieces.end(), pl.tail.begin(), pl.tail.end());
    }
    const unsigned long long *d_s, *d_e;
    const int* d_z0;
    const int* d_cols = upload_int(c, ip, pieces, &d_s, &d_e, &d_z0);
    ck(cudaEventRecord(c.e0, c.stream), "event record");
    // i192 buffers are carved from the dd workspaces (24 B <= 32 B per dd pair)
    if (g_cnt > 0 && ip.sparse) {
      ensure(c.groups, c.groups_cap, i192_slots(g_cnt));
      pk::SpaIntSpec sp;
      sp.n = ip.n;
      sp.zcols = ip.zcols;
      sp.zmax = ip.zmax;
      pk::SpaIntLaunch a{};
      a.d_cols = d_cols;
      a.d_z0 = d_z0;
      a.group_part = c.groups;
      a.out = c.out;
      a.counter = c.counter;
      a.chunk_lo = pl.chunk_lo + 32 * g_lo;
      a.num_groups = g_cnt;
      a.g_end = g_end;
      a.k = pl.k;
      a.stream = c.stream;
      a.sms = c.sms;
      std::string err;
      const int rc = pk::spa_int_launch(sp, a, err);
      if (rc != 0) fail(PK_ERR_CUDA, err);
      ++r.launches;
    } else if (g_cnt > 0) {
      ensure(c.groups, c.groups_cap, i192_slots(g_cnt));
      pk::IntLaunch a{};
      a.d_cols = d_cols;
      a.z0 = ip.z0.data();
      a.zb = ip.zb;
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
      ck((cudaError_t)dispatch_int(ip.n, a), "int register kernel launch");
      ++r.launches;
    }
    if (!pieces.empty()) {
      ensure(c.chunks, c.chunks_cap, i192_slots(pieces.size()));
      launch_walk_int(c, ip, d_cols, d_z0, d_s, d_e, (int)pieces.size(), (pk::i192*)c.chunks);
      ++r.launches;
    }
    ck(cudaEventRecord(c.e1, c.stream), "event record");
    ck(cudaStreamSynchronize(c.stream), "kernel execution");
    ck(cudaEventElapsedTime(&r.ms, c.e0, c.e1), "event time");
    if (g_cnt > 0) {
      pk::i192 t;
      ck(cudaMemcpy(&t, c.out, sizeof(t), cudaMemcpyDeviceToHost), "D2H total");
      h_i192_add(r.sum, t);
    }
    if (!pieces.empty()) {
      std::vector<pk::i192> w(pieces.size());
      ck(cudaMemcpy(w.data(), c.chunks, w.size() * sizeof(pk::i192), cudaMemcpyDeviceToHost), "D2H walkers");
      for (auto& v : w) h_i192_add(r.sum, v);
    }
  } catch (const PkError& e) {
    r.code = e.code;
    r.err = e.msg;
  }
}

void fill_info(const IntPrep& ip, pk_int_info* info) {
  if (!info) return;
  info->zbits = ip.zb;
  info->even_rows = ip.even_rows;
  info->exact_terms = ip.exact_terms ? 1 : 0;
  info->reserved = 0;
  info->log2_term_bound = ip.log2_bound;
}

}  // namespace

// ===========================================================================
// exported C ABI

namespace {
// CCS (cptrs[n+1], rids, vals) -> dense (n-1) x n toggled columns; the
// reference's StructureError conditions (matrix.py:198-222, :256-259)
std::vector<double> ccs_to_cols(const int64_t* cptrs, const int64_t* rids, const double* vals,
                                int n, int comps) {
  if (!cptrs || (cptrs[n] > 0 && (!rids || !vals))) fail(PK_ERR_ARG, "null pointer argument");
  if (cptrs[0] != 0) fail(PK_ERR_STRUCTURE, "cptrs[0] must be 0");
  std::vector<double> cols(ncols_of(n) * comps, 0.0);
  for (int j = 0; j < n; ++j) {
    if (cptrs[j + 1] < cptrs[j]) fail(PK_ERR_STRUCTURE, "cptrs must be non-decreasing");
    for (int64_t t = cptrs[j]; t < cptrs[j + 1]; ++t) {
      const int64_t r = rids[t];
      if (r < 0 || r >= n) fail(PK_ERR_STRUCTURE, "row index out of range");
      if (t > cptrs[j] && rids[t - 1] >= r)
        fail(PK_ERR_STRUCTURE, "row indices must be strictly ascending within a column");
      if (j < n - 1)
        for (int q = 0; q < comps; ++q) cols[((size_t)j * n + r) * comps + q] = vals[t * comps + q];
    }
  }
  return cols;
}

}  // namespace

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
    check_n(n);
    check_policy(policy);
    if (!x0 || !out_dd || (n > 1 && !cols)) fail(PK_ERR_ARG, "null pointer argument");
    check_range(n, start, end);
    Kind kd = dense_f64_kind(cols, x0, n, policy, (flags & PK_FLAG_EXACT) != 0,
                             (flags & PK_FLAG_SPARSE) != 0, (flags & PK_FLAG_PRECISE) != 0);
    dd_t out[2];
    drive(kd, start, end, log2_chunk, device_list(devices, ndev), out, stats);
    out_dd[0] = out[0].hi;
    out_dd[1] = out[0].lo;
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
    Kind kd = dense_f64_kind(cols, x0, n, policy, true);
    drive_ranges(kd, starts, ends, nranges, device, reinterpret_cast<dd_t*>(out_dd));
  });
}

int pk_dense_f64_chunks(const double* cols, const double* x0, int n, int log2_chunk,
                        uint64_t chunk_lo, uint64_t nchunks, int policy, uint32_t flags,
                        int device, double* out_chunks, double out_total[2]) {
  return guarded([&] {
    check_n(n);
    check_policy(policy);
    if (!x0 || !cols || !out_total) fail(PK_ERR_ARG, "null pointer argument");
    Kind kd = dense_f64_kind(cols, x0, n, policy, (flags & PK_FLAG_EXACT) != 0,
                             (flags & PK_FLAG_SPARSE) != 0, (flags & PK_FLAG_PRECISE) != 0);
    dd_t tot[2];
    drive_chunks(kd, log2_chunk, chunk_lo, nchunks, device, reinterpret_cast<dd_t*>(out_chunks), tot);
    out_total[0] = tot[0].hi;
    out_total[1] = tot[0].lo;
  });
}

int pk_dense_c128(const double* cols, const double* x0, int n, uint64_t start, uint64_t end,
                  uint32_t flags, int log2_chunk, const int* devices, int ndev, double out[4],
                  pk_run_stats* stats) {
  return guarded([&] {
    check_n(n);
    if (!x0 || !out || (n > 1 && !cols)) fail(PK_ERR_ARG, "null pointer argument");
    check_range(n, start, end);
    Kind kd = dense_c128_kind(cols, x0, n, (flags & PK_FLAG_EXACT) != 0,
                              (flags & PK_FLAG_SPARSE) != 0, (flags & PK_FLAG_PRECISE) != 0);
    dd_t res[2];
    drive(kd, start, end, log2_chunk, device_list(devices, ndev), res, stats);
    out[0] = res[0].hi;
    out[1] = res[0].lo;
    out[2] = res[1].hi;
    out[3] = res[1].lo;
  });
}

int pk_dense_c128_ranges(const double* cols, const double* x0, int n, const uint64_t* starts,
                         const uint64_t* ends, int nranges, int device, double* out) {
  return guarded([&] {
    check_n(n);
    if (nranges < 0) fail(PK_ERR_ARG, "negative range count");
    if (nranges == 0) return;
    if (!x0 || !out || !starts || !ends || (n > 1 && !cols)) fail(PK_ERR_ARG, "null pointer argument");
    Kind kd = dense_c128_kind(cols, x0, n, true);
    drive_ranges(kd, starts, ends, nranges, device, reinterpret_cast<dd_t*>(out));
  });
}

int pk_dense_c128_chunks(const double* cols, const double* x0, int n, int log2_chunk,
                         uint64_t chunk_lo, uint64_t nchunks, uint32_t flags, int device,
                         double* out_chunks, double out_total[4]) {
  return guarded([&] {
    check_n(n);
    if (!x0 || !cols || !out_total) fail(PK_ERR_ARG, "null pointer argument");
    Kind kd = dense_c128_kind(cols, x0, n, (flags & PK_FLAG_EXACT) != 0,
                              (flags & PK_FLAG_SPARSE) != 0, (flags & PK_FLAG_PRECISE) != 0);
    dd_t tot[2];
    drive_chunks(kd, log2_chunk, chunk_lo, nchunks, device, reinterpret_cast<dd_t*>(out_chunks), tot);
    out_total[0] = tot[0].hi;
    out_total[1] = tot[0].lo;
    out_total[2] = tot[1].hi;
    out_total[3] = tot[1].lo;
  });
}

int pk_int(const int64_t* a, int n, uint64_t start, uint64_t end, uint32_t flags, int log2_chunk,
           const int* devices, int ndev, uint64_t out_z[3], pk_int_info* info,
           pk_run_stats* stats) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    check_n(n);
    if (!a || !out_z) fail(PK_ERR_ARG, "null pointer argument");
    check_range(n, start, end);
    IntPrep ip = prep_int(a, n);
    ip.sparse = (flags & PK_FLAG_SPARSE) != 0 && n >= pk::kIntNMin;
    fill_info(ip, info);
    std::vector<int> devs = device_list(devices, ndev);
    const int logu = n >= pk::kIntNMin ? (ip.sparse ? pk::kSpaLogU : pk::int_logu(n)) : 0;
    DensePlan pl = plan_dense(n, logu, start, end, log2_chunk, (int)devs.size());
    const int nd = pl.num_groups ? (int)devs.size() : 1;
    std::vector<IntDevResult> res(nd);
    auto work = [&](int i) {
      const uint64_t lo = pl.num_groups * i / nd, hi = pl.num_groups * (i + 1) / nd;
      run_int_on_device(devs[i], ip, pl, lo, hi - lo, i == 0, end, res[i]);
    };
    if (nd == 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (int i = 0; i < nd; ++i) th.emplace_back(work, i);
      for (auto& t : th) t.join();
    }
    pk::i192 total{0, 0, 0};
    for (auto& r : res) {
      if (r.code != PK_OK) fail(r.code, r.err);
      h_i192_add(total, r.sum);
    }
    out_z[0] = total.w0;
    out_z[1] = total.w1;
    out_z[2] = total.w2;
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

int pk_int_ranges(const int64_t* a, int n, const uint64_t* starts, const uint64_t* ends,
                  int nranges, int device, uint64_t* out_z, pk_int_info* info) {
  return guarded([&] {
    check_n(n);
    if (nranges < 0) fail(PK_ERR_ARG, "negative range count");
    if (!a || (nranges > 0 && (!out_z || !starts || !ends))) fail(PK_ERR_ARG, "null pointer argument");
    IntPrep ip = prep_int(a, n);
    fill_info(ip, info);
    if (nranges == 0) return;
    std::vector<Range> rs(nranges);
    for (int i = 0; i < nranges; ++i) {
      check_range(n, starts[i], ends[i]);
      rs[i] = Range(starts[i], ends[i]);
    }
    DevCtx& c = dev_ctx(device);
    std::lock_guard<std::mutex> lock(c.mu);
    ck(cudaSetDevice(device), "cudaSetDevice");
    const unsigned long long *d_s, *d_e;
    const int* d_z0;
    const int* d_cols = upload_int(c, ip, rs, &d_s, &d_e, &d_z0);
    ensure(c.chunks, c.chunks_cap, i192_slots(rs.size()));
    launch_walk_int(c, ip, d_cols, d_z0, d_s, d_e, nranges, (pk::i192*)c.chunks);
    ck(cudaStreamSynchronize(c.stream), "walker execution");
    ck(cudaMemcpy(out_z, c.chunks, rs.size() * sizeof(pk::i192), cudaMemcpyDeviceToHost), "D2H");
  });
}

int pk_dense_f64_batch(const double* cols, const double* x0, int n, int batch, int policy,
                       uint32_t flags, int device, double* out_dd, pk_run_stats* stats) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    check_n(n);
    check_policy(policy);
    if (batch < 0) fail(PK_ERR_ARG, "negative batch");
    if (batch == 0) return;
    if (!x0 || !out_dd || (n > 1 && !cols)) fail(PK_ERR_ARG, "null pointer argument");
    const size_t ncol = (size_t)(n > 1 ? n - 1 : 0) * n;
    DevCtx& c = dev_ctx(device);
    std::lock_guard<std::mutex> lock(c.mu);
    ck(cudaSetDevice(device), "cudaSetDevice");
    // fast modes: every matrix rounded onto its per-row grids (exact states)
    std::vector<double> qcols, qx0;
    if ((flags & PK_FLAG_EXACT) == 0 && n >= pk::kDenseNMin) {
      qcols.resize(ncol * batch);
      qx0.resize((size_t)n * batch);
      for (int b = 0; b < batch; ++b)
        quantize_walk(cols + (size_t)b * ncol, x0 + (size_t)b * n, n, 1,
                      qcols.data() + (size_t)b * ncol, qx0.data() + (size_t)b * n);
      cols = qcols.data();
      x0 = qx0.data();
    }
    const size_t in_doubles = ncol * batch + (size_t)n * batch;
    ensure(c.scratch, c.scratch_cap, in_doubles * 8 + 64);
    double* d_cols = (double*)c.scratch;
    double* d_x0 = d_cols + ncol * batch;
    if (ncol) ck(cudaMemcpyAsync(d_cols, cols, ncol * batch * 8, cudaMemcpyHostToDevice, c.stream), "H2D cols");
    ck(cudaMemcpyAsync(d_x0, x0, (size_t)n * batch * 8, cudaMemcpyHostToDevice, c.stream), "H2D x0");
    ensure(c.chunks, c.chunks_cap, (size_t)batch);
    ck(cudaEventRecord(c.e0, c.stream), "event record");
    int k = 0;
    if (n >= pk::kDenseNMin) {
      k = pk::batch_log2_chunk(n, pk::dense_logu(n));
      const size_t groups = (size_t)((1ull << (n - 1 - k)) / 32);
      ensure(c.groups, c.groups_cap, groups * batch);
      pk::DenseBatchLaunch a{};
      a.d_cols = d_cols;
      a.d_x0 = d_x0;
      a.policy = policy;
      a.exact = (flags & PK_FLAG_EXACT) != 0;
      a.batch = batch;
      a.k = k;
      a.group_part = c.groups;
      a.out = c.chunks;
      a.stream = c.stream;
      a.sms = c.sms;
      ck((cudaError_t)dispatch_dense_batch(n, a), "dense_f64 batch launch");
    } else {
      const unsigned grid = (unsigned)((batch + pk::kWalkBlock - 1) / pk::kWalkBlock);
      switch (policy) {
        case PK_POLICY_DD: pk::walk_dense_f64_multi<pk::POL_DD><<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, batch, c.chunks); break;
        case PK_POLICY_KAHAN: pk::walk_dense_f64_multi<pk::POL_KAHAN><<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, batch, c.chunks); break;
        case PK_POLICY_DQ: pk::walk_dense_f64_multi<pk::POL_DQ><<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, batch, c.chunks); break;
        default: pk::walk_dense_f64_multi<pk::POL_QQ><<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, batch, c.chunks); break;
      }
      ck(cudaGetLastError(), "walk_dense_f64_multi launch");
    }
    ck(cudaEventRecord(c.e1, c.stream), "event record");
    ck(cudaStreamSynchronize(c.stream), "kernel execution");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, c.e0, c.e1), "event time");
    ck(cudaMemcpy(out_dd, c.chunks, (size_t)batch * sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H");
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->kernel_ms = ms;
      stats->iterates = total_iterates(n) * (uint64_t)batch;
      stats->log2_chunk = k;
      stats->devices = 1;
      stats->launches = 1;
      stats->chunks = k ? (uint64_t)batch << (n - 1 - k) : 0;
      stats->wall_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

int pk_int_spa_source(const int64_t* a, int n, char* buf, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    check_n(n);
    if (!a || !len) fail(PK_ERR_ARG, "null pointer argument");
    if (n < pk::kIntNMin) fail(PK_ERR_ARG, "SpaRyser kernels need n >= 11");
    IntPrep ip = prep_int(a, n);
    pk::SpaIntSpec sp;
    sp.n = n;
    sp.zcols = ip.zcols;
    sp.zmax = ip.zmax;
    const std::string src = pk::spa_int_source(sp);
    *len = src.size();
    if (buf && cap > 0) {
      const size_t m = src.size() < cap - 1 ? src.size() : (size_t)cap - 1;
      std::memcpy(buf, src.data(), m);
      buf[m] = '\0';
    }
  });
}

int pk_sparse_f64(const int64_t* cptrs, const int64_t* rids, const double* vals, int n,
                  const double* x0, uint64_t start, uint64_t end, int policy, uint32_t flags,
                  int log2_chunk, const int* devices, int ndev, double out_dd[2],
                  pk_run_stats* stats) {
  return guarded([&] {
    check_n(n);
    check_policy(policy);
    if (!x0 || !out_dd) fail(PK_ERR_ARG, "null pointer argument");
    check_range(n, start, end);
    const std::vector<double> cols = ccs_to_cols(cptrs, rids, vals, n, 1);
    Kind kd = dense_f64_kind(cols.data(), x0, n, policy, (flags & PK_FLAG_EXACT) != 0, true);
    dd_t out[2];
    drive(kd, start, end, log2_chunk, device_list(devices, ndev), out, stats);
    out_dd[0] = out[0].hi;
    out_dd[1] = out[0].lo;
  });
}

int pk_spa_f64_source(const double* cols, int n, int policy, uint32_t flags, char* buf,
                      uint64_t cap, uint64_t* len) {
  return guarded([&] {
    check_n(n);
    check_policy(policy);
    if (!cols || !len) fail(PK_ERR_ARG, "null pointer argument");
    if (n < pk::kDenseNMin) fail(PK_ERR_ARG, "SpaRyser kernels need n >= 11");
    pk::SpaF64Spec sp;
    sp.n = n;
    sp.policy = policy;
    sp.exact = (flags & PK_FLAG_EXACT) != 0;
    sp.rows.resize(n - 1);
    for (int j = 0; j < n - 1; ++j)
      for (int i = 0; i < n; ++i)
        if (cols[(size_t)j * n + i] != 0.0) sp.rows[j].push_back(i);
    const std::string src = pk::spa_f64_source(sp);
    *len = src.size();
    if (buf && cap > 0) {
      const size_t m = src.size() < cap - 1 ? src.size() : (size_t)cap - 1;
      std::memcpy(buf, src.data(), m);
      buf[m] = '\0';
    }
  });
}

int pk_sparse_c128(const int64_t* cptrs, const int64_t* rids, const double* vals, int n,
                   const double* x0, uint64_t start, uint64_t end, uint32_t flags,
                   int log2_chunk, const int* devices, int ndev, double out[4],
                   pk_run_stats* stats) {
  return guarded([&] {
    check_n(n);
    if (!x0 || !out) fail(PK_ERR_ARG, "null pointer argument");
    check_range(n, start, end);
    const std::vector<double> cols = ccs_to_cols(cptrs, rids, vals, n, 2);
    Kind kd = dense_c128_kind(cols.data(), x0, n, (flags & PK_FLAG_EXACT) != 0, true);
    dd_t o[2];
    drive(kd, start, end, log2_chunk, device_list(devices, ndev), o, stats);
    out[0] = o[0].hi;
    out[1] = o[0].lo;
    out[2] = o[1].hi;
    out[3] = o[1].lo;
  });
}

int pk_spa_c128_source(const double* cols, int n, uint32_t flags, char* buf, uint64_t cap,
                       uint64_t* len) {
  return guarded([&] {
    check_n(n);
    if (!cols || !len) fail(PK_ERR_ARG, "null pointer argument");
    if (n < pk::kC128NMin || n > pk::kC128NMax)
      fail(PK_ERR_ARG, "complex SpaRyser kernels need 11 <= n <= 40");
    const std::string src = pk::spa_c128_source(spa_c128_spec(cols, n, (flags & PK_FLAG_EXACT) != 0));
    *len = src.size();
    if (buf && cap > 0) {
      const size_t m = src.size() < cap - 1 ? src.size() : (size_t)cap - 1;
      std::memcpy(buf, src.data(), m);
      buf[m] = '\0';
    }
  });
}

int pk_dense_c128_batch(const double* cols, const double* x0, int n, int batch, uint32_t flags,
                        int device, double* out, pk_run_stats* stats) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    check_n(n);
    if (batch < 0) fail(PK_ERR_ARG, "negative batch");
    if (batch == 0) return;
    if (!x0 || !out || (n > 1 && !cols)) fail(PK_ERR_ARG, "null pointer argument");
    const size_t ncol = 2 * (size_t)(n > 1 ? n - 1 : 0) * n;
    DevCtx& c = dev_ctx(device);
    std::lock_guard<std::mutex> lock(c.mu);
    ck(cudaSetDevice(device), "cudaSetDevice");
    // fast modes: every matrix rounded onto its per-row, per-component grids
    std::vector<double> qcols, qx0;
    if ((flags & PK_FLAG_EXACT) == 0 && n >= pk::kC128NMin) {
      qcols.resize(ncol * batch);
      qx0.resize(2 * (size_t)n * batch);
      for (int b = 0; b < batch; ++b)
        quantize_walk(cols + (size_t)b * ncol, x0 + 2 * (size_t)b * n, n, 2,
                      qcols.data() + (size_t)b * ncol, qx0.data() + 2 * (size_t)b * n);
      cols = qcols.data();
      x0 = qx0.data();
    }
    const size_t in_doubles = ncol * batch + 2 * (size_t)n * batch;
    ensure(c.scratch, c.scratch_cap, in_doubles * 8 + 64);
    double* d_cols = (double*)c.scratch;
    double* d_x0 = d_cols + ncol * batch;
    if (ncol) ck(cudaMemcpyAsync(d_cols, cols, ncol * batch * 8, cudaMemcpyHostToDevice, c.stream), "H2D cols");
    ck(cudaMemcpyAsync(d_x0, x0, 2 * (size_t)n * batch * 8, cudaMemcpyHostToDevice, c.stream), "H2D x0");
    ensure(c.chunks, c.chunks_cap, 2 * (size_t)batch);
    ck(cudaEventRecord(c.e0, c.stream), "event record");
    int k = 0;
    if (n >= pk::kC128NMin) {
      const bool pair = c128_use_pair(n);  // K3p above K3's register limit
      k = pk::batch_log2_chunk(n, pair ? ((flags & PK_FLAG_EXACT) ? pk::c128_pair_logu(n)
                                                                 : pk::c128_pair_fast_logu(n))
                                  : (flags & PK_FLAG_EXACT) ? pk::c128_logu(n)
                                                            : pk::c128_fast_logu(n));
      const size_t groups = (size_t)((1ull << (n - 1 - k)) / 32);
      ensure(c.groups, c.groups_cap, 2 * groups * batch);
      pk::C128BatchLaunch a{};
      a.d_cols = d_cols;
      a.d_x0 = d_x0;
      a.exact = (flags & PK_FLAG_EXACT) != 0;
      a.batch = batch;
      a.k = k;
      a.group_part = c.groups;
      a.out = c.chunks;
      a.stream = c.stream;
      a.sms = c.sms;
      ck((cudaError_t)(pair ? dispatch_c128_pair_batch(n, a) : dispatch_c128_batch(n, a)),
         "dense_c128 batch launch");
    } else {
      const unsigned grid = (unsigned)((batch + pk::kWalkBlock - 1) / pk::kWalkBlock);
      pk::walk_dense_c128_multi<<<grid, pk::kWalkBlock, 0, c.stream>>>(d_cols, d_x0, n, batch, c.chunks);
      ck(cudaGetLastError(), "walk_dense_c128_multi launch");
    }
    ck(cudaEventRecord(c.e1, c.stream), "event record");
    ck(cudaStreamSynchronize(c.stream), "kernel execution");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, c.e0, c.e1), "event time");
    if (k) {
      // register kernels: (re dd, im dd) per matrix
      ck(cudaMemcpy(out, c.chunks, (size_t)batch * 2 * sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H");
    } else {
      // walkers: plain (re, im) per matrix -> (re, 0, im, 0)
      std::vector<dd_t> w((size_t)batch);
      ck(cudaMemcpy(w.data(), c.chunks, (size_t)batch * sizeof(dd_t), cudaMemcpyDeviceToHost), "D2H");
      for (int b = 0; b < batch; ++b) {
        out[4 * b] = w[b].hi;
        out[4 * b + 1] = 0.0;
        out[4 * b + 2] = w[b].lo;
        out[4 * b + 3] = 0.0;
      }
    }
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->kernel_ms = ms;
      stats->iterates = total_iterates(n) * (uint64_t)batch;
      stats->log2_chunk = k;
      stats->devices = 1;
      stats->launches = 1;
      stats->chunks = k ? (uint64_t)batch << (n - 1 - k) : 0;
      stats->wall_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

// acc = dd_add(acc, (v_k, 0)) over k in order, from acc = (0, 0): the
// reference's leaf combination (preprocess.py:398-417) for one component
int pk_quantize_walk(const double* cols, const double* x0, int n, int comps, double* qcols,
                     double* qx0) {
  return guarded([&] {
    check_n(n);
    if (comps != 1 && comps != 2) fail(PK_ERR_ARG, "comps must be 1 (real) or 2 (complex)");
    if (!x0 || !qx0 || (n > 1 && (!cols || !qcols))) fail(PK_ERR_ARG, "null pointer argument");
    const size_t nc = (size_t)comps * (n > 1 ? n - 1 : 0) * n;
    std::vector<double> c(cols, cols + nc), x(x0, x0 + (size_t)comps * n);  // outputs may alias
    quantize_walk(c.data(), x.data(), n, comps, qcols, qx0);
  });
}

int pk_dd_accumulate(const double* vals, int64_t count, double out[2]) {
  return guarded([&] {
    if ((!vals && count > 0) || !out || count < 0) fail(PK_ERR_ARG, "bad arguments");
    dd_t acc{0.0, 0.0};
    for (int64_t k = 0; k < count; ++k) acc = h_dd_add(acc, dd_t{vals[k], 0.0});
    out[0] = acc.hi;
    out[1] = acc.lo;
  });
}

int pk_int_batch(const int64_t* a, int n, int batch, int device, uint64_t* out_z,
                 pk_int_info* info, pk_run_stats* stats) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    check_n(n);
    if (batch < 0) fail(PK_ERR_ARG, "negative batch");
    if (batch == 0) return;
    if (!a || !out_z) fail(PK_ERR_ARG, "null pointer argument");
    const size_t nn = (size_t)n * n, nc = (size_t)(n > 1 ? n - 1 : 0) * n;
    std::vector<int> hcols(nc * batch), hz0((size_t)n * batch);
    int zb = 5;
    for (int b = 0; b < batch; ++b) {
      IntPrep ip = prep_int(a + nn * b, n);
      if (!ip.exact_terms)
        fail(PK_ERR_OVERFLOW, "batched integer walk: a term may reach 2^127 (matrix " +
                                  std::to_string(b) + ")");
      if (nc) std::memcpy(hcols.data() + nc * b, ip.zcols.data(), nc * sizeof(int));
      std::memcpy(hz0.data() + (size_t)n * b, ip.z0.data(), (size_t)n * sizeof(int));
      if (ip.zb > zb) zb = ip.zb;
      if (info) fill_info(ip, info + b);
    }
    DevCtx& c = dev_ctx(device);
    std::lock_guard<std::mutex> lock(c.mu);
    ck(cudaSetDevice(device), "cudaSetDevice");
    const size_t ints = ((nc + n) * batch + 3) & ~size_t(3);
    ensure(c.scratch, c.scratch_cap, ints * 4 + 64);
    int* d_cols = (int*)c.scratch;
    int* d_z0 = d_cols + nc * batch;
    if (nc) ck(cudaMemcpyAsync(d_cols, hcols.data(), nc * batch * 4, cudaMemcpyHostToDevice, c.stream), "H2D cols");
    ck(cudaMemcpyAsync(d_z0, hz0.data(), (size_t)n * batch * 4, cudaMemcpyHostToDevice, c.stream), "H2D z0");
    // i192 outputs in the dd workspaces (24 B <= 32 B per dd pair)
    ensure(c.chunks, c.chunks_cap, i192_slots((size_t)batch));
    ck(cudaEventRecord(c.e0, c.stream), "event record");
    int k = 0;
    if (n >= pk::kIntNMin) {
      k = pk::batch_log2_chunk(n, pk::int_logu(n));
      const size_t groups = (size_t)((1ull << (n - 1 - k)) / 32);
      ensure(c.groups, c.groups_cap, i192_slots(groups * batch));
      pk::IntBatchLaunch l{};
      l.d_cols = d_cols;
      l.d_z0 = d_z0;
      l.zb = zb;
      l.batch = batch;
      l.k = k;
      l.group_part = c.groups;
      l.out = c.chunks;
      l.stream = c.stream;
      l.sms = c.sms;
      ck((cudaError_t)dispatch_int_batch(n, l), "int batch launch");
    } else {
      const unsigned grid = (unsigned)((batch + 127) / 128);
      pk::walk_int_multi<<<grid, 128, 0, c.stream>>>(d_cols, d_z0, n, batch, (pk::i192*)c.chunks);
      ck(cudaGetLastError(), "walk_int_multi launch");
    }
    ck(cudaEventRecord(c.e1, c.stream), "event record");
    ck(cudaStreamSynchronize(c.stream), "kernel execution");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, c.e0, c.e1), "event time");
    std::vector<pk::i192> hv((size_t)batch);
    ck(cudaMemcpy(hv.data(), c.chunks, (size_t)batch * sizeof(pk::i192), cudaMemcpyDeviceToHost), "D2H");
    for (int b = 0; b < batch; ++b) {
      out_z[3 * b] = hv[b].w0;
      out_z[3 * b + 1] = hv[b].w1;
      out_z[3 * b + 2] = hv[b].w2;
    }
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->kernel_ms = ms;
      stats->iterates = total_iterates(n) * (uint64_t)batch;
      stats->log2_chunk = k;
      stats->devices = 1;
      stats->launches = 1;
      stats->wall_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

}  // extern "C"
