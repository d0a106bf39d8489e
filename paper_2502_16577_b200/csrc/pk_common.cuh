// Shared device arithmetic for the Gray-walk kernels.
//
// Every floating-point operation that the reference performs with a separate
// rounding is spelled here with an explicit __d*_rn intrinsic so that nvcc
// can neither contract it into an FMA nor reassociate it. That is what makes
// the per-chunk partials bit-identical to permkit's chunk loops
// (/root/reference/pkg/src/permkit/_loops.py:35-107) when the product is
// evaluated sequentially.
#pragma once
#if defined(__CUDACC_RTC__)
// NVRTC (generated SpaRyser kernels, pk_spa_codegen.cu) has no system headers
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned int uint32_t;
typedef int int32_t;
#else
#include <cstdint>
#endif

namespace pk {

enum Policy : int { POL_DD = 0, POL_KAHAN = 1, POL_DQ = 2, POL_QQ = 3 };

struct dd_t {
  double hi;
  double lo;
};

// ---------------------------------------------------------------------------
// error-free transforms (precision.py:52-64)

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

__device__ __forceinline__ void quick_two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  e = __dsub_rn(b, __dsub_rn(s, a));
}

// Robust double-double add (precision.py:84-96): both component pairs get an
// error-free sum, then two renormalisations.
__device__ __forceinline__ dd_t dd_add(dd_t a, dd_t b) {
  double s1, s2, t1, t2;
  two_sum(a.hi, b.hi, s1, s2);
  two_sum(a.lo, b.lo, t1, t2);
  s2 = __dadd_rn(s2, t1);
  quick_two_sum(s1, s2, s1, s2);
  s2 = __dadd_rn(s2, t2);
  quick_two_sum(s1, s2, s1, s2);
  return dd_t{s1, s2};
}

__device__ __forceinline__ dd_t shfl_down_dd(dd_t v, int off) {
  dd_t r;
  r.hi = __shfl_down_sync(0xffffffffu, v.hi, off);
  r.lo = __shfl_down_sync(0xffffffffu, v.lo, off);
  return r;
}

// Balanced pairwise tree over the 32 lanes of a warp (lane 0 ends up with
// ((p0+p1)+(p2+p3))+...). The shape is fixed, so the result is independent
// of scheduling; it is the bottom five levels of the global chunk tree.
__device__ __forceinline__ dd_t warp_tree_dd(dd_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const dd_t o = shfl_down_dd(v, off);
    if ((lane & (2 * off - 1)) == 0) v = dd_add(v, o);
  }
  return v;
}

// ---------------------------------------------------------------------------
// per-thread partial-sum accumulators, one per policy (_loops.py:88-105).
// add(p) folds +p, sub(p) folds -p: the term sign is the iterate parity.

template <int POL>
struct Acc;

template <>
struct Acc<POL_DD> {
  double a = 0.0;
  __device__ __forceinline__ void add(double p) { a = __dadd_rn(a, p); }
  __device__ __forceinline__ void sub(double p) { a = __dsub_rn(a, p); }
  __device__ __forceinline__ dd_t partial() const { return dd_t{a, 0.0}; }
};

// Compensated: y = term + c; t = s + y; c = (s - t) + y; s = t  (_loops.py:94-98)
template <>
struct Acc<POL_KAHAN> {
  double a = 0.0, b = 0.0;
  __device__ __forceinline__ void fold(double term) {
    const double y = __dadd_rn(term, b);
    const double t = __dadd_rn(a, y);
    b = __dadd_rn(__dsub_rn(a, t), y);
    a = t;
  }
  __device__ __forceinline__ void add(double p) { fold(p); }
  __device__ __forceinline__ void sub(double p) { fold(-p); }
  // run_range normalises a compensated partial with two_sum (parallel.py:284-286)
  __device__ __forceinline__ dd_t partial() const {
    dd_t r;
    two_sum(a, b, r.hi, r.lo);
    return r;
  }
};

// double-double partial, plain-double products (_loops.py:99-105)
template <>
struct Acc<POL_DQ> {
  double a = 0.0, b = 0.0;
  __device__ __forceinline__ void fold(double term) {
    const double s1 = __dadd_rn(a, term);
    const double bb = __dsub_rn(s1, a);
    double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s1, bb)), __dsub_rn(term, bb));
    e = __dadd_rn(e, b);
    a = __dadd_rn(s1, e);
    b = __dsub_rn(e, __dsub_rn(a, s1));
  }
  __device__ __forceinline__ void add(double p) { fold(p); }
  __device__ __forceinline__ void sub(double p) { fold(-p); }
  __device__ __forceinline__ dd_t partial() const { return dd_t{a, b}; }
};

// double-double partial fed by double-double products (_loops.py:50-83)
template <>
struct Acc<POL_QQ> {
  double a = 0.0, b = 0.0;
  __device__ __forceinline__ void fold(double th, double tl) {
    const double s1 = __dadd_rn(a, th);
    const double bb = __dsub_rn(s1, a);
    double s2 = __dadd_rn(__dsub_rn(a, __dsub_rn(s1, bb)), __dsub_rn(th, bb));
    const double t1 = __dadd_rn(b, tl);
    const double bb2 = __dsub_rn(t1, b);
    const double t2e = __dadd_rn(__dsub_rn(b, __dsub_rn(t1, bb2)), __dsub_rn(tl, bb2));
    s2 = __dadd_rn(s2, t1);
    const double sh = __dadd_rn(s1, s2);
    double sl = __dsub_rn(s2, __dsub_rn(sh, s1));
    sl = __dadd_rn(sl, t2e);
    a = __dadd_rn(sh, sl);
    b = __dsub_rn(sl, __dsub_rn(a, sh));
  }
  __device__ __forceinline__ void add2(double ph, double pl) { fold(ph, pl); }
  __device__ __forceinline__ void sub2(double ph, double pl) { fold(-ph, -pl); }
  __device__ __forceinline__ dd_t partial() const { return dd_t{a, b}; }
};

// One double-double product step ph:pl *= xi. The reference splits with
// Dekker's constant because the interpreter has no fma (precision.py:10-11);
// Dekker's error term is exact, and so is fma(ph, xi, -p), so the two agree
// bit for bit. The pl*xi correction keeps its own rounding, as in
// _loops.py:62-65.
__device__ __forceinline__ void qq_mul_step(double& ph, double& pl, double xi) {
  const double p = __dmul_rn(ph, xi);
  double e = __fma_rn(ph, xi, -p);
  e = __dadd_rn(e, __dmul_rn(pl, xi));
  ph = __dadd_rn(p, e);
  pl = __dsub_rn(e, __dsub_rn(ph, p));
}

// compile-time trailing-zero count (column of local step q >= 1)
__host__ __device__ constexpr int ctz_c(int q) {
  int j = 0;
  while (((q >> j) & 1) == 0) ++j;
  return j;
}

// Changed column and direction for iterate g >= 1 (graycode.py:26-37):
// j = ctz(g); the Gray bit j is set after the flip iff bit j+1 of g is 0.
__device__ __forceinline__ int changed_col(uint64_t g) { return __ffsll((long long)g) - 1; }
__device__ __forceinline__ bool flip_on(uint64_t g, int j) { return ((g >> (j + 1)) & 1ull) == 0; }

// ---------------------------------------------------------------------------
// complex, plain double (_loops.py:186-235). Values interleaved (re, im).
// The reference multiplies as CPython/numba do: (ac - bd) + (ad + bc)i, one
// rounding per operation; the column update promotes s to complex(s, 0).

__device__ __forceinline__ void cmul_ref(double ar, double ai, double br, double bi, double& cr,
                                         double& ci) {
  cr = __dsub_rn(__dmul_rn(ar, br), __dmul_rn(ai, bi));
  ci = __dadd_rn(__dmul_rn(ar, bi), __dmul_rn(ai, br));
}

__device__ __forceinline__ void c_update_ref(double& xr, double& xi, double s, double cr,
                                             double ci) {
  double tr, ti;
  cmul_ref(s, 0.0, cr, ci, tr, ti);
  xr = __dadd_rn(xr, tr);
  xi = __dadd_rn(xi, ti);
}

__device__ __forceinline__ void c_fold_ref(double& accr, double& acci, const double* x, int n,
                                           bool odd) {
  double pr = 1.0, pi = 0.0;
  for (int i = 0; i < n; ++i) {
    double r, im;
    cmul_ref(pr, pi, x[2 * i], x[2 * i + 1], r, im);
    pr = r;
    pi = im;
  }
  if (odd) {
    accr = __dsub_rn(accr, pr);
    acci = __dsub_rn(acci, pi);
  } else {
    accr = __dadd_rn(accr, pr);
    acci = __dadd_rn(acci, pi);
  }
}

}  // namespace pk
