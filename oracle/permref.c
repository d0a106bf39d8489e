/*
 * permref.c -- CPU restatement of permkit's Gray-walk permanent hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity oracle: tests/, the smoke()
 * entry and bench.py's cpu_baseline leg may call it, nothing in the product
 * path may. It restates, operation for operation, the reference algorithm in
 * /root/reference/pkg/src/permkit (a pure Python + numba package; no native
 * sources exist to compile, so there is no oracle/_ref build):
 *
 *   state builders   kernels.py:75-163    (dense/sparse x0, doubled int state)
 *   jump-in          parallel.py:162-229  (init_x_at / _y_init_at)
 *   chunk loops      _loops.py:35-284     (policies DD/KAHAN/DQ/QQ, c128, int)
 *   run_range        parallel.py:232-289  (partial normalisation)
 *
 * Pinned against the reference itself: the JSON fixtures under tests/golden/ were made by
 * tools/make_golden.py importing permkit, and tests/test_oracle.py checks this
 * file bit for bit against them.
 *
 * Compile: cc -O2 -fPIC -shared -ffp-contract=off -o liboracle.so permref.c -lpthread
 * -ffp-contract=off matters: the reference's float arithmetic has one rounding
 * per operation (CPython / numba without fastmath never fuse a*b+c).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

enum { POL_DD = 0, POL_KAHAN = 1, POL_DQ = 2, POL_QQ = 3 };

static const double SPLITTER = 134217729.0; /* 2^27 + 1, precision.py:21 */

/* iterate g >= 1: changed column = ctz(g); direction +1 iff Gray bit j is
 * set after the flip (graycode.py:26-37, _loops.py:39-46) */
static inline int changed_col(uint64_t g) { return __builtin_ctzll(g); }
static inline double flip_sign(uint64_t g, int j) {
  uint64_t gray = g ^ (g >> 1);
  return ((gray >> j) & 1ull) ? 1.0 : -1.0;
}

/* ------------------------------------------------------------------------ */
/* accumulators (_loops.py:50-105)                                           */

typedef struct { double a, b; } acc2;

static inline void acc_fold(acc2* acc, double term, int policy) {
  if (policy == POL_DD) {
    acc->a = acc->a + term;
  } else if (policy == POL_KAHAN) {
    double y = term + acc->b;
    double t = acc->a + y;
    acc->b = (acc->a - t) + y;
    acc->a = t;
  } else { /* DQ */
    double s1 = acc->a + term;
    double bb = s1 - acc->a;
    double e = (acc->a - (s1 - bb)) + (term - bb);
    e = e + acc->b;
    acc->a = s1 + e;
    acc->b = e - (acc->a - s1);
  }
}

static inline void acc_fold_qq(acc2* acc, double th, double tl) {
  double s1 = acc->a + th;
  double bb = s1 - acc->a;
  double s2 = (acc->a - (s1 - bb)) + (th - bb);
  double t1 = acc->b + tl;
  double bb2 = t1 - acc->b;
  double t2e = (acc->b - (t1 - bb2)) + (tl - bb2);
  s2 = s2 + t1;
  double sh = s1 + s2;
  double sl = s2 - (sh - s1);
  sl = sl + t2e;
  acc->a = sh + sl;
  acc->b = sl - (acc->a - sh);
}

/* double-double product of the state, Dekker split (_loops.py:50-66) */
static inline void qq_product(const double* x, int n, double* ph_out, double* pl_out) {
  double ph = 1.0, pl = 0.0;
  for (int i = 0; i < n; ++i) {
    double xi = x[i];
    double p = ph * xi;
    double t = SPLITTER * ph;
    double ahi = t - (t - ph);
    double alo = ph - ahi;
    double t2 = SPLITTER * xi;
    double bhi = t2 - (t2 - xi);
    double blo = xi - bhi;
    double e = ((ahi * bhi - p) + ahi * blo + alo * bhi) + alo * blo;
    e = e + pl * xi;
    ph = p + e;
    pl = e - (ph - p);
  }
  *ph_out = ph;
  *pl_out = pl;
}

static inline void fold_state(acc2* acc, const double* x, int n, uint64_t g, int policy) {
  if (policy == POL_QQ) {
    double ph, pl;
    qq_product(x, n, &ph, &pl);
    if (g & 1ull) acc_fold_qq(acc, -ph, -pl);
    else acc_fold_qq(acc, ph, pl);
  } else {
    double prod = 1.0;
    for (int i = 0; i < n; ++i) prod = prod * x[i];
    acc_fold(acc, (g & 1ull) ? -prod : prod, policy);
  }
}

/* run_range's lossless normalisation to a double-double (parallel.py:282-289) */
static void normalise(acc2 acc, int policy, double out[2]) {
  if (policy == POL_DD) {
    out[0] = acc.a;
    out[1] = 0.0;
  } else if (policy == POL_KAHAN) {
    double s = acc.a + acc.b;
    double bb = s - acc.a;
    double e = (acc.a - (s - bb)) + (acc.b - bb);
    out[0] = s;
    out[1] = e;
  } else {
    out[0] = acc.a;
    out[1] = acc.b;
  }
}

/* ------------------------------------------------------------------------ */
/* state builders                                                            */

/* dense_float_state (kernels.py:75-89): cols[j*n+i] = a_ij (j < n-1),
 * x0 = a_{i,n-1} - rowsum_i/2 with left-to-right row sums (matrix.py:333-343).
 * a is row major. */
void oracle_dense_f64_state(const double* a, int n, double* cols, double* x0) {
  for (int j = 0; j < n - 1; ++j)
    for (int i = 0; i < n; ++i) cols[j * n + i] = a[i * n + j];
  for (int i = 0; i < n; ++i) {
    double rs = a[i * n];
    for (int j = 1; j < n; ++j) rs = rs + a[i * n + j];
    x0[i] = a[i * n + n - 1] - rs / 2.0;
  }
}

/* ------------------------------------------------------------------------ */
/* dense real: run_range (parallel.py:232-289) over chunk_dense_f64          */

int oracle_dense_f64_range(const double* cols, const double* x0, int n, uint64_t start,
                           uint64_t end, int policy, double out[2]) {
  if (n < 1 || n > 63 || start < 1 || end < start) return -1;
  if (end > ((1ull << (n - 1)) - 1ull)) return -1;
  double x[64];
  memcpy(x, x0, sizeof(double) * (size_t)n);
  /* init_x_at(start - 1): ascending columns of gray(start-1) */
  uint64_t code = (start - 1) ^ ((start - 1) >> 1);
  for (int j = 0; code; ++j, code >>= 1)
    if (code & 1ull)
      for (int i = 0; i < n; ++i) x[i] = x[i] + cols[j * n + i];
  acc2 acc = {0.0, 0.0};
  for (uint64_t g = start; g <= end; ++g) {
    int j = changed_col(g);
    double s = flip_sign(g, j);
    const double* c = cols + (size_t)j * n;
    for (int i = 0; i < n; ++i) x[i] = x[i] + s * c[i];
    fold_state(&acc, x, n, g, policy);
    if (g == UINT64_MAX) break;
  }
  normalise(acc, policy, out);
  return 0;
}

/* g = 0 term in the policy's inner precision (parallel.py:292-315,
 * kernels.py:166-180). out = (hi, lo); lo = 0 unless QQ. */
void oracle_dense_f64_p0(const double* x0, int n, int policy, double out[2]) {
  if (policy == POL_QQ) {
    qq_product(x0, n, &out[0], &out[1]);
  } else {
    double p = 1.0;
    for (int i = 0; i < n; ++i) p = p * x0[i];
    out[0] = p;
    out[1] = 0.0;
  }
}

/* ------------------------------------------------------------------------ */
/* sparse real (CCS): chunk_sparse_f64 (_loops.py:110-183). x0 comes from
 * sparse_float_state (kernels.py:113-127), built by the caller.             */

int oracle_sparse_f64_range(const int64_t* cptrs, const int64_t* rids, const double* vals,
                            const double* x0, int n, uint64_t start, uint64_t end, int policy,
                            double out[2]) {
  if (n < 1 || n > 63 || start < 1 || end < start) return -1;
  if (end > ((1ull << (n - 1)) - 1ull)) return -1;
  double x[64];
  memcpy(x, x0, sizeof(double) * (size_t)n);
  uint64_t code = (start - 1) ^ ((start - 1) >> 1);
  for (int j = 0; code; ++j, code >>= 1)
    if (code & 1ull)
      for (int64_t p = cptrs[j]; p < cptrs[j + 1]; ++p) x[rids[p]] = x[rids[p]] + vals[p];
  acc2 acc = {0.0, 0.0};
  for (uint64_t g = start; g <= end; ++g) {
    int j = changed_col(g);
    double s = flip_sign(g, j);
    for (int64_t p = cptrs[j]; p < cptrs[j + 1]; ++p) x[rids[p]] = x[rids[p]] + s * vals[p];
    fold_state(&acc, x, n, g, policy);
  }
  normalise(acc, policy, out);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* complex, plain double only (_loops.py:186-235). Interleaved (re, im).
 * Complex product as CPython/numba evaluate it: (ac - bd) + (ad + bc)i with
 * one rounding per operation. s*col with s = +-1 is exact per component.    */

static inline void cmul(double ar, double ai, double br, double bi, double* cr, double* ci) {
  *cr = ar * br - ai * bi;
  *ci = ar * bi + ai * br;
}

static void c128_fold(double* accr, double* acci, const double* x, int n, uint64_t g) {
  double pr = 1.0, pi = 0.0;
  for (int i = 0; i < n; ++i) {
    double r, im;
    cmul(pr, pi, x[2 * i], x[2 * i + 1], &r, &im);
    pr = r;
    pi = im;
  }
  if (g & 1ull) {
    *accr = *accr - pr;
    *acci = *acci - pi;
  } else {
    *accr = *accr + pr;
    *acci = *acci + pi;
  }
}

int oracle_dense_c128_range(const double* cols, const double* x0, int n, uint64_t start,
                            uint64_t end, double out[2]) {
  if (n < 1 || n > 63 || start < 1 || end < start) return -1;
  if (end > ((1ull << (n - 1)) - 1ull)) return -1;
  double x[128];
  memcpy(x, x0, sizeof(double) * 2 * (size_t)n);
  uint64_t code = (start - 1) ^ ((start - 1) >> 1);
  for (int j = 0; code; ++j, code >>= 1)
    if (code & 1ull)
      for (int i = 0; i < n; ++i) {
        x[2 * i] = x[2 * i] + cols[2 * (j * n + i)];
        x[2 * i + 1] = x[2 * i + 1] + cols[2 * (j * n + i) + 1];
      }
  double accr = 0.0, acci = 0.0;
  for (uint64_t g = start; g <= end; ++g) {
    int j = changed_col(g);
    double s = flip_sign(g, j);
    const double* c = cols + 2 * (size_t)j * n;
    for (int i = 0; i < n; ++i) {
      /* x + s*c with s promoted to complex(s, 0): full complex product, as
       * CPython 3.12 / numba evaluate float * complex */
      double sr, si;
      cmul(s, 0.0, c[2 * i], c[2 * i + 1], &sr, &si);
      x[2 * i] = x[2 * i] + sr;
      x[2 * i + 1] = x[2 * i + 1] + si;
    }
    c128_fold(&accr, &acci, x, n, g);
  }
  out[0] = accr;
  out[1] = acci;
  return 0;
}

int oracle_sparse_c128_range(const int64_t* cptrs, const int64_t* rids, const double* vals,
                             const double* x0, int n, uint64_t start, uint64_t end,
                             double out[2]) {
  if (n < 1 || n > 63 || start < 1 || end < start) return -1;
  if (end > ((1ull << (n - 1)) - 1ull)) return -1;
  double x[128];
  memcpy(x, x0, sizeof(double) * 2 * (size_t)n);
  uint64_t code = (start - 1) ^ ((start - 1) >> 1);
  for (int j = 0; code; ++j, code >>= 1)
    if (code & 1ull)
      for (int64_t p = cptrs[j]; p < cptrs[j + 1]; ++p) {
        int64_t r = rids[p];
        x[2 * r] = x[2 * r] + vals[2 * p];
        x[2 * r + 1] = x[2 * r + 1] + vals[2 * p + 1];
      }
  double accr = 0.0, acci = 0.0;
  for (uint64_t g = start; g <= end; ++g) {
    int j = changed_col(g);
    double s = flip_sign(g, j);
    for (int64_t p = cptrs[j]; p < cptrs[j + 1]; ++p) {
      int64_t r = rids[p];
      double sr, si;
      cmul(s, 0.0, vals[2 * p], vals[2 * p + 1], &sr, &si);
      x[2 * r] = x[2 * r] + sr;
      x[2 * r + 1] = x[2 * r + 1] + si;
    }
    c128_fold(&accr, &acci, x, n, g);
  }
  out[0] = accr;
  out[1] = acci;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* exact integers: y = 2x walk (_loops.py:238-284, _y_init_at parallel.py:204-229).
 * Python ints are unbounded; here products and the running total use
 * __int128 with overflow detection, which covers every test size (the caller
 * gets -2 if a value would not fit). out = (lo, hi) two's complement words.  */

typedef __int128 i128;

static int int_fold(i128* total, const int64_t* y, int n, uint64_t g) {
  i128 prod = 1;
  for (int i = 0; i < n; ++i)
    if (__builtin_mul_overflow(prod, (i128)y[i], &prod)) return -2;
  if (g & 1ull) {
    if (__builtin_sub_overflow(*total, prod, total)) return -2;
  } else {
    if (__builtin_add_overflow(*total, prod, total)) return -2;
  }
  return 0;
}

static void put_i128(i128 v, int64_t out[2]) {
  out[0] = (int64_t)(uint64_t)((unsigned __int128)v);
  out[1] = (int64_t)(uint64_t)(((unsigned __int128)v) >> 64);
}

/* cols2[j*n+i] = 2*a_ij (j < n-1); y0 = 2*a_{i,n-1} - rowsum_i (kernels.py:104-110) */
int oracle_dense_int_range(const int64_t* cols2, const int64_t* y0, int n, uint64_t start,
                           uint64_t end, int64_t out[2]) {
  if (n < 1 || n > 63 || start < 1 || end < start) return -1;
  if (end > ((1ull << (n - 1)) - 1ull)) return -1;
  int64_t y[64];
  memcpy(y, y0, sizeof(int64_t) * (size_t)n);
  uint64_t code = (start - 1) ^ ((start - 1) >> 1);
  for (int j = 0; code; ++j, code >>= 1)
    if (code & 1ull)
      for (int i = 0; i < n; ++i) y[i] += cols2[j * n + i];
  i128 total = 0;
  for (uint64_t g = start; g <= end; ++g) {
    int j = changed_col(g);
    uint64_t gray = g ^ (g >> 1);
    const int64_t* c = cols2 + (size_t)j * n;
    if ((gray >> j) & 1ull)
      for (int i = 0; i < n; ++i) y[i] += c[i];
    else
      for (int i = 0; i < n; ++i) y[i] -= c[i];
    if (int_fold(&total, y, n, g)) return -2;
  }
  put_i128(total, out);
  return 0;
}

/* sparse integer: CCS with doubled values for columns < n-1 (kernels.py:146-163) */
int oracle_sparse_int_range(const int64_t* cptrs, const int64_t* rids, const int64_t* vals2,
                            const int64_t* y0, int n, uint64_t start, uint64_t end,
                            int64_t out[2]) {
  if (n < 1 || n > 63 || start < 1 || end < start) return -1;
  if (end > ((1ull << (n - 1)) - 1ull)) return -1;
  int64_t y[64];
  memcpy(y, y0, sizeof(int64_t) * (size_t)n);
  uint64_t code = (start - 1) ^ ((start - 1) >> 1);
  for (int j = 0; code; ++j, code >>= 1)
    if (code & 1ull)
      for (int64_t p = cptrs[j]; p < cptrs[j + 1]; ++p) y[rids[p]] += vals2[p];
  i128 total = 0;
  for (uint64_t g = start; g <= end; ++g) {
    int j = changed_col(g);
    uint64_t gray = g ^ (g >> 1);
    if ((gray >> j) & 1ull)
      for (int64_t p = cptrs[j]; p < cptrs[j + 1]; ++p) y[rids[p]] += vals2[p];
    else
      for (int64_t p = cptrs[j]; p < cptrs[j + 1]; ++p) y[rids[p]] -= vals2[p];
    if (int_fold(&total, y, n, g)) return -2;
  }
  put_i128(total, out);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* threaded plan execution for the CPU baseline: the ranges of a plan run on
 * a pthread pool, partials land in range order (execute_plan,
 * parallel.py:318-341); the caller reduces them.                            */

typedef struct {
  const double* cols;
  const double* x0;
  int n, policy, nranges;
  const uint64_t* starts;
  const uint64_t* ends;
  double* out; /* 2 per range */
  int next;
  pthread_mutex_t mu;
  int rc;
} plan_job;

static void* plan_worker(void* arg) {
  plan_job* pj = (plan_job*)arg;
  for (;;) {
    pthread_mutex_lock(&pj->mu);
    int r = pj->next++;
    pthread_mutex_unlock(&pj->mu);
    if (r >= pj->nranges) break;
    if (oracle_dense_f64_range(pj->cols, pj->x0, pj->n, pj->starts[r], pj->ends[r], pj->policy,
                               pj->out + 2 * r))
      pj->rc = -1;
  }
  return NULL;
}

int oracle_dense_f64_ranges_mt(const double* cols, const double* x0, int n,
                               const uint64_t* starts, const uint64_t* ends, int nranges,
                               int policy, int threads, double* out) {
  plan_job pj = {cols, x0, n, policy, nranges, starts, ends, out, 0, PTHREAD_MUTEX_INITIALIZER, 0};
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, plan_worker, &pj);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  return pj.rc;
}
