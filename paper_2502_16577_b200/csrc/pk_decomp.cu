// Native decomposition worklist (host C++): the task tree of permkit's
// decomp_run (/root/reference/pkg/src/permkit/preprocess.py:420-507) with the
// d1 / d2 / d34 compressions of :289-364, on dense n x n task matrices.
//
// The Python worklist (paper_2502_16577_b200/preprocess.py) spends ~4 us per
// task in the interpreter; trees reach millions of tasks while the GPU leaf
// batches take milliseconds. This unit walks the same tree natively and hands
// back (a) the trivial contributions (n = 1 tasks) and (b) the kernel leaves
// (task id, multiplier, dense matrix), which the Python side evaluates in
// batched GPU launches and combines in task-id order exactly like permkit.
//
// Every value is produced by the scalar operations permkit performs, in the
// same order: float products and sums rounded once each (host code is built
// with -ffp-contract=off), complex products as CPython's
// (ar*br - ai*bi, ar*bi + ai*br), integers exact in 128 bits with overflow
// detection (PK_ERR_OVERFLOW lets the caller fall back to the Python
// worklist, which has arbitrary precision). tests/test_preprocess.py checks
// the tree against the reference's own leaves.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "permkit_b200.h"

namespace {

thread_local std::string g_derr;

struct Fail {
  int code;
  std::string msg;
};

// ------------------------------------------------------------------ scalars

struct Real {
  double v;
  static Real zero() { return {0.0}; }
  bool nz() const { return v != 0.0; }
  Real mul(const Real& b) const { return {v * b.v}; }
  Real add(const Real& b) const { return {v + b.v}; }
};

struct Cplx {
  double r, i;
  static Cplx zero() { return {0.0, 0.0}; }
  bool nz() const { return r != 0.0 || i != 0.0; }
  Cplx mul(const Cplx& b) const { return {r * b.r - i * b.i, r * b.i + i * b.r}; }
  Cplx add(const Cplx& b) const { return {r + b.r, i + b.i}; }
};

struct Int {
  __int128 v;
  static Int zero() { return {0}; }
  bool nz() const { return v != 0; }
  Int mul(const Int& b) const {
    __int128 r;
    if (__builtin_mul_overflow(v, b.v, &r)) throw Fail{PK_ERR_OVERFLOW, "integer overflow"};
    return {r};
  }
  Int add(const Int& b) const {
    __int128 r;
    if (__builtin_add_overflow(v, b.v, &r)) throw Fail{PK_ERR_OVERFLOW, "integer overflow"};
    return {r};
  }
};

// ------------------------------------------------------------------- tasks

template <class T>
struct Task {
  int n;
  std::vector<T> a;  // row-major n x n, zero = no stored entry
  T mult;
  int depth;
  int64_t id;
};

template <class T>
struct Out {
  std::vector<int64_t> triv_id;
  std::vector<T> triv_val;
  std::vector<int64_t> leaf_id;
  std::vector<int32_t> leaf_n;
  std::vector<T> leaf_mult;
  std::vector<T> leaf_vals;  // concatenated n*n matrices
  pk_decomp_stats st{};
};

struct Pick {
  bool row;
  int index;
  int count;
};

template <class T>
Pick min_nnz(const Task<T>& t) {
  const int n = t.n;
  Pick best{true, 0, n + 1};
  for (int i = 0; i < n; ++i) {
    int c = 0;
    for (int j = 0; j < n; ++j) c += t.a[i * n + j].nz();
    if (c < best.count) best = {true, i, c};
  }
  for (int j = 0; j < n; ++j) {
    int c = 0;
    for (int i = 0; i < n; ++i) c += t.a[i * n + j].nz();
    if (c < best.count) best = {false, j, c};
  }
  return best;
}

// minor without row r and column c
template <class T>
std::vector<T> drop(const std::vector<T>& a, int n, int r, int c) {
  std::vector<T> m((size_t)(n - 1) * (n - 1));
  size_t k = 0;
  for (int i = 0; i < n; ++i) {
    if (i == r) continue;
    for (int j = 0; j < n; ++j)
      if (j != c) m[k++] = a[i * n + j];
  }
  return m;
}

// drop `row`; columns j1 < j2 become a2*col(j1) + a1*col(j2) at index 0
// (preprocess.py:304-326: comb = (0 + a2*v1) + a1*v2, zero results dropped)
template <class T>
std::vector<T> fold_cols(const std::vector<T>& a, int n, int row, int j1, const T& a1, int j2,
                         const T& a2) {
  const int m = n - 1;
  std::vector<T> out((size_t)m * m, T::zero());
  int ii = 0;
  for (int i = 0; i < n; ++i) {
    if (i == row) continue;
    const T& v1 = a[i * n + j1];
    const T& v2 = a[i * n + j2];
    bool have = false;
    T comb = T::zero();
    if (v1.nz()) {
      comb = T::zero().add(a2.mul(v1));
      have = true;
    }
    if (v2.nz()) {
      comb = (have ? comb : T::zero()).add(a1.mul(v2));
      have = true;
    }
    if (have && comb.nz()) out[(size_t)ii * m] = comb;
    int jj = 1;
    for (int j = 0; j < n; ++j) {
      if (j == j1 || j == j2) continue;
      out[(size_t)ii * m + jj++] = a[i * n + j];
    }
    ++ii;
  }
  return out;
}

// transposed fold: drop column `col`; rows i1 < i2 become a2*row(i1) +
// a1*row(i2) at index 0, the other rows follow in order
template <class T>
std::vector<T> fold_rows(const std::vector<T>& a, int n, int col, int i1, const T& a1, int i2,
                         const T& a2) {
  const int m = n - 1;
  std::vector<T> out((size_t)m * m, T::zero());
  int jj = 0;
  for (int j = 0; j < n; ++j) {
    if (j == col) continue;
    const T& v1 = a[i1 * n + j];
    const T& v2 = a[i2 * n + j];
    bool have = false;
    T comb = T::zero();
    if (v1.nz()) {
      comb = T::zero().add(a2.mul(v1));
      have = true;
    }
    if (v2.nz()) {
      comb = (have ? comb : T::zero()).add(a1.mul(v2));
      have = true;
    }
    if (have && comb.nz()) out[jj] = comb;
    ++jj;
  }
  int ii = 1;
  for (int i = 0; i < n; ++i) {
    if (i == i1 || i == i2) continue;
    int kk = 0;
    for (int j = 0; j < n; ++j)
      if (j != col) out[(size_t)ii * m + kk++] = a[i * n + j];
    ++ii;
  }
  return out;
}

// the two lowest-index nonzeros of row / column `index`
template <class T>
void first_two(const Task<T>& t, bool row, int index, int& p1, T& v1, int& p2, T& v2) {
  const int n = t.n;
  int k = 0;
  for (int q = 0; q < n && k < 2; ++q) {
    const T& v = row ? t.a[index * n + q] : t.a[q * n + index];
    if (!v.nz()) continue;
    if (k == 0) {
      p1 = q;
      v1 = v;
    } else {
      p2 = q;
      v2 = v;
    }
    ++k;
  }
}

template <class T>
void walk(Task<T> root, int threshold, uint64_t task_limit, double time_limit,
          double dense_density, Out<T>& out) {
  const auto t0 = std::chrono::steady_clock::now();
  pk_decomp_stats& st = out.st;
  std::vector<Task<T>> stack;
  stack.push_back(std::move(root));
  int64_t next_id = 1;
  st.tasks_created = 1;
  uint64_t polls = 0;
  while (!stack.empty()) {
    if (st.tasks_created > task_limit)
      throw Fail{PK_ERR_TIMEOUT, "task budget of " + std::to_string(task_limit) + " exhausted"};
    if ((++polls & 1023) == 0 &&
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > time_limit)
      throw Fail{PK_ERR_TIMEOUT, "wall-clock budget exhausted"};
    Task<T> t = std::move(stack.back());
    stack.pop_back();
    if (t.depth > st.max_depth) st.max_depth = t.depth;
    const int n = t.n;
    const Pick p = min_nnz(t);
    if (p.count == 0) {
      ++st.trivial_leaves;
      continue;
    }
    if (n == 1) {
      ++st.trivial_leaves;
      out.triv_id.push_back(t.id);
      out.triv_val.push_back(t.mult.mul(t.a[0]));
      continue;
    }
    if (p.count == 1) {
      int r = -1, c = -1;
      for (int q = 0; q < n; ++q) {
        if (p.row && t.a[p.index * n + q].nz()) {
          r = p.index;
          c = q;
        }
        if (!p.row && t.a[q * n + p.index].nz()) {
          r = q;
          c = p.index;
        }
      }
      const T alpha = t.a[r * n + c];
      ++st.d1_applied;
      stack.push_back(Task<T>{n - 1, drop(t.a, n, r, c), t.mult.mul(alpha), t.depth + 1, next_id++});
      ++st.tasks_created;
      continue;
    }
    if (p.count == 2 || p.count <= threshold) {  // d2 regardless of the threshold
      int q1 = -1, q2 = -1;
      T v1 = T::zero(), v2 = T::zero();
      first_two(t, p.row, p.index, q1, v1, q2, v2);
      std::vector<T> folded = p.row ? fold_cols(t.a, n, p.index, q1, v1, q2, v2)
                                    : fold_rows(t.a, n, p.index, q1, v1, q2, v2);
      if (p.count == 2) {
        ++st.d2_applied;
        stack.push_back(Task<T>{n - 1, std::move(folded), t.mult, t.depth + 1, next_id++});
        ++st.tasks_created;
        continue;
      }
      std::vector<T> zeroed = t.a;
      if (p.row) {
        zeroed[p.index * n + q1] = T::zero();
        zeroed[p.index * n + q2] = T::zero();
      } else {
        zeroed[q1 * n + p.index] = T::zero();
        zeroed[q2 * n + p.index] = T::zero();
      }
      ++st.d34_applied;
      stack.push_back(Task<T>{n, std::move(zeroed), t.mult, t.depth + 1, next_id});
      stack.push_back(Task<T>{n - 1, std::move(folded), t.mult, t.depth + 1, next_id + 1});
      next_id += 2;
      st.tasks_created += 2;
      continue;
    }
    // dense enough everywhere: a kernel leaf
    int nnz = 0;
    for (const T& v : t.a) nnz += v.nz();
    ++st.kernel_leaves;
    if ((double)nnz / ((double)n * n) >= dense_density) ++st.dense_kernel_leaves;
    out.leaf_id.push_back(t.id);
    out.leaf_n.push_back(n);
    out.leaf_mult.push_back(t.mult);
    out.leaf_vals.insert(out.leaf_vals.end(), t.a.begin(), t.a.end());
  }
  st.elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

struct Handle {
  int kind = 0;
  Out<Real> r;
  Out<Cplx> c;
  Out<Int> z;
};

template <class T>
void copy_out(const Out<T>& o, pk_decomp_result* res) {
  res->stats = o.st;
  res->trivial = (int64_t)o.triv_id.size();
  res->leaves = (int64_t)o.leaf_id.size();
  res->leaf_values = (int64_t)o.leaf_vals.size();
}

}  // namespace

extern "C" {

int pk_decomp_tree(int kind, int n, const void* a, int threshold, uint64_t task_limit,
                   double time_limit, double dense_density, void** handle,
                   pk_decomp_result* res) {
  try {
    if (!a || !handle || !res) throw Fail{PK_ERR_ARG, "null pointer argument"};
    if (n < 1 || n > 63) throw Fail{n > 63 ? PK_ERR_IMPOSSIBLE : PK_ERR_ARG, "bad order"};
    auto* h = new Handle();
    h->kind = kind;
    try {
      const size_t nn = (size_t)n * n;
      if (kind == PK_KIND_REAL) {
        Task<Real> t{n, std::vector<Real>(nn), Real{1.0}, 0, 0};
        for (size_t k = 0; k < nn; ++k) t.a[k].v = ((const double*)a)[k];
        walk(std::move(t), threshold, task_limit, time_limit, dense_density, h->r);
        copy_out(h->r, res);
      } else if (kind == PK_KIND_COMPLEX) {
        Task<Cplx> t{n, std::vector<Cplx>(nn), Cplx{1.0, 0.0}, 0, 0};
        for (size_t k = 0; k < nn; ++k) t.a[k] = {((const double*)a)[2 * k], ((const double*)a)[2 * k + 1]};
        walk(std::move(t), threshold, task_limit, time_limit, dense_density, h->c);
        copy_out(h->c, res);
      } else if (kind == PK_KIND_INT) {
        Task<Int> t{n, std::vector<Int>(nn), Int{1}, 0, 0};
        for (size_t k = 0; k < nn; ++k) t.a[k].v = ((const int64_t*)a)[k];
        walk(std::move(t), threshold, task_limit, time_limit, dense_density, h->z);
        copy_out(h->z, res);
      } else {
        throw Fail{PK_ERR_ARG, "unknown kind"};
      }
    } catch (...) {
      delete h;
      throw;
    }
    *handle = h;
    g_derr.clear();
    return PK_OK;
  } catch (const Fail& f) {
    g_derr = f.msg;
    return f.code;
  } catch (const std::exception& e) {
    g_derr = e.what();
    return PK_ERR_ARG;
  }
}

// Copy the tree's outputs. Scalars are 1 double (real), 2 doubles (complex,
// re/im) or 2 int64 words (integer, little-endian two's complement 128-bit).
int pk_decomp_fetch(void* handle, int64_t* triv_id, void* triv_val, int64_t* leaf_id,
                    int32_t* leaf_n, void* leaf_mult, void* leaf_vals) {
  auto* h = (Handle*)handle;
  if (!h) return PK_ERR_ARG;
  auto put = [&](const auto& o) {
    using T = typename std::decay_t<decltype(o.leaf_mult)>::value_type;
    static_assert(sizeof(T) % 8 == 0, "scalar layout");
    if (triv_id) std::memcpy(triv_id, o.triv_id.data(), o.triv_id.size() * 8);
    if (triv_val) std::memcpy(triv_val, o.triv_val.data(), o.triv_val.size() * sizeof(T));
    if (leaf_id) std::memcpy(leaf_id, o.leaf_id.data(), o.leaf_id.size() * 8);
    if (leaf_n) std::memcpy(leaf_n, o.leaf_n.data(), o.leaf_n.size() * 4);
    if (leaf_mult) std::memcpy(leaf_mult, o.leaf_mult.data(), o.leaf_mult.size() * sizeof(T));
    if (leaf_vals) std::memcpy(leaf_vals, o.leaf_vals.data(), o.leaf_vals.size() * sizeof(T));
  };
  if (h->kind == PK_KIND_REAL) put(h->r);
  else if (h->kind == PK_KIND_COMPLEX) put(h->c);
  else put(h->z);
  return PK_OK;
}

void pk_decomp_free(void* handle) { delete (Handle*)handle; }

const char* pk_decomp_last_error(void) { return g_derr.c_str(); }

}  // extern "C"
