/*
 * permkit_b200.h -- C ABI of the B200-native Gray-walk permanent kernels.
 *
 * The entry points replace the inner machinery of the reference package
 * permkit (/root/reference/pkg/src/permkit), whose Python surface
 * (permanent, perm_nw, perm_spa, permanent_chunked, run_range, execute_plan)
 * is mirrored one to one by the Python package paper_2502_16577_b200 on top
 * of this ABI (see INTEGRATION.md for the ctypes binding a permkit
 * maintainer would add).
 *
 * Conventions
 *   - All arrays are host memory, C contiguous, owned by the caller. The
 *     library copies what it needs to the device on every call (matrices are
 *     at most 62*63*16 bytes) and keeps only per-device workspace.
 *   - Calls are synchronous and thread safe; results go to caller buffers.
 *   - Every function returns PK_OK (0) or a PK_ERR_* code; pk_last_error()
 *     then holds a message (thread local). There is no CPU fallback: a
 *     missing or failing device is PK_ERR_CUDA.
 *   - Iterates follow the reference: g in [1, 2^(n-1) - 1]; g = 0 (the
 *     initial product) is never part of a range (parallel.py:232-289).
 *   - A range partial is what run_range returns (parallel.py:144-159):
 *     a double-double (hi, lo) for real kinds, (re, im) for complex, and the
 *     exact signed y-space integer (two's complement, little-endian 64-bit
 *     words) for the integer kind.
 */
#ifndef PERMKIT_B200_H
#define PERMKIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PK_ABI_VERSION 1

/* status codes -> permkit exceptions (errors.py:11-47) */
#define PK_OK 0
#define PK_ERR_ARG 1        /* ValueError: bad n, range, pointer or count    */
#define PK_ERR_POLICY 2     /* PolicyError (kernels.py:309-310)               */
#define PK_ERR_STRUCTURE 3  /* StructureError: inconsistent CCS arrays        */
#define PK_ERR_IMPOSSIBLE 4 /* ImpossibleError: n > 63 (matrix.py:35-42)      */
#define PK_ERR_CUDA 5       /* device missing or a CUDA call failed           */
#define PK_ERR_OVERFLOW 6   /* exact integer path cannot represent the values */
#define PK_ERR_TIMEOUT 7    /* DecompTimeout: task or wall-clock budget spent */

/* matrix kinds (matrix.py:25-28) */
#define PK_KIND_REAL 0
#define PK_KIND_COMPLEX 1
#define PK_KIND_INT 2

/* accumulator policies, same codes as _loops.py:27-30 */
#define PK_POLICY_DD 0
#define PK_POLICY_KAHAN 1
#define PK_POLICY_DQ 2
#define PK_POLICY_QQ 3

/* flags */
#define PK_FLAG_EXACT 1u /* per-chunk arithmetic identical to the reference loop
                            (one policy fold per term); default folds a body
                            of 16 terms in plain double first */
#define PK_FLAG_SPARSE 2u /* real and integer walks: generate, compile (NVRTC) and cache a
                             per-matrix SpaRyser kernel that updates only the
                             flipped column's nonzeros (_loops.py:263-284) */
#define PK_FLAG_PRECISE 4u /* dense real and complex walks (pk_dense_f64[_chunks], pk_dense_c128[_chunks]):
                              exact fixed-point row sums, double-double products
                              and sums -- reference-grade values (policy ignored,
                              ~12x the fast walk); the accuracy anchor at orders
                              the reference cannot run */

typedef struct pk_run_stats {
  double kernel_ms;       /* device time of the call's kernels, max over devices */
  double wall_ms;         /* host wall time spent inside the call */
  uint64_t iterates;      /* Gray iterates walked */
  uint64_t chunks;        /* aligned chunks walked by the register kernels */
  uint64_t walker_ranges; /* unaligned pieces walked by the range walkers */
  int32_t log2_chunk;     /* chunk size exponent k */
  int32_t devices;        /* devices used */
  int32_t launches;       /* kernel launches issued */
  int32_t reserved;
} pk_run_stats;

int pk_abi_version(void);
/* number of visible CUDA devices; < 0 on error */
int pk_device_count(void);
/* message for the last failing call on this thread ("" if none) */
const char* pk_last_error(void);

/* measured FP64 peak (DFMA chains, 2 flops each) of `device` in TFLOP/s: the
 * roofline denominator of the FP64-bound walk kernels. iters ~ 20000 gives a
 * ~40 ms measurement on a B200. */
int pk_fp64_peak(int device, int iters, double* tflops, double* ms);

/* ---------------------------------------------------------------- dense real
 * cols[j*n + i] = a_ij for j < n-1; x0[i] = a_{i,n-1} - rowsum_i / 2
 * (dense_float_state, kernels.py:75-89).
 *
 * pk_dense_f64: one partial over iterates [start, end], reduced on the
 * device(s) in a fixed tree order. Replaces run_range (parallel.py:232-289)
 * for large ranges and the whole execute_plan + reduce_partials pipeline
 * (parallel.py:318-387) when [start, end] = [1, 2^(n-1)-1].
 * devices/ndev: CUDA device ordinals to spread the aligned chunks over
 * (NULL/0 = device 0). log2_chunk: 0 = automatic.
 */
int pk_dense_f64(const double* cols, const double* x0, int n, uint64_t start, uint64_t end,
                 int policy, uint32_t flags, int log2_chunk, const int* devices, int ndev,
                 double out_dd[2], pk_run_stats* stats);

/* nranges independent run_range partials, bit-identical to permkit's
 * chunk_dense_f64 over each range (_loops.py:35-107). out: 2 doubles per range. */
int pk_dense_f64_ranges(const double* cols, const double* x0, int n, const uint64_t* starts,
                        const uint64_t* ends, int nranges, int policy, int device,
                        double* out_dd);

/* Per-chunk partials of the register kernel, for parity checks: chunks
 * [chunk_lo, chunk_lo + nchunks) of size 2^log2_chunk (nchunks a multiple of
 * 32), chunk c covering [1 + c*2^k, (c+1)*2^k] clipped to 2^(n-1)-1.
 * out_chunks: 2 doubles per chunk; out_total: the device tree over them. */
int pk_dense_f64_chunks(const double* cols, const double* x0, int n, int log2_chunk,
                        uint64_t chunk_lo, uint64_t nchunks, int policy, uint32_t flags,
                        int device, double* out_chunks, double out_total[2]);

/* Whole walks of `batch` matrices of one order n in one launch (decomposition
 * leaves, boson-sampling submatrices). cols/x0 hold the
 * matrices back to back in the pk_dense_f64 layout; out_dd[2*b] is matrix b's
 * partial over [1, 2^(n-1)-1] (add its g = 0 product and the sign, as
 * reduce_partials does). One block per matrix at a time, its 2^10 aligned
 * chunks tree-reduced like a single launch; n < 11 walks one thread per
 * matrix. */
int pk_dense_f64_batch(const double* cols, const double* x0, int n, int batch, int policy,
                       uint32_t flags, int device, double* out_dd, pk_run_stats* stats);

/* --------------------------------------------------------------- sparse real
 * SpaRyser (chunk_sparse_f64, _loops.py:110-183; state of sparse_float_state,
 * kernels.py:113-127): CCS of the whole matrix, cptrs[n+1] / rids / vals as
 * the reference's CcsMatrix (rows strictly ascending within a column, else
 * PK_ERR_STRUCTURE); column n-1 is already folded into x0 by the caller.
 * The aligned middle of [start, end] runs a kernel generated and compiled
 * (NVRTC, cached per pattern and device) for the nonzero pattern: each step
 * adds only the flipped column's nonzeros. Same arithmetic, chunking and
 * reduction as pk_dense_f64 on the densified matrix, hence the same bits.
 * pk_dense_f64 / pk_dense_f64_chunks with PK_FLAG_SPARSE do the same for a
 * dense column array (pattern = its nonzero entries). */
int pk_sparse_f64(const int64_t* cptrs, const int64_t* rids, const double* vals, int n,
                  const double* x0, uint64_t start, uint64_t end, int policy, uint32_t flags,
                  int log2_chunk, const int* devices, int ndev, double out_dd[2],
                  pk_run_stats* stats);
/* the generated CUDA source for the nonzero pattern of `cols` (n >= 11) */
int pk_spa_f64_source(const double* cols, int n, int policy, uint32_t flags, char* buf,
                      uint64_t cap, uint64_t* len);

/* ------------------------------------------------------------- dense complex
 * Interleaved (re, im) doubles: cols[2*(j*n + i) + {0,1}] = a_ij (j < n-1),
 * x0[2*i + {0,1}] = a_{i,n-1} - rowsum_i / 2 (dense_complex_state,
 * kernels.py:92-101). Complex runs use the plain-double policy only
 * (kernels.py:309-310); the register kernels keep (re, im) partials per
 * chunk and reduce each component as a double-double tree.
 *
 * pk_dense_c128: out = (re_hi, re_lo, im_hi, im_lo) over [start, end]
 * (register kernels for 11 <= n <= 63 -- one thread per chunk to n = 40,
 * a lane pair per chunk above -- range walkers otherwise).
 * pk_dense_c128_ranges: bit-identical run_range partials, out = (re, im) per
 * range (chunk_dense_c128, _loops.py:186-209).
 * pk_dense_c128_chunks: per-chunk (re, im) partials, out_total as above. */
int pk_dense_c128(const double* cols, const double* x0, int n, uint64_t start, uint64_t end,
                  uint32_t flags, int log2_chunk, const int* devices, int ndev, double out[4],
                  pk_run_stats* stats);
int pk_dense_c128_ranges(const double* cols, const double* x0, int n, const uint64_t* starts,
                         const uint64_t* ends, int nranges, int device, double* out);
int pk_dense_c128_chunks(const double* cols, const double* x0, int n, int log2_chunk,
                         uint64_t chunk_lo, uint64_t nchunks, uint32_t flags, int device,
                         double* out_chunks, double out_total[4]);

/* Whole complex walks of `batch` matrices of one order n <= 63 in one launch
 * (boson-sampling submatrices). cols/x0 back to back in the
 * pk_dense_c128 layout; out[4*b .. 4*b+3] = (re_hi, re_lo, im_hi, im_lo) of
 * matrix b's partial over [1, 2^(n-1)-1] (add the g = 0 product and the
 * sign). Equal bit for bit to pk_dense_c128 with the same chunk exponent. */
int pk_dense_c128_batch(const double* cols, const double* x0, int n, int batch, uint32_t flags,
                        int device, double* out, pk_run_stats* stats);

/* SpaRyser for complex pairs (chunk_sparse_c128, _loops.py:212-235; state of
 * sparse_complex_state, kernels.py:130-143): vals interleaved (re, im) per
 * stored entry, otherwise as pk_sparse_f64. out as pk_dense_c128. The
 * generated kernel keeps K3's arithmetic, body length and reduction, so the
 * result equals pk_dense_c128 on the densified pair bit for bit.
 * pk_dense_c128 / pk_dense_c128_chunks accept PK_FLAG_SPARSE likewise. */
int pk_sparse_c128(const int64_t* cptrs, const int64_t* rids, const double* vals, int n,
                   const double* x0, uint64_t start, uint64_t end, uint32_t flags,
                   int log2_chunk, const int* devices, int ndev, double out[4],
                   pk_run_stats* stats);
int pk_spa_c128_source(const double* cols, int n, uint32_t flags, char* buf, uint64_t cap,
                       uint64_t* len);

/* --------------------------------------------------------- exact integers
 * a: row-major n*n int64 matrix (integer kind, matrix.py:53-63). The walk
 * runs on z_i = y_i / 2 (even row sum) or y_i (odd row sum), y = 2x the
 * reference's doubled state (kernels.py:104-110), so
 *     y-space partial (run_range's PartialResult.value) = z-partial * 2^even_rows.
 * out_z: z-space partial over [start, end] as a 192-bit two's complement
 * integer (3 little-endian words). Exact whenever info->exact_terms is 1
 * (every term below 2^127 in magnitude); otherwise only the low 128 bits are
 * meaningful (the partial mod 2^128, enough to recover a whole-walk total
 * under a permanent bound). PK_ERR_OVERFLOW if a row's absolute sum exceeds
 * 2^31 (32-bit state). Register kernels for 11 <= n <= 63, walkers below. */
typedef struct pk_int_info {
  int32_t zbits;          /* |z| < 2^zbits: 5, 7, 15 or 31 */
  int32_t even_rows;      /* rows with even sum: y-space scale 2^even_rows */
  int32_t exact_terms;    /* 1 if the product of the row bounds is < 2^127 */
  int32_t reserved;
  double log2_term_bound; /* log2 of that product */
} pk_int_info;

int pk_int(const int64_t* a, int n, uint64_t start, uint64_t end, uint32_t flags, int log2_chunk,
           const int* devices, int ndev, uint64_t out_z[3], pk_int_info* info,
           pk_run_stats* stats);
/* Whole exact walks of `batch` integer matrices of one order in one launch
 * (decomposition leaves): a holds the matrices back to back (n*n int64
 * each); out_z[3*b..3*b+2] = matrix b's z-space partial over
 * [1, 2^(n-1)-1] (add its g = 0 term and rescale as pk_int's), info[b] its
 * z-space facts. Every matrix must have exact_terms (else PK_ERR_OVERFLOW;
 * the caller then walks it alone, which has the modular route). */
int pk_int_batch(const int64_t* a, int n, int batch, int device, uint64_t* out_z,
                 pk_int_info* info, pk_run_stats* stats);
/* the CUDA source of the generated SpaRyser kernel for `a` (n >= 11): copies
 * at most cap-1 bytes + NUL into buf, *len = full length */
int pk_int_spa_source(const int64_t* a, int n, char* buf, uint64_t cap, uint64_t* len);
/* one exact partial per range (walkers, one device thread each): 3 words each */
int pk_int_ranges(const int64_t* a, int n, const uint64_t* starts, const uint64_t* ends,
                  int nranges, int device, uint64_t* out_z, pk_int_info* info);

/* ------------------------------------------------ decomposition worklist
 * The task tree of permkit's decomp_run (preprocess.py:420-507): LIFO
 * worklist of d1 / d2 / d34 compressions (:289-364) on the sparsest row or
 * column, until every row and column has more than `threshold` nonzeros.
 * Host code (no device work): the caller evaluates the kernel leaves (e.g.
 * in batched launches) and combines contributions in task-id order.
 * a: dense row-major n x n matrix, zeros = absent entries; doubles (real),
 * interleaved (re, im) doubles (complex) or int64 (integer). Integers are
 * exact in 128 bits; beyond that PK_ERR_OVERFLOW. Budgets: PK_ERR_TIMEOUT.
 * On success *handle owns the outputs: fetch them, then free the handle. */
typedef struct pk_decomp_stats {
  uint64_t tasks_created;
  uint64_t d1_applied;
  uint64_t d2_applied;
  uint64_t d34_applied;
  uint64_t trivial_leaves;
  uint64_t kernel_leaves;
  uint64_t dense_kernel_leaves;
  int64_t max_depth;
  double elapsed_s;
} pk_decomp_stats;

typedef struct pk_decomp_result {
  pk_decomp_stats stats;
  int64_t trivial;      /* n = 1 contributions (task id, multiplier * a_00) */
  int64_t leaves;       /* kernel leaves (task id, order, multiplier, matrix) */
  int64_t leaf_values;  /* total scalars of the concatenated leaf matrices */
} pk_decomp_result;

/* The fast modes' input rounding (host only, no device needed): every
 * value of row i (component c of interleaved complex data when comps = 2) is
 * rounded to the grid 2^-F, F = 52 - e, B = |x0_i| + sum_j |a_ij| < 2^e, on
 * which every subset sum x0_i + sum_{j in S} a_ij -- every state of the
 * walk -- is a double. cols are the n-1 walked columns (dense_float_state /
 * dense_complex_state layout), x0 the seed; outputs may alias the inputs.
 * Replaces nothing in the reference: its walk rounds x at every step
 * (_loops.py:47-48); DESIGN.md §3 "Exact states". */
int pk_quantize_walk(const double* cols, const double* x0, int n, int comps, double* qcols,
                     double* qx0);

/* acc = dd_add(acc, (vals[k], 0)) for k in order from (0, 0) (the robust
 * double-double add of precision.py:84-96): permkit's leaf combination */
int pk_dd_accumulate(const double* vals, int64_t count, double out[2]);

int pk_decomp_tree(int kind, int n, const void* a, int threshold, uint64_t task_limit,
                   double time_limit, double dense_density, void** handle,
                   pk_decomp_result* res);
/* scalars: 1 double (real), 2 doubles (complex), 2 int64 words (integer,
 * little-endian two's complement 128-bit); any pointer may be NULL */
int pk_decomp_fetch(void* handle, int64_t* triv_id, void* triv_val, int64_t* leaf_id,
                    int32_t* leaf_n, void* leaf_mult, void* leaf_vals);
void pk_decomp_free(void* handle);
const char* pk_decomp_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* PERMKIT_B200_H */
