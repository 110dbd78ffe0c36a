/*
 * rac_b200.h — C ABI of the B200-native RAC-MBADMM sweep (arXiv 1907.01995).
 *
 * The reference (`racml` 0.1.0, pure Python over numpy/scipy) has no
 * FFI/plugin layer: its boundary is three Python entry points.  This ABI sits
 * *underneath* their drop-in replacements (paper_1907_01995_b200.{elastic_net,
 * svm,engine}) and replaces the numpy/LAPACK calls each of them makes.  Every
 * entry point cites the reference code it replaces.
 *
 * Conventions
 *   - All pointers are DEVICE pointers unless the name ends in `_host`.
 *   - All arithmetic is IEEE FP64; indices are int64 on input, int32 inside.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - Every function returns RAC_OK (0) or an error code; no exceptions cross
 *     the ABI.  rac_last_error() returns a thread-local message.
 *   - Work is enqueued asynchronously on `stream` unless stated otherwise.
 */
#ifndef RAC_B200_H
#define RAC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RAC_OK 0
#define RAC_ERR_ARG 1          /* invalid argument (reference: ValueError)               */
#define RAC_ERR_CUDA 2         /* CUDA runtime error / no sm_100 device                   */
#define RAC_ERR_NOT_PD 3       /* block not positive definite (BlockDefinitenessError)    */
#define RAC_ERR_UNSUPPORTED 4  /* shape outside what this build supports                  */

/* sweep modes (problems.py:318-323 Mode) */
#define RAC_MODE_RAC 0
#define RAC_MODE_RP 1
#define RAC_MODE_CYCLIC 2

/* solve status (problems.py:326-329 Status) */
#define RAC_STATUS_MAX_ITERS 0
#define RAC_STATUS_CONVERGED 1
#define RAC_STATUS_DIVERGED 2

/* kernel kinds (svm.py:37-48 KernelSpec.kind) */
#define RAC_KERNEL_LINEAR 0
#define RAC_KERNEL_GAUSSIAN 1

/* how rac_en forms the block systems and the coupling term */
#define RAC_GRAM_BLOCKS 0     /* per sweep: X_b'X_b of every block from X (the reference's recompute) */
#define RAC_GRAM_COVARIANCE 1 /* once: G = X'X/m (n x n); blocks gather G, chain updates q = G beta */

/* design-matrix layouts accepted by rac_en_set_data */
#define RAC_LAYOUT_ROW_MAJOR 0 /* numpy C order, X[i*n + j]                                */
#define RAC_LAYOUT_COL_MAJOR 1 /* Fortran order with leading dim m, X[i + j*m]             */

const char* rac_version(void);
const char* rac_last_error(void);
/* Number of kernels this library has launched since load (all contexts, all
 * streams); used by bench.py to report gpu_launches inside a timed region. */
uint64_t rac_launch_count(void);

/* Return freed context memory of the current device's stream-ordered pool to the
 * driver, keeping at most keep_bytes mapped (the pool itself keeps <= 8 GiB across
 * synchronisations).  No reference counterpart: numpy frees eagerly. */
int rac_trim_pool(uint64_t keep_bytes);
/* 0 if `device` is an sm_100 part this library was built for. */
int rac_device_check(int device);

/* ------------------------------------------------------------------ K1
 * Random without-replacement block assembly.
 * Replaces problems.py:234-243 chunk_indices(rng.permutation(n), s) as used at
 * elastic_net.py:195, svm.py:231, engine.py:318-319.  `perms` holds `count`
 * permutations of 0..n-1 (int64, the host PCG64 stream); `idx_out` receives,
 * per permutation, p = ceil(n/s) rows of s int32 indices, each row sorted
 * ascending (the last row holds n - (p-1)s valid entries, the rest are -1). */
int rac_chunk_sort(const int64_t* perms, int64_t n, int32_t s, int32_t count,
                   int32_t* idx_out, void* stream);

/* ------------------------------------------------------------------ K2/K3
 * Batched block systems for one partition (p blocks of s indices):
 *   sys_b = scale * V_b' V_b + shift * I         (elastic_net.py:210-212)
 * where V_b gathers vectors idx[b*s + j] of V (vector k = V[k*ldv .. +len]).
 * Then L_b = chol(sys_b) and inv_b = sys_b^{-1}, written to `inv`
 * (p x s x s, row-major).  `info[b]` = 0, or k+1 if the k-th leading minor of
 * block b is not positive (np.linalg.cholesky failure, elastic_net.py:213-219).
 * `ws` must hold rac_gram_workspace_bytes(...) bytes. */
size_t rac_gram_workspace_bytes(int64_t len, int32_t s, int32_t p);
int rac_gram_inverse(const double* V, int64_t ldv, int64_t len, const int32_t* idx,
                     int32_t s, int32_t p, int64_t n_valid, double scale, double shift,
                     double* ws, double* inv, int32_t* info, void* stream);

/* Elementwise z-prox (elastic_net.py:102-131, z_update): z = S(xi - g*beta, thr)/den. */
int rac_z_prox(const double* beta, const double* xi, int64_t n, double gamma, double thr,
               double den, double* z, void* stream);

/* ------------------------------------------------------------------ fit()
 * Elastic-net / LASSO / ridge sweep engine behind elastic_net.fit
 * (elastic_net.py:150-232).  One context per solve. */
typedef struct rac_en_ctx rac_en_ctx;

int rac_en_create(rac_en_ctx** out, int64_t m, int64_t n, int32_t block_size, int32_t mode,
                  double lam, double alpha, double gamma, void* stream);
/* X: m x n design (layout RAC_LAYOUT_*), y: m.  Copies X into the context's
 * column-major HBM layout and computes c = -X'y/m (elastic_net.py:177). */
int rac_en_set_data(rac_en_ctx* ctx, const double* X, int32_t layout, const double* y);
/* RP mode only: the fixed partition from one permutation of n
 * (elastic_net.py:187-189); block systems are factored once. */
/* Streaming ingest of a row-major design matrix in row chunks (device
 * pointers), in increasing row order covering [0, m): row0 a multiple of 32,
 * rows a multiple of 32 except for the last chunk, which also passes y and
 * finalises c (and, in covariance mode, G = X'X/m accumulated chunk by chunk,
 * so forming G overlaps the host->device transfer of the following chunks).
 * Equivalent to rac_en_set_data up to the summation order of G. */
int rac_en_set_data_rows(rac_en_ctx* ctx, const double* X_rows, int64_t row0, int64_t rows, const double* y);
/* Select RAC_GRAM_BLOCKS (default) or RAC_GRAM_COVARIANCE.  Covariance mode
 * forms G = X'X/m on the next rac_en_run / rac_en_set_partition (n x n doubles
 * of HBM) and runs the chain on G in one thread-block cluster; selecting it
 * again re-forms G.  RAC_ERR_UNSUPPORTED if the single-cluster chain does not
 * fit (large n or s).  In rp mode the partition must be set again afterwards. */
/* Sparse design (scipy CSC, canonical: rows sorted within a column, no duplicates):
 * indptr int64[n+1], rows int32[nnz], vals double[nnz] (device).  Expanded into the
 * context's column-major X on the device; replaces elastic_net.py:144-147 _col_block on
 * sparse X (the reference densifies each block's columns per sweep). */
int rac_en_set_data_csc(rac_en_ctx* ctx, const int64_t* indptr, const int32_t* rows, const double* vals,
                        const double* y);
int rac_en_set_gram_mode(rac_en_ctx* ctx, int32_t mode);
int rac_en_set_partition(rac_en_ctx* ctx, const int64_t* perm);
/* Enqueue `count` sweeps.  RAC: `perms` = count permutations of n.  RP: count
 * permutations of p (block visit orders, elastic_net.py:197-198).  tol < 0
 * means fixed sweeps (spec.tol None).  Sweeps after convergence are no-ops. */
int rac_en_run(rac_en_ctx* ctx, const int64_t* perms, int32_t count, double tol);
/* Non-blocking status (no reference counterpart): the control word as it stood after
 * the latest run (lag 0) or the one before it (lag 1), waiting only for that run's work —
 * lets a driver enqueue the next batch of sweeps before reading the previous batch's
 * status (launches after convergence or a non-PD block are no-ops on the device).
 * Fields as in rac_en_progress. */
int rac_en_poll(rac_en_ctx* ctx, int32_t lag, int32_t* iterations_host, int32_t* converged_host,
                int32_t* failed_block_host);
/* Synchronizes the stream.  iterations = sweeps executed so far. */
int rac_en_progress(rac_en_ctx* ctx, int32_t* iterations_host, int32_t* converged_host,
                    double* residual_host, int32_t* failed_block_host);
/* Device-to-device copies of the iterate (any pointer may be NULL). */
int rac_en_get(rac_en_ctx* ctx, double* beta, double* z, double* xi, double* r);
/* per-sweep ||beta - z||_1 history (count = iterations) and gamma*||dz||_inf */
int rac_en_history(rac_en_ctx* ctx, double* primal, double* dual, int32_t capacity);
/* Optional per-stage CUDA-event timing of subsequent sweeps; rac_en_timing
 * synchronizes and returns the summed milliseconds of [assembly, gram,
 * factor, chain] over the timed sweeps, then resets. */
int rac_en_set_timing(rac_en_ctx* ctx, int32_t enable);
int rac_en_timing(rac_en_ctx* ctx, double* stage_ms_host4, int32_t* sweeps_host);
/* The digit-slicing share (ms, summed over the sweeps of the last rac_en_timing call) of
 * the gram stage when the block Grams ran on the int8 tensor cores; 0 otherwise. */
int rac_en_timing_slicing(rac_en_ctx* ctx, double* slice_ms_host);
/* enable >= 2 in rac_en_set_timing also records %globaltimer at every chain
 * phase boundary of each sweep (CTA 0), up to 8 + 16p stamps (the last
 * sweep's are kept).  Streaming chain: [start, R0, then per block bar, S1,
 * bar, S2, bar, R].  Resident chain: [start, 3 row-pass stamps, R0, then per
 * block cluster sync, cluster reduce, grid barrier, commit, rhs loads, solve
 * data wait, rhs, delta + cluster sync, tile wait, row pass 1, row sync, row
 * pass 2, row pass 3, next-block issue]. */
int rac_en_trace(rac_en_ctx* ctx, int64_t* host, int32_t capacity);
/* Debugging aid (no reference counterpart): progress markers of the lookahead
 * covariance chain are written to `mapped_host`, a device-accessible pinned host
 * buffer of >= 16 int64 (NULL switches it off); readable while a kernel runs. */
int rac_debug_buffer(void* mapped_host);
/* Utility (no reference counterpart): G (n x n, row-major, device) = Xc'Xc over the
 * samples [0, len) of the column-major device matrix Xc (leading dimension ld;
 * with method 0 len is rounded up to 32 and rows up to that must be readable),
 * divided by div when div > 0, else ADDED to G.  method 0: FP64 DMMA tiles;
 * method 1: exact int8 digit slices on the tcgen05 tensor cores (the covariance
 * mode's default).  Synchronous. */
int rac_gram_covariance(const double* Xc, int64_t ld, int64_t len, int32_t n, double* G, double div,
                        int32_t method);
/* [chain variant (0 streaming, 1 resident-tile cluster), CTAs, rows per chunk, chunks per CTA] */
int rac_en_info(rac_en_ctx* ctx, int32_t* info_host4);
/* Digit slices of the context's int8 tensor-core Grams (block Grams, else the last
 * covariance G): 7 or 8 (chosen on the device per data set from the columns' max/rms),
 * 0 when the Grams run on the FP64 DMMA tiles.  Synchronises the context's stream. */
int rac_en_gram_slices(rac_en_ctx* ctx, int32_t* slices_host);
/* Re-arm a context for a new fit with the same shape (m, n, block size, mode):
 * iterates, history and failure state cleared, data / partition / G must be set
 * again; buffers, plans and streams are kept (fit()'s context pool).  The tags
 * of the lookahead chain's messages keep increasing across resets. */
int rac_en_reset(rac_en_ctx* ctx, double lam, double alpha, double gamma);
int rac_en_destroy(rac_en_ctx* ctx);

/* ------------------------------------------------------------------ train()/solve()
 * Dense box-QP sweep engine behind engine.solve (engine.py:322-405) and
 * svm.train (svm.py:181-284): min 1/2 x'Hx + c'x  s.t. Ax = b, lo <= x <= hi. */
typedef struct rac_qp_ctx rac_qp_ctx;

/* ridge_rel > 0 adds ridge_rel * max(diag(M_b)) to every block matrix
 * (svm.py:242-246 uses 1e-9).  running_residual != 0 reports the primal
 * residual from the running Ax (svm.py:256,260) instead of recomputing. */
int rac_qp_create(rac_qp_ctx** out, int64_t n, int64_t m, int32_t block_size, int32_t mode,
                  double beta, double ridge_rel, void* stream);
/* H: n x n row-major symmetric (may be NULL), A: m x n row-major (NULL iff m == 0),
 * b: m, c: n, lower/upper: n (+-inf allowed).  Copies into context storage. */
int rac_qp_set_problem(rac_qp_ctx* ctx, const double* H, const double* A, const double* b,
                       const double* c, const double* lower, const double* upper);
/* Use an externally owned H (e.g. the SVM Q built by rac_svm_build_q) without copying. */
int rac_qp_borrow_h(rac_qp_ctx* ctx, const double* H);
/* Replaces engine.py:284-315's inputs (x, y) of run_sweep: the next sweep starts from the
 * device vectors x (n) and y (m) instead of (clip(0, lower, upper), 0). */
int rac_qp_set_state(rac_qp_ctx* ctx, const double* x, const double* y);
/* Kernel strips on the fly instead of a resident n x n H (SVM dual, svm.py:96-143 — the
 * reference assembles each block's s x n strip from data rows): H_ij = labels_i labels_j
 * K(X_i, X_j) with X n x d row-major (device), kind RAC_KERNEL_*; per sweep the blocks' H_bb,
 * then the strip rows of up to max_strip_bytes worth of blocks at a time.  Before
 * rac_qp_set_problem (with H = null; every box must contain 0); RAC / CYCLIC modes. */
int rac_qp_set_kernel_strips(rac_qp_ctx* ctx, const double* X, int64_t d, const double* labels, int32_t kind,
                             double sigma, uint64_t max_strip_bytes);
/* Divergence bar (engine.py:361-362): set_problem uses 1e8*max(primal0, 1);
 * svm.train has no guard and passes +inf. */
int rac_qp_set_divergence_bar(rac_qp_ctx* ctx, double bar);
int rac_qp_set_partition(rac_qp_ctx* ctx, const int64_t* perm);   /* RP / CYCLIC */
int rac_qp_run(rac_qp_ctx* ctx, const int64_t* perms, int32_t count, double tol_primal,
               double tol_dual, int32_t fixed_iterations);
int rac_qp_progress(rac_qp_ctx* ctx, int32_t* iterations_host, int32_t* status_host,
                    int32_t* failed_block_host);
int rac_qp_get(rac_qp_ctx* ctx, double* x, double* y, double* hx, double* ax);
int rac_qp_history(rac_qp_ctx* ctx, double* primal, double* primal_l1, double* dual,
                   int32_t capacity);
/* Optional chain trace of the most recent sweep (CTA 0), 14p int64: per block
 * %globaltimer at [S start, gather done, M/N resident, unconstrained x done,
 * box solve done, S end, G start, G end, next H_bb x_b done, strip done], then
 * per block the box-solver counters [reduced solves, active-set passes, ns in
 * reduced solves, ns in box]. */
int rac_qp_set_trace(rac_qp_ctx* ctx, int32_t enable);
int rac_qp_trace(rac_qp_ctx* ctx, int64_t* host, int32_t capacity);
int rac_qp_destroy(rac_qp_ctx* ctx);

/* Label-weighted kernel matrix Q_ij = y_i y_j K(x_i, x_j) (svm.py:82-93,139),
 * X: N x d row-major.  Built once with FP64 tensor-core tiles. */
int rac_svm_build_q(const double* X, int64_t N, int64_t d, const double* labels, int32_t kind,
                    double sigma, double* Q, void* stream);
/* out_i = sum_j Q_ij * w_j (one HBM pass; used for the SVM bias, svm.py:287-305). */
/* Label-weighted kernel strip rows of s samples against all N:
 *   strip[i * N + j] = labels[rows[i]] * labels[j] * K(X[rows[i]], X[j])
 * X row-major N x d (device), rows int32 (-1 = zero padding row).  FP64 tensor cores with
 * the kernel epilogue fused.  Replaces svm.py:121-143 assemble_kernel_block(with_strip=True)
 * / KernelRowCache.row (svm.py:107-118); Q_bb = strip[:, rows]. */
int rac_svm_kernel_strip(const double* X, int64_t N, int64_t d, const double* labels, const int32_t* rows,
                         int32_t s, int32_t kind, double sigma, double* strip, void* stream);
/* ------------------------------------------------------------------ consensus baseline
 * Per-sweep part of elastic_net.py:252-316 consensus_fit (the paper's Table-1 two-block
 * baseline): `count` sweeps of copy solves, z-shrink, dual step and residual, all on the
 * device; sweeps after state[1] (stop flag: residual <= tol, tol < 0 = never) are no-ops.
 * S_i^{-1} (direct, p x p) / W_i^{-1} (Woodbury, n_i x n_i) are formed by the caller. */
typedef struct rac_consensus_args {
  int32_t N;               /* copies (sample groups) */
  int64_t p;               /* features */
  const int32_t* kind;     /* [N] 0 direct, 1 Woodbury */
  const int32_t* ni;       /* [N] samples per group */
  const int64_t* off_inv;  /* [N] offsets into inv */
  const int64_t* off_x;    /* [N] offsets of X_i (n_i x p row-major) into xg (Woodbury) */
  const int64_t* off_u;    /* [N] offsets of group i's n_i-vectors into u / inner (increasing) */
  const double* inv;
  const double* xg;
  const double* w0;        /* [N][p] X_i' y_i / n */
  double* copies;          /* [N][p] */
  double* duals;           /* [N][p] */
  double* z;               /* [p] */
  double* u;               /* [wb_rows] */
  double* inner;           /* [wb_rows] */
  double* part;            /* [part_cap] */
  double* hist;            /* residual per sweep */
  int32_t* state;          /* [0] sweeps done, [1] stop flag */
  int64_t wb_rows;         /* sum of n_i over Woodbury groups' u slots (0: none) */
  int32_t direct_groups;
  int32_t part_cap;
  double gamma, thr, denom, tol;
} rac_consensus_args;
int rac_consensus_run(const rac_consensus_args* args, int32_t count, void* stream);

int rac_gemv(const double* Q, int64_t rows, int64_t cols, const double* w, double* out,
             void* stream);

/* Exact box-QP minimizer for ONE block on the device (engine.py:189-245),
 * exposed for testing: M s x s row-major SPD, r, lo, hi -> x.  info as above. */
int rac_box_block_min(const double* M, const double* r, const double* lo, const double* hi,
                      int32_t s, double* x, int32_t* info, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RAC_B200_H */
