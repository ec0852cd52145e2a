/*
 * spmvtune_b200.h — C ABI of libspmvtune_b200.so, the B200 (sm_100a) engine
 * behind the spmvtune drop-in API.
 *
 * The reference (`/root/reference/pkg/src/spmvtune`, pure Python/numpy) has
 * no FFI of its own; every entry point below replaces one reference function
 * or container operation, cited as file:line relative to that directory.
 * The Python host package (paper_2411_10143_b200/) binds these with ctypes
 * (see INTEGRATION.md for the binding a reference maintainer would add).
 *
 * Conventions
 *   - Every function returns an int status (svb_status); nothing throws
 *     across the ABI.  svb_last_error() returns the calling thread's message
 *     for the most recent non-zero status.
 *   - Status -> reference exception (errors.py:4-29):
 *       SVB_UNSUPPORTED_CONFIG -> UnsupportedConfigError
 *       SVB_INAPPLICABLE       -> FormatInapplicableError
 *       SVB_DIM_MISMATCH       -> ValueError
 *       SVB_NONFINITE          -> SolverNumericalError
 *       SVB_OOM                -> MemoryError
 *       SVB_CUDA / SVB_INVALID -> RuntimeError / ValueError
 *   - Matrices (svb_matrix*) are immutable after creation and may be read
 *     concurrently from several streams (kernels.py:14-17).  The caller owns
 *     the handle and releases it with svb_matrix_destroy.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *   - Pointers named *_dev are device pointers; *_host are host pointers.
 *   - Index arrays cross the ABI as int64 (the reference's dtype,
 *     formats.py:34-38); on the device, column indices are int32 and
 *     row pointers int32 unless nnz >= 2^31 (then int64).
 */
#ifndef SPMVTUNE_B200_H
#define SPMVTUNE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVB_ABI_VERSION 1

typedef enum {
  SVB_OK = 0,
  SVB_UNSUPPORTED_CONFIG = 1,
  SVB_INAPPLICABLE = 2,
  SVB_DIM_MISMATCH = 3,
  SVB_NONFINITE = 4,
  SVB_OOM = 5,
  SVB_CUDA = 6,
  SVB_INVALID = 7,
  SVB_FORMAT_ERROR = 8   /* -> MatrixMarketError */
} svb_status;

/* FormatTag (formats.py:21-26) */
typedef enum { SVB_COO = 0, SVB_CSR = 1, SVB_ELL = 2, SVB_DIA = 3, SVB_HYB = 4 } svb_format;
/* Library (kernels.py:37-40) */
typedef enum { SVB_LIBA = 0, SVB_LIBB = 1, SVB_LIBC = 2 } svb_library;
/* value precision of an SpMV call */
typedef enum { SVB_F64 = 0, SVB_F32 = 1 } svb_dtype;

typedef struct svb_matrix svb_matrix;

typedef struct {
  int32_t format;        /* svb_format */
  int32_t ptr64;         /* CSR/COO-derived row pointer is int64 on device */
  int64_t nrows, ncols;
  int64_t nnz;           /* stored entries (ELL: non-sentinel cells) */
  int64_t width;         /* ELL / HYB ELL-part width */
  int64_t ndiag;         /* DIA */
  int64_t spill_nnz;     /* HYB COO part */
  int64_t device_bytes;  /* bytes held on the device by this handle */
} svb_matrix_info;

/* which host array svb_matrix_download copies out (int64 / float64) */
typedef enum {
  SVB_ARR_ROW_PTR = 0,   /* CSR row_ptr, int64[nrows+1] */
  SVB_ARR_ROWS = 1,      /* COO rows / HYB spill rows, int64[nnz] */
  SVB_ARR_COLS = 2,      /* CSR/COO cols, int64[nnz]; ELL cols int64[width*nrows] col-major */
  SVB_ARR_VALS = 3,      /* values, float64 (same layouts) */
  SVB_ARR_OFFSETS = 4,   /* DIA offsets, int64[ndiag] */
  SVB_ARR_DATA = 5,      /* DIA data, float64[ndiag*nrows] row-major */
  SVB_ARR_SPILL_COLS = 6,/* HYB spill cols, int64[spill_nnz] */
  SVB_ARR_SPILL_VALS = 7 /* HYB spill values, float64[spill_nnz] */
} svb_array;

/* ---- library ------------------------------------------------------------ */
const char* svb_last_error(void);
int svb_abi_version(void);
/* Number of this library's kernels launched so far by the process. */
int svb_launch_count(int64_t* out);
/* Select the device for the calling thread and warm the allocator. */
int svb_init(int device);
/* Block until `stream` drains (used by host wrappers at API boundaries). */
int svb_stream_sync(void* stream);
/* Stream / event / memory plumbing for the host layer (no reference
 * counterpart: the reference is single-address-space numpy). */
int svb_stream_create(int priority, void** out);   /* non-blocking stream */
int svb_stream_destroy(void* stream);
int svb_event_record(void* stream, void** out);    /* new event, recorded on stream */
int svb_event_query(void* event);                  /* SVB_OK when complete, else SVB_INVALID */
int svb_event_sync(void* event);                   /* block until the event completes */
int svb_stream_wait_event(void* stream, void* event);
int svb_event_destroy(void* event);
/* CUDA graph capture of work enqueued on `stream` by this thread (B200
 * runtime: CG batches replay as one launch); replays count their kernels
 * into svb_launch_count. */
int svb_graph_begin(void* stream);
int svb_graph_end(void* stream, void** graph_out);
int svb_graph_launch(void* graph, void* stream);
int svb_graph_destroy(void* graph);
int svb_malloc(int64_t bytes, void** out);         /* device memory (pool) */
int svb_free(void* ptr);
int svb_host_alloc(int64_t bytes, void** out);     /* pinned host memory */
int svb_host_free(void* ptr);
int svb_copy(void* dst, const void* src, int64_t bytes, void* stream);  /* any direction, async */
/* Host numpy buffer <-> device: device -> pageable host copies of >= 12 MB
 * go through a pinned staging buffer drained by several host threads;
 * everything else copies directly.  Blocking like cudaMemcpy from pageable
 * memory: returns when `src` may be reused (to_device) or `dst` holds the
 * data. */
int svb_copy_host(void* dst, const void* src, int64_t bytes, int32_t to_device, void* stream);
int svb_memset(void* dst, int value, int64_t bytes, void* stream);
int svb_device_info(int32_t* sm_count, int64_t* free_bytes, int64_t* total_bytes);
/* stream-ordered pool: bytes reserved from the driver / currently in use */
int svb_pool_info(int64_t* reserved_bytes, int64_t* used_bytes);

/* ---- containers (formats.py:50-260) ------------------------------------ */
/* CooMatrix(nrows, ncols, rows, cols, values): row-major sorted, no dups. */
int svb_coo_create(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows_host,
                   const int64_t* cols_host, const double* vals_host, void* stream,
                   svb_matrix** out);
/* CsrMatrix(nrows, ncols, row_ptr, col_idx, values) */
int svb_csr_create(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* row_ptr_host,
                   const int64_t* col_idx_host, const double* vals_host, void* stream,
                   svb_matrix** out);
/* Rows [r0, r1) of a CSR matrix as a new CSR (same ncols, rebased row
 * pointer): the interior / boundary row blocks of a row-partitioned rank,
 * whose interior SpMV overlaps the halo exchange. */
int svb_csr_row_slice(const svb_matrix* src, int64_t r0, int64_t r1, void* stream,
                      svb_matrix** out);
/* A row-partitioned rank's own host slab (distributed_solve_slab, the
 * per-rank form of distributed_solve's CsrMatrix input, formats.py:103-146):
 * rows [r0, r0 + nrows) of a matrix with ncols_global columns; row_ptr is
 * slab-local (row_ptr[0] = 0, row_ptr[nrows] = nnz); col_idx holds GLOBAL
 * column indices, int64 (the reference's dtype) when cols_i64 != 0, else
 * int32.  Uploaded and validated on the device with the CsrMatrix rules
 * and messages (endpoints, non-decreasing row_ptr, column range, strictly
 * increasing columns -> SVB_DIM_MISMATCH); stored with columns relative to
 * the rank's window [cmin, cmax] (hull of the columns and the own rows),
 * returned in window[2]. */
int svb_csr_create_slab(int64_t nrows, int64_t ncols_global, int64_t nnz, int64_t r0,
                        const int64_t* row_ptr_host, const void* col_idx_host, int32_t cols_i64,
                        const double* vals_host, void* stream, int64_t* window, svb_matrix** out);
/* CSR handle -> caller-owned host slab: row_ptr int64[nrows+1], columns
 * int32[nnz] plus col_shift (window-relative -> global), values f64[nnz]. */
int svb_csr_export(const svb_matrix* m, int64_t col_shift, int64_t* row_ptr_host, int32_t* cols_host,
                   double* vals_host, void* stream);
/* EllMatrix(nrows, ncols, width, col_idx, values): column-major (nrows x width)
 * arrays, i.e. cell (i, k) at k*nrows + i; sentinel column = ncols. */
int svb_ell_create(int64_t nrows, int64_t ncols, int64_t width, const int64_t* cols_host,
                   const double* vals_host, void* stream, svb_matrix** out);
/* DiaMatrix(nrows, ncols, offsets, data): data[k*nrows + i] = A[i, i+offsets[k]] */
int svb_dia_create(int64_t nrows, int64_t ncols, int64_t ndiag, const int64_t* offsets_host,
                   const double* data_host, void* stream, svb_matrix** out);
/* HybMatrix(ell_part, coo_part, split_width): composes copies of two handles */
int svb_hyb_create(const svb_matrix* ell, const svb_matrix* coo, void* stream,
                   svb_matrix** out);
int svb_matrix_destroy(svb_matrix* m);
int svb_matrix_info_get(const svb_matrix* m, svb_matrix_info* info);
/* Copy one array back to caller-owned host memory (int64 or float64). */
int svb_matrix_download(const svb_matrix* m, int which, void* dst_host, void* stream);

/* On-device constant-coefficient stencil generator (configs 1, 2, 5 of
 * BASELINE.json; no reference counterpart — the reference builds its test
 * matrices on the host, tests/helpers.py:42-84).  dims[ndim] with the fastest
 * axis last; offsets[nst*ndim]; weights[nst]. */
int svb_csr_stencil(int ndim, const int64_t* dims, int nst, const int32_t* offsets,
                    const double* weights, void* stream, svb_matrix** out);
/* Rows [r0, r1) of the same stencil matrix as a row-partitioned rank's local
 * block: ncols = cmax - cmin + 1 and column c is stored as
 * c - cmin (the rank's column window, which must cover rows [r0, r1)).
 * Generated on the device, so a 600^3 slab never exists on the host. */
int svb_csr_stencil_rows(int ndim, const int64_t* dims, int nst, const int32_t* offsets,
                         const double* weights, int64_t r0, int64_t r1, int64_t cmin, int64_t cmax,
                         void* stream, svb_matrix** out);

/* ---- Matrix Market ingest (mmio.py:32-126) + from_triplets on the device
 * (formats.py:86-100).  svb_mm_open reads the file and validates banner and
 * size line (dims = {nrows, ncols, nnz}, flags = {pattern, symmetric});
 * svb_mm_parse fills caller-owned 0-based rows/cols/vals[nnz] with nthreads
 * host threads (0 = all cores), reporting the lowest failing entry with the
 * reference's message; status SVB_FORMAT_ERROR maps to MatrixMarketError.
 * svb_coo_from_triplets sorts (stable radix sort on the device) and, with
 * sum_duplicates, merges repeated coordinates in np.add.reduceat order. */
typedef struct svb_mm svb_mm;
int svb_mm_open(const char* path, int64_t* dims, int32_t* flags, svb_mm** out);
int svb_mm_parse(svb_mm* h, int64_t* rows_host, int64_t* cols_host, double* vals_host, int32_t nthreads);
int svb_mm_close(svb_mm* h);
int svb_coo_from_triplets(int64_t nrows, int64_t ncols, int64_t n, const int64_t* rows_host,
                          const int64_t* cols_host, const double* vals_host, int32_t sum_duplicates,
                          void* stream, svb_matrix** out);

/* ---- conversion: convert(m, target) (formats.py:302-320) ----------------
 * Bit-exact with the reference arrays.  DIA above 4096 diagonals returns
 * SVB_INAPPLICABLE (formats.py:351-356).  `max_ell_cells` (0 = unlimited)
 * caps nrows*width for ELL (a B200-side memory guard the reference lacks). */
int svb_convert(const svb_matrix* src, int target, int64_t max_ell_cells, void* stream,
                svb_matrix** out);
/* hyb_split_width over the row lengths of m (formats.py:364-370) */
int svb_hyb_split_width(const svb_matrix* m, void* stream, int64_t* width_out);

/* ---- SpMV: execute_spmv(cfg, m, x, workers=, out=) (kernels.py:274-312) --
 * y = A x with the (format, library, lane) kernel of the configuration; the
 * matrix must be stored in `format` (else SVB_UNSUPPORTED_CONFIG, kernels.py:
 * 125-128).  `workers` is the LibC chunk count (kernels.py:202-248).  All
 * kernels except COO/LibB reproduce the reference's fp64 summation order
 * bit-for-bit.  x_dev/y_dev: device vectors of `dtype`. */
int svb_spmv(const svb_matrix* m, int format, int library, int lane, int workers,
             int dtype, const void* x_dev, void* y_dev, void* stream);
/* Same product with host buffers: H2D of x, kernel, D2H of y (the e2e path
 * of bench.py); staging lives in pinned/device pools owned by the library. */
int svb_spmv_host(const svb_matrix* m, int format, int library, int lane, int workers,
                  const double* x_host, double* y_host, void* stream);
/* spmv_reference(m, x) (formats.py:419-435): sequential row order (CSR). */
int svb_spmv_sequential(const svb_matrix* csr, const double* x_dev, double* y_dev,
                        void* stream);

/* ---- features: extract_features(csr) (features.py:68-156) ----------------
 * agg[7] = {sum r, sum r^2, max r, min r, sum(last-first), sum longest-run,
 * ndiag}; the host evaluates the 15 float features with the reference's own
 * expressions (features.py:103-110, 147-150), making them bit-exact. */
int svb_features(const svb_matrix* csr, int64_t* agg_host, void* stream);
/* The same pass as a job, for extract_features(csr, cancel, counter=...)
 * (features.py:68-156): start enqueues it on `stream` and returns at once;
 * cancel raises a device flag the kernel polls once per 256-row tile
 * (it then stops reading row_ptr/col_idx; the reference checks every
 * row_chunk rows, features.py:89-91) and may be called from any thread
 * while another blocks in wait; query reports completion without
 * blocking; wait blocks until the pass ends (no result, the job stays
 * live); finish waits, writes agg[7], counters[2] = {row_ptr elements,
 * col_idx elements} actually read (TraversalCounter, features.py:60-65) and
 * *cancelled, and releases the job.  precancelled != 0 reads nothing.  An
 * uncancelled pass leaves its diagonal bitmap and sorted offsets on the
 * handle for a later DIA conversion. */
typedef struct svb_features_job svb_features_job;
int svb_features_start(const svb_matrix* csr, int precancelled, void* stream, svb_features_job** job);
int svb_features_cancel(svb_features_job* job);
int svb_features_query(svb_features_job* job, int* done);
int svb_features_wait(svb_features_job* job);
int svb_features_finish(svb_features_job* job, int64_t* agg_host, int64_t* counters_host, int* cancelled);
/* The distinct diagonal offsets (col - row) of a CSR handle plus `shift`,
 * ascending (the ndiag feature's set, features.py:118-126; a row-partitioned
 * rank passes shift = cmin - r0 for global offsets so the ranks' sets can be
 * united exactly).  *count = number of offsets; min(count, cap) are copied. */
int svb_diag_offsets(const svb_matrix* csr, int64_t shift, int64_t* out_host, int64_t cap, int64_t* count,
                     void* stream);

/* ---- Krylov workspaces (solver.py:219-342; CG is new) ---- */
typedef struct svb_krylov svb_krylov;
typedef struct {
  double beta;       /* ||r|| of the last restart/residual call */
  double hnext;      /* ||w|| after MGS (GMRES) */
  double estimate;   /* |g[j+1]|/||b|| (GMRES) or ||r||/||b|| (CG) */
  double hjj;        /* rotated H[j,j] (GMRES breakdown check) */
  double pq;         /* p.Ap (CG) */
  int32_t nonfinite; /* a non-finite scalar was produced */
  int32_t done;      /* batched CG: 0 running, 1 tol met, 2 p.Ap == 0, 3 non-finite */
  int64_t count;     /* batched CG: iterations executed since svb_cg_batch_reset */
} svb_krylov_status;

/* n rows, restart m (GMRES, 1 <= m <= 24000; m = 0 for CG).  Owns
 * V[(m+1) x n], H, Givens state, CG vectors and the mapped status block.
 * SVB_INVALID above 24000 (y of the x update is staged in shared memory);
 * SVB_OOM when V does not fit the device. */
int svb_krylov_create(int64_t n, int32_t m, svb_krylov** out);
int svb_krylov_destroy(svb_krylov* k);
/* device pointers of workspace vectors: 0..m = V rows; -1 = x; -2 = b;
 * -3 = tmp (matvec target); -4 = CG p; -5 = CG q; -6 = CG r */
int svb_krylov_vec(svb_krylov* k, int which, double** out);
int svb_krylov_status_get(svb_krylov* k, void* stream, svb_krylov_status* out);
/* re-record the status event on `stream` (after a graph replay: an event
 * recorded during stream capture is not a usable event afterwards) */
int svb_krylov_mark(svb_krylov* k, void* stream);
/* ||b|| into status.beta */
int svb_krylov_bnorm(svb_krylov* k, void* stream);
/* GMRES cycle start: r = b - tmp; beta = ||r||; V0 = r/beta; g = beta e1 */
int svb_gmres_restart(svb_krylov* k, void* stream);
/* GMRES Arnoldi step j after the matvec wrote V[j+1] = A V[j]: fused
 * modified Gram-Schmidt (axpy_i + dot_{i+1} per pass), ||w||, Givens
 * rotations and the residual estimate, all on device. */
int svb_gmres_arnoldi(svb_krylov* k, int32_t j, double bnorm, void* stream);
/* V[j+1] /= hnext */
int svb_gmres_normalize(svb_krylov* k, int32_t j, void* stream);
/* x += V[:j+1]^T y with y from the rotated triangular system (solver.py:211-216) */
int svb_gmres_update_x(svb_krylov* k, int32_t j, void* stream);
/* status.beta = ||b - tmp|| (explicit residual confirmation) */
int svb_krylov_residual(svb_krylov* k, void* stream);
/* CG: r = b - tmp, p = r, rr = r.r  (tmp = A x) */
int svb_cg_restart(svb_krylov* k, void* stream);
/* CG after q = A p: alpha = rr/(p.q); x += alpha p; r -= alpha q; rr' = r.r;
 * estimate = sqrt(rr')/bnorm; p = r + (rr'/rr) p */
int svb_cg_step(svb_krylov* k, double bnorm, void* stream);

/* Batched CG: the host enqueues many iterations (SpMV + svb_cg_step_batched)
 * without reading status in between; once an iteration meets `tol` (or hits
 * p.Ap == 0 / a non-finite value) the remaining kernels of the batch are
 * no-ops, so x and r stay at that iteration.  Estimates are logged on device. */
int svb_cg_batch_reset(svb_krylov* k, double tol, int64_t history_cap, void* stream);
int svb_cg_batch_resume(svb_krylov* k, void* stream);   /* clear `done`, keep count */
int svb_cg_step_batched(svb_krylov* k, double bnorm, void* stream);
/* One batched CG iteration for a DIA operator with q = A p fused with p.q
 * (same q as svb_spmv DIA/LibA; saves the separate p.q pass). */
int svb_cg_step_batched_dia(svb_krylov* k, const svb_matrix* dia, double bnorm, void* stream);
int svb_cg_history(svb_krylov* k, int64_t first, int64_t count, double* host, void* stream);

/* ---- generic fused vector ops (device vectors of length n) -------------- */
int svb_dot(const double* x_dev, const double* y_dev, int64_t n, double* out_host,
            void* stream);

/* Building blocks of the row-partitioned (multi-GPU) solvers: every
 * reduction writes its LOCAL result to a device scalar, which the caller
 * all-reduces in place (NCCL) before the next primitive reads it — scalars
 * never visit the host inside a step.  Deterministic fixed-order sums. */
typedef struct svb_vecops svb_vecops;
int svb_vecops_create(int64_t n, svb_vecops** out);
int svb_vecops_destroy(svb_vecops* v);
/* *out_dev = x . y */
int svb_vec_dot(svb_vecops* v, const double* x_dev, const double* y_dev, double* out_dev,
                void* stream);
/* y += sign * (*alpha_dev) * x;  *out_dev = (z ? z : y) . y   (out_dev may be NULL) */
int svb_vec_axpy_dot(svb_vecops* v, const double* alpha_dev, double sign, const double* x_dev,
                     double* y_dev, const double* z_dev, double* out_dev, void* stream);
/* y = a x + b y */
int svb_vec_axpby(svb_vecops* v, double a, const double* x_dev, double b, double* y_dev,
                  void* stream);
/* x *= s */
int svb_vec_scale(svb_vecops* v, double* x_dev, double s, void* stream);
/* Row-partitioned CG on device scalars sc[] (NCCL all-reduces them in place
 * between calls), the two vector passes that follow the SpMV + p.Ap pass:
 *   svb_dcg_rupdate: a = sc[icur]/sc[ipq] -> sc[ialpha], r -= a q, local
 *                    r.r -> sc[out] (a zero/non-finite sc[ipq]: a = 0, r
 *                    untouched, sc[out] = sc[icur]);
 *   svb_dcg_xp:      x += sc[ialpha] p, then p = r + (sc[inew]/sc[iold]) p.
 * Oracle: oracle/cpu_oracle.py:cg (x += a p; r -= a q; p = r + b p). */
int svb_dcg_rupdate(svb_vecops* v, double* sc_dev, int32_t icur, int32_t ipq, int32_t out, int32_t ialpha,
                    const double* q_dev, double* r_dev, void* stream);
int svb_dcg_xp(svb_vecops* v, const double* sc_dev, int32_t ialpha, int32_t inew, int32_t iold,
               const double* r_dev, double* p_dev, double* x_dev, void* stream);
/* y = A x in the configuration, fused with *out_dev = dsrc . y (CG's p.Ap,
 * oracle/cpu_oracle.py:cg) — one pass for DIA (the dot folded into the
 * TMA-staged SpMV), SpMV + dot otherwise; `accumulate` adds into *out_dev
 * (the interior / boundary row parts of one local SpMV, in a fixed order). */
int svb_vec_spmv_dot(svb_vecops* v, const svb_matrix* m, int format, int library, int lane, int workers,
                     const double* x_dev, double* y_dev, const double* dsrc_dev, double* out_dev,
                     int32_t accumulate, void* stream);
/* Row-partitioned GMRES, classical Gram-Schmidt twice (CGS2; the reference's
 * MGS loop solver.py:294-297 needs j+2 sequential all-reduces per Arnoldi
 * step across ranks, CGS2 two).  V = basis rows (row i at V_dev + i*ld),
 * the first k used; h_dev, div_dev, out_dev are device scalars.  Modes:
 *   0 DOT:    out[i] = V_i . w                                (i < k)
 *   1 UPDATE: dst = w - sum h_i V_i; out[i] = V_i . dst; out[k] = dst . dst
 *   2 FINISH: dst = (w - sum h_i V_i) / *div
 *   3 AXPY:   dst = w + sum h_i V_i   (x += V y)
 * dst may alias w.  Fixed-order sums (deterministic). */
int svb_vec_gs(svb_vecops* v, int32_t mode, const double* V_dev, int64_t ld, int32_t k, const double* h_dev,
               const double* div_dev, const double* w_dev, double* dst_dev, double* out_dev, void* stream);
/* *hn_dev = sqrt(max(*nrm_dev - sum h2_i^2, 0)): the norm after CGS2's
 * second pass from the first pass's w.w and the correction coefficients. */
int svb_vec_gs_hn(const double* h2_dev, int32_t k, const double* nrm_dev, double* hn_dev, void* stream);
/* x[0..n) = v on the device (row-partitioned setup: windows of ones) */
int svb_fill(double* x_dev, int64_t n, double v, void* stream);

/* ---- compiled cascade inference (inference.py:55-125, model_schema.md) ---
 * Flattened tree ensemble: node arrays in the reference's flattening order;
 * leaves carry feature = -1.  Evaluation: `<=` goes left, per-class sums in
 * list order as float64, argmax ties to the lowest index. */
typedef struct svb_forest svb_forest;
int svb_forest_create(int32_t nclasses, int32_t ntrees, const int32_t* tree_class,
                      const int32_t* roots, int32_t nnodes, const int32_t* feature,
                      const double* threshold, const int32_t* left, const int32_t* right,
                      const double* score, svb_forest** out);
int svb_forest_destroy(svb_forest* f);
int svb_forest_predict(const svb_forest* f, const double* x15, double* scores_out,
                       int32_t* label_out);

/* ---- native solver drivers + configuration mailbox -------
 * svb_gmres_run / svb_cg_run: the whole solve loop of gmres_solve / cg_solve
 * (solver.py:345-362; reference _gmres_core, solver.py:219-342) in C++ for
 * hosts without Python.  b_dev/x_dev: device vectors (x0 = 0); A is read,
 * never modified.  history_host: capacity max_iters doubles (per-iteration
 * residual estimates); timeline_host: up to timeline_cap swaps, the first
 * being the initial configuration at iteration 1.  A non-finite scalar
 * returns SVB_NONFINITE with the reference's message; a breakdown whose
 * explicit residual stays above tol reports stagnated = 1 (StagnationError).
 * The mailbox (ConfigMailbox, solver.py:126-185) is polled between
 * iterations: svb_mailbox_publish (any thread, last writer wins) offers a
 * matrix handle already stored in cfg.format and an optional CUDA event it
 * is complete at; a different configuration is swapped in for the next
 * iteration.  The handle must outlive the solve.  svb_mailbox_finished
 * reports the solver done (the advisor's cancel flag). */
typedef struct {
  int32_t format, library, lane, workers;   /* SpmvConfig + LibC chunk count */
} svb_config;
typedef struct {
  int32_t restart_m;   /* GMRES(m); ignored by CG */
  int32_t max_iters;
  double tol;
} svb_solve_params;
typedef struct {
  int32_t iteration;   /* first iteration run with `config` */
  svb_config config;
  double prep_seconds;
} svb_swap;
typedef struct {
  int32_t converged;
  int32_t stagnated;
  int32_t iterations;
  int32_t history_len;
  int32_t nswaps;         /* timeline entries (may exceed timeline_cap) */
  double final_residual;  /* NaN when max_iters == 0 (reference: None) */
} svb_solve_report;
typedef struct svb_mailbox svb_mailbox;
int svb_mailbox_create(svb_mailbox** out);
int svb_mailbox_destroy(svb_mailbox* mb);
int svb_mailbox_publish(svb_mailbox* mb, const svb_matrix* m, svb_config cfg, void* ready_event,
                        double prep_seconds);
int svb_mailbox_finished(svb_mailbox* mb, int32_t* out);
int svb_gmres_run(const svb_matrix* A, svb_config cfg, const double* b_dev, double* x_dev,
                  const svb_solve_params* params, svb_mailbox* mb, void* stream, double* history_host,
                  svb_swap* timeline_host, int32_t timeline_cap, svb_solve_report* out);
int svb_cg_run(const svb_matrix* A, svb_config cfg, const double* b_dev, double* x_dev,
               const svb_solve_params* params, svb_mailbox* mb, void* stream, double* history_host,
               svb_swap* timeline_host, int32_t timeline_cap, svb_solve_report* out);


/* ---- peer-memory collectives (csrc/peer.cu; distributed.py PeerComm) ----
 * The row-partitioned CG's per-iteration exchanges done by the solver's own
 * kernels over NVLink/NVSwitch peer memory instead of NCCL: an all-reduce
 * of <= 64 device doubles through per-rank mailboxes (every rank stores its
 * values into every mailbox, release-tags them, sums its own mailbox in rank
 * order: bit-identical on all ranks), and the halo pushed by the x/p pass
 * straight into the neighbours' windows with a release tag the neighbour's
 * boundary SpMV waits for (svb_peer_wait_halo).  Mailboxes and windows are
 * cudaMalloc'd (CUDA IPC exportable: svb_peer_ipc_handle/open); every wait
 * has a 30 s deadline that raises svb_peer_error instead of hanging.
 * Replaces the NCCL calls of the reference-shaped loop (oracle/cpu_oracle.py:cg;
 * the reference itself has no distributed solver). */
typedef struct svb_peer svb_peer;
int svb_peer_create(int rank, int world, svb_peer** out);
int svb_peer_destroy(svb_peer* g);
int svb_peer_mailbox(const svb_peer* g, void** dev_ptr);
int svb_peer_set_mailbox(svb_peer* g, int rank, void* dev_ptr);
int svb_peer_alloc(int64_t bytes, void** out);
int svb_peer_free(void* dev_ptr);
int svb_peer_ipc_handle(void* dev_ptr, void* handle64);
int svb_peer_ipc_open(const void* handle64, void** dev_ptr);
int svb_peer_ipc_close(void* dev_ptr);
int svb_peer_error(const svb_peer* g, int* err);
int svb_peer_allreduce(svb_peer* g, double* v_dev, int count, void* stream);
int svb_peer_wait_halo(svb_peer* g, const int32_t* peers, int npeers, void* stream);
int svb_dcg_xp_push(svb_peer* g, int64_t n, const double* sc_dev, int32_t ialpha, int32_t inew, int32_t iold,
                    const double* r_dev, double* p_dev, double* x_dev, int nseg, const int64_t* lo,
                    const int64_t* cnt, double* const* dst_dev, const int32_t* peer, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPMVTUNE_B200_H */
