/*
 * smat.h — C ABI of the B200-native structured-operator engine (libsmat.so).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `linopkit` (a fastmat-style structured-matrix library): the validated
 * matrix-free forward (A·x) and backward (A^H·y) transforms of batched column
 * blocks.  The reference reaches its numpy transform kernels through
 *
 *   LinearOperator.forward / backward   pkg/src/linopkit/core.py:128-167
 *   subclass _forward / _backward hooks pkg/src/linopkit/core.py:114-118
 *   leaves / composites                 pkg/src/linopkit/leaves.py, composites.py
 *   kernels dft / fwht / get_plan       pkg/src/linopkit/kernels.py:127-190
 *
 * Here the whole operator tree is serialised once into an array of
 * `smat_node`, compiled into an immutable device plan (`smat_plan_build`,
 * replacing the per-node recursion of composites.py:49-61 and the plan cache
 * of kernels.py:150-153), and every application is ONE `smat_apply` call that
 * launches the plan's fused passes on a CUDA stream.  No torch types cross
 * this boundary: plain pointers, sizes and a `cudaStream_t` passed as void*.
 *
 * Layout: x and y are (rows, ncols) blocks — by default row-major
 * (SMAT_ROW_MAJOR, the numpy/torch C order the reference uses,
 * core.py:128-149): element (i, col) at i*ld + col with a leading dimension
 * ld >= ncols (ld = ncols: C-contiguous; ld > ncols: a column slice of a wider
 * block, read and written in place).  SMAT_COL_MAJOR blocks (Fortran order,
 * element (i, col) at col*ld + i) are accepted too.  Columns are independent.
 *
 * Ownership: callers own x, y and the workspace; the plan owns every device
 * parameter (spectra, twiddles, chirps, diagonals, dense factors).  A plan is
 * immutable after build; `smat_apply` is reentrant across streams when each
 * stream uses its own workspace (reference threading contract: core.py:5-7).
 *
 * Errors: every entry point returns an `smat_status`; the message of the last
 * failure on the calling thread is available from `smat_last_error()`.  The
 * Python layer maps the codes to the reference exception classes
 * (errors.py:4-65) after doing the reference's own validation first.
 */
#ifndef SMAT_H_
#define SMAT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMAT_ABI_VERSION 3  /* 3: leading dimensions + layout on apply, peak probe */

#if defined(__GNUC__)
#define SMAT_API __attribute__((visibility("default")))
#else
#define SMAT_API
#endif

typedef enum smat_status {
  SMAT_OK = 0,
  SMAT_BAD_SHAPE = 1,    /* DimensionMismatch / ChainMismatch (errors.py:8, 32) */
  SMAT_NOT_POW2 = 2,     /* NotPowerOfTwo (errors.py:16)                        */
  SMAT_BAD_DTYPE = 3,    /* TypeError in coerce_array (core.py:66-68)            */
  SMAT_CUDA_ERROR = 4,   /* a CUDA runtime failure                               */
  SMAT_BAD_ARG = 5,      /* ValueError                                           */
  SMAT_UNSUPPORTED = 6,  /* operator/size combination with no device path       */
  SMAT_OOM = 7           /* device allocation failed                             */
} smat_status;

typedef enum smat_layout {
  SMAT_ROW_MAJOR = 0, /* element (i, col) at i*ld + col, ld >= ncols (0: ld = ncols) */
  SMAT_COL_MAJOR = 1  /* element (i, col) at col*ld + i, ld >= rows  (0: ld = rows)  */
} smat_layout;

typedef enum smat_dtype {
  SMAT_F32 = 0,
  SMAT_F64 = 1,
  SMAT_C64 = 2,
  SMAT_C128 = 3,
  SMAT_I32 = 4,
  SMAT_I64 = 5
} smat_dtype;

/* Operator kinds.  Leaves: leaves.py:28-322; composites: composites.py:30-398. */
typedef enum smat_kind {
  SMAT_IDENTITY = 0,   /* Identity(n)                      leaves.py:68-79   */
  SMAT_ZERO = 1,       /* Zero(rows, cols)                 leaves.py:52-65   */
  SMAT_DIAGONAL = 2,   /* Diagonal(d)  (alias Diag)        leaves.py:82-97   */
  SMAT_DENSE = 3,      /* Dense(entries) (alias Matrix)    leaves.py:28-49   */
  SMAT_HADAMARD = 4,   /* Hadamard(order)                  leaves.py:181-204 */
  SMAT_FOURIER = 5,    /* Fourier(n)                       leaves.py:162-178 */
  SMAT_CIRCULANT = 6,  /* Circulant(c)                     leaves.py:207-234 */
  SMAT_TOEPLITZ = 7,   /* Toeplitz(first_col, row_rest)    leaves.py:237-290 */
  SMAT_LOWRANK = 8,    /* LowRank(U, V[, s]) = U diag(s) V^H   (new type)     */
  SMAT_PRODUCT = 9,    /* Product(*factors)                composites.py:30-67  */
  SMAT_SUM = 10,       /* Sum(*terms)                      (new type)           */
  SMAT_KRON = 11,      /* Kron(*factors)                   composites.py:70-121 */
  SMAT_PARTIAL = 12,   /* Partial(base, rows, cols)        composites.py:239-320*/
  SMAT_ADJOINT = 13,   /* Adjoint(base)                    core.py:229-253      */
  SMAT_BLOCKDIAG = 14, /* BlockDiag(*blocks)               composites.py:196-236*/
  SMAT_BLOCKS = 15,    /* Blocks(grid)                     composites.py:124-193*/
  SMAT_SCALED = 16,    /* scalar * base (Polynomial/Power building block)       */
  SMAT_SPARSE = 17,    /* Sparse(rows, cols, triplets) CSR  leaves.py:100-159   */
  SMAT_POLYNOMIAL = 18 /* Polynomial(base, coeffs) Horner   composites.py:323-365*/
} smat_kind;

/* A host-resident parameter array (copied to the device by plan build). */
typedef struct smat_param {
  const void* data; /* host pointer, C-contiguous                     */
  int64_t len;      /* number of elements                             */
  int32_t dtype;    /* smat_dtype of `data`                           */
  int32_t _pad;
} smat_param;

/*
 * One node of the serialised operator tree.
 *   kind     smat_kind
 *   rows/cols operator shape (core.py:96-106)
 *   children index range [first_child, first_child + n_children) into the
 *            `children` array passed to smat_plan_build
 *   iparam   kind-specific integers:
 *              HADAMARD: iparam[0] = order
 *              BLOCKS:   iparam[0] = grid rows, iparam[1] = grid cols
 *              PARTIAL:  iparam[0] = has_rows, iparam[1] = has_cols,
 *                        iparam[2] = rows unique, iparam[3] = cols unique
 *              LOWRANK:  iparam[0] = rank r
 *   dparam   kind-specific scalars (SCALED: dparam[0] + i dparam[1])
 *   param    kind-specific arrays:
 *              DIAGONAL: param[0] = d
 *              DENSE:    param[0] = entries (rows x cols)
 *              CIRCULANT:param[0] = first column c
 *              TOEPLITZ: param[0] = first column, param[1] = first row rest
 *              LOWRANK:  param[0] = U (rows x r), param[1] = V (cols x r),
 *                        param[2] = s (r) or empty
 *              PARTIAL:  param[0] = row indices (I64), param[1] = col indices
 *              SPARSE:   param[0] = row_ptr (I64, rows+1), param[1] = col_idx
 *                        (I64, nnz), param[2] = values (nnz), duplicates summed
 *                        (the reference's csr_matrix.sum_duplicates)
 *              POLYNOMIAL: one child (square base), param[0] = ascending
 *                        coefficients (F64 or C128)
 */
typedef struct smat_node {
  int32_t kind;
  int32_t n_children;
  int32_t first_child;
  int32_t _pad;
  int64_t rows;
  int64_t cols;
  int64_t iparam[4];
  double dparam[2];
  smat_param param[4];
} smat_node;

typedef struct smat_plan smat_plan;

/* Compile a serialised operator tree into an immutable device plan for the
 * working dtype `dtype` on CUDA device `device`.  Replaces operator
 * construction-time precomputation (Circulant spectrum leaves.py:216, Toeplitz
 * embedding leaves.py:253-261, DftPlan tables kernels.py:68-93) and the
 * lru-cached plan registry get_plan (kernels.py:150-153). */
SMAT_API int smat_plan_build(const smat_node* nodes, int32_t n_nodes, const int32_t* children,
                    int32_t n_children, int32_t root, int32_t dtype, int32_t device,
                    smat_plan** out);

/* Device workspace (bytes) one smat_apply of `ncols` columns with leading
 * dimensions ldx / ldy (0 = dense) in `layout` needs.  Row-major blocks with
 * ld > ncols are transformed in place where every pass of the plan can
 * address the strided rows; otherwise (and for SMAT_COL_MAJOR) the apply
 * stages the block through the workspace with one device copy each way. */
SMAT_API int smat_workspace_bytes(const smat_plan* plan, int32_t direction, int64_t ncols, int64_t ldx,
                                  int64_t ldy, int32_t layout, size_t* out_bytes);

/* y = A·x (direction 0, forward — core.py:128-149) or y = A^H·x (direction 1,
 * backward — core.py:151-167) on device buffers; asynchronous on `stream`,
 * no allocation, CUDA-graph capturable.  x is (cols, ncols) for direction 0
 * and (rows, ncols) for direction 1, in the plan dtype except that a real
 * input to a complex plan may be passed with `x_dtype` = the matching real
 * dtype (it is promoted on load, core.py:145).  y is written in the plan
 * dtype.  ldx / ldy / layout: see "Layout" above (x and y must not overlap). */
SMAT_API int smat_apply(const smat_plan* plan, int32_t direction, const void* x, int32_t x_dtype,
                        int64_t ldx, void* y, int64_t ldy, int64_t ncols, int32_t layout,
                        void* workspace, size_t workspace_bytes, void* stream);

/* End-to-end application on HOST buffers (the reference's numpy-in/numpy-out
 * contract, core.py:128-149): pinned or pageable host x, host y.  Columns are
 * streamed through the device in chunks so that host->device copies, the
 * device passes and device->host copies overlap on separate streams. */
SMAT_API int smat_apply_host(const smat_plan* plan, int32_t direction, const void* x_host,
                             int32_t x_dtype, int64_t ldx, void* y_host, int64_t ldy, int64_t ncols,
                             int32_t layout, int32_t chunk_cols);

/* smat_apply with a CUDA event recorded on `stream` before every launch and
 * after the last one; synchronises the stream and returns the duration (ms) and
 * a kernel label of each launch (at most `max_launches`; labels are written
 * '\n'-separated into `labels`).  Measurement helper for bench.py's roofline. */
SMAT_API int smat_apply_profiled(const smat_plan* plan, int32_t direction, const void* x,
                                 int32_t x_dtype, void* y, int64_t ncols, void* workspace,
                                 size_t workspace_bytes, void* stream, float* launch_ms,
                                 int32_t max_launches, int32_t* n_launches, char* labels,
                                 size_t labels_len);

/* Number of kernel launches one smat_apply issues, and a human-readable
 * description of the compiled passes (diagnostics, bench gpu_launches). */
SMAT_API int smat_plan_launches(const smat_plan* plan, int32_t direction, int64_t ncols,
                       int64_t* out_launches);
SMAT_API int smat_plan_describe(const smat_plan* plan, char* buf, size_t buf_len);

/* Rows/cols/dtype of a compiled plan. */
SMAT_API int smat_plan_shape(const smat_plan* plan, int64_t* rows, int64_t* cols, int32_t* dtype);

SMAT_API void smat_plan_free(smat_plan* plan);

/* Thread-local message of the last failing call on this thread. */
SMAT_API const char* smat_last_error(void);

SMAT_API int smat_abi_version(void);

/* Arithmetic peak of device `device` in TFLOP/s, measured by a short
 * register-only kernel: kind 0 DFMA (FP64 vector), 1 DMMA m8n8k4 (FP64 tensor
 * core), 2 DFMA and DMMA warps side by side, 3 FFMA2 (packed FP32).  The
 * compute-roofline denominators of bench.py. */
SMAT_API int smat_probe_peak(int32_t kind, int32_t device, double* tflops);

/* ---------------------------------------------------------------------------
 * Device-resident solver steps (pkg/src/linopkit/solvers.py).  Every vector is
 * an (n, ncols) C-contiguous float64 (SMAT_F64) or complex128 (SMAT_C128)
 * device block; `scratch` is caller device memory of at least
 * smat_solver_scratch_bytes(n, ncols) bytes; all calls are asynchronous on
 * `stream` and CUDA-graph capturable.  The operator applications in between
 * are ordinary smat_apply calls.
 * ------------------------------------------------------------------------- */

/* Scratch bytes the solver steps need for (n, ncols) blocks. */
SMAT_API size_t smat_solver_scratch_bytes(int64_t n, int64_t ncols);

/* Per-column CG state: `state` is a device double[ncols][SMAT_CG_STATE] array,
 * fields in order: rs_old, threshold, alpha, beta, iterations, status
 * (0 running, 1 converged, 2 breakdown — non-positive curvature, 3 iteration
 * limit reached), residual norm, curvature at breakdown. */
#define SMAT_CG_STATE 8

/* x = 0, r = p = b, rs_old = |b|^2, threshold = tol * |b| per column; a zero
 * column is converged at iteration 0 (solvers.py:75-84). */
SMAT_API int smat_cg_init(int32_t dtype, int64_t n, int64_t ncols, const void* b, void* x, void* r, void* p,
                          double* state, double tol, void* scratch, size_t scratch_bytes, void* stream);

/* One conjugate-gradient iteration on every running column given ap = A p
 * (solvers.py:85-102): curvature / breakdown test, x += alpha p,
 * r -= alpha ap, convergence test, p = r + beta p. */
SMAT_API int smat_cg_step(int32_t dtype, int64_t n, int64_t ncols, void* x, void* r, void* p, const void* ap,
                          double* state, int64_t max_iter, void* scratch, size_t scratch_bytes, void* stream);

/* ISTA halves (solvers.py:182-192) on length-n vectors.  state = device
 * double[2]: l1 norm of the current x, step counter k.
 * residual: r = b - mx, trace[k] = lam * l1 + |r|^2 / 2, k += 1.
 * update:   x = soft_threshold(x + alpha * g, level), l1 = sum |x|. */
SMAT_API int smat_ista_residual(int32_t dtype, int64_t n, const void* b, const void* mx, void* r, double* trace,
                                double* state, double lam, void* scratch, size_t scratch_bytes, void* stream);
SMAT_API int smat_ista_update(int32_t dtype, int64_t n, void* x, const void* g, double alpha, double level,
                              double* state, void* scratch, size_t scratch_bytes, void* stream);

/* One power-method step given w = A v (or A^H A v) (solvers.py:318-332).
 * state = device double[6]: estimate |v^H w|, iterations, done, converged,
 * (internal), zero-iterate flag; v = w / |w| unless done. */
SMAT_API int smat_power_step(int32_t dtype, int64_t n, void* v, const void* w, double* state, double tol,
                             void* scratch, size_t scratch_bytes, void* stream);

/* y = soft_threshold(x, c) elementwise (solvers.py:22-34); y may alias x. */
SMAT_API int smat_soft_threshold(int32_t dtype, int64_t n, const void* x, void* y, double c, void* stream);

/* out_index[0] = argmax_i |g[i]| over i with excluded[i] == 0 (excluded may be
 * null), lowest index on ties — OMP's atom pick (solvers.py:233-235). */
SMAT_API int smat_abs_argmax(int32_t dtype, int64_t n, const void* g, const unsigned char* excluded,
                             int64_t* out_index, void* scratch, size_t scratch_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SMAT_H_ */
