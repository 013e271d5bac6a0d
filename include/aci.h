/*
 * aci.h — C-ABI of libaci.so, the B200-native (sm_100a) hot path of
 * alternating cross interpolation (ACI), M. K. Ritter, arxiv 2604.00037.
 *
 * Citation keys: P:n = PAPER.md line n (Ritter 2026), R# = reading # in
 * DESIGN.md §2. All floating point is IEEE binary64 (FP64).
 *
 * Conventions shared by every call:
 *  - A tensor train (TT) x has L >= 1 cores; core s (0-based) is a row-major
 *    array of shape [r_s][d_s][r_{s+1}] with r_0 = r_L = 1.
 *  - Local indices are 0-based; a full multi-index is L uint8 values.
 *  - Return value: ACI_OK (0), a negative ACI_ERR_* code, or ACI_NOT_CONVERGED
 *    (> 0, still a valid result). On error aci_last_error() describes it.
 *  - Host pointers are only read during the call; nothing is retained.
 *  - All device work is enqueued on the caller's stream (NULL = the library's
 *    internal stream); calls return after the stream work they enqueued is
 *    complete unless noted.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    call returns ACI_ERR_CUDA.
 */
#ifndef ACI_B200_H
#define ACI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACI_OK 0
#define ACI_NOT_CONVERGED 1      /* max_sweeps exhausted or rank cap bound; output valid */
#define ACI_ERR_INVALID -1       /* null pointer, bad size, bad option */
#define ACI_ERR_SHAPE -2         /* inputs disagree in L or d_s */
#define ACI_ERR_NONFINITE -3     /* NaN/Inf in an input core, y_init, or produced by f */
#define ACI_ERR_OOM -4           /* device allocation failed or caller workspace too small */
#define ACI_ERR_CUDA -5          /* CUDA runtime/driver error, or no sm_100 device */
#define ACI_ERR_UNSUPPORTED -6   /* size outside the compiled kernel envelope (see aci_limits) */

typedef struct tt_s tt_t; /* opaque; device-resident cores */

/* ---------------------------------------------------------------- TT objects */

/* Create a device-resident TT from host cores (x_sigma = X_1[sigma_1]...X_L[sigma_L]).
 * L: number of sites (>= 1); d[L]: local dimensions (1..255); ranks[L+1]: bond dimensions
 * with ranks[0] = ranks[L] = 1; cores[L]: host pointers, core s holds ranks[s]*d[s]*ranks[s+1]
 * doubles row-major [alpha][sigma][beta]. The cores are copied (host -> device) before return.
 * Errors: ACI_ERR_INVALID (null, L < 1, d or rank < 1, boundary rank != 1),
 * ACI_ERR_NONFINITE (NaN/Inf in a core), ACI_ERR_OOM, ACI_ERR_CUDA. *out is owned by the caller. */
int tt_create(int L, const int *d, const int *ranks, const double *const *cores, tt_t **out);

/* Same, from ONE contiguous device buffer holding core 0, core 1, ... back to back
 * (device pointer). The data are copied device -> device. */
int tt_create_device(int L, const int *d, const int *ranks, const double *dev_cores, void *stream, tt_t **out);

/* Complex TTs (f: C^N -> C; the random Fourier series of P:289-296). Arguments as
 * tt_create / tt_create_device, but every core entry is a complex number stored as two
 * consecutive doubles (re, im) (C99 double complex / numpy complex128 layout): core s holds
 * 2*ranks[s]*d[s]*ranks[s+1] doubles. Every other call accepts complex handles: tt_get_cores and
 * tt_evaluate(_device) then read/write 2 doubles per entry / per point, and aci_elementwise(_ex)
 * requires all inputs (and y_init) to be complex and returns a complex TT (readings RZ1-RZ6 of
 * pivots by |z|^2 = re^2 + im^2, complex Schur updates). Complex 2-site blocks
 * are limited to 512 rows (aci_elementwise returns ACI_ERR_UNSUPPORTED beyond). */
int tt_create_z(int L, const int *d, const int *ranks, const double *const *cores, tt_t **out);
int tt_create_device_z(int L, const int *d, const int *ranks, const double *dev_cores, void *stream, tt_t **out);

/* 1 if tt holds complex cores, else 0 (NULL: 0). */
int tt_is_complex(const tt_t *tt);

/* Free a TT (device memory included; it returns to the library's stream-ordered pool). NULL is a
 * no-op. Returns ACI_OK. Every library call that reads or writes a TT has finished with it when it
 * returns; work the caller enqueued itself on tt_device_cores() must be complete before this call
 * (there is no device-wide synchronisation here: it would break stream captures in other host
 * threads). */
int tt_destroy(tt_t *tt);

/* Shape query: *L, and if non-NULL d[L], ranks[L+1]. */
int tt_shape(const tt_t *tt, int *L, int *d, int *ranks);

/* Copy the cores to host buffers host_cores[s] (each ranks[s]*d[s]*ranks[s+1] doubles; twice
 * that, interleaved (re, im), for a complex TT). */
int tt_get_cores(const tt_t *tt, double *const *host_cores);

/* Device pointer to the contiguous core storage (core s at offset sum_{t<s} r_t d_t r_{t+1}).
 * Valid until tt_destroy; the caller synchronises its own work on it before destroying. */
const double *tt_device_cores(const tt_t *tt);

/* Evaluate x at npts full multi-indices (O(L chi^2) per point).
 * idx: host, npts*L uint8 (row-major, point-major), out: host, npts doubles (2*npts,
 * interleaved (re, im), for a complex TT).
 * Errors: ACI_ERR_INVALID (index >= d_s, null), ACI_ERR_CUDA. */
int tt_evaluate(const tt_t *tt, int64_t npts, const uint8_t *idx, double *out);

/* Same with device buffers (idx: device npts*L uint8; out: device npts doubles), enqueued on stream. */
int tt_evaluate_device(const tt_t *tt, int64_t npts, const uint8_t *dev_idx, double *dev_out, void *stream);

/* ---------------------------------------------------------------- the operation f */

/* f(x_1..x_N) = sum_t coef[t] * prod_n x_n^expo[t*N + n]. This covers Hadamard
 * products (one term, all exponents 1), sums, psi^3 and a*b + a^2. n_terms <= ACI_MAX_TERMS,
 * exponents 0..ACI_MAX_EXPO. N is the n_inputs of the call that uses the op. */
#define ACI_MAX_INPUTS 4
#define ACI_MAX_TERMS 8
#define ACI_MAX_EXPO 4
typedef struct {
  int n_terms;
  const double *coef; /* n_terms */
  const int *expo;    /* n_terms x n_inputs, row-major */
} aci_op;

/* ---------------------------------------------------------------- the ACI product */

typedef struct {
  double error_estimate;     /* max_l eps_l / s of the last iteration (absolute mode: max eps_l) */
  double scale;              /* s = max |Pi| seen (R1) */
  int iterations;            /* full iterations (L->R + R->L) performed (R10) */
  int converged;             /* no rank grew and max eps <= tau*s */
  int max_rank;              /* max output bond dimension */
  int n_updates;             /* 2-site updates performed (= 2 (L-1) iterations) */
  int64_t pivot_steps;       /* accepted pivots over all prrLU calls */
  double flops_contraction;  /* SURVEY 8(d) model, per distinct input, from the live ranks */
  double flops_prrlu;        /* sum_k 2 (m-k-1)(n-k-1) */
  double flops_trsm;         /* output cores: r^2 (n - r) per bond */
  double flops_init;         /* canonicalisation GEMMs */
  float ms;                  /* host wall time of the call (includes the final sync) */
  int64_t n_launches;        /* kernels this call launched */
  int graph_iterations;      /* iterations replayed from one captured CUDA graph (0 = direct launches) */
  float ms_graph_setup;      /* host time spent capturing + instantiating that graph */
} aci_report;

/* Optional per-kernel-class device timing (CUDA events around each launch on the call's
 * stream; adds a few microseconds per launch). Classes: */
#define ACI_PROF_CANON 0     /* a0: canonicalisation (all its kernels) */
#define ACI_PROF_GEMM_AB 1   /* a1/a2: A = L X, B = X R */
#define ACI_PROF_GEMM_PI 2   /* a3+a4: Pi = f(A1 B1, ...) */
#define ACI_PROF_PRRLU 3     /* a5: prrLU */
#define ACI_PROF_UPDATE 4    /* a6/a7: index sets + frames (+ planning) */
#define ACI_PROF_CONV 5      /* a9: convergence */
#define ACI_PROF_TRSM 6      /* a8: output cores */
#define ACI_PROF_NCLASS 7
typedef struct {
  double ms[ACI_PROF_NCLASS];        /* out: summed event time per class */
  int64_t launches[ACI_PROF_NCLASS]; /* out: launches per class */
} aci_profile;

/* Optional per-update log (for parity tests): entries in update order. */
typedef struct {
  int capacity_updates;      /* entries the buffers below can hold */
  int capacity_pivots;       /* pivots per entry the row/col buffers can hold (>= maxrank) */
  int *info;                 /* capacity_updates x 5: bond, dir (0 = L->R, 1 = R->L), rl, rr, r */
  double *eps_scale;         /* capacity_updates x 2: eps_l, s */
  int *rows;                 /* capacity_updates x capacity_pivots: pivot rows in Pi's matricisation */
  int *cols;                 /* capacity_updates x capacity_pivots: pivot columns */
  int n_written;             /* out: entries written */
  /* canonicalisation pivots: for s = 1..L-1, |J_s| and the pivot columns */
  int *canon_n;              /* L+1 (entries 1..L-1 used) */
  int *canon_cols;           /* (L+1) x capacity_pivots */
} aci_pivot_log;

#define ACI_TOL_RELATIVE 0   /* R1: reject |c| <= tol * s (default) */
#define ACI_TOL_ABSOLUTE 1   /* paper-literal absolute tau */

typedef struct {
  uint64_t seed;             /* y_init seed when y_init == NULL (counter-based N(0,1), R9) */
  const tt_t *y_init;        /* initial guess; ranks are capped at maxrank */
  int tol_mode;              /* ACI_TOL_RELATIVE | ACI_TOL_ABSOLUTE */
  aci_pivot_log *log;        /* optional */
  void *stream;              /* cudaStream_t; NULL = the calling thread's library stream. A stream
                              * carries one call at a time: a call on a stream another call is
                              * still using returns ACI_ERR_INVALID (concurrent calls: one stream
                              * each) */
  void *workspace;           /* optional caller device memory (e.g. a torch tensor), >= the bytes
                              * aci_workspace_query returns, 256-byte aligned (else ACI_ERR_INVALID;
                              * cudaMalloc and the torch caching allocator return 512-byte aligned
                              * blocks). The library owns it for the duration of the call. */
  size_t workspace_bytes;
  /* optional: multi-indices of the final index sets, host buffers:
   * I_sets[b] must hold (>= out rank of bond b) x (b+1) bytes; J_sets[s] (>= rank) x (L-s). */
  uint8_t **I_sets;
  uint8_t **J_sets;
  aci_profile *profile;      /* optional: per-class device times of this call */
  float *iter_ms;            /* optional, max_sweeps floats: device time of each iteration (both
                              * half-sweeps + convergence test; CUDA events on the call's stream) */
  int concurrent;            /* 1: this call may run concurrently with other aci calls on other
                              * streams (host threads). prrLU launches then never span several
                              * thread-block clusters: blocks that fit one 16-CTA cluster (real:
                              * 128 x 1024, 256 x 512, 512 x 512, 1024 x 256; complex: 128 x 1024,
                              * 256 x 512, 512 x 256) use exactly one cluster, which the hardware
                              * schedules as a unit; larger blocks (e.g. the 1024 x 1024 blocks of
                              * configs[3] at chi = 256) use the L2 grid tier launched cooperatively,
                              * i.e. gang-scheduled (all CTAs resident or none). So concurrent
                              * products cannot deadlock on each other's spinning CTAs. Results are
                              * bit-identical to the default tiers (same keys and arithmetic).
                              * 0 (default): the fastest tiers, which may span several clusters
                              * (not gang-scheduled); such calls from several host threads are
                              * serialised by the library (a process-wide lock). Another PROCESS
                              * sharing the GPU (MPS) is not covered by that lock: a multi-cluster
                              * grid assumes its clusters can all be resident at once (checked once
                              * with cudaOccupancyMaxActiveClusters on an idle GPU); use concurrent
                              * mode there. */
  int pivoting;              /* ACI_PIVOT_FULL (default): full pivoting, Alg. 2 as written.
                              * ACI_PIVOT_ROOK: rook pivoting in every prrLU of the call (B:5
                              * "full/rook"; reading R23 of DESIGN.md §2): the pivot is an entry that
                              * is the largest of its active row and column, found from the smallest
                              * active column by alternating column / row maxima; eps is the magnitude
                              * of the first rejected rook candidate. Pivots (hence outputs) differ
                              * from full pivoting. Real values only and blocks within the
                              * `concurrent` envelope (one CTA or one 16-CTA cluster), else
                              * ACI_ERR_UNSUPPORTED. */
} aci_options;

#define ACI_PIVOT_FULL 0
#define ACI_PIVOT_ROOK 1

/*
 * aci_elementwise — Alg. 1: y ~ f(x^1, ..., x^N) with ||y - f(x)||_inf ~ tau
 * (Eq. ydef:maxnorm), by 2-site updates (Eq. pifromframes, prrLU Alg. 2
 * P:504-545, cross interpolation Alg. 3, frames Alg. 5).
 *
 * inputs[n_inputs]: borrowed, unmodified, may alias (aliases are merged into the exponents);
 *   all must share L and d_s (else ACI_ERR_SHAPE). n_inputs <= ACI_MAX_INPUTS distinct.
 * tol >= 0 (relative to s by default, R1); maxrank >= 1 (chi-hat); max_sweeps >= 1 iterations.
 * *out: new TT owned by the caller (valid also when ACI_NOT_CONVERGED is returned).
 * rep: nullable.
 * Errors: ACI_ERR_INVALID, ACI_ERR_SHAPE, ACI_ERR_NONFINITE (f produced NaN/Inf),
 *   ACI_ERR_OOM, ACI_ERR_CUDA, ACI_ERR_UNSUPPORTED (a 2-site block larger than aci_limits).
 */
int aci_elementwise(aci_op op, const tt_t *const *inputs, int n_inputs, double tol, int maxrank,
                    int max_sweeps, tt_t **out, aci_report *rep);

/* Same with options (opts may be NULL). */
int aci_elementwise_ex(aci_op op, const tt_t *const *inputs, int n_inputs, double tol, int maxrank,
                       int max_sweeps, tt_t **out, aci_report *rep, const aci_options *opts);

/* One product of a batch (aci_elementwise_batch). */
typedef struct {
  aci_op op;
  const tt_t *const *inputs;
  int n_inputs;
  double tol;
  int maxrank;
  int max_sweeps;
  const aci_options *options; /* nullable; `concurrent` is forced on and `stream`/`workspace` are
                               * ignored: every product runs on a library stream of its worker */
  tt_t **out;                  /* out: new TT owned by the caller */
  aci_report *rep;             /* out, nullable */
  int status;                  /* out: this product's return code (ACI_OK, ACI_NOT_CONVERGED, < 0) */
} aci_job;

/*
 * aci_elementwise_batch — several independent products (concurrent products
 * on one GPU, P:74 time stepping, several nonlinear terms) run concurrently: min(n_jobs,
 * max_parallel) library threads (max_parallel <= 0: 8) each take the next job and run it with
 * aci_options.concurrent on their own stream, so the products overlap on the GPU (every prrLU
 * launch stays within one thread-block cluster). Each job's result is exactly what the
 * corresponding aci_elementwise_ex call returns. Returns ACI_OK if every job returned >= 0,
 * else the first negative status in job order (the other jobs still ran; see jobs[i].status).
 */
int aci_elementwise_batch(aci_job *jobs, int n_jobs, int max_parallel);

/* Device workspace (bytes) aci_elementwise_ex needs for these inputs, maxrank and max_sweeps (the
 * per-update pivot log holds max_sweeps iterations; a call with more sweeps than the query was
 * made for returns ACI_ERR_OOM "caller workspace too small"). y_init: nullable (the default
 * initial guess's ranks are assumed). Errors: ACI_ERR_INVALID (null, maxrank < 1, max_sweeps < 1),
 * ACI_ERR_SHAPE, ACI_ERR_UNSUPPORTED. */
int aci_workspace_query(const tt_t *const *inputs, int n_inputs, int maxrank, int max_sweeps, const tt_t *y_init,
                        size_t *bytes);

/* Compiled envelope: the largest Pi block (rows, cols) the prrLU kernels accept. */
int aci_limits(int *max_rows, int *max_cols);

/*
 * aci_prrlu — the prrLU step alone (a5; Alg. 2, readings R1-R4, R17): partial-rank LU
 * with full pivoting of a device-resident row-major m x n FP64 block (leading dimension n),
 * exactly as a 2-site update runs it (same kernel, tiers, tie-break and arithmetic), for tests and
 * for callers that factorise their own blocks.
 *
 * dev_M: device, m x n, row-major, read only. maxrank >= 1: at most min(maxrank, m, n) pivots.
 * tol >= 0, tol_mode: ACI_TOL_RELATIVE -> a candidate c is rejected when |c| <= tol * |first
 *   candidate| (= tol * max|M|, R8); ACI_TOL_ABSOLUTE -> when |c| <= tol. The first pivot is
 *   always kept (R2); a zero block gives rank 1 with pivot (0, 0) (R17).
 * static_m, static_n: the launch's static capacity (>= m, n; 0 = m, n) — the product launches every
 *   bond for its largest possible block and the kernel picks its tier from the live size.
 * dev_rows, dev_cols: device, >= min(maxrank, m, n) ints: the pivots in selection order (R21).
 * dev_U: device, nullable, >= min(maxrank, m, n) x n doubles, ld n: U_k = S_k[p_k, :] / S_k[p_k, q_k].
 * *rank, *eps (host): the rank r and the first rejected candidate's |c| (0 when none, R2).
 * stream: a cudaStream_t or NULL (the library stream); the call synchronises it.
 * Errors: ACI_ERR_INVALID, ACI_ERR_UNSUPPORTED (static size beyond aci_limits), ACI_ERR_OOM,
 *   ACI_ERR_CUDA.
 */
int aci_prrlu(const double *dev_M, int m, int n, int maxrank, double tol, int tol_mode, int static_m, int static_n,
              int *dev_rows, int *dev_cols, double *dev_U, int *rank, double *eps, void *stream);

/* Thread-local description of the last error of this thread. */
const char *aci_last_error(void);

/* Library version string. */
const char *aci_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ACI_B200_H */
