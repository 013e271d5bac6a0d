// Internal declarations shared by the translation units of libaci.so.
// Nothing here is part of the C-ABI (include/aci.h is).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define ACI_GEMM_MAX_IN 4

// One GEMM problem C = sum over inputs (FUSE: f of) A_n (M x K_n) * B_n (K_n x N), row-major.
// Written by the planner kernels on the device (M, N, leading dims depend on live ranks).
struct GemmDesc {
  double *C;
  int M, N, ldc;
  const double *S;  // EPI_SUB: C = S - A B (S has leading dimension lds)
  int lds;
  int nin;
  const double *A[ACI_GEMM_MAX_IN];
  const double *B[ACI_GEMM_MAX_IN];
  int K[ACI_GEMM_MAX_IN], lda[ACI_GEMM_MAX_IN], ldb[ACI_GEMM_MAX_IN];
  // complex GEMMs run as real GEMMs on interleaved (re, im) storage against a right operand in
  // 2x2-block EXPANDED form (row 2k: re, im; row 2k+1: -im, re), so that
  // [a_re a_im] [[b_re, b_im], [-b_im, b_re]] = [re(ab), im(ab)].
  // EPI_STORE_X writes the complex result C ((K' xd) x n, viewed K' x (xd n)) in expanded form:
  // row i -> block row i / xd, column block (i % xd) n + j; ldc is the expanded leading dim.
  int xd;
};

// Elementwise f = sum_t coef[t] prod_n x_n^expo[t][n].
struct FOp {
  int T, N;
  double coef[8];
  int expo[8 * ACI_GEMM_MAX_IN];
  int monomial_all_ones;  // 1: f = coef[0] * x_0 * ... * x_{N-1} (fast epilogue path)
};

// Live sizes of one prrLU problem, written by the planner on the device.
struct LuDims {
  int m, n, ldm;      // matrix rows, cols, leading dimension
  int kmax;           // min(maxrank, m, n)
  int ldu;            // leading dimension of the U rows output
};

// prrLU arguments (Alg. 2, readings R1-R4, R17).
struct LuArgs {
  const double *M;            // row-major matrix (device)
  const LuDims *dims;         // live sizes
  double tol;
  int thr_mode;               // 0: thr = tol * s (R1); 1: thr = tol * |first candidate| (R8); 2: thr = tol
  const unsigned long long *scale_bits;  // s as IEEE bits (non-negative double)
  int *rows, *cols;           // pivots out (selection order, R21)
  int *r_out;                 // rank out
  double *eps_out;            // first rejected candidate (R2)
  double *U;                  // optional U rows out (r x n, ld = dims->ldu), U_k = S_k[p,:]/c
  // grid tier exchange: every published word carries a tag (epoch << 12 | step + 1) in its
  // upper 32 bits, so readers validate data without release/acquire fences
  unsigned long long *colpub; // 2 x G x colcap x 2 x prrlu_col_spread() words: (tag|lo32, tag|hi32) per element
  int colcap;
  unsigned long long *keys;   // 2 x G x 4 words: tag|hi, tag|lo, tag|id, pad
  unsigned int *counter;      // zeroed before launch
  unsigned int *epoch;        // incremented by every grid-tier launch (tags stay unique)
  long long *dbg;             // development timing (ACI_PRRLU_TIMING builds only)
};

// ---- launchers (defined in gemm.cu / prrlu.cu / sweep.cu) ----
void launch_gemm(const GemmDesc *d_descs, int ndesc, int max_m, int max_n, int nin, bool fuse, const FOp &op,
                 unsigned long long *scale_bits, int *nonfinite, cudaStream_t st);
// Pi launch with the inputs split by inner dimension: descriptors 0..nbig-1 run the DMMA main
// loop, nbig..nbig+nsmall-1 (K <= gemm_small_k()) are evaluated in the epilogue.
void launch_gemm_split(const GemmDesc *d_descs, int ndesc, int max_m, int max_n, int nbig, int nsmall, bool fuse,
                       const FOp &op, unsigned long long *scale_bits, int *nonfinite, cudaStream_t st);
int gemm_small_k();
// Sets kernel attributes (dynamic shared memory) once; call before any stream capture.
void gemm_init();
// Complex GEMMs (interleaved storage, expanded right operand): mode 0 = plain store, 1 = expanded
// store (GemmDesc::xd), 2 = complex f of nin inputs (max |Pi| into sb, NaN flag into nf).
void launch_gemm_z(const GemmDesc *d, int ndesc, int max_m, int max_n, int mode, int nin, const FOp &op,
                   unsigned long long *sb, int *nf, cudaStream_t st);
// C = S - A B for every descriptor (blocked triangular solve updates).
void launch_gemm_sub(const GemmDesc *d_descs, int ndesc, int max_m, int max_n, cudaStream_t st);

// a3+a4 of the next L->R bond streamed while this bond's prrLU runs (DESIGN.md §5 "streamed Pi"):
// rows of Pi_{b+1} = f(A^1_{b+1} B^1_{b+1}, ...) are computed as the pivot rows I_b they need are
// taken. A^n_{b+1} row (k, sigma) = Ahat^n[rows[k]][sigma c2 .. sigma c2 + c2) (Ahat^n = A^n_b X^n_{b+1},
// the look-ahead product, W = d1 c2 doubles per row); the gathered rows are also stored to Anext^n.
// Inputs in Pi order: 0..nbig-1 through the DMMA main loop, the rest (c2 <= gemm_small_k()) in the
// epilogue. rows[] and *r_in read -1 until the prrLU writes them.
struct PiStreamArgs {
  const int *rows;    // pivot rows of bond b (written one by one by the prrLU)
  const int *r_in;    // final rank of bond b
  const int *rk;      // live ranks: n' = db2 * rk[b + 3]
  int kcap;           // capacity of rows[] (the prrLU takes at most kcap pivots)
  int ntmax;          // 32-column tiles of the static n' (grid = ntmax x P)
  unsigned poll_ns;   // back-off between polls
  unsigned long long *ts;  // development timestamps (ACI_STREAM_TS builds only)
  int b, d1, db2, N, nbig;
  const double *Ahat[ACI_GEMM_MAX_IN];
  double *Anext[ACI_GEMM_MAX_IN];  // null: not stored
  const double *B[ACI_GEMM_MAX_IN];  // B^n_{b+1} (c2 x n', ld n')
  int c2[ACI_GEMM_MAX_IN];
  double *Pi;         // Pi_{b+1}, ld n'
  unsigned long long *sp;  // max |Pi_{b+1}| (bits) of this stream, merged into *scale by its last CTA
  unsigned long long *scale;  // the running s: snapshot into info[4..5] at the start, merged at the end
  int *info;          // bond b's index-kernel snapshot (info + 4: s as Pi_b left it)
  unsigned *done;     // CTA exit counter (reset by the last CTA)
  int *nonfinite;
};
// c2: the inputs' K in Pi order; ntmax = ceil(static n' / 32) (<= 64), sum of the DMMA inputs'
// K <= 256 (shared-memory panels)
bool pi_stream_supported(int nbig, int nsmall, const int *c2, int ntmax);
// grid = ntmax x P persistent CTAs (column tile q % ntmax, chunks q / ntmax + P t)
void launch_pi_stream(const PiStreamArgs &a, int nsmall, const FOp &op, int grid, cudaStream_t st);

// Picks the tier for a (max_m x max_n) problem; returns false if it is out of the envelope.
bool prrlu_supported(int max_m, int max_n, bool cplx = false);
size_t prrlu_exchange_bytes(int max_m, int max_n);
// cplx: complex entries (interleaved; ldm/ldu in complex elements; colcap >= 2 m).
// one: single-cluster mode (aci_options.concurrent): at most one 16-CTA cluster per launch.
// `started` (optional, created with cudaEventDisableTiming) fires once every CTA has begun.
// Returns the launch's own error (a rejected configuration leaves the outputs unwritten).
// rook: rook pivoting (R23, NEXT-4; prrlu_supported_rook envelope, real values) instead of full.
cudaError_t launch_prrlu(const LuArgs &a, int max_m, int max_n, cudaStream_t st, bool cplx = false, bool one = false,
                         cudaEvent_t started = nullptr, bool rook = false);
bool prrlu_supported_one(int m, int n, bool cplx);
bool prrlu_supported_rook(int m, int n);
// true when concurrent-mode products may factorise blocks beyond one cluster (they then use the
// cooperative, gang-scheduled L2 grid tier)
bool prrlu_coop_multicluster();
// Chooses the prrLU exchange tier (cluster size) once; call before any stream capture.
void prrlu_init();
void prrlu_envelope(int *max_rows, int *max_cols);
// Column-slot stride factor of the exchange buffer: a slot holds colcap * 2 * factor u64 words.
int prrlu_col_spread();
