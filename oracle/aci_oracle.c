/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of alternating cross
 * interpolation (ACI), written from PAPER.md (Ritter, arxiv 2604.00037),
 * Appendix B, Algorithms 1-5, with the readings of DESIGN.md §2
 * (= SURVEY.md §8(c) R1-R22). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library. It
 * shares no code with the CUDA path (paper_2604_00037_b200/csrc).
 *
 * Conventions:
 *  - sites s = 0..L-1, bonds b = 0..L-2 (bond b joins sites b and b+1);
 *  - cores row-major [alpha][sigma][beta];
 *  - Pi matricisation (Alg. 4): row = a*d_b + sigma,
 *    col = sigma' * |J_{b+2}| + j;
 *  - tolerance: relative to s = running max |Pi| (R1) unless absolute;
 *  - prrLU stop rule / epsilon / tie-break / elimination arithmetic: R2-R4;
 *  - orientation: final cores from the last right-to-left half-sweep,
 *    Y_{b+1} = U_J^{-1} U, Y_0 = Pi_0[:, J] (R5).
 *
 * Every step is a naive loop. No blocking, no BLAS.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_INVALID -1
#define ORC_ERR_NONFINITE -3
#define ORC_ERR_OOM -4

/* ------------------------------------------------------------------ */
/* Dense helpers (naive loops)                                         */
/* ------------------------------------------------------------------ */

/* C (M x N) = A (M x K) * B (K x N), all row-major, plain triple loop
 * (the "Einstein summation" convention of P:397). */
static void matmul(int M, int N, int K, const double *A, const double *B, double *C) {
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double acc = 0.0;
      for (int k = 0; k < K; ++k) acc += A[(size_t)i * K + k] * B[(size_t)k * N + j];
      C[(size_t)i * N + j] = acc;
    }
}

/* ------------------------------------------------------------------ */
/* Alg. 2 — LDU / prrLU with full pivoting                 */
/* ------------------------------------------------------------------ */

typedef struct {
  int r;        /* number of accepted pivots (>= 1) */
  int *rows;    /* pivot rows, in selection order (R21) */
  int *cols;    /* pivot columns */
  double *D;    /* pivot values */
  double *U;    /* r x n, U_k = S_k[p_k, :] * [S_k[p_k, q_k]]^{-1}, U_k[q_k] = 1 (R4) */
  double *Lc;   /* m x r, L_k = S_k[:, q_k] * [S_k[p_k, q_k]]^{-1}, L_k[p_k] = 1 (R4) */
  double eps;   /* |c| of the first rejected candidate; 0 if exhausted (R2) */
  double first; /* |c| of the first candidate = max |M| */
} ldu_t;

static void ldu_free(ldu_t *f) {
  free(f->rows); free(f->cols); free(f->D); free(f->U); free(f->Lc);
  memset(f, 0, sizeof(*f));
}

/*
 * Alg. 2 with the readings R1-R4, R17:
 *   k = 0, 1, ...:
 *     if k == min(m,n): eps = 0, stop (exhausted)
 *     (p,q) = argmax_{active} |S| ; ties -> smallest (row, col) (R3)
 *     c = S[p][q]
 *     if k == maxrank: eps = |c|, stop
 *     if k > 0 and |c| <= thr: eps = |c|, stop (candidate rejected, R2)
 *     if k == 0 and c == 0: dummy pivot (p,q), D=0, U = e_q, eps = 0, stop (R17)
 *     accept; inv = 1/c; U_k = S[p,:]*inv (U_k[q] = 1) ; L_k = S[:,q]*inv (L_k[p] = 1) ;
 *     S_ij <- fma(-l_i, S_pj, S_ij) on the active trailing block (R4)
 * thr_mode: 0 = absolute thr; 1 = thr * |first candidate| (relative to own max, R8).
 * Returns ORC_ERR_NONFINITE if M contains NaN/Inf.
 */
/*
 * Rook pivot search (SURVEY 8(f) NEXT-4, B:5 "full/rook"; reading R23 of DESIGN.md §2 — the paper
 * only uses full pivoting, and does not define rook). Textbook rook pivoting (Neal & Poole):
 * start at the smallest active column c; r = argmax over active rows of |S[i][c]|; then alternate
 * row and column maxima until an entry is the largest in both its row and its column. Ties go to
 * the smallest index (R3); an alternation stops as soon as the new extremum does not exceed the
 * current entry, so the accepted (p, q) is maximal in its active row AND its active column.
 */
static int col_argmax(int m, int n, const double *S, const char *rowdone, int c) {
  int r = -1;
  double best = -1.0;
  for (int i = 0; i < m; ++i)
    if (!rowdone[i] && fabs(S[(size_t)i * n + c]) > best) { best = fabs(S[(size_t)i * n + c]); r = i; }
  return r;
}
static int row_argmax(int n, const double *S, const char *coldone, int r) {
  int c = -1;
  double best = -1.0;
  for (int j = 0; j < n; ++j)
    if (!coldone[j] && fabs(S[(size_t)r * n + j]) > best) { best = fabs(S[(size_t)r * n + j]); c = j; }
  return c;
}
static void rook_search(int m, int n, const double *S, const char *rowdone, const char *coldone, int *pp, int *pq) {
  int c = 0;
  while (coldone[c]) ++c;
  int r = col_argmax(m, n, S, rowdone, c);
  for (;;) {
    int c2 = row_argmax(n, S, coldone, r);
    if (fabs(S[(size_t)r * n + c2]) <= fabs(S[(size_t)r * n + c])) break; /* (r,c): max of its column and row */
    c = c2;
    int r2 = col_argmax(m, n, S, rowdone, c);
    if (fabs(S[(size_t)r2 * n + c]) <= fabs(S[(size_t)r * n + c])) break; /* (r,c): max of its row and column */
    r = r2;
  }
  *pp = r;
  *pq = c;
}

static int ldu_p(int m, int n, const double *M, double thr, int thr_mode, int maxrank, int pivoting, ldu_t *out);
static int ldu(int m, int n, const double *M, double thr, int thr_mode, int maxrank, ldu_t *out) {
  return ldu_p(m, n, M, thr, thr_mode, maxrank, 0, out);
}

/* pivoting: 0 = full, 1 = rook (R23); everything else (stop rule, eps, elimination) as Alg. 2 */
static int ldu_p(int m, int n, const double *M, double thr, int thr_mode, int maxrank, int pivoting, ldu_t *out) {
  memset(out, 0, sizeof(*out));
  for (size_t t = 0; t < (size_t)m * n; ++t)
    if (!isfinite(M[t])) return ORC_ERR_NONFINITE;
  double *S = (double *)malloc(sizeof(double) * (size_t)m * n);
  char *rowdone = (char *)calloc(m, 1), *coldone = (char *)calloc(n, 1);
  int kcap = m < n ? m : n;
  if (maxrank < kcap) kcap = maxrank;
  out->rows = (int *)malloc(sizeof(int) * (kcap + 1));
  out->cols = (int *)malloc(sizeof(int) * (kcap + 1));
  out->D = (double *)malloc(sizeof(double) * (kcap + 1));
  out->U = (double *)calloc((size_t)(kcap + 1) * n, sizeof(double));
  out->Lc = (double *)calloc((size_t)m * (kcap + 1), sizeof(double));
  if (!S || !rowdone || !coldone || !out->rows || !out->U || !out->Lc) return ORC_ERR_OOM;
  memcpy(S, M, sizeof(double) * (size_t)m * n);
  int mn = m < n ? m : n;
  int k = 0;
  for (;;) {
    if (k == mn) { out->eps = 0.0; break; }
    int p = -1, q = -1;
    if (pivoting == 1) {
      rook_search(m, n, S, rowdone, coldone, &p, &q);
    } else {
      double best = -1.0;
      for (int i = 0; i < m; ++i) {
        if (rowdone[i]) continue;
        for (int j = 0; j < n; ++j) {
          if (coldone[j]) continue;
          double a = fabs(S[(size_t)i * n + j]);
          if (a > best) { best = a; p = i; q = j; } /* strict '>' keeps the smallest (row, col) on ties */
        }
      }
    }
    double c = S[(size_t)p * n + q];
    if (k == 0) out->first = fabs(c);
    double t = thr_mode == 1 ? thr * out->first : thr;
    if (k == maxrank) { out->eps = fabs(c); break; }
    if (k > 0 && fabs(c) <= t) { out->eps = fabs(c); break; }
    out->rows[k] = p; out->cols[k] = q; out->D[k] = c;
    if (k == 0 && c == 0.0) {
      /* R17: zero matrix -> rank 1, dummy pivot, B = e_q, eps = 0 */
      out->U[q] = 1.0;
      out->eps = 0.0;
      k = 1;
      break;
    }
    /* P:535 multiplies by [M_{chi,chi}]^{-1}: one reciprocal per pivot (R4) */
    const double inv = 1.0 / c;
    for (int j = 0; j < n; ++j) out->U[(size_t)k * n + j] = coldone[j] ? 0.0 : S[(size_t)p * n + j] * inv;
    for (int i = 0; i < m; ++i) out->Lc[(size_t)i * (kcap + 1) + k] = rowdone[i] ? 0.0 : S[(size_t)i * n + q] * inv;
    out->U[(size_t)k * n + q] = 1.0;
    out->Lc[(size_t)p * (kcap + 1) + k] = 1.0;
    /* Schur complement on the active block, l_i = S_iq * [S_pq]^{-1}, fma order fixed (R4) */
    for (int i = 0; i < m; ++i) {
      if (rowdone[i] || i == p) continue;
      double l = S[(size_t)i * n + q] * inv;
      for (int j = 0; j < n; ++j) {
        if (coldone[j] || j == q) continue;
        S[(size_t)i * n + j] = fma(-l, S[(size_t)p * n + j], S[(size_t)i * n + j]);
      }
    }
    rowdone[p] = 1; coldone[q] = 1;
    ++k;
  }
  out->r = k;
  free(S); free(rowdone); free(coldone);
  return ORC_OK;
}

/* Exported for the pin tests: prrLU of a dense row-major m x n matrix (pivoting 0 full, 1 rook). */
int oracle_ldu_p(int m, int n, const double *M, double thr, int thr_mode, int maxrank, int pivoting,
                 int *r, int *rows, int *cols, double *D, double *U /* maxr x n */,
                 double *Lc /* m x maxr */, int maxr, double *eps) {
  if (m < 1 || n < 1 || maxrank < 1 || thr < 0 || pivoting < 0 || pivoting > 1) return ORC_ERR_INVALID;
  ldu_t f;
  int st = ldu_p(m, n, M, thr, thr_mode, maxrank, pivoting, &f);
  if (st != ORC_OK) return st;
  int kcap = (m < n ? m : n);
  if (maxrank < kcap) kcap = maxrank;
  *r = f.r;
  *eps = f.eps;
  for (int k = 0; k < f.r && k < maxr; ++k) {
    rows[k] = f.rows[k]; cols[k] = f.cols[k]; D[k] = f.D[k];
    if (U) for (int j = 0; j < n; ++j) U[(size_t)k * n + j] = f.U[(size_t)k * n + j];
    if (Lc) for (int i = 0; i < m; ++i) Lc[(size_t)i * maxr + k] = f.Lc[(size_t)i * (kcap + 1) + k];
  }
  ldu_free(&f);
  return ORC_OK;
}

int oracle_ldu(int m, int n, const double *M, double thr, int thr_mode, int maxrank,
               int *r, int *rows, int *cols, double *D, double *U, double *Lc, int maxr, double *eps) {
  return oracle_ldu_p(m, n, M, thr, thr_mode, maxrank, 0, r, rows, cols, D, U, Lc, maxr, eps);
}

/* ------------------------------------------------------------------ */
/* Alg. 3, right-orthogonal branch (R6):                   */
/*   B = [U_{1:r, J}]^{-1} U  (unit upper triangular back substitution) */
/* ------------------------------------------------------------------ */
static void ci_right_B(int r, int n, const double *U, const int *cols, double *B) {
  for (int k = r - 1; k >= 0; --k)
    for (int j = 0; j < n; ++j) {
      double acc = U[(size_t)k * n + j];
      for (int i = k + 1; i < r; ++i) acc -= U[(size_t)k * n + cols[i]] * B[(size_t)i * n + j];
      B[(size_t)k * n + j] = acc;
    }
}

/* Exported for pins: cross interpolation (Alg. 3), right orientation.
 * A = M[:, J] (m x r), B = U_J^{-1} U (r x n). */
int oracle_ci_right(int m, int n, const double *M, double thr, int thr_mode, int maxrank,
                    int *r, int *rows, int *cols, double *A, double *B, int maxr, double *eps) {
  ldu_t f;
  int st = ldu(m, n, M, thr, thr_mode, maxrank, &f);
  if (st != ORC_OK) return st;
  *r = f.r; *eps = f.eps;
  double *Bt = (double *)malloc(sizeof(double) * (size_t)f.r * n);
  ci_right_B(f.r, n, f.U, f.cols, Bt);
  for (int k = 0; k < f.r && k < maxr; ++k) {
    rows[k] = f.rows[k]; cols[k] = f.cols[k];
    for (int j = 0; j < n; ++j) B[(size_t)k * n + j] = Bt[(size_t)k * n + j];
    for (int i = 0; i < m; ++i) A[(size_t)i * maxr + k] = M[(size_t)i * n + f.cols[k]];
  }
  free(Bt);
  ldu_free(&f);
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Elementwise f: polynomial sum_t coef_t prod_n x_n^{expo[t][n]}     */
/* (covers Hadamard products, psi^3 and a*b + a^2)          */
/* ------------------------------------------------------------------ */
typedef struct {
  int N, T;
  const double *coef; /* T */
  const int *expo;    /* T x N */
} op_t;

static double apply_f(const op_t *op, const double *x /* N */) {
  double y = 0.0;
  for (int t = 0; t < op->T; ++t) {
    double p = op->coef[t];
    for (int n = 0; n < op->N; ++n)
      for (int e = 0; e < op->expo[t * op->N + n]; ++e) p *= x[n];
    y += p;
  }
  return y;
}

/* ------------------------------------------------------------------ */
/* ACI state                                                          */
/* ------------------------------------------------------------------ */
typedef struct {
  int b, dir, rl, rr, r;
  double eps, scale;
  int *rows, *cols;
} logent_t;

typedef struct {
  int L, N;
  int *d;           /* L */
  int *xr;          /* N x (L+1) input ranks */
  double ***X;      /* N x L cores */
  op_t op;
  /* index sets, materialised (R21/R22): I[b] is chi[b] x (b+1); J[s] is |J_s| x (L-s) */
  unsigned char **I, **J;
  int *chi;         /* chi[b] = |I_b| = |J_{b+1}|, b = 0..L-2 */
  int *Jn;          /* Jn[s] = |J_s| for s = 1..L (Jn[L] = 1) */
  /* frames: Lf[n][b] = L^n_b (chi[b] x xr[n][b+1]); Rf[n][s] = R^n_s (xr[n][s] x Jn[s]) */
  double ***Lf, ***Rf;
  /* output cores */
  int *yr;          /* L+1 */
  double **Y;
  /* report */
  double scale, err_estimate;
  int iterations, converged;
  double flops_contraction, flops_prrlu;
  long long pivot_steps;
  int nlog, caplog;
  logent_t *log;
  /* canonicalisation J sets, for parity (R22) */
  int *canon_Jn;
  unsigned char **canon_J;
  int *canon_cols_log_n;
  int **canon_cols_log;
  int pivoting;     /* 0 full, 1 rook (R23): every prrLU of the run */
} aci_t;

static void log_push(aci_t *S, int b, int dir, int rl, int rr, const ldu_t *f, double scale) {
  if (S->nlog == S->caplog) {
    S->caplog = S->caplog ? 2 * S->caplog : 256;
    S->log = (logent_t *)realloc(S->log, sizeof(logent_t) * S->caplog);
  }
  logent_t *e = &S->log[S->nlog++];
  e->b = b; e->dir = dir; e->rl = rl; e->rr = rr; e->r = f->r; e->eps = f->eps; e->scale = scale;
  e->rows = (int *)malloc(sizeof(int) * f->r);
  e->cols = (int *)malloc(sizeof(int) * f->r);
  memcpy(e->rows, f->rows, sizeof(int) * f->r);
  memcpy(e->cols, f->cols, sizeof(int) * f->r);
}

/* Alg. 5 Leftframe: L'_{i sigma, beta} = L_{i,gamma} X^sigma_{gamma,beta}; keep rows I. */
static double *leftframe(int rl, int chiL, int d, int chiR, const double *Lprev, const double *X,
                         int r, const int *rows) {
  double *full = (double *)malloc(sizeof(double) * (size_t)rl * d * chiR);
  /* Lprev (rl x chiL) * X (chiL x d*chiR) -> rl x (d*chiR) = (rl*d) x chiR row-major */
  matmul(rl, d * chiR, chiL, Lprev, X, full);
  double *out = (double *)malloc(sizeof(double) * (size_t)r * chiR);
  for (int k = 0; k < r; ++k)
    memcpy(out + (size_t)k * chiR, full + (size_t)rows[k] * chiR, sizeof(double) * chiR);
  free(full);
  return out;
}

/* Alg. 5 Rightframe: R'_{alpha, sigma j} = X^sigma_{alpha,gamma} R_{gamma,j}; keep columns J. */
static double *rightframe(int chiL, int d, int chiR, int rr, const double *X, const double *Rnext,
                          int r, const int *cols) {
  double *full = (double *)malloc(sizeof(double) * (size_t)chiL * d * rr);
  /* X viewed (chiL*d) x chiR times Rnext (chiR x rr) -> (chiL*d) x rr = chiL x (d*rr) */
  matmul(chiL * d, rr, chiR, X, Rnext, full);
  double *out = (double *)malloc(sizeof(double) * (size_t)chiL * r);
  for (int a = 0; a < chiL; ++a)
    for (int k = 0; k < r; ++k) out[(size_t)a * r + k] = full[(size_t)a * d * rr + cols[k]];
  free(full);
  return out;
}

/* Eq. pifromframes (Alg. 1): Pi^n = L^n_{b-1} X^n_b X^n_{b+1} R^n_{b+2},
 * evaluated as A = L X_b, B = X_{b+1} R, Pi^n = A B (the association of Appendix A item 1).
 * Then Pi = f(Pi^1..Pi^N) entrywise. Also returns A^n, B^n (caller frees). */
static double *assemble_pi(aci_t *S, int b, int rl, int rr, double **A, double **B, double *flops) {
  int L = S->L;
  (void)L;
  int db = S->d[b], db1 = S->d[b + 1];
  int m = rl * db, n = db1 * rr;
  double **P = (double **)malloc(sizeof(double *) * S->N);
  for (int nn = 0; nn < S->N; ++nn) {
    int c0 = S->xr[nn * (S->L + 1) + b], c1 = S->xr[nn * (S->L + 1) + b + 1], c2 = S->xr[nn * (S->L + 1) + b + 2];
    const double *Lp = b == 0 ? NULL : S->Lf[nn][b - 1];
    const double *Rn = (b + 2 == S->L) ? NULL : S->Rf[nn][b + 2];
    double one = 1.0;
    A[nn] = (double *)malloc(sizeof(double) * (size_t)rl * db * c1);
    matmul(rl, db * c1, c0, Lp ? Lp : &one, S->X[nn][b], A[nn]);
    B[nn] = (double *)malloc(sizeof(double) * (size_t)c1 * db1 * rr);
    matmul(c1 * db1, rr, c2, S->X[nn][b + 1], Rn ? Rn : &one, B[nn]);
    P[nn] = (double *)malloc(sizeof(double) * (size_t)m * n);
    /* A viewed (rl*db) x c1, B viewed c1 x (db1*rr) */
    matmul(m, n, c1, A[nn], B[nn], P[nn]);
    *flops += 2.0 * rl * c0 * db * c1 + 2.0 * c1 * db1 * c2 * rr + 2.0 * m * c1 * n;
  }
  double *Pi = (double *)malloc(sizeof(double) * (size_t)m * n);
  double *x = (double *)malloc(sizeof(double) * S->N);
  for (size_t t = 0; t < (size_t)m * n; ++t) {
    for (int nn = 0; nn < S->N; ++nn) x[nn] = P[nn][t];
    Pi[t] = apply_f(&S->op, x);
  }
  for (int nn = 0; nn < S->N; ++nn) free(P[nn]);
  free(P); free(x);
  return Pi;
}

/* Index-set update for bond b from the pivots (R21):
 * I_b[k] = (I_{b-1}[row/d_b], row % d_b) ; J_{b+1}[k] = (col / rr, J_{b+2}[col % rr]). */
static void update_index_sets(aci_t *S, int b, int rl, int rr, const ldu_t *f) {
  int L = S->L, db = S->d[b];
  (void)rl;
  unsigned char *In = (unsigned char *)malloc((size_t)f->r * (b + 1));
  unsigned char *Jn = (unsigned char *)malloc((size_t)f->r * (L - b - 1));
  for (int k = 0; k < f->r; ++k) {
    int a = f->rows[k] / db, sg = f->rows[k] % db;
    if (b > 0) memcpy(In + (size_t)k * (b + 1), S->I[b - 1] + (size_t)a * b, b);
    In[(size_t)k * (b + 1) + b] = (unsigned char)sg;
    int sp = f->cols[k] / rr, j = f->cols[k] % rr;
    Jn[(size_t)k * (L - b - 1)] = (unsigned char)sp;
    if (b + 2 < L) memcpy(Jn + (size_t)k * (L - b - 1) + 1, S->J[b + 2] + (size_t)j * (L - b - 2), L - b - 2);
  }
  free(S->I[b]); free(S->J[b + 1]);
  S->I[b] = In; S->J[b + 1] = Jn;
  S->chi[b] = f->r;
  S->Jn[b + 1] = f->r;
}

static void aci_free(aci_t *S) {
  if (!S) return;
  for (int nn = 0; nn < S->N; ++nn) {
    for (int s = 0; s <= S->L; ++s) { if (S->Lf[nn][s]) free(S->Lf[nn][s]); if (S->Rf[nn][s]) free(S->Rf[nn][s]); }
    free(S->Lf[nn]); free(S->Rf[nn]);
    for (int s = 0; s < S->L; ++s) free(S->X[nn][s]);
    free(S->X[nn]);
  }
  free(S->Lf); free(S->Rf); free(S->X);
  for (int s = 0; s <= S->L; ++s) { free(S->I[s]); free(S->J[s]); }
  free(S->I); free(S->J);
  for (int s = 0; s < S->L; ++s) if (S->Y) free(S->Y[s]);
  free(S->Y); free(S->yr);
  for (int i = 0; i < S->nlog; ++i) { free(S->log[i].rows); free(S->log[i].cols); }
  free(S->log);
  for (int s = 0; s <= S->L; ++s) { if (S->canon_J) free(S->canon_J[s]); if (S->canon_cols_log) free(S->canon_cols_log[s]); }
  free(S->canon_J); free(S->canon_Jn); free(S->canon_cols_log); free(S->canon_cols_log_n);
  free(S->chi); free(S->Jn); free(S->d); free(S->xr);
  free((void *)S->op.coef); free((void *)S->op.expo);
  free(S);
}

void oracle_free(void *h) { aci_free((aci_t *)h); }

/* ------------------------------------------------------------------ */
/* Alg. 1 — AlternatingCrossInterpolation                 */
/* ------------------------------------------------------------------ */
/*
 * inputs: N distinct TTs (aliases already merged into the exponents),
 * xranks: N x (L+1), xcores: N*L pointers (row-major cores),
 * op: T terms with coef[T], expo[T x N],
 * y_init: ranks yr0[L+1] and cores (R9: the initial guess is an input),
 * tol, tol_mode (0 relative (R1), 1 absolute), maxrank, maxiter.
 * Returns a handle (NULL on allocation failure); *status receives the code.
 */
void *oracle_aci_p(int L, const int *d, int N, const int *xranks, const double *const *xcores,
                   int T, const double *coef, const int *expo, const int *yr0, const double *const *ycores,
                   double tol, int tol_mode, int maxrank, int maxiter, int pivoting, int *status) {
  *status = ORC_OK;
  if (L < 2 || N < 1 || T < 1 || maxrank < 1 || maxiter < 1 || tol < 0 || pivoting < 0 || pivoting > 1) {
    *status = ORC_ERR_INVALID;
    return NULL;
  }
  aci_t *S = (aci_t *)calloc(1, sizeof(aci_t));
  S->L = L; S->N = N;
  S->pivoting = pivoting;
  S->d = (int *)malloc(sizeof(int) * L); memcpy(S->d, d, sizeof(int) * L);
  S->xr = (int *)malloc(sizeof(int) * N * (L + 1)); memcpy(S->xr, xranks, sizeof(int) * N * (L + 1));
  double *cf = (double *)malloc(sizeof(double) * T); memcpy(cf, coef, sizeof(double) * T);
  int *ex = (int *)malloc(sizeof(int) * T * N); memcpy(ex, expo, sizeof(int) * T * N);
  S->op.N = N; S->op.T = T; S->op.coef = cf; S->op.expo = ex;
  S->X = (double ***)malloc(sizeof(double **) * N);
  S->Lf = (double ***)malloc(sizeof(double **) * N);
  S->Rf = (double ***)malloc(sizeof(double **) * N);
  for (int nn = 0; nn < N; ++nn) {
    S->X[nn] = (double **)malloc(sizeof(double *) * L);
    double **Xn = S->X[nn];
    for (int s = 0; s < L; ++s) {
      size_t sz = (size_t)xranks[nn * (L + 1) + s] * d[s] * xranks[nn * (L + 1) + s + 1];
      Xn[s] = (double *)malloc(sizeof(double) * sz);
      memcpy(Xn[s], xcores[nn * L + s], sizeof(double) * sz);
    }
    S->Lf[nn] = (double **)calloc(L + 1, sizeof(double *));
    S->Rf[nn] = (double **)calloc(L + 1, sizeof(double *));
  }
  S->I = (unsigned char **)calloc(L + 1, sizeof(unsigned char *));
  S->J = (unsigned char **)calloc(L + 1, sizeof(unsigned char *));
  S->chi = (int *)calloc(L, sizeof(int));
  S->Jn = (int *)calloc(L + 1, sizeof(int));
  S->Jn[L] = 1;
  S->canon_J = (unsigned char **)calloc(L + 1, sizeof(unsigned char *));
  S->canon_Jn = (int *)calloc(L + 1, sizeof(int));
  S->canon_cols_log = (int **)calloc(L + 1, sizeof(int *));
  S->canon_cols_log_n = (int *)calloc(L + 1, sizeof(int));

  /* ---- CI-canonicalise y_init; J_L..J_2 (0-based: J[L-1]..J[1]); R^n_s ---- */
  double **Y = (double **)malloc(sizeof(double *) * L);
  int *yr = (int *)malloc(sizeof(int) * (L + 1));
  memcpy(yr, yr0, sizeof(int) * (L + 1));
  for (int s = 0; s < L; ++s) {
    size_t sz = (size_t)yr[s] * d[s] * yr[s + 1];
    Y[s] = (double *)malloc(sizeof(double) * sz);
    memcpy(Y[s], ycores[s], sizeof(double) * sz);
  }
  for (int s = L - 1; s >= 1; --s) {
    int rows_ = yr[s], jn = S->Jn[s + 1];
    int cols_ = d[s] * jn; /* M_{alpha, sigma j}; Y[s] already has right bond |J_{s+1}| */
    ldu_t f;
    /* R8: tolerance relative to M's own max (or absolute in absolute mode).
     * R9': |J_s| never exceeds the full-tensor bond bound prod_{t<s} d_t (a no-op for a
     * minimal y_init, which is what the generators produce). */
    int cap = maxrank;
    {
      long long pl = 1;
      for (int t = 0; t < s && pl < cap; ++t) pl *= d[t];
      if (pl < cap) cap = (int)pl;
    }
    int st = ldu_p(rows_, cols_, Y[s], tol, tol_mode == 0 ? 1 : 0, cap, S->pivoting, &f);
    if (st != ORC_OK) { *status = st; aci_free(S); return NULL; }
    /* J_s[k] = (sigma, J_{s+1}[j]) */
    unsigned char *Js = (unsigned char *)malloc((size_t)f.r * (L - s));
    for (int k = 0; k < f.r; ++k) {
      int sg = f.cols[k] / jn, j = f.cols[k] % jn;
      Js[(size_t)k * (L - s)] = (unsigned char)sg;
      if (s + 1 < L) memcpy(Js + (size_t)k * (L - s) + 1, S->J[s + 1] + (size_t)j * (L - s - 1), L - s - 1);
    }
    S->J[s] = Js; S->Jn[s] = f.r;
    S->canon_J[s] = (unsigned char *)malloc((size_t)f.r * (L - s));
    memcpy(S->canon_J[s], Js, (size_t)f.r * (L - s));
    S->canon_Jn[s] = f.r;
    S->canon_cols_log[s] = (int *)malloc(sizeof(int) * f.r);
    memcpy(S->canon_cols_log[s], f.cols, sizeof(int) * f.r);
    S->canon_cols_log_n[s] = f.r;
    /* M' = M[:, J] (rows_ x r); Y_{s-1} <- Y_{s-1} M' */
    double *Mp = (double *)malloc(sizeof(double) * (size_t)rows_ * f.r);
    for (int a = 0; a < rows_; ++a)
      for (int k = 0; k < f.r; ++k) Mp[(size_t)a * f.r + k] = Y[s][(size_t)a * cols_ + f.cols[k]];
    double *Ynew = (double *)malloc(sizeof(double) * (size_t)yr[s - 1] * d[s - 1] * f.r);
    matmul(yr[s - 1] * d[s - 1], f.r, rows_, Y[s - 1], Mp, Ynew);
    free(Y[s - 1]); Y[s - 1] = Ynew;
    free(Mp);
    /* R^n_s = Rightframe(X^n_s, R^n_{s+1}, J_s) */
    for (int nn = 0; nn < N; ++nn) {
      int c0 = xranks[nn * (L + 1) + s], c1 = xranks[nn * (L + 1) + s + 1];
      double one = 1.0;
      const double *Rn = (s + 1 == L) ? &one : S->Rf[nn][s + 1];
      S->Rf[nn][s] = rightframe(c0, d[s], c1, jn, S->X[nn][s], Rn, f.r, f.cols);
    }
    ldu_free(&f);
  }
  for (int s = 0; s < L; ++s) free(Y[s]);
  free(Y); free(yr);
  int *prev = (int *)malloc(sizeof(int) * L);
  for (int b = 0; b < L - 1; ++b) prev[b] = S->Jn[b + 1];

  /* ---- main loop ---- */
  S->yr = (int *)calloc(L + 1, sizeof(int));
  S->Y = (double **)calloc(L, sizeof(double *));
  double scale = 0.0;
  int it;
  for (it = 1; it <= maxiter; ++it) {
    double maxeps = 0.0;
    for (int dir = 0; dir < 2; ++dir) {
      for (int step = 0; step < L - 1; ++step) {
        int b = dir == 0 ? step : L - 2 - step;
        int rl = b == 0 ? 1 : S->chi[b - 1];
        int rr = (b + 2 == L) ? 1 : S->Jn[b + 2];
        int m = rl * d[b], n = d[b + 1] * rr;
        double **A = (double **)malloc(sizeof(double *) * N), **B = (double **)malloc(sizeof(double *) * N);
        double *Pi = assemble_pi(S, b, rl, rr, A, B, &S->flops_contraction);
        for (size_t t = 0; t < (size_t)m * n; ++t) {
          if (!isfinite(Pi[t])) { *status = ORC_ERR_NONFINITE; aci_free(S); return NULL; }
          if (fabs(Pi[t]) > scale) scale = fabs(Pi[t]);
        }
        double thr = tol_mode == 0 ? tol * scale : tol;
        ldu_t f;
        ldu_p(m, n, Pi, thr, 0, maxrank, S->pivoting, &f);
        for (int k = 0; k < f.r; ++k) S->flops_prrlu += 2.0 * (m - k - 1) * (n - k - 1);
        S->pivot_steps += f.r;
        if (f.eps > maxeps) maxeps = f.eps;
        log_push(S, b, dir, rl, rr, &f, scale);
        update_index_sets(S, b, rl, rr, &f);
        if (dir == 0) {
          /* L^n_b = Leftframe(X^n_b, L^n_{b-1}, I_b) */
          for (int nn = 0; nn < N; ++nn) {
            int c0 = S->xr[nn * (L + 1) + b], c1 = S->xr[nn * (L + 1) + b + 1];
            double one = 1.0;
            double *nl = leftframe(rl, c0, d[b], c1, b == 0 ? &one : S->Lf[nn][b - 1], S->X[nn][b], f.r, f.rows);
            free(S->Lf[nn][b]); S->Lf[nn][b] = nl;
          }
        } else {
          /* R^n_{b+1} = Rightframe(X^n_{b+1}, R^n_{b+2}, J_{b+1}) */
          for (int nn = 0; nn < N; ++nn) {
            int c1 = S->xr[nn * (L + 1) + b + 1], c2 = S->xr[nn * (L + 1) + b + 2];
            double one = 1.0;
            double *nr = rightframe(c1, d[b + 1], c2, rr, S->X[nn][b + 1], (b + 2 == L) ? &one : S->Rf[nn][b + 2], f.r, f.cols);
            free(S->Rf[nn][b + 1]); S->Rf[nn][b + 1] = nr;
          }
          /* R5: output cores of the right-to-left half-sweep: Y_{b+1} = U_J^{-1} U ; Y_0 = Pi[:, J] */
          free(S->Y[b + 1]);
          S->Y[b + 1] = (double *)malloc(sizeof(double) * (size_t)f.r * n);
          ci_right_B(f.r, n, f.U, f.cols, S->Y[b + 1]);
          S->yr[b + 1] = f.r;
          if (b == 0) {
            free(S->Y[0]);
            S->Y[0] = (double *)malloc(sizeof(double) * (size_t)m * f.r);
            for (int i = 0; i < m; ++i)
              for (int k = 0; k < f.r; ++k) S->Y[0][(size_t)i * f.r + k] = Pi[(size_t)i * n + f.cols[k]];
          }
        }
        ldu_free(&f);
        for (int nn = 0; nn < N; ++nn) { free(A[nn]); free(B[nn]); }
        free(A); free(B); free(Pi);
      }
    }
    /* P:497-499 with R10: converged iff no bond rank increased and max eps <= tau*s */
    int grew = 0;
    for (int b = 0; b < L - 1; ++b) { if (S->chi[b] > prev[b]) grew = 1; prev[b] = S->chi[b]; }
    double thr = tol_mode == 0 ? tol * scale : tol;
    S->err_estimate = scale > 0 ? maxeps / scale : 0.0;
    if (tol_mode == 1) S->err_estimate = maxeps;
    S->iterations = it;
    if (!grew && maxeps <= thr) { S->converged = 1; break; }
  }
  free(prev);
  S->yr[0] = 1; S->yr[L] = 1;
  S->scale = scale;
  return S;
}

void *oracle_aci(int L, const int *d, int N, const int *xranks, const double *const *xcores,
                 int T, const double *coef, const int *expo, const int *yr0, const double *const *ycores,
                 double tol, int tol_mode, int maxrank, int maxiter, int *status) {
  return oracle_aci_p(L, d, N, xranks, xcores, T, coef, expo, yr0, ycores, tol, tol_mode, maxrank, maxiter, 0, status);
}

/* ---- accessors (ctypes) ---- */
void oracle_report(void *h, double *scale, double *err, int *iters, int *conv, double *fc, double *fp, long long *piv) {
  aci_t *S = (aci_t *)h;
  *scale = S->scale; *err = S->err_estimate; *iters = S->iterations; *conv = S->converged;
  *fc = S->flops_contraction; *fp = S->flops_prrlu; *piv = S->pivot_steps;
}
void oracle_out_ranks(void *h, int *ranks) { aci_t *S = (aci_t *)h; memcpy(ranks, S->yr, sizeof(int) * (S->L + 1)); }
void oracle_out_core(void *h, int s, double *dst) {
  aci_t *S = (aci_t *)h;
  size_t sz = (size_t)S->yr[s] * S->d[s] * S->yr[s + 1];
  memcpy(dst, S->Y[s], sizeof(double) * sz);
}
int oracle_log_count(void *h) { return ((aci_t *)h)->nlog; }
void oracle_log_entry(void *h, int u, int *info /* b, dir, rl, rr, r */, double *eps_scale, int *rows, int *cols) {
  logent_t *e = &((aci_t *)h)->log[u];
  info[0] = e->b; info[1] = e->dir; info[2] = e->rl; info[3] = e->rr; info[4] = e->r;
  eps_scale[0] = e->eps; eps_scale[1] = e->scale;
  if (rows) memcpy(rows, e->rows, sizeof(int) * e->r);
  if (cols) memcpy(cols, e->cols, sizeof(int) * e->r);
}
int oracle_chi(void *h, int b) { return ((aci_t *)h)->chi[b]; }
int oracle_jn(void *h, int s) { return ((aci_t *)h)->Jn[s]; }
void oracle_Iset(void *h, int b, unsigned char *dst) { aci_t *S = (aci_t *)h; memcpy(dst, S->I[b], (size_t)S->chi[b] * (b + 1)); }
void oracle_Jset(void *h, int s, unsigned char *dst) { aci_t *S = (aci_t *)h; memcpy(dst, S->J[s], (size_t)S->Jn[s] * (S->L - s)); }
int oracle_canon_jn(void *h, int s) { return ((aci_t *)h)->canon_Jn[s]; }
void oracle_canon_Jset(void *h, int s, unsigned char *dst) { aci_t *S = (aci_t *)h; memcpy(dst, S->canon_J[s], (size_t)S->canon_Jn[s] * (S->L - s)); }
void oracle_canon_cols(void *h, int s, int *dst) { aci_t *S = (aci_t *)h; memcpy(dst, S->canon_cols_log[s], sizeof(int) * S->canon_cols_log_n[s]); }
/* frames: L^n_b is chi[b] x xr[n][b+1]; R^n_s is xr[n][s] x Jn[s] */
void oracle_Lframe(void *h, int n, int b, double *dst) {
  aci_t *S = (aci_t *)h;
  memcpy(dst, S->Lf[n][b], sizeof(double) * (size_t)S->chi[b] * S->xr[n * (S->L + 1) + b + 1]);
}
void oracle_Rframe(void *h, int n, int s, double *dst) {
  aci_t *S = (aci_t *)h;
  memcpy(dst, S->Rf[n][s], sizeof(double) * (size_t)S->xr[n * (S->L + 1) + s] * S->Jn[s]);
}

/* Exported for the Pi pin: Eq. pifromframes + f for explicit frames. Lp: N pointers (rl x c0,
 * NULL = [1]); Rn: N pointers (c2 x rr, NULL = [1]); X0, X1: N pointers to cores of sites b, b+1. */
int oracle_assemble_pi(int N, const int *c /* N x 3: c0, c1, c2 */, int db, int db1, int rl, int rr,
                       const double *const *Lp, const double *const *X0, const double *const *X1,
                       const double *const *Rn, int T, const double *coef, const int *expo, double *Pi) {
  int m = rl * db, n = db1 * rr;
  op_t op = {N, T, coef, expo};
  double **P = (double **)malloc(sizeof(double *) * N);
  for (int nn = 0; nn < N; ++nn) {
    int c0 = c[3 * nn], c1 = c[3 * nn + 1], c2 = c[3 * nn + 2];
    double one = 1.0;
    double *A = (double *)malloc(sizeof(double) * (size_t)rl * db * c1);
    double *B = (double *)malloc(sizeof(double) * (size_t)c1 * db1 * rr);
    matmul(rl, db * c1, c0, Lp[nn] ? Lp[nn] : &one, X0[nn], A);
    matmul(c1 * db1, rr, c2, X1[nn], Rn[nn] ? Rn[nn] : &one, B);
    P[nn] = (double *)malloc(sizeof(double) * (size_t)m * n);
    matmul(m, n, c1, A, B, P[nn]);
    free(A); free(B);
  }
  double *x = (double *)malloc(sizeof(double) * N);
  for (size_t t = 0; t < (size_t)m * n; ++t) {
    for (int nn = 0; nn < N; ++nn) x[nn] = P[nn][t];
    Pi[t] = apply_f(&op, x);
  }
  for (int nn = 0; nn < N; ++nn) free(P[nn]);
  free(P); free(x);
  return ORC_OK;
}
