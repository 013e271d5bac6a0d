/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Complex-valued ACI (f: C^N -> C; the random Fourier series of P:289-296 have complex
 * coefficients): Alg. 1-5 as naive loops, the same steps and readings as
 * aci_oracle.c (R1-R22) with the complex-arithmetic readings RZ1-RZ6 of
 * DESIGN.md §2 (the paper does not spell complex arithmetic out):
 *   RZ1  pivot magnitude (P:529 argmax |M_ij|): w = fl(fl(re*re) + fl(im*im)); argmax w, ties to
 *        the smallest (row, col) (R3); |c| = sqrt(w) (correctly rounded) for the threshold,
 *        epsilon and the scale s (R1, R2).
 *   RZ2  inverse pivot (P:535 [M_{chi,chi}]^{-1}): inv = (c_re / w, (-c_im) / w).
 *   RZ3  product z*y: (fl(fl(z_re y_re) - fl(z_im y_im)), fl(fl(z_re y_im) + fl(z_im y_re))).
 *        Used for l_i = S_iq * inv and U_k[j] = S_pj * inv.
 *   RZ4  Schur update S_ij <- S_ij - l_i u_j:
 *        re = fma(l_im, u_im, fma(-l_re, u_re, S_re)), im = fma(-l_im, u_re, fma(-l_re, u_im, S_im)).
 *   RZ5  contractions and f: plain loops with RZ3 products, real and imaginary parts summed
 *        separately (roundoff-level only; parity is on pivots and tolerances).
 *   RZ6  f has real coefficients: f = sum_t coef_t prod_n x_n^{e_tn}.
 * Complex arrays are interleaved (re, im) doubles (numpy complex128 layout).
 * Only tests/, __graft_entry__.smoke() and bench.py may load this library; it shares no code with
 * the CUDA path.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_INVALID -1
#define ORC_ERR_NONFINITE -3
#define ORC_ERR_OOM -4

typedef struct { double re, im; } cz;

static cz cz_mul(cz a, cz b) { /* RZ3 */
  cz r;
  double t1 = a.re * b.re, t2 = a.im * b.im, t3 = a.re * b.im, t4 = a.im * b.re;
  r.re = t1 - t2;
  r.im = t3 + t4;
  return r;
}
static double cz_w(cz a) { /* RZ1 */
  double x = a.re * a.re, y = a.im * a.im;
  return x + y;
}

/* C (M x N) = A (M x K) * B (K x N), complex row-major, plain triple loop (RZ5). */
static void zmatmul(int M, int N, int K, const cz *A, const cz *B, cz *C) {
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double ar = 0.0, ai = 0.0;
      for (int k = 0; k < K; ++k) {
        cz p = cz_mul(A[(size_t)i * K + k], B[(size_t)k * N + j]);
        ar += p.re;
        ai += p.im;
      }
      C[(size_t)i * N + j].re = ar;
      C[(size_t)i * N + j].im = ai;
    }
}

/* ---------------- Alg. 2, complex, readings R2-R4/R17 + RZ1-RZ4 ---------------- */
typedef struct {
  int r;
  int *rows, *cols;
  cz *D;
  cz *U;       /* r x n, U_k = S_k[p,:] * inv, U_k[q] = 1 */
  double eps;  /* |c| of the first rejected candidate (R2) */
  double first;
  double *gap; /* per accepted pivot: (w1 - w2) / w1, w1 >= w2 the two largest candidate |z|^2
                * (diagnostic for ties within roundoff; 1 if there is a single candidate) */
} zldu_t;

static void zldu_free(zldu_t *f) {
  free(f->rows); free(f->cols); free(f->D); free(f->U); free(f->gap);
  memset(f, 0, sizeof(*f));
}

static int zldu(int m, int n, const cz *M, double thr, int thr_mode, int maxrank, zldu_t *out) {
  memset(out, 0, sizeof(*out));
  for (size_t t = 0; t < (size_t)m * n; ++t)
    if (!isfinite(M[t].re) || !isfinite(M[t].im)) return ORC_ERR_NONFINITE;
  cz *S = (cz *)malloc(sizeof(cz) * (size_t)m * n);
  char *rowdone = (char *)calloc(m, 1), *coldone = (char *)calloc(n, 1);
  int kcap = m < n ? m : n;
  if (maxrank < kcap) kcap = maxrank;
  out->rows = (int *)malloc(sizeof(int) * (kcap + 1));
  out->cols = (int *)malloc(sizeof(int) * (kcap + 1));
  out->D = (cz *)malloc(sizeof(cz) * (kcap + 1));
  out->U = (cz *)calloc((size_t)(kcap + 1) * n, sizeof(cz));
  out->gap = (double *)calloc(kcap + 1, sizeof(double));
  if (!S || !rowdone || !coldone || !out->rows || !out->U || !out->gap) return ORC_ERR_OOM;
  memcpy(S, M, sizeof(cz) * (size_t)m * n);
  int mn = m < n ? m : n;
  int k = 0;
  for (;;) {
    if (k == mn) { out->eps = 0.0; break; }
    int p = -1, q = -1;
    double best = -1.0, second = -1.0;
    for (int i = 0; i < m; ++i) {
      if (rowdone[i]) continue;
      for (int j = 0; j < n; ++j) {
        if (coldone[j]) continue;
        double w = cz_w(S[(size_t)i * n + j]);
        if (w > best) { second = best; best = w; p = i; q = j; } /* strict '>': smallest (row, col) (R3) */
        else if (w > second) second = w;
      }
    }
    out->gap[k] = (best > 0 && second >= 0) ? (best - second) / best : 1.0;
    cz c = S[(size_t)p * n + q];
    double w = cz_w(c);
    double absc = sqrt(w);
    if (k == 0) out->first = absc;
    double t = thr_mode == 1 ? thr * out->first : thr;
    if (k == maxrank) { out->eps = absc; break; }
    if (k > 0 && absc <= t) { out->eps = absc; break; }
    out->rows[k] = p; out->cols[k] = q; out->D[k] = c;
    if (k == 0 && w == 0.0) { /* R17 */
      out->U[q].re = 1.0; out->U[q].im = 0.0;
      out->eps = 0.0;
      k = 1;
      break;
    }
    cz inv; /* RZ2 */
    inv.re = c.re / w;
    inv.im = (-c.im) / w;
    for (int j = 0; j < n; ++j) {
      cz z = {0.0, 0.0};
      if (!coldone[j]) z = cz_mul(S[(size_t)p * n + j], inv);
      out->U[(size_t)k * n + j] = z;
    }
    out->U[(size_t)k * n + q].re = 1.0; out->U[(size_t)k * n + q].im = 0.0;
    for (int i = 0; i < m; ++i) {
      if (rowdone[i] || i == p) continue;
      cz l = cz_mul(S[(size_t)i * n + q], inv);
      for (int j = 0; j < n; ++j) {
        if (coldone[j] || j == q) continue;
        cz u = S[(size_t)p * n + j];
        cz *s = &S[(size_t)i * n + j];
        double tr = fma(-l.re, u.re, s->re); /* RZ4 */
        double ti = fma(-l.re, u.im, s->im);
        s->re = fma(l.im, u.im, tr);
        s->im = fma(-l.im, u.re, ti);
      }
    }
    rowdone[p] = 1; coldone[q] = 1;
    ++k;
  }
  out->r = k;
  free(S); free(rowdone); free(coldone);
  return ORC_OK;
}

int oraclez_ldu(int m, int n, const double *M, double thr, int thr_mode, int maxrank, int *r, int *rows, int *cols,
                double *D, double *U /* maxr x n complex */, int maxr, double *eps) {
  if (m < 1 || n < 1 || maxrank < 1 || thr < 0) return ORC_ERR_INVALID;
  zldu_t f;
  int st = zldu(m, n, (const cz *)M, thr, thr_mode, maxrank, &f);
  if (st != ORC_OK) return st;
  *r = f.r;
  *eps = f.eps;
  for (int k = 0; k < f.r && k < maxr; ++k) {
    rows[k] = f.rows[k]; cols[k] = f.cols[k];
    D[2 * k] = f.D[k].re; D[2 * k + 1] = f.D[k].im;
    if (U) memcpy(U + (size_t)2 * k * n, f.U + (size_t)k * n, sizeof(cz) * n);
  }
  zldu_free(&f);
  return ORC_OK;
}

/* Alg. 3 right branch (R6): B = U_J^{-1} U (unit upper triangular back substitution). */
static void zci_right_B(int r, int n, const cz *U, const int *cols, cz *B) {
  for (int k = r - 1; k >= 0; --k)
    for (int j = 0; j < n; ++j) {
      double ar = U[(size_t)k * n + j].re, ai = U[(size_t)k * n + j].im;
      for (int i = k + 1; i < r; ++i) {
        cz p = cz_mul(U[(size_t)k * n + cols[i]], B[(size_t)i * n + j]);
        ar -= p.re;
        ai -= p.im;
      }
      B[(size_t)k * n + j].re = ar;
      B[(size_t)k * n + j].im = ai;
    }
}

/* ---------------- f (RZ6) ---------------- */
typedef struct {
  int N, T;
  const double *coef;
  const int *expo;
} zop_t;

static cz apply_fz(const zop_t *op, const cz *x) {
  cz y = {0.0, 0.0};
  for (int t = 0; t < op->T; ++t) {
    cz p = {op->coef[t], 0.0};
    for (int n = 0; n < op->N; ++n)
      for (int e = 0; e < op->expo[t * op->N + n]; ++e) p = cz_mul(p, x[n]);
    y.re += p.re;
    y.im += p.im;
  }
  return y;
}

/* ---------------- ACI state (as aci_oracle.c) ---------------- */
typedef struct {
  int b, dir, rl, rr, r;
  double eps, scale;
  int *rows, *cols;
  double *gap;
} zlogent_t;

typedef struct {
  int L, N;
  int *d, *xr;
  cz ***X;
  zop_t op;
  unsigned char **I, **J;
  int *chi, *Jn;
  cz ***Lf, ***Rf;
  int *yr;
  cz **Y;
  double scale, err_estimate;
  int iterations, converged;
  double flops_contraction, flops_prrlu;
  long long pivot_steps;
  int nlog, caplog;
  zlogent_t *log;
  int *canon_Jn;
  int **canon_cols_log;
} zaci_t;

static void zlog_push(zaci_t *S, int b, int dir, int rl, int rr, const zldu_t *f, double scale) {
  if (S->nlog == S->caplog) {
    S->caplog = S->caplog ? 2 * S->caplog : 256;
    S->log = (zlogent_t *)realloc(S->log, sizeof(zlogent_t) * S->caplog);
  }
  zlogent_t *e = &S->log[S->nlog++];
  e->b = b; e->dir = dir; e->rl = rl; e->rr = rr; e->r = f->r; e->eps = f->eps; e->scale = scale;
  e->rows = (int *)malloc(sizeof(int) * f->r);
  e->cols = (int *)malloc(sizeof(int) * f->r);
  memcpy(e->rows, f->rows, sizeof(int) * f->r);
  memcpy(e->cols, f->cols, sizeof(int) * f->r);
  e->gap = (double *)malloc(sizeof(double) * f->r);
  memcpy(e->gap, f->gap, sizeof(double) * f->r);
}

/* Alg. 5 Leftframe */
static cz *zleftframe(int rl, int chiL, int d, int chiR, const cz *Lprev, const cz *X, int r, const int *rows) {
  cz *full = (cz *)malloc(sizeof(cz) * (size_t)rl * d * chiR);
  zmatmul(rl, d * chiR, chiL, Lprev, X, full);
  cz *out = (cz *)malloc(sizeof(cz) * (size_t)r * chiR);
  for (int k = 0; k < r; ++k) memcpy(out + (size_t)k * chiR, full + (size_t)rows[k] * chiR, sizeof(cz) * chiR);
  free(full);
  return out;
}

/* Alg. 5 Rightframe */
static cz *zrightframe(int chiL, int d, int chiR, int rr, const cz *X, const cz *Rnext, int r, const int *cols) {
  cz *full = (cz *)malloc(sizeof(cz) * (size_t)chiL * d * rr);
  zmatmul(chiL * d, rr, chiR, X, Rnext, full);
  cz *out = (cz *)malloc(sizeof(cz) * (size_t)chiL * r);
  for (int a = 0; a < chiL; ++a)
    for (int k = 0; k < r; ++k) out[(size_t)a * r + k] = full[(size_t)a * d * rr + cols[k]];
  free(full);
  return out;
}

/* Eq. pifromframes then f */
static cz *zassemble_pi(zaci_t *S, int b, int rl, int rr, double *flops) {
  int db = S->d[b], db1 = S->d[b + 1];
  int m = rl * db, n = db1 * rr;
  cz **P = (cz **)malloc(sizeof(cz *) * S->N);
  const cz one = {1.0, 0.0};
  for (int nn = 0; nn < S->N; ++nn) {
    int c0 = S->xr[nn * (S->L + 1) + b], c1 = S->xr[nn * (S->L + 1) + b + 1], c2 = S->xr[nn * (S->L + 1) + b + 2];
    const cz *Lp = b == 0 ? &one : S->Lf[nn][b - 1];
    const cz *Rn = (b + 2 == S->L) ? &one : S->Rf[nn][b + 2];
    cz *A = (cz *)malloc(sizeof(cz) * (size_t)rl * db * c1);
    cz *B = (cz *)malloc(sizeof(cz) * (size_t)c1 * db1 * rr);
    zmatmul(rl, db * c1, c0, Lp, S->X[nn][b], A);
    zmatmul(c1 * db1, rr, c2, S->X[nn][b + 1], Rn, B);
    P[nn] = (cz *)malloc(sizeof(cz) * (size_t)m * n);
    zmatmul(m, n, c1, A, B, P[nn]);
    free(A); free(B);
    /* real flops of the complex contraction model: 4x the real count (4 real products per
     * complex product) */
    *flops += 4.0 * (2.0 * rl * c0 * db * c1 + 2.0 * c1 * db1 * c2 * rr + 2.0 * m * c1 * n);
  }
  cz *Pi = (cz *)malloc(sizeof(cz) * (size_t)m * n);
  cz *x = (cz *)malloc(sizeof(cz) * S->N);
  for (size_t t = 0; t < (size_t)m * n; ++t) {
    for (int nn = 0; nn < S->N; ++nn) x[nn] = P[nn][t];
    Pi[t] = apply_fz(&S->op, x);
  }
  for (int nn = 0; nn < S->N; ++nn) free(P[nn]);
  free(P); free(x);
  return Pi;
}

static void zupdate_index_sets(zaci_t *S, int b, int rr, const zldu_t *f) {
  int L = S->L, db = S->d[b];
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

static void zaci_free(zaci_t *S) {
  if (!S) return;
  for (int nn = 0; nn < S->N; ++nn) {
    for (int s = 0; s <= S->L; ++s) { free(S->Lf[nn][s]); free(S->Rf[nn][s]); }
    free(S->Lf[nn]); free(S->Rf[nn]);
    for (int s = 0; s < S->L; ++s) free(S->X[nn][s]);
    free(S->X[nn]);
  }
  free(S->Lf); free(S->Rf); free(S->X);
  for (int s = 0; s <= S->L; ++s) { free(S->I[s]); free(S->J[s]); }
  free(S->I); free(S->J);
  for (int s = 0; s < S->L; ++s) if (S->Y) free(S->Y[s]);
  free(S->Y); free(S->yr);
  for (int i = 0; i < S->nlog; ++i) { free(S->log[i].rows); free(S->log[i].cols); free(S->log[i].gap); }
  free(S->log);
  for (int s = 0; s <= S->L; ++s) if (S->canon_cols_log) free(S->canon_cols_log[s]);
  free(S->canon_cols_log); free(S->canon_Jn);
  free(S->chi); free(S->Jn); free(S->d); free(S->xr);
  free((void *)S->op.coef); free((void *)S->op.expo);
  free(S);
}

void oraclez_free(void *h) { zaci_free((zaci_t *)h); }

/* Alg. 1, complex; arguments as oracle_aci (cores interleaved complex). */
void *oraclez_aci(int L, const int *d, int N, const int *xranks, const double *const *xcores, int T,
                  const double *coef, const int *expo, const int *yr0, const double *const *ycores, double tol,
                  int tol_mode, int maxrank, int maxiter, int *status) {
  *status = ORC_OK;
  if (L < 2 || N < 1 || T < 1 || maxrank < 1 || maxiter < 1 || tol < 0) { *status = ORC_ERR_INVALID; return NULL; }
  zaci_t *S = (zaci_t *)calloc(1, sizeof(zaci_t));
  S->L = L; S->N = N;
  S->d = (int *)malloc(sizeof(int) * L); memcpy(S->d, d, sizeof(int) * L);
  S->xr = (int *)malloc(sizeof(int) * N * (L + 1)); memcpy(S->xr, xranks, sizeof(int) * N * (L + 1));
  double *cf = (double *)malloc(sizeof(double) * T); memcpy(cf, coef, sizeof(double) * T);
  int *ex = (int *)malloc(sizeof(int) * T * N); memcpy(ex, expo, sizeof(int) * T * N);
  S->op.N = N; S->op.T = T; S->op.coef = cf; S->op.expo = ex;
  S->X = (cz ***)malloc(sizeof(cz **) * N);
  S->Lf = (cz ***)malloc(sizeof(cz **) * N);
  S->Rf = (cz ***)malloc(sizeof(cz **) * N);
  for (int nn = 0; nn < N; ++nn) {
    S->X[nn] = (cz **)malloc(sizeof(cz *) * L);
    for (int s = 0; s < L; ++s) {
      size_t sz = (size_t)xranks[nn * (L + 1) + s] * d[s] * xranks[nn * (L + 1) + s + 1];
      S->X[nn][s] = (cz *)malloc(sizeof(cz) * sz);
      memcpy(S->X[nn][s], xcores[nn * L + s], sizeof(cz) * sz);
    }
    S->Lf[nn] = (cz **)calloc(L + 1, sizeof(cz *));
    S->Rf[nn] = (cz **)calloc(L + 1, sizeof(cz *));
  }
  S->I = (unsigned char **)calloc(L + 1, sizeof(unsigned char *));
  S->J = (unsigned char **)calloc(L + 1, sizeof(unsigned char *));
  S->chi = (int *)calloc(L, sizeof(int));
  S->Jn = (int *)calloc(L + 1, sizeof(int));
  S->Jn[L] = 1;
  S->canon_Jn = (int *)calloc(L + 1, sizeof(int));
  S->canon_cols_log = (int **)calloc(L + 1, sizeof(int *));
  const cz one = {1.0, 0.0};

  /* ---- CI-canonicalise y_init (R8, R9') ---- */
  cz **Y = (cz **)malloc(sizeof(cz *) * L);
  int *yr = (int *)malloc(sizeof(int) * (L + 1));
  memcpy(yr, yr0, sizeof(int) * (L + 1));
  for (int s = 0; s < L; ++s) {
    size_t sz = (size_t)yr[s] * d[s] * yr[s + 1];
    Y[s] = (cz *)malloc(sizeof(cz) * sz);
    memcpy(Y[s], ycores[s], sizeof(cz) * sz);
  }
  for (int s = L - 1; s >= 1; --s) {
    int rows_ = yr[s], jn = S->Jn[s + 1];
    int cols_ = d[s] * jn;
    int cap = maxrank;
    {
      long long pl = 1;
      for (int t = 0; t < s && pl < cap; ++t) pl *= d[t];
      if (pl < cap) cap = (int)pl;
    }
    zldu_t f;
    int st = zldu(rows_, cols_, Y[s], tol, tol_mode == 0 ? 1 : 0, cap, &f);
    if (st != ORC_OK) { *status = st; zaci_free(S); return NULL; }
    unsigned char *Js = (unsigned char *)malloc((size_t)f.r * (L - s));
    for (int k = 0; k < f.r; ++k) {
      int sg = f.cols[k] / jn, j = f.cols[k] % jn;
      Js[(size_t)k * (L - s)] = (unsigned char)sg;
      if (s + 1 < L) memcpy(Js + (size_t)k * (L - s) + 1, S->J[s + 1] + (size_t)j * (L - s - 1), L - s - 1);
    }
    S->J[s] = Js; S->Jn[s] = f.r;
    S->canon_Jn[s] = f.r;
    S->canon_cols_log[s] = (int *)malloc(sizeof(int) * f.r);
    memcpy(S->canon_cols_log[s], f.cols, sizeof(int) * f.r);
    cz *Mp = (cz *)malloc(sizeof(cz) * (size_t)rows_ * f.r);
    for (int a = 0; a < rows_; ++a)
      for (int k = 0; k < f.r; ++k) Mp[(size_t)a * f.r + k] = Y[s][(size_t)a * cols_ + f.cols[k]];
    cz *Ynew = (cz *)malloc(sizeof(cz) * (size_t)yr[s - 1] * d[s - 1] * f.r);
    zmatmul(yr[s - 1] * d[s - 1], f.r, rows_, Y[s - 1], Mp, Ynew);
    free(Y[s - 1]); Y[s - 1] = Ynew;
    free(Mp);
    for (int nn = 0; nn < N; ++nn) {
      int c0 = xranks[nn * (L + 1) + s], c1 = xranks[nn * (L + 1) + s + 1];
      const cz *Rn = (s + 1 == L) ? &one : S->Rf[nn][s + 1];
      S->Rf[nn][s] = zrightframe(c0, d[s], c1, jn, S->X[nn][s], Rn, f.r, f.cols);
    }
    zldu_free(&f);
  }
  for (int s = 0; s < L; ++s) free(Y[s]);
  free(Y); free(yr);
  int *prev = (int *)malloc(sizeof(int) * L);
  for (int b = 0; b < L - 1; ++b) prev[b] = S->Jn[b + 1];

  /* ---- P:447-500 ---- */
  S->yr = (int *)calloc(L + 1, sizeof(int));
  S->Y = (cz **)calloc(L, sizeof(cz *));
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
        cz *Pi = zassemble_pi(S, b, rl, rr, &S->flops_contraction);
        for (size_t t = 0; t < (size_t)m * n; ++t) {
          if (!isfinite(Pi[t].re) || !isfinite(Pi[t].im)) { *status = ORC_ERR_NONFINITE; zaci_free(S); return NULL; }
          double a = sqrt(cz_w(Pi[t])); /* RZ1 */
          if (a > scale) scale = a;
        }
        double thr = tol_mode == 0 ? tol * scale : tol;
        zldu_t f;
        zldu(m, n, Pi, thr, 0, maxrank, &f);
        for (int k = 0; k < f.r; ++k) S->flops_prrlu += 8.0 * (m - k - 1) * (n - k - 1);
        S->pivot_steps += f.r;
        if (f.eps > maxeps) maxeps = f.eps;
        zlog_push(S, b, dir, rl, rr, &f, scale);
        zupdate_index_sets(S, b, rr, &f);
        if (dir == 0) {
          for (int nn = 0; nn < N; ++nn) {
            int c0 = S->xr[nn * (L + 1) + b], c1 = S->xr[nn * (L + 1) + b + 1];
            cz *nl = zleftframe(rl, c0, d[b], c1, b == 0 ? &one : S->Lf[nn][b - 1], S->X[nn][b], f.r, f.rows);
            free(S->Lf[nn][b]); S->Lf[nn][b] = nl;
          }
        } else {
          for (int nn = 0; nn < N; ++nn) {
            int c1 = S->xr[nn * (L + 1) + b + 1], c2 = S->xr[nn * (L + 1) + b + 2];
            cz *nr = zrightframe(c1, d[b + 1], c2, rr, S->X[nn][b + 1], (b + 2 == L) ? &one : S->Rf[nn][b + 2], f.r,
                                 f.cols);
            free(S->Rf[nn][b + 1]); S->Rf[nn][b + 1] = nr;
          }
          free(S->Y[b + 1]);
          S->Y[b + 1] = (cz *)malloc(sizeof(cz) * (size_t)f.r * n);
          zci_right_B(f.r, n, f.U, f.cols, S->Y[b + 1]);
          S->yr[b + 1] = f.r;
          if (b == 0) {
            free(S->Y[0]);
            S->Y[0] = (cz *)malloc(sizeof(cz) * (size_t)m * f.r);
            for (int i = 0; i < m; ++i)
              for (int k = 0; k < f.r; ++k) S->Y[0][(size_t)i * f.r + k] = Pi[(size_t)i * n + f.cols[k]];
          }
        }
        zldu_free(&f);
        free(Pi);
      }
    }
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

void oraclez_report(void *h, double *scale, double *err, int *iters, int *conv, double *fc, double *fp, long long *piv) {
  zaci_t *S = (zaci_t *)h;
  *scale = S->scale; *err = S->err_estimate; *iters = S->iterations; *conv = S->converged;
  *fc = S->flops_contraction; *fp = S->flops_prrlu; *piv = S->pivot_steps;
}
void oraclez_out_ranks(void *h, int *ranks) { zaci_t *S = (zaci_t *)h; memcpy(ranks, S->yr, sizeof(int) * (S->L + 1)); }
void oraclez_out_core(void *h, int s, double *dst) {
  zaci_t *S = (zaci_t *)h;
  memcpy(dst, S->Y[s], sizeof(cz) * (size_t)S->yr[s] * S->d[s] * S->yr[s + 1]);
}
int oraclez_log_count(void *h) { return ((zaci_t *)h)->nlog; }
void oraclez_log_entry(void *h, int u, int *info, double *eps_scale, int *rows, int *cols) {
  zlogent_t *e = &((zaci_t *)h)->log[u];
  info[0] = e->b; info[1] = e->dir; info[2] = e->rl; info[3] = e->rr; info[4] = e->r;
  eps_scale[0] = e->eps; eps_scale[1] = e->scale;
  if (rows) memcpy(rows, e->rows, sizeof(int) * e->r);
  if (cols) memcpy(cols, e->cols, sizeof(int) * e->r);
}
void oraclez_log_gaps(void *h, int u, double *gap) {
  zlogent_t *e = &((zaci_t *)h)->log[u];
  memcpy(gap, e->gap, sizeof(double) * e->r);
}
int oraclez_canon_jn(void *h, int s) { return ((zaci_t *)h)->canon_Jn[s]; }
void oraclez_canon_cols(void *h, int s, int *dst) {
  zaci_t *S = (zaci_t *)h;
  memcpy(dst, S->canon_cols_log[s], sizeof(int) * S->canon_Jn[s]);
}
