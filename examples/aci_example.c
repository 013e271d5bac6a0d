/*
 * Minimal C use of the libaci.so C-ABI (include/aci.h), no Python: two random tensor trains,
 * their Hadamard product by ACI, and a check of the result at random points against the
 * product of the inputs' values (tt_evaluate). Prints one line; exit code 0 iff the relative
 * max error is within 10 * tol.
 *
 *   gcc -O2 -I include examples/aci_example.c -L paper_2604_00037_b200 -laci \
 *       -Wl,-rpath,$PWD/paper_2604_00037_b200 -lm -o examples/aci_example
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "aci.h"

static uint64_t rng_state = 88172645463325252ull;
static double urand(void) { /* xorshift64*, uniform in [-1, 1) */
  rng_state ^= rng_state >> 12;
  rng_state ^= rng_state << 25;
  rng_state ^= rng_state >> 27;
  return (double)((rng_state * 2685821657736338717ull) >> 11) / 4503599627370496.0 - 1.0;
}

static tt_t *random_tt(int L, int d, int chi) {
  int *dims = malloc(sizeof(int) * L), *ranks = malloc(sizeof(int) * (L + 1));
  double **cores = malloc(sizeof(double *) * L);
  ranks[0] = ranks[L] = 1;
  for (int s = 1; s < L; ++s) ranks[s] = chi;
  for (int s = 0; s < L; ++s) {
    dims[s] = d;
    size_t n = (size_t)ranks[s] * d * ranks[s + 1];
    cores[s] = malloc(sizeof(double) * n);
    for (size_t i = 0; i < n; ++i) cores[s][i] = urand() / sqrt((double)chi * d);
  }
  tt_t *t = NULL;
  int st = tt_create(L, dims, ranks, (const double *const *)cores, &t);
  for (int s = 0; s < L; ++s) free(cores[s]);
  free(cores);
  free(dims);
  free(ranks);
  if (st != ACI_OK) {
    fprintf(stderr, "tt_create: %s\n", aci_last_error());
    exit(2);
  }
  return t;
}

int main(void) {
  const int L = 24, d = 2, npts = 4096;
  const double tol = 1e-10;
  tt_t *a = random_tt(L, d, 16), *b = random_tt(L, d, 2);
  const tt_t *inputs[2] = {a, b};
  const double coef[1] = {1.0};
  const int expo[2] = {1, 1}; /* f(x1, x2) = x1 * x2 */
  aci_op op = {1, coef, expo};
  tt_t *y = NULL;
  aci_report rep;
  int st = aci_elementwise(op, inputs, 2, tol, 32, 20, &y, &rep);
  if (st < 0) {
    fprintf(stderr, "aci_elementwise: %s\n", aci_last_error());
    return 2;
  }
  uint8_t *idx = malloc((size_t)npts * L);
  for (size_t i = 0; i < (size_t)npts * L; ++i) idx[i] = (uint8_t)(urand() > 0.0);
  double *va = malloc(sizeof(double) * npts), *vb = malloc(sizeof(double) * npts), *vy = malloc(sizeof(double) * npts);
  if (tt_evaluate(a, npts, idx, va) || tt_evaluate(b, npts, idx, vb) || tt_evaluate(y, npts, idx, vy)) {
    fprintf(stderr, "tt_evaluate: %s\n", aci_last_error());
    return 2;
  }
  double err = 0.0, ref = 0.0;
  for (int p = 0; p < npts; ++p) {
    double e = fabs(vy[p] - va[p] * vb[p]), r = fabs(va[p] * vb[p]);
    if (e > err) err = e;
    if (r > ref) ref = r;
  }
  printf("aci_example: %s, status %d, iterations %d, max rank %d, %lld pivots, %.2f ms, rel max error %.3e\n",
         aci_version(), st, rep.iterations, rep.max_rank, (long long)rep.pivot_steps, rep.ms, err / ref);
  int ok = err <= 10 * tol * ref;

  /* the same product three times as one batch (concurrent products on library streams): each
   * result must equal the single run's at the sample points */
  aci_job jobs[3];
  tt_t *ys[3] = {NULL, NULL, NULL};
  aci_report reps[3];
  for (int j = 0; j < 3; ++j) {
    aci_job J = {op, inputs, 2, tol, 32, 20, NULL, &ys[j], &reps[j], 0};
    jobs[j] = J;
  }
  st = aci_elementwise_batch(jobs, 3, 0);
  if (st < 0) {
    fprintf(stderr, "aci_elementwise_batch: %s\n", aci_last_error());
    return 2;
  }
  double *vz = malloc(sizeof(double) * npts);
  double berr = 0.0;
  for (int j = 0; j < 3; ++j) {
    if (tt_evaluate(ys[j], npts, idx, vz)) return 2;
    for (int p = 0; p < npts; ++p) berr = fmax(berr, fabs(vz[p] - vy[p]));
    tt_destroy(ys[j]);
  }
  printf("aci_example: batch of 3, max |batch - single| = %.3e\n", berr);
  ok = ok && berr == 0.0;
  free(vz);
  tt_destroy(y);
  tt_destroy(a);
  tt_destroy(b);
  free(idx);
  free(va);
  free(vb);
  free(vy);
  return ok ? 0 : 1;
}
