/* tools/implicit_cpu.c — CPU implicit application of the dual operator (measurement baseline for the
 * amortization point; not the oracle, not the GPU path).
 *
 * q = sum_i scatter( B~_i L_i^{-T} L_i^{-1} B~_i^T gather(lambda) )   (eq.
 * dualop_apply_impl: SpMV, forward TRSV, backward TRSV, SpMV), with the same CSC factor L_i and
 * permutation the GPU path receives.  OpenMP over subdomains (one subdomain per thread, like the
 * paper's "threads handle subdomains"); each subdomain writes its own local result, the
 * scatter into q is serial (deterministic).
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t n, m;
  const int64_t* Lp;
  const int32_t* Li;
  const double* Lx;
  const int32_t* iperm; /* iperm[old] = new */
  const int32_t* Bp;    /* CSC of B~^T, rows in original numbering */
  const int32_t* Bi;
  const double* Bx;
  const int64_t* lmap;
} implicit_sd;

static void apply_one(const implicit_sd* s, const double* lambda, double* x, double* y) {
  const int32_t n = s->n, m = s->m;
  memset(x, 0, sizeof(double) * (size_t)n);
  for (int32_t j = 0; j < m; j++) {
    const double l = lambda[s->lmap[j]];
    for (int32_t p = s->Bp[j]; p < s->Bp[j + 1]; p++) x[s->iperm[s->Bi[p]]] += s->Bx[p] * l;
  }
  for (int32_t c = 0; c < n; c++) { /* L y = x (column oriented) */
    const int64_t a = s->Lp[c], b = s->Lp[c + 1];
    const double xc = x[c] / s->Lx[a];
    x[c] = xc;
    if (xc != 0.0)
      for (int64_t p = a + 1; p < b; p++) x[s->Li[p]] -= s->Lx[p] * xc;
  }
  for (int32_t c = n - 1; c >= 0; c--) { /* L^T z = y */
    const int64_t a = s->Lp[c], b = s->Lp[c + 1];
    double t = x[c];
    for (int64_t p = a + 1; p < b; p++) t -= s->Lx[p] * x[s->Li[p]];
    x[c] = t / s->Lx[a];
  }
  for (int32_t j = 0; j < m; j++) {
    double t = 0.0;
    for (int32_t p = s->Bp[j]; p < s->Bp[j + 1]; p++) t += s->Bx[p] * x[s->iperm[s->Bi[p]]];
    y[j] = t;
  }
}

/* q (n_lambda) = implicit apply over nsub subdomains.  ybuf: sum_i m_i doubles (scratch),
   xbuf: nthreads * max_n doubles (scratch).  Returns the number of threads used. */
int implicit_apply(int32_t nsub, const implicit_sd* sds, const double* lambda, double* q, int64_t n_lambda,
                   double* ybuf, const int64_t* yoff, double* xbuf, int32_t max_n, int nthreads) {
  if (nthreads > 0) omp_set_num_threads(nthreads);
  int used = 1;
#pragma omp parallel
  {
#pragma omp single
    used = omp_get_num_threads();
    double* x = xbuf + (size_t)omp_get_thread_num() * (size_t)max_n;
#pragma omp for schedule(dynamic, 1)
    for (int32_t i = 0; i < nsub; i++) apply_one(&sds[i], lambda, x, ybuf + yoff[i]);
  }
  memset(q, 0, sizeof(double) * (size_t)n_lambda);
  for (int32_t i = 0; i < nsub; i++)
    for (int32_t j = 0; j < sds[i].m; j++) q[sds[i].lmap[j]] += ybuf[yoff[i] + j];
  return used;
}
