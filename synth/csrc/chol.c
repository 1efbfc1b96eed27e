/* synth/csrc/chol.c — INPUT GENERATOR ONLY (not the method, not the oracle).
 *
 * Produces the precomputed sparse Cholesky factor L of P*K_reg*P^T that the paper
 * takes as the *input* of Schur-complement assembly (§3 "The input for the
 * algorithm is the matrix B~_i^T together with the factor L_i"; §2.2 two-stage
 * symbolic/numeric factorization).  This plays the role CHOLMOD plays in the paper.
 *
 * Up-looking (row-by-row) sparse Cholesky: for each row k the pattern of L(k,0:k-1) is the
 * elimination-tree reach of the pattern of A(0:k-1,k); the row is computed by a sparse
 * triangular solve with the already-computed columns.  Output is CSC with the diagonal first
 * and row indices ascending in every column (the layout sc_plan expects).
 *
 * The oracle (oracle/) never calls this file: it factors K_reg itself, densely, in the
 * natural order.  The GPU path never calls it either; it only receives its output.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Elimination tree of a symmetric matrix given by its upper pattern (column j holds rows i<=j),
   Liu's algorithm with path compression. Acp/Aci: CSC of the full symmetric pattern. */
static void etree(int32_t n, const int64_t* Ap, const int32_t* Ai, int32_t* parent, int32_t* anc) {
  for (int32_t k = 0; k < n; k++) {
    parent[k] = -1;
    anc[k] = -1;
    for (int64_t p = Ap[k]; p < Ap[k + 1]; p++) {
      int32_t i = Ai[p];
      while (i != -1 && i < k) {
        int32_t next = anc[i];
        anc[i] = k;
        if (next == -1) {
          parent[i] = k;
          break;
        }
        i = next;
      }
    }
  }
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* Pattern of row k of L (excluding the diagonal): the etree reach of the pattern of A(0:k-1,k).
   Returned ascending in s[0..top), which is a topological order (a child index is always smaller
   than its parent's, and every column j feeding x[i] is an etree descendant of i). */
static int32_t ereach(int32_t k, const int64_t* Ap, const int32_t* Ai, const int32_t* parent,
                      int32_t* s, int32_t* mark) {
  int32_t top = 0;
  mark[k] = k;
  for (int64_t p = Ap[k]; p < Ap[k + 1]; p++) {
    int32_t i = Ai[p];
    if (i > k) continue;
    while (i >= 0 && mark[i] != k) {
      s[top++] = i;
      mark[i] = k;
      i = parent[i];
    }
  }
  qsort(s, (size_t)top, sizeof(int32_t), cmp_i32);
  return top;
}

/* Symbolic + numeric factorization.
   Input: n, CSC of the full symmetric matrix C = P K P^T (both triangles, any row order).
   Two-call protocol: call with Lx == NULL to obtain nnz(L) in *nnz_out and Lp filled;
   then call again with Li/Lx allocated to nnz(L).
   Returns 0 on success, k+1 if the pivot at column k is not positive. */
int synth_cholesky(int32_t n, const int64_t* Ap, const int32_t* Ai, const double* Ax, int64_t* Lp,
                   int32_t* Li, double* Lx, int64_t* nnz_out) {
  int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int32_t* anc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int32_t* s = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int32_t* mark = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int64_t* cnt = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  int rc = 0;
  etree(n, Ap, Ai, parent, anc);
  for (int32_t k = 0; k < n; k++) mark[k] = -1;
  /* column counts: row k contributes one entry to each column in ereach(k), plus diagonal */
  for (int32_t k = 0; k < n; k++) {
    int32_t top = ereach(k, Ap, Ai, parent, s, mark);
    for (int32_t t = 0; t < top; t++) cnt[s[t]]++;
    cnt[k]++;
  }
  Lp[0] = 0;
  for (int32_t k = 0; k < n; k++) Lp[k + 1] = Lp[k] + cnt[k];
  *nnz_out = Lp[n];
  if (Lx == NULL || Li == NULL) goto done;
  {
    double* x = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    int64_t* c = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int32_t k = 0; k < n; k++) {
      c[k] = Lp[k];
      mark[k] = -1;
    }
    for (int32_t k = 0; k < n; k++) {
      int32_t top = ereach(k, Ap, Ai, parent, s, mark);
      x[k] = 0.0;
      for (int64_t p = Ap[k]; p < Ap[k + 1]; p++)
        if (Ai[p] <= k) x[Ai[p]] += Ax[p];
      double d = x[k];
      x[k] = 0.0;
      for (int32_t t = 0; t < top; t++) {
        int32_t i = s[t];
        double lki = x[i] / Lx[Lp[i]];
        x[i] = 0.0;
        for (int64_t p = Lp[i] + 1; p < c[i]; p++) x[Li[p]] -= Lx[p] * lki;
        d -= lki * lki;
        int64_t q = c[i]++;
        Li[q] = k;
        Lx[q] = lki;
      }
      if (!(d > 0.0)) {
        rc = k + 1;
        break;
      }
      int64_t q = c[k]++;
      Li[q] = k;
      Lx[q] = sqrt(d);
    }
    free(x);
    free(c);
  }
done:
  free(parent);
  free(anc);
  free(s);
  free(mark);
  free(cnt);
  return rc;
}
