/* oracle/oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * The CPU oracle for the local FETI dual operator.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it.  It shares no code, header, table
 * or helper with the CUDA path (paper_2509_21037_b200/); it never sees L, the fill-reducing
 * permutation, the stepped order, supernodes or tiles.
 *
 * What it computes is the plain definition
 *     F_i = B~_i K_i^+ B~_i^T,   K_i^+ = K_{i,reg}^{-1} = L^{-T} L^{-1}
 * (PAPER.md P:258-262 eq. localdualoperator; P:285-290 eq. localdualoperatorwithU), evaluated as
 * the implicit operator of eq. dualop_apply_impl applied to each unit vector:
 *   O1  K_reg (natural DOF order, as generated) is stored in band form (half-bandwidth b = max|i-j|
 *       over its nonzeros).  Cholesky fill of a band matrix stays inside the band, so this is the
 *       textbook dense Cholesky with its loops restricted to where entries can be nonzero.
 *   O2  unpivoted Cholesky K_reg = L L^T, row by row:  L_ij = (A_ij - sum_{k<j} L_ik L_jk) / L_jj,
 *       L_ii = sqrt(A_ii - sum_{k<i} L_ik^2); a pivot <= 0 is reported (not SPD).
 *   O3  for each requested multiplier column j: z = L^{-T} (L^{-1} B~^T(:,j))  (forward, backward).
 *   O4  F(a,j) = sum_d B~^T(d,a) z(d)  for every multiplier a  (explicit product, full m x m,
 *       not symmetrised).
 * Everything is FP64.  Parity pins for this file live in tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Band storage: row i holds columns j in [i-b, i] at Lb[i*(b+1) + (j - i + b)]. */
#define BAND(Lb, b, i, j) (Lb)[(int64_t)(i) * ((b) + 1) + ((j) - (i) + (b))]

int32_t oracle_bandwidth(int32_t n, const int64_t* rowptr, const int32_t* colidx) {
  int32_t b = 0;
  for (int32_t i = 0; i < n; i++)
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; p++) {
      int32_t d = i - colidx[p];
      if (d < 0) d = -d;
      if (d > b) b = d;
    }
  return b;
}

/* O1+O2: band Cholesky of the symmetric matrix given in CSR (both triangles or lower only; only
   entries with j <= i are read).  Lb must hold n*(b+1) doubles.  Returns 0, or k+1 when the pivot of
   row k is not positive. */
int oracle_cholesky_band(int32_t n, int32_t b, const int64_t* rowptr, const int32_t* colidx,
                         const double* vals, double* Lb) {
  memset(Lb, 0, sizeof(double) * (size_t)n * (size_t)(b + 1));
  for (int32_t i = 0; i < n; i++)
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; p++) {
      int32_t j = colidx[p];
      if (j <= i && i - j <= b) BAND(Lb, b, i, j) += vals[p];
    }
  for (int32_t i = 0; i < n; i++) {
    int32_t j0 = i - b > 0 ? i - b : 0;
    for (int32_t j = j0; j <= i; j++) {
      int32_t k0 = j - b > j0 ? j - b : j0; /* L_ik != 0 needs k >= i-b, L_jk needs k >= j-b */
      double s = BAND(Lb, b, i, j);
      for (int32_t k = k0; k < j; k++) s -= BAND(Lb, b, i, k) * BAND(Lb, b, j, k);
      if (j == i) {
        if (!(s > 0.0)) return i + 1;
        BAND(Lb, b, i, i) = sqrt(s);
      } else {
        BAND(Lb, b, i, j) = s / BAND(Lb, b, j, j);
      }
    }
  }
  return 0;
}

/* O3 forward: y = L^{-1} x, in place. */
void oracle_forward(int32_t n, int32_t b, const double* Lb, double* x) {
  for (int32_t i = 0; i < n; i++) {
    int32_t k0 = i - b > 0 ? i - b : 0;
    double s = x[i];
    for (int32_t k = k0; k < i; k++) s -= BAND(Lb, b, i, k) * x[k];
    x[i] = s / BAND(Lb, b, i, i);
  }
}

/* O3 backward: z = L^{-T} y, in place. */
void oracle_backward(int32_t n, int32_t b, const double* Lb, double* x) {
  for (int32_t i = n - 1; i >= 0; i--) {
    int32_t k1 = i + b < n - 1 ? i + b : n - 1;
    double s = x[i];
    for (int32_t k = i + 1; k <= k1; k++) s -= BAND(Lb, b, k, i) * x[k];
    x[i] = s / BAND(Lb, b, i, i);
  }
}

/* Whole oracle for one subdomain: columns `cols[0..ncols)` of F (or all m columns when cols is
   NULL) written to F[c*m + a] (column-major m x ncols).  K_reg in CSR (natural order); B~^T in CSC
   (n x m).  Returns 0, -1 on allocation failure, or k+1 when K_reg is not SPD at row k. */
int oracle_dual_operator(int32_t n, const int64_t* K_rowptr, const int32_t* K_colidx, const double* K_vals,
                         int32_t m, const int32_t* Bt_colptr, const int32_t* Bt_rowidx, const double* Bt_vals,
                         int32_t ncols, const int32_t* cols, double* F) {
  int32_t b = oracle_bandwidth(n, K_rowptr, K_colidx);
  double* Lb = (double*)malloc(sizeof(double) * (size_t)n * (size_t)(b + 1) + 8);
  double* z = (double*)malloc(sizeof(double) * (size_t)n + 8);
  if (!Lb || !z) {
    free(Lb);
    free(z);
    return -1;
  }
  int rc = oracle_cholesky_band(n, b, K_rowptr, K_colidx, K_vals, Lb);
  if (rc == 0) {
    int32_t nc = cols ? ncols : m;
    for (int32_t c = 0; c < nc; c++) {
      int32_t j = cols ? cols[c] : c;
      memset(z, 0, sizeof(double) * (size_t)n);
      for (int32_t p = Bt_colptr[j]; p < Bt_colptr[j + 1]; p++) z[Bt_rowidx[p]] += Bt_vals[p];
      oracle_forward(n, b, Lb, z);
      oracle_backward(n, b, Lb, z);
      for (int32_t a = 0; a < m; a++) {
        double s = 0.0;
        for (int32_t p = Bt_colptr[a]; p < Bt_colptr[a + 1]; p++) s += Bt_vals[p] * z[Bt_rowidx[p]];
        F[(int64_t)c * m + a] = s;
      }
    }
  }
  free(Lb);
  free(z);
  return rc;
}
