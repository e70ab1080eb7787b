/*
 * rsim/blockops.h — b×b block arithmetic with a FIXED operation order, plus
 * the canonical reduction layout.  Shared by the sm_100a kernels and the CPU
 * oracle so that block-Jacobi scaling, SpMV rows, ILU(0) and every Krylov
 * dot product produce identical bits on both sides.
 *
 * Canonical reduction (sum of per-row values v_0..v_{n-1}):
 *   rows are cut into consecutive chunks of RSIM_RED_CHUNK = 256; inside a
 *   chunk, "thread" t holds v[256c + t] (+0.0 past the end) and the 256 values
 *   are combined by the tree
 *     for off in 16,8,4,2,1:  s[lane] += s[lane+off]   (inside each warp)
 *     for off in 4,2,1:       w[k]   += w[k+off]        (over the 8 warp sums)
 *   giving one partial per chunk.  If there is more than one chunk the
 *   partials are reduced again with the same rule (recursively).
 * On the GPU a chunk is exactly 8 warps doing __shfl_down_sync, so any CTA
 * that owns whole chunks reduces them locally; oracle/ replays the same tree
 * in plain loops.  Per-row values for b>1 are the in-order component sums
 * (row dot = Σ_c a_c b_c, c ascending).
 */
#ifndef RSIM_BLOCKOPS_H
#define RSIM_BLOCKOPS_H

#include "physics.h"

#define RSIM_RED_CHUNK 256

namespace rsim {
namespace blk {

/* Inverse of a b×b block by the adjugate; false if singular / non-finite. */
RSIM_HD bool inv(const double (*D)[1], double (*Di)[1]) {
  double d = D[0][0];
  if (!(d != 0.0) || !(fabs(d) < HUGE_VAL)) return false;
  Di[0][0] = 1.0 / d;
  return true;
}
RSIM_HD bool inv(const double (*D)[2], double (*Di)[2]) {
  double det = D[0][0] * D[1][1] - D[0][1] * D[1][0];
  if (!(det != 0.0) || !(fabs(det) < HUGE_VAL)) return false;
  Di[0][0] = D[1][1] / det;
  Di[0][1] = -(D[0][1] / det);
  Di[1][0] = -(D[1][0] / det);
  Di[1][1] = D[0][0] / det;
  return true;
}
RSIM_HD bool inv(const double (*D)[3], double (*Di)[3]) {
  double c00 = D[1][1] * D[2][2] - D[1][2] * D[2][1];
  double c01 = D[1][2] * D[2][0] - D[1][0] * D[2][2];
  double c02 = D[1][0] * D[2][1] - D[1][1] * D[2][0];
  double det = (D[0][0] * c00 + D[0][1] * c01) + D[0][2] * c02;
  if (!(det != 0.0) || !(fabs(det) < HUGE_VAL)) return false;
  Di[0][0] = c00 / det;
  Di[1][0] = c01 / det;
  Di[2][0] = c02 / det;
  Di[0][1] = (D[0][2] * D[2][1] - D[0][1] * D[2][2]) / det;
  Di[0][2] = (D[0][1] * D[1][2] - D[0][2] * D[1][1]) / det;
  Di[1][1] = (D[0][0] * D[2][2] - D[0][2] * D[2][0]) / det;
  Di[1][2] = (D[0][2] * D[1][0] - D[0][0] * D[1][2]) / det;
  Di[2][1] = (D[0][1] * D[2][0] - D[0][0] * D[2][1]) / det;
  Di[2][2] = (D[0][0] * D[1][1] - D[0][1] * D[1][0]) / det;
  return true;
}

/* y = M x  (row r: ((M_r0 x_0) + M_r1 x_1) + ...). */
template <int B>
RSIM_HD void gemv(const double (*M)[B], const double* x, double* y) {
  for (int r = 0; r < B; ++r) {
    double s = M[r][0] * x[0];
    for (int c = 1; c < B; ++c) s = s + M[r][c] * x[c];
    y[r] = s;
  }
}

/* "Pressure-only" block: every entry outside column 0 is (±)0.  This is the
 * off-diagonal block of a row whose own cell is the upwind side of the
 * connection (physics.h flux_terms: ∂F_ij/∂u_j then has the p_j column only),
 * about half of all off-diagonal blocks.  The assembly counts them with exactly
 * this test (one bit per block in ell_po).  They are multiplied like any other
 * block: skipping their zero columns in the Krylov kernels was measured in round 2
 * and loses on whole runs (lanes of a warp disagree on the block shape). */
template <int B>
RSIM_HD bool col0_only(const double* M) {
  bool z = B > 1;
  for (int r = 0; r < B; ++r)
    for (int c = 1; c < B; ++c) z = z && (M[r * B + c] == 0.0);
  return z;
}

/* y += M x, flat row-major block (as stored in the BSR/ELL value arrays). */
template <int B>
RSIM_HD void gemv_acc_flat(const double* M, const double* x, double* y) {
  for (int r = 0; r < B; ++r) {
    double s = M[r * B] * x[0];
    for (int c = 1; c < B; ++c) s = s + M[r * B + c] * x[c];
    y[r] = y[r] + s;
  }
}

/* y = M x, flat row-major block. */
template <int B>
RSIM_HD void gemv_flat(const double* M, const double* x, double* y) {
  for (int r = 0; r < B; ++r) {
    double s = M[r * B] * x[0];
    for (int c = 1; c < B; ++c) s = s + M[r * B + c] * x[c];
    y[r] = s;
  }
}

/* y -= M x, flat row-major block. */
template <int B>
RSIM_HD void gemv_sub_flat(const double* M, const double* x, double* y) {
  for (int r = 0; r < B; ++r) {
    double s = M[r * B] * x[0];
    for (int c = 1; c < B; ++c) s = s + M[r * B + c] * x[c];
    y[r] = y[r] - s;
  }
}

/* C = A B (all b×b, row-major arrays). */
template <int B>
RSIM_HD void gemm(const double (*A)[B], const double (*Bm)[B], double (*C)[B]) {
  for (int r = 0; r < B; ++r)
    for (int c = 0; c < B; ++c) {
      double s = A[r][0] * Bm[0][c];
      for (int k = 1; k < B; ++k) s = s + A[r][k] * Bm[k][c];
      C[r][c] = s;
    }
}

/* Flat variants used by ILU(0): C -= A B ; C = A B. */
template <int B>
RSIM_HD void gemm_sub_flat(const double* A, const double* Bm, double* C) {
  for (int r = 0; r < B; ++r)
    for (int c = 0; c < B; ++c) {
      double s = A[r * B] * Bm[c];
      for (int k = 1; k < B; ++k) s = s + A[r * B + k] * Bm[k * B + c];
      C[r * B + c] = C[r * B + c] - s;
    }
}
template <int B>
RSIM_HD void gemm_flat(const double* A, const double* Bm, double* C) {
  for (int r = 0; r < B; ++r)
    for (int c = 0; c < B; ++c) {
      double s = A[r * B] * Bm[c];
      for (int k = 1; k < B; ++k) s = s + A[r * B + k] * Bm[k * B + c];
      C[r * B + c] = s;
    }
}
template <int B>
RSIM_HD bool inv_flat(const double* D, double* Di) {
  double a[B][B], ai[B][B];
  for (int r = 0; r < B; ++r)
    for (int c = 0; c < B; ++c) a[r][c] = D[r * B + c];
  if (!inv(a, ai)) return false;
  for (int r = 0; r < B; ++r)
    for (int c = 0; c < B; ++c) Di[r * B + c] = ai[r][c];
  return true;
}

/* Row-local dot product Σ_c a_c b_c (c ascending, starting with the c=0 term). */
template <int B>
RSIM_HD double rowdot(const double* a, const double* b) {
  double s = a[0] * b[0];
  for (int c = 1; c < B; ++c) s = s + a[c] * b[c];
  return s;
}

}  // namespace blk
}  // namespace rsim

#endif /* RSIM_BLOCKOPS_H */
