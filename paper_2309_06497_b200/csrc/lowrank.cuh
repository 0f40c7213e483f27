// Root inverse of structurally low-rank factors (eigh semantics, matfun.py:139-157).
//
// A factor accumulated over s steps from mode unfoldings with K columns has rank <= r = s K; early in
// training (every vector block before step d, every order-2 block at its first refreshes) r << d.
// Then, with Q (d x r') an orthonormal basis containing range(A) and B = Q^T A Q (r' x r'),
//
//     f(A) = f(0) I + Q (f(B) - f(0) I) Q^T,      f(lambda) = (lambda - min(lambda_min, 0) + eps)^(-eta/p),
//
// exactly (the null space of A is the orthogonal complement of range(Q) plus the junk directions of
// Q, on which B vanishes).  Pipeline (FP64; the n^2 r' GEMMs on the tcgen05 Ozaki engine):
//   Y = Omega^T A (Gaussian Omega, r' = r + 8 columns) -> CGS2 (one CTA per factor, rows of Y^T,
//   numerically dependent rows replaced by unit vectors) -> T = Q^T A, B = T Q -> f(B) by the
//   batched Jacobi eigensolver -> X = f(0) I + Q^T^T (f(B) - f(0) I) Q^T, symmetrised.
// Cost ~6 n^2 r' instead of ~100 n^3 for the Jacobi rounds on the full factor.
#pragma once

#include <vector>

#include "common.cuh"

namespace shampoo {

struct LowRankJob {
  int32_t d;         // factor size
  int32_t r;         // structural rank bound
  int32_t root_p;
  int32_t has_prev;  // out already holds a previous inverse (guard fallback)
  const double* in;  // d x d factor (float64)
  double* out;       // d x d inverse root (float64)
};

// Runs every job; stats[4] accumulates the guard branches like RootInverseBatch::run.
int low_rank_root_inverse(const std::vector<LowRankJob>& jobs, double in_scale, double eta, double eps,
                          cudaStream_t s, int64_t* stats);

}  // namespace shampoo
