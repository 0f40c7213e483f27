// Root inverse of structurally low-rank factors (eigh semantics, matfun.py:139-157).
//
// A factor accumulated over s steps from mode unfoldings with K columns has rank <= r = s K; early in
// training (every vector block before step d, every order-2 block at its first refreshes) r << d.
// Then, with Q (d x r') an orthonormal basis containing range(A) and B = Q^T A Q (r' x r'),
//
//     f(A) = f(0) I + Q (f(B) - f(0) I) Q^T,      f(lambda) = (lambda - min(lambda_min, 0) + eps)^(-eta/p),
//
// exactly (the null space of A is the orthogonal complement of range(Q) plus the junk directions of
// Q, on which B vanishes).  r is the structural rank bound itself (no oversampling: Y = Omega^T A has
// rank <= r, so r rows span range(A)).  Pipeline (FP64; the n^2 r GEMMs on the tcgen05 Ozaki engine):
//   Y = Omega^T A (Gaussian Omega, r rows) -> block CGS2 (64-row blocks: projections on the earlier
//   blocks as Ozaki GEMMs, the in-block pass on an 8-CTA cluster holding the block in shared memory;
//   numerically dependent rows replaced by unit vectors and re-projected) -> T = Q A, B = T Q^T ->
//   f(B) by RootInverseBatch (B is full rank: Newton pre-pass, Jacobi if gated) ->
//   X = f(0) I + Q^T (f(B) - f(0) I) Q (symmetric-output GEMM).
// Cost ~6 n^2 r + r^3-class solve instead of the full-size Jacobi rounds.
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
