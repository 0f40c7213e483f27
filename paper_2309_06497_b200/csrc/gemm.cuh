// Grouped, strided GEMM problem descriptors (executed by the tcgen05 Ozaki engine, tcgen05.cuh, or
// the thin-problem kernels, thin.cuh) and a grouped GEMV.  One launch covers every problem of a
// phase (all blocks, all modes) through a device-side tile table, so a step costs O(phases)
// launches, not O(blocks).
//
//   C[i,j] = alpha * sum_k A(i,k) * B(j,k) + beta * C[i,j]
//   X(r,k) = X + idx2(r; rdiv, rhi, rlo) + idx2(k; kdiv, khi, klo)
//   idx2(x; div, hi, lo) = (x / div) * hi + (x % div) * lo
//
// The two-level indices express every mode-k unfolding of a row-major block
// (outer x d_k x inner) without copies: the factor statistics
// (precond.py:161-165) contract over k = (o, n) and the mode products
// (precond.py:168-174) run over output columns c = (o, n).
#pragma once

#include <vector>

#include "common.cuh"

namespace shampoo {

enum GemmFlags : int32_t {
  kGemmSym = 1,    // C symmetric: compute tiles tm >= tn, mirror-write the rest (A==B except on the Ozaki path)
  kGemmReadC = 2,  // C = alpha*AB + beta*C (else beta ignored)
  kGemmMasked = 4, // skip unless mask[mask_index] != 0
  kGemmConstA = 8,  // operand A changes rarely (an inverse factor): tensor-core packs are cached
  kGemmConstB = 16, // same for operand B
  kGemmXformA = 32, // operand A packed as xa * A + xb * I with the fixed row exponent a_fexp (Ozaki path)
  kGemmXformB = 64, // same for operand B (b_xa, b_xb, b_fexp)
  kGemmLowerOnly = 128, // with kGemmSym: write the lower triangle only (the factor statistics; the upper
                        // triangle is restored by symmetrize before anything reads the full factor)
};

struct Idx2 {
  int32_t div;  // 0x7fffffff = single level
  int32_t pad;
  int64_t hi, lo;
};

inline Idx2 idx1(int64_t stride) { return Idx2{0x7fffffff, 0, 0, stride}; }
inline Idx2 idx2(int64_t div, int64_t hi, int64_t lo) { return Idx2{(int32_t)div, 0, hi, lo}; }

struct GemmProblem {
  int32_t M, N, K;
  int32_t flags;
  int32_t tiles_m, tiles_n;
  int32_t mask_index;
  int32_t ksplit;   // K chunks (split-K); filled by upload()
  int32_t kchunk;   // K per chunk
  int32_t pad;
  int64_t tiles;
  int64_t ws_off;   // split-K workspace offset (doubles)
  const void* A;
  Idx2 a_r, a_k;
  const void* B;
  Idx2 b_r, b_k;
  void* C;
  Idx2 c_r, c_c;
  double alpha, beta;
  // kGemmXform*: the operand entering the product is xa * X + xb * delta(row, k), sliced with the fixed
  // exponent fexp (|entries| < 2^fexp guaranteed by the caller) -- no row-maximum pass
  double a_xa, a_xb, b_xa, b_xb;
  int32_t a_fexp, b_fexp;
};

struct GemvProblem {
  int32_t n;  // square matrix size
  int32_t mask_index;
  const void* X;  // n x n row-major
  const void* x;  // n
  void* y;        // n
  double alpha;
};

template <typename T>
class GemvBatch {
 public:
  std::vector<GemvProblem> host;
  GemvBatch() = default;
  GemvBatch(const GemvBatch&) = delete;
  GemvBatch& operator=(const GemvBatch&) = delete;
  ~GemvBatch();
  void add(const GemvProblem& p) { host.push_back(p); }
  bool empty() const { return host.empty(); }
  int upload();
  int launch(cudaStream_t s, const int32_t* mask = nullptr) const;

 private:
  GemvProblem* d_prob_ = nullptr;
  int64_t* d_begin_ = nullptr;  // row-group prefix
  int64_t total_groups_ = 0;
};

// Symmetric mode-k Gram of a row-major block viewed as (outer, d, inner):
//   C(d x d) = beta*C + alpha * unfold_k(X) unfold_k(X)^T
GemmProblem make_mode_gram(const void* X, int64_t outer, int64_t d, int64_t inner, void* C,
                           double alpha, double beta);
// Mode-k product Y = Mat x_k X on (outer, d, inner) blocks:
//   Y[o,i,n] = alpha * sum_j Mat[i,j] X[o,j,n]
GemmProblem make_mode_product(const void* Mat, const void* X, void* Y, int64_t outer, int64_t d,
                              int64_t inner, double alpha);
// Row-major C(MxN) = alpha * opA(A) opB(B) + beta*C; ta/tb: operand stored transposed.
GemmProblem make_gemm(bool ta, bool tb, int32_t M, int32_t N, int32_t K, const void* A, int64_t lda,
                      const void* B, int64_t ldb, void* C, int64_t ldc, double alpha, double beta);

}  // namespace shampoo
