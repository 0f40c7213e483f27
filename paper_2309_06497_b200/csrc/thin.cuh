// Thin problems of the grouped GEMM phases: a dimension too small for a 128 x 64 tensor-core tile.
//   rank-1 SYRK      (factor updates of vector blocks): CTA per row, contiguous vector accesses;
//   K <= 32          (3x3 / 7x7 kernel-mode products): one thread per output element;
//   M, N <= 8        (factors of 3x3 / 7x7 kernel modes, K up to 786k): CTA per 4096-wide k
//                    chunk, FP64 partials reduced in chunk order.
// Both are HBM-bound; products are exact and sums FP64 (deterministic), for float or double
// storage.  SYM problems are computed on the full square (bitwise symmetric, coalesced).
#pragma once

#include <vector>

#include "gemm.cuh"

namespace shampoo {

bool ThinGemmBatch_accepts(const GemmProblem& p);

template <typename T>
class ThinGemmBatch {
 public:
  std::vector<GemmProblem> host;
  ThinGemmBatch() = default;
  ThinGemmBatch(const ThinGemmBatch&) = delete;
  ThinGemmBatch& operator=(const ThinGemmBatch&) = delete;
  ~ThinGemmBatch();
  void add(const GemmProblem& p) { host.push_back(p); }
  int upload();
  int launch(cudaStream_t s, const int32_t* mask = nullptr) const;
  double flops() const;

 private:
  GemmProblem* d_r1_ = nullptr;      // rank-1 symmetric updates (vector-block factors)
  int64_t* d_r1begin_ = nullptr;
  int64_t n_r1_ctas_ = 0;
  int n_r1_ = 0;
  GemmProblem* d_out_ = nullptr;
  int64_t* d_obegin_ = nullptr;
  GemmProblem* d_red_ = nullptr;
  int64_t* d_rbegin_ = nullptr;
  int64_t* d_rbegin8_ = nullptr;  // CTA prefix of the M, N <= 8 reduction problems (after the <= 4 ones)
  int64_t* d_woff_ = nullptr;
  int32_t* d_nch_ = nullptr;
  double* ws_ = nullptr;
  int64_t n_out_items_ = 0, n_red_ctas_ = 0;
  int n_out_ = 0, n_red_ = 0, n_red4_ = 0;
  int64_t n_red4_ctas_ = 0;
};

}  // namespace shampoo
