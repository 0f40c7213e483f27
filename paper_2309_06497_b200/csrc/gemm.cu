// Grouped GEMV (order-1 blocks: P = X g with the n x n inverse factor, FP64 sums) and the problem
// builders that express every mode-k unfolding of a row-major block as a strided GEMM (see
// gemm.cuh).  The GEMMs themselves run on the tcgen05 Ozaki engine (tcgen05.cu) or, when too thin
// for a tensor-core tile, on the HBM-bound kernels of thin.cu.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "gemm.cuh"

namespace shampoo {

namespace {

// One warp per output row; CTA = 8 rows.
template <typename T>
__global__ void __launch_bounds__(256) grouped_gemv_kernel(const GemvProblem* __restrict__ probs,
                                                           const int64_t* __restrict__ begin, int nprob,
                                                           const int32_t* __restrict__ mask) {
  const int64_t gi = blockIdx.x;
  int lo = 0, hi = nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (begin[mid] <= gi) lo = mid;
    else hi = mid - 1;
  }
  const GemvProblem& P = probs[lo];
  if (mask && mask[P.mask_index] == 0) return;
  const int row = (int)(gi - begin[lo]) * 8 + (threadIdx.x >> 5);
  if (row >= P.n) return;
  const T* __restrict__ X = static_cast<const T*>(P.X) + (int64_t)row * P.n;
  const T* __restrict__ x = static_cast<const T*>(P.x);
  double s = 0;
  for (int j = threadIdx.x & 31; j < P.n; j += 32) s = fma((double)X[j], (double)x[j], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) static_cast<T*>(P.y)[row] = T(P.alpha * s);
}

}  // namespace

template <typename T>
GemvBatch<T>::~GemvBatch() {
  dev_free(d_prob_);
  dev_free(d_begin_);
}

template <typename T>
int GemvBatch<T>::upload() {
  dev_free(d_prob_);
  dev_free(d_begin_);
  d_prob_ = nullptr;
  d_begin_ = nullptr;
  total_groups_ = 0;
  if (host.empty()) return SHAMPOO_OK;
  std::vector<int64_t> begin(host.size());
  for (size_t i = 0; i < host.size(); ++i) {
    begin[i] = total_groups_;
    total_groups_ += (host[i].n + 7) / 8;
  }
  SH_CUDA_CHECK(dev_malloc(&d_prob_, host.size() * sizeof(GemvProblem)));
  SH_CUDA_CHECK(dev_malloc(&d_begin_, host.size() * sizeof(int64_t)));
  SH_CUDA_CHECK(cudaMemcpy(d_prob_, host.data(), host.size() * sizeof(GemvProblem), cudaMemcpyHostToDevice));
  SH_CUDA_CHECK(cudaMemcpy(d_begin_, begin.data(), begin.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  return SHAMPOO_OK;
}

template <typename T>
int GemvBatch<T>::launch(cudaStream_t s, const int32_t* mask) const {
  if (total_groups_ == 0) return SHAMPOO_OK;
  grouped_gemv_kernel<T><<<(unsigned)total_groups_, 256, 0, s>>>(d_prob_, d_begin_, (int)host.size(), mask);
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

template class GemvBatch<double>;
template class GemvBatch<float>;

GemmProblem make_mode_gram(const void* X, int64_t outer, int64_t d, int64_t inner, void* C, double alpha,
                           double beta) {
  GemmProblem p{};
  p.M = p.N = (int32_t)d;
  p.K = (int32_t)(outer * inner);
  p.flags = kGemmSym | (beta != 0.0 ? kGemmReadC : 0);
  p.A = p.B = X;
  p.a_r = p.b_r = idx1(inner);
  // contraction index k = (o, n): address o*d*inner + n
  p.a_k = p.b_k = (inner == 1) ? idx1(d) : (outer == 1 ? idx1(1) : idx2(inner, d * inner, 1));
  p.C = C;
  p.c_r = idx1(d);
  p.c_c = idx1(1);
  p.alpha = alpha;
  p.beta = beta;
  return p;
}

GemmProblem make_mode_product(const void* Mat, const void* X, void* Y, int64_t outer, int64_t d, int64_t inner,
                              double alpha) {
  GemmProblem p{};
  p.alpha = alpha;
  p.beta = 0.0;
  if (inner == 1) {
    // last mode: Y(o, i) = sum_j X(o, j) Mat(i, j)   (rows o contiguous, coalesced stores)
    p.M = (int32_t)outer;
    p.N = (int32_t)d;
    p.K = (int32_t)d;
    p.A = X;
    p.a_r = idx1(d);
    p.a_k = idx1(1);
    p.B = Mat;
    p.b_r = idx1(d);
    p.b_k = idx1(1);
    p.C = Y;
    p.c_r = idx1(d);
    p.c_c = idx1(1);
    p.flags |= kGemmConstB;
    return p;
  }
  // Y(i, c) with c = (o, n): sum_j Mat(i, j) X(c, j)
  p.M = (int32_t)d;
  p.N = (int32_t)(outer * inner);
  p.K = (int32_t)d;
  p.flags |= kGemmConstA;
  p.A = Mat;
  p.a_r = idx1(d);
  p.a_k = idx1(1);
  p.B = X;
  p.b_r = (outer == 1) ? idx1(1) : idx2(inner, d * inner, 1);
  p.b_k = idx1(inner);
  p.C = Y;
  p.c_r = idx1(inner);
  p.c_c = (outer == 1) ? idx1(1) : idx2(inner, d * inner, 1);
  return p;
}

GemmProblem make_gemm(bool ta, bool tb, int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, const void* B,
                      int64_t ldb, void* C, int64_t ldc, double alpha, double beta) {
  GemmProblem p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.flags = beta != 0.0 ? kGemmReadC : 0;
  p.A = A;
  p.a_r = ta ? idx1(1) : idx1(lda);
  p.a_k = ta ? idx1(lda) : idx1(1);
  p.B = B;
  p.b_r = tb ? idx1(ldb) : idx1(1);
  p.b_k = tb ? idx1(1) : idx1(ldb);
  p.C = C;
  p.c_r = idx1(ldc);
  p.c_c = idx1(1);
  p.alpha = alpha;
  p.beta = beta;
  return p;
}

}  // namespace shampoo
