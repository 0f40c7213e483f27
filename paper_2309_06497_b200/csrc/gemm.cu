// Grouped strided GEMM / GEMV kernels (see gemm.cuh).
//
// Tile 64x64x16, 256 threads, 4x4 register micro-tile per thread.  Each warp
// covers a 16x32 sub-tile (4 row groups x 8 column groups) so that the
// per-k shared-memory reads are broadcast-friendly: 4 wavefronts per 16 DFMA
// issue slots, i.e. the FP64 pipe, not shared memory, is the limiter.
// Global->register prefetch of the next k-slab overlaps the current one.
#include <algorithm>
#include <cmath>

#include "gemm.cuh"

namespace shampoo {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256, PAD = 4;

__device__ __forceinline__ int64_t ev(const Idx2& x, int32_t v) {
  if (x.div == 0x7fffffff) return (int64_t)v * x.lo;
  return (int64_t)(v / x.div) * x.hi + (int64_t)(v % x.div) * x.lo;
}

// Load 4 elements of a 64x16 operand slab into registers.
template <typename T>
__device__ __forceinline__ void load_slab(const T* __restrict__ X, const Idx2& xr, const Idx2& xk,
                                          int rows, int K, int r0, int k0, bool kfast, T (&v)[4]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    int r, k;
    if (kfast) {
      const int f = tid * 4 + e;  // 4 consecutive k per thread
      r = f / BK;
      k = f % BK;
    } else {
      r = tid % BM;  // consecutive threads -> consecutive rows
      k = tid / BM + 4 * e;
    }
    const int gr = r0 + r, gk = k0 + k;
    v[e] = (gr < rows && gk < K) ? X[ev(xr, gr) + ev(xk, gk)] : T(0);
  }
}

template <typename T>
__device__ __forceinline__ void store_slab(T (*S)[BM + PAD], bool kfast, const T (&v)[4]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    int r, k;
    if (kfast) {
      const int f = tid * 4 + e;
      r = f / BK;
      k = f % BK;
    } else {
      r = tid % BM;
      k = tid / BM + 4 * e;
    }
    S[k][r] = v[e];
  }
}

__device__ __forceinline__ void tri_index(int64_t l, int& tm, int& tn) {
  // l -> (tm, tn) with tm >= tn, row-major over the lower triangle
  int r = (int)((sqrt(8.0 * (double)l + 1.0) - 1.0) * 0.5);
  while ((int64_t)(r + 1) * (r + 2) / 2 <= l) ++r;
  while ((int64_t)r * (r + 1) / 2 > l) --r;
  tm = r;
  tn = (int)(l - (int64_t)r * (r + 1) / 2);
}

template <typename T>
__global__ void __launch_bounds__(NT) grouped_gemm_kernel(const GemmProblem* __restrict__ probs,
                                                          const int64_t* __restrict__ begin,
                                                          int nprob, const int32_t* __restrict__ mask) {
  __shared__ __align__(16) T As[2][BK][BM + PAD];
  __shared__ __align__(16) T Bs[2][BK][BN + PAD];

  // locate problem: last p with begin[p] <= blockIdx.x
  const int64_t tile = blockIdx.x;
  int lo = 0, hi = nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (begin[mid] <= tile) lo = mid;
    else hi = mid - 1;
  }
  const GemmProblem& P = probs[lo];
  if ((P.flags & kGemmMasked) && mask && mask[P.mask_index] == 0) return;
  const int64_t lt = tile - begin[lo];
  int tm, tn;
  if (P.flags & kGemmSym) {
    tri_index(lt, tm, tn);
  } else {
    tm = (int)(lt / P.tiles_n);
    tn = (int)(lt % P.tiles_n);
  }
  const int m0 = tm * BM, n0 = tn * BN;
  const T* __restrict__ A = static_cast<const T*>(P.A);
  const T* __restrict__ B = static_cast<const T*>(P.B);
  const bool akf = (P.a_k.lo == 1), bkf = (P.b_k.lo == 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ty = (warp >> 1) * 4 + (lane >> 3);  // 0..15
  const int tx = (warp & 1) * 8 + (lane & 7);    // 0..15

  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);

  T ra[4], rb[4];
  const int nk = (P.K + BK - 1) / BK;
  load_slab<T>(A, P.a_r, P.a_k, P.M, P.K, m0, 0, akf, ra);
  load_slab<T>(B, P.b_r, P.b_k, P.N, P.K, n0, 0, bkf, rb);
  store_slab<T>(As[0], akf, ra);
  store_slab<T>(Bs[0], bkf, rb);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) {
      load_slab<T>(A, P.a_r, P.a_k, P.M, P.K, m0, (kt + 1) * BK, akf, ra);
      load_slab<T>(B, P.b_r, P.b_k, P.N, P.K, n0, (kt + 1) * BK, bkf, rb);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[cur][kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[cur][kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (kt + 1 < nk) {
      store_slab<T>(As[cur ^ 1], akf, ra);
      store_slab<T>(Bs[cur ^ 1], bkf, rb);
    }
    __syncthreads();
  }

  T* __restrict__ C = static_cast<T*>(P.C);
  const T alpha = T(P.alpha), beta = T(P.beta);
  const bool readc = (P.flags & kGemmReadC) != 0;
  const bool mirror = (P.flags & kGemmSym) && tm != tn;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gi = m0 + ty * 4 + i;
    if (gi >= P.M) continue;
    const int64_t ri = ev(P.c_r, gi);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gj = n0 + tx * 4 + j;
      if (gj >= P.N) continue;
      const int64_t at = ri + ev(P.c_c, gj);
      T v = alpha * acc[i][j];
      if (readc) v = fma(beta, C[at], v);
      C[at] = v;
      if (mirror) C[ev(P.c_r, gj) + ev(P.c_c, gi)] = v;
    }
  }
}

// One warp per output row; CTA = 8 rows.
template <typename T>
__global__ void __launch_bounds__(256) grouped_gemv_kernel(const GemvProblem* __restrict__ probs,
                                                           const int64_t* __restrict__ begin,
                                                           int nprob, const int32_t* __restrict__ mask) {
  const int64_t g = blockIdx.x;
  int lo = 0, hi = nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (begin[mid] <= g) lo = mid;
    else hi = mid - 1;
  }
  const GemvProblem& P = probs[lo];
  if (mask && mask[P.mask_index] == 0) return;
  const int row = (int)(g - begin[lo]) * 8 + (threadIdx.x >> 5);
  if (row >= P.n) return;
  const T* __restrict__ X = static_cast<const T*>(P.X) + (int64_t)row * P.n;
  const T* __restrict__ x = static_cast<const T*>(P.x);
  T s = 0;
  for (int j = threadIdx.x & 31; j < P.n; j += 32) s = fma(X[j], x[j], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) static_cast<T*>(P.y)[row] = T(P.alpha) * s;
}

}  // namespace

template <typename T>
GemmBatch<T>::~GemmBatch() {
  cudaFree(d_prob_);
  cudaFree(d_begin_);
}

template <typename T>
int GemmBatch<T>::upload() {
  cudaFree(d_prob_);
  cudaFree(d_begin_);
  d_prob_ = nullptr;
  d_begin_ = nullptr;
  total_tiles_ = 0;
  if (host.empty()) return SHAMPOO_OK;
  std::vector<int64_t> begin(host.size());
  for (size_t i = 0; i < host.size(); ++i) {
    GemmProblem& p = host[i];
    p.tiles_m = (p.M + BM - 1) / BM;
    p.tiles_n = (p.N + BN - 1) / BN;
    p.tiles = (p.flags & kGemmSym) ? (int64_t)p.tiles_m * (p.tiles_m + 1) / 2
                                   : (int64_t)p.tiles_m * p.tiles_n;
    if (p.M == 0 || p.N == 0) p.tiles = 0;
    begin[i] = total_tiles_;
    total_tiles_ += p.tiles;
  }
  SH_CUDA_CHECK(cudaMalloc(&d_prob_, host.size() * sizeof(GemmProblem)));
  SH_CUDA_CHECK(cudaMalloc(&d_begin_, host.size() * sizeof(int64_t)));
  SH_CUDA_CHECK(cudaMemcpy(d_prob_, host.data(), host.size() * sizeof(GemmProblem), cudaMemcpyHostToDevice));
  SH_CUDA_CHECK(cudaMemcpy(d_begin_, begin.data(), begin.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  return SHAMPOO_OK;
}

template <typename T>
int GemmBatch<T>::launch(cudaStream_t s, const int32_t* mask) const {
  if (total_tiles_ == 0) return SHAMPOO_OK;
  grouped_gemm_kernel<T><<<(unsigned)total_tiles_, NT, 0, s>>>(d_prob_, d_begin_, (int)host.size(), mask);
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

template <typename T>
double GemmBatch<T>::flops() const {
  double f = 0;
  for (const auto& p : host) f += 2.0 * p.M * (double)p.N * p.K;
  return f;
}

template <typename T>
GemvBatch<T>::~GemvBatch() {
  cudaFree(d_prob_);
  cudaFree(d_begin_);
}

template <typename T>
int GemvBatch<T>::upload() {
  cudaFree(d_prob_);
  cudaFree(d_begin_);
  d_prob_ = nullptr;
  d_begin_ = nullptr;
  total_groups_ = 0;
  if (host.empty()) return SHAMPOO_OK;
  std::vector<int64_t> begin(host.size());
  for (size_t i = 0; i < host.size(); ++i) {
    begin[i] = total_groups_;
    total_groups_ += (host[i].n + 7) / 8;
  }
  SH_CUDA_CHECK(cudaMalloc(&d_prob_, host.size() * sizeof(GemvProblem)));
  SH_CUDA_CHECK(cudaMalloc(&d_begin_, host.size() * sizeof(int64_t)));
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

template class GemmBatch<double>;
template class GemmBatch<float>;
template class GemvBatch<double>;
template class GemvBatch<float>;

GemmProblem make_mode_gram(const void* X, int64_t outer, int64_t d, int64_t inner, void* C,
                           double alpha, double beta) {
  GemmProblem p{};
  p.M = p.N = (int32_t)d;
  p.K = (int32_t)(outer * inner);
  p.flags = kGemmSym | (beta != 0.0 ? kGemmReadC : 0);
  p.A = p.B = X;
  p.a_r = p.b_r = idx1(inner);
  p.a_k = p.b_k = (inner == 1) ? idx1(d) : idx2(inner, d * inner, 1);
  if (inner == 1) p.a_k = p.b_k = Idx2{0x7fffffff, 0, 0, d};
  p.C = C;
  p.c_r = idx1(d);
  p.c_c = idx1(1);
  p.alpha = alpha;
  p.beta = beta;
  return p;
}

GemmProblem make_mode_product(const void* Mat, const void* X, void* Y, int64_t outer, int64_t d,
                              int64_t inner, double alpha) {
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
    return p;
  }
  // Y(i, c) with c = (o, n): sum_j Mat(i, j) X(c, j)
  p.M = (int32_t)d;
  p.N = (int32_t)(outer * inner);
  p.K = (int32_t)d;
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

GemmProblem make_gemm(bool ta, bool tb, int32_t M, int32_t N, int32_t K, const void* A, int64_t lda,
                      const void* B, int64_t ldb, void* C, int64_t ldc, double alpha, double beta) {
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
