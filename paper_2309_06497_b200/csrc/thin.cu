// Thin problems of the grouped GEMM phases (see thin.cuh): HBM-bound CUDA-core kernels with
// exact products and FP64 accumulation in a fixed order (deterministic).
#include <algorithm>

#include "thin.cuh"

namespace shampoo {

namespace {

constexpr int KRED_CHUNK = 4096;  // k per CTA of the small-M/N reduction
constexpr int TMAX = 8;           // M, N <= 8 for the reduction kernel
constexpr int KOUT_ITEMS = 2048;  // outputs per CTA of the small-K kernel

__device__ __forceinline__ int64_t ev(const Idx2& x, int64_t v) {
  if (x.div == 0x7fffffff) return v * x.lo;
  const uint32_t q = (uint32_t)v / (uint32_t)x.div;  // indices are < 2^31: 32-bit division
  return (int64_t)q * x.hi + (int64_t)((uint32_t)v - q * (uint32_t)x.div) * x.lo;
}

__device__ __forceinline__ int find64(const int64_t* __restrict__ begin, int n, int64_t x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (begin[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

template <typename T>
__device__ __forceinline__ void thin_store(const GemmProblem& P, int i, int j, double acc) {
  T* __restrict__ C = static_cast<T*>(P.C);
  const int64_t at = ev(P.c_r, i) + ev(P.c_c, j);
  double v = P.alpha * acc;
  if (P.flags & kGemmReadC) v = fma(P.beta, (double)C[at], v);
  C[at] = (T)v;
}

// Small K: one thread per output element; a CTA covers rows [r0, r0 + R) of one problem
// (R * N ~ 2048 outputs).  SYM problems are computed on the full square: the (i,j) and (j,i)
// sums see the same products in the same order, so C stays exactly symmetric with fully
// coalesced stores (no mirror writes).
template <typename T>
__global__ void __launch_bounds__(256) k_thin_kout(const GemmProblem* __restrict__ probs,
                                                   const int64_t* __restrict__ begin, int nprob,
                                                   const int32_t* __restrict__ mask) {
  const int p = find64(begin, nprob, blockIdx.x);
  const GemmProblem P = probs[p];  // by value: fields stay in registers across the stores to C
  if ((P.flags & kGemmMasked) && mask && !mask[P.mask_index]) return;
  // CTA item = (block of R rows, chunk of KOUT_ITEMS columns): wide problems spread over many CTAs
  const int R = max(1, KOUT_ITEMS / P.N);
  const int nchunk = (P.N + KOUT_ITEMS - 1) / KOUT_ITEMS;
  const int64_t item = blockIdx.x - begin[p];
  const int r0 = (int)(item / nchunk) * R;
  const int cbeg = (int)(item % nchunk) * KOUT_ITEMS, cend = min(P.N, cbeg + KOUT_ITEMS);
  const int rows = min(R, P.M - r0);
  const T* __restrict__ A = static_cast<const T*>(P.A);
  const T* __restrict__ B = static_cast<const T*>(P.B);
  T* __restrict__ C = static_cast<T*>(P.C);
  const bool readc = (P.flags & kGemmReadC) != 0;
  if (P.N <= 8 && P.K <= 8) {
    // tall and narrow (the 3x3 / 7x7 kernel modes: M up to ~10^6, N = K = 3): a thread per row,
    // its K inputs loaded once, the N x K operand in shared memory; same k order as below
    __shared__ double bs[64];
    for (int t = threadIdx.x; t < P.N * P.K; t += blockDim.x) bs[t] = (double)B[ev(P.b_r, t / P.K) + ev(P.b_k, t % P.K)];
    __syncthreads();
    for (int i = r0 + threadIdx.x; i < r0 + rows; i += blockDim.x) {
      const int64_t ai = ev(P.a_r, i), ci = ev(P.c_r, i);
      double a[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = k < P.K ? (double)A[ai + ev(P.a_k, k)] : 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j >= P.N) break;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < P.K) acc = fma(a[k], bs[j * P.K + k], acc);
        const int64_t at = ci + ev(P.c_c, j);
        double v = P.alpha * acc;
        if (readc) v = fma(P.beta, (double)C[at], v);
        C[at] = (T)v;
      }
    }
    return;
  }
  if (P.N >= 64) {  // wide rows: row loop outside, coalesced column loop inside (no divisions)
    for (int i = r0; i < r0 + rows; ++i) {
      const int64_t ai = ev(P.a_r, i), ci = ev(P.c_r, i);
      for (int j = cbeg + threadIdx.x; j < cend; j += blockDim.x) {
        const int64_t bj = ev(P.b_r, j);
        double acc = 0.0;
        for (int k = 0; k < P.K; ++k) acc = fma((double)A[ai + ev(P.a_k, k)], (double)B[bj + ev(P.b_k, k)], acc);
        const int64_t at = ci + ev(P.c_c, j);
        double v = P.alpha * acc;
        if (readc) v = fma(P.beta, (double)C[at], v);
        C[at] = (T)v;
      }
    }
    return;
  }
  for (int e = threadIdx.x; e < rows * P.N; e += blockDim.x) {
    const int i = r0 + e / P.N, j = e % P.N;
    const int64_t ai = ev(P.a_r, i), bj = ev(P.b_r, j);
    double acc = 0.0;
    for (int k = 0; k < P.K; ++k) acc = fma((double)A[ai + ev(P.a_k, k)], (double)B[bj + ev(P.b_k, k)], acc);
    const int64_t at = ev(P.c_r, i) + ev(P.c_c, j);
    double v = P.alpha * acc;
    if (readc) v = fma(P.beta, (double)C[at], v);
    C[at] = (T)v;
  }
}

// Rank-1 symmetric update C = beta C + alpha x x^T of a contiguous row-major C (the factor EMA of
// a vector block, precond.py:232-242): CTA per (problem, row), 16-byte accesses.  With
// kGemmLowerOnly only columns j <= i are written (the statistics keep lower triangles; k_symmetrize
// restores the upper ones), else the full row -- x_i x_j == x_j x_i exactly, so the square stays
// bitwise symmetric.
template <typename T>
__global__ void __launch_bounds__(256) k_thin_rank1(const GemmProblem* __restrict__ probs,
                                                    const int64_t* __restrict__ begin, int nprob,
                                                    const int32_t* __restrict__ mask) {
  const int p = find64(begin, nprob, blockIdx.x);
  const GemmProblem P = probs[p];  // by value: fields stay in registers across the stores to C
  if ((P.flags & kGemmMasked) && mask && !mask[P.mask_index]) return;
  // lower-only: CTA per row pair (i, N-1-i), i + 1 + N - i = N + 1 elements -- balanced work
  const bool lower = (P.flags & kGemmLowerOnly) != 0;
  const int item = (int)(blockIdx.x - begin[p]);
  for (int h = 0; h < (lower ? 2 : 1); ++h) {
  const int i = lower ? (h == 0 ? item : P.N - 1 - item) : item;
  if (h == 1 && i == item) break;  // odd N: the middle row once
  const T* __restrict__ x = static_cast<const T*>(P.A);
  T* __restrict__ row = static_cast<T*>(P.C) + (int64_t)i * P.N;
  const double xi = (double)x[ev(P.a_r, i)];
  const bool readc = (P.flags & kGemmReadC) != 0;
  const int64_t step = P.a_r.lo;
  const int jend = lower ? i + 1 : P.N;
  if (sizeof(T) == 8 && step == 1 && ((reinterpret_cast<uintptr_t>(row) | reinterpret_cast<uintptr_t>(x)) & 15) == 0) {
    const double2* __restrict__ x2 = reinterpret_cast<const double2*>(x);
    double2* __restrict__ r2 = reinterpret_cast<double2*>(row);
    const int npair = jend / 2;
    for (int q = threadIdx.x; q < npair; q += blockDim.x) {
      const double2 xv = x2[q];
      double2 cv = readc ? r2[q] : make_double2(0.0, 0.0);
      double v0 = P.alpha * (xi * xv.x), v1 = P.alpha * (xi * xv.y);
      if (readc) {
        v0 = fma(P.beta, cv.x, v0);
        v1 = fma(P.beta, cv.y, v1);
      }
      r2[q] = make_double2(v0, v1);
    }
    if ((jend & 1) && threadIdx.x == 0) {  // odd tail (the diagonal of an even row)
      const int j = jend - 1;
      double v = P.alpha * (xi * (double)x[j]);
      if (readc) v = fma(P.beta, (double)row[j], v);
      row[j] = (T)v;
    }
    continue;
  }
  for (int j = threadIdx.x; j < jend; j += blockDim.x) {
    double v = P.alpha * (xi * (double)x[j * step]);
    if (readc) v = fma(P.beta, (double)row[j], v);
    row[j] = (T)v;
  }
  }
}

// Small M and N (<= TB <= 8), any K: CTA per (problem, 4096-wide k chunk) -> FP64 partials (layout
// TMAX x TMAX per chunk).  TB = 4 for the 3 x 3 kernel modes: 16 accumulators instead of 64 (the
// 8 x 8 variant ran at one CTA per SM on its 187 registers).
template <typename T, int TB>
__global__ void __launch_bounds__(256) k_thin_kred(const GemmProblem* __restrict__ probs,
                                                   const int64_t* __restrict__ begin, int nprob,
                                                   const int32_t* __restrict__ mask, const int64_t* __restrict__ woff,
                                                   double* __restrict__ ws) {
  __shared__ double red[TB * TB][8];
  const int p = find64(begin, nprob, blockIdx.x);
  const GemmProblem P = probs[p];  // by value: fields stay in registers across the stores to C
  if ((P.flags & kGemmMasked) && mask && !mask[P.mask_index]) return;
  const int chunk = (int)(blockIdx.x - begin[p]);
  const T* __restrict__ A = static_cast<const T*>(P.A);
  const T* __restrict__ B = static_cast<const T*>(P.B);
  double acc[TB][TB];
#pragma unroll
  for (int i = 0; i < TB; ++i)
#pragma unroll
    for (int j = 0; j < TB; ++j) acc[i][j] = 0.0;
  const int k0 = chunk * KRED_CHUNK, k1 = min(P.K, k0 + KRED_CHUNK);
  int64_t ar[TB], br[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    ar[i] = i < P.M ? ev(P.a_r, i) : 0;
    br[i] = i < P.N ? ev(P.b_r, i) : 0;
  }
  for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
    double a[TB], b[TB];
    const int64_t ak = ev(P.a_k, k), bk = ev(P.b_k, k);
#pragma unroll
    for (int i = 0; i < TB; ++i) {
      a[i] = i < P.M ? (double)A[ar[i] + ak] : 0.0;
      b[i] = i < P.N ? (double)B[br[i] + bk] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < TB; ++i)
#pragma unroll
      for (int j = 0; j < TB; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
  }
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < TB; ++i)
#pragma unroll
    for (int j = 0; j < TB; ++j) {
      const double v = warp_sum(acc[i][j]);
      if (ln == 0) red[i * TB + j][w] = v;
    }
  __syncthreads();
  if (threadIdx.x < TMAX * TMAX) {
    const int i = threadIdx.x / TMAX, j = threadIdx.x % TMAX;
    double v = 0.0;
    if (i < TB && j < TB)
      for (int q = 0; q < 8; ++q) v += red[i * TB + j][q];
    ws[woff[p] + (int64_t)chunk * TMAX * TMAX + threadIdx.x] = v;
  }
}

// Chunk partials -> C: a warp per output element, lanes over the chunks (fixed order), then a
// fixed-shape warp tree (deterministic).
template <typename T>
__global__ void __launch_bounds__(256) k_thin_kred_final(const GemmProblem* __restrict__ probs, int nprob,
                                                         const int32_t* __restrict__ mask,
                                                         const int64_t* __restrict__ woff,
                                                         const int32_t* __restrict__ nchunks,
                                                         const double* __restrict__ ws) {
  const int p = blockIdx.x;
  const GemmProblem P = probs[p];  // by value: fields stay in registers across the stores to C
  if ((P.flags & kGemmMasked) && mask && !mask[P.mask_index]) return;
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  for (int e = w; e < TMAX * TMAX; e += 8) {
    const int i = e / TMAX, j = e % TMAX;
    if (i >= P.M || j >= P.N) continue;
    double acc = 0.0;
    for (int c = ln; c < nchunks[p]; c += 32) acc += ws[woff[p] + (int64_t)c * TMAX * TMAX + e];
    acc = warp_sum(acc);
    if (ln == 0) thin_store<T>(P, i, j, acc);
  }
}

}  // namespace

bool ThinGemmBatch_accepts(const GemmProblem& p) { return p.K <= 32 || (p.M <= TMAX && p.N <= TMAX); }

// x x^T with x contiguous (stride a_r.lo), C row-major contiguous: the vector-block factor update
static bool is_rank1(const GemmProblem& p) {
  return p.K == 1 && (p.flags & kGemmSym) && p.A == p.B && p.M == p.N && p.a_r.div == 0x7fffffff &&
         p.c_r.div == 0x7fffffff && p.c_c.div == 0x7fffffff && p.c_r.lo == p.N && p.c_c.lo == 1;
}

template <typename T>
ThinGemmBatch<T>::~ThinGemmBatch() {
  dev_free(d_r1_);
  dev_free(d_r1begin_);
  dev_free(d_out_);
  dev_free(d_obegin_);
  dev_free(d_red_);
  dev_free(d_rbegin_);
  dev_free(d_rbegin8_);
  dev_free(d_woff_);
  dev_free(d_nch_);
  dev_free(ws_);
}

template <typename T>
int ThinGemmBatch<T>::upload() {
  std::vector<GemmProblem> outp, redp, r1p;
  std::vector<GemmProblem> red8;
  for (const auto& p : host) {
    if (is_rank1(p)) r1p.push_back(p);
    else if (p.K <= 32) outp.push_back(p);
    else if (p.M <= 4 && p.N <= 4) redp.push_back(p);
    else red8.push_back(p);
  }
  n_red4_ = (int)redp.size();
  redp.insert(redp.end(), red8.begin(), red8.end());
  std::vector<int64_t> r1b;
  n_r1_ctas_ = 0;
  for (const auto& p : r1p) {  // CTA per row (lower-only: per row pair)
    r1b.push_back(n_r1_ctas_);
    n_r1_ctas_ += (p.flags & kGemmLowerOnly) ? (p.M + 1) / 2 : p.M;
  }
  n_r1_ = (int)r1p.size();
  if (n_r1_) {
    SH_CUDA_CHECK(dev_malloc(&d_r1_, r1p.size() * sizeof(GemmProblem)));
    SH_CUDA_CHECK(dev_malloc(&d_r1begin_, r1b.size() * sizeof(int64_t)));
    SH_CUDA_CHECK(cudaMemcpy(d_r1_, r1p.data(), r1p.size() * sizeof(GemmProblem), cudaMemcpyHostToDevice));
    SH_CUDA_CHECK(cudaMemcpy(d_r1begin_, r1b.data(), r1b.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  std::vector<int64_t> ob, rb, wo;
  std::vector<int32_t> nch;
  n_out_items_ = 0;  // CTAs
  for (const auto& p : outp) {
    ob.push_back(n_out_items_);
    const int R = std::max(1, KOUT_ITEMS / std::max(p.N, 1));
    const int nchunk = std::max(1, (p.N + KOUT_ITEMS - 1) / KOUT_ITEMS);
    n_out_items_ += (int64_t)((p.M + R - 1) / R) * nchunk;
  }
  n_red_ctas_ = 0;
  n_red4_ctas_ = 0;
  int64_t wsz = 0;
  for (size_t q = 0; q < redp.size(); ++q) {
    const GemmProblem& p = redp[q];
    const int c = std::max(1, (p.K + KRED_CHUNK - 1) / KRED_CHUNK);
    if ((int)q == n_red4_) n_red4_ctas_ = n_red_ctas_;
    rb.push_back(n_red_ctas_);
    wo.push_back(wsz);
    nch.push_back(c);
    n_red_ctas_ += c;
    wsz += (int64_t)c * TMAX * TMAX;
  }
  if (n_red4_ == (int)redp.size()) n_red4_ctas_ = n_red_ctas_;
  n_out_ = (int)outp.size();
  n_red_ = (int)redp.size();
  if (n_out_) {
    SH_CUDA_CHECK(dev_malloc(&d_out_, outp.size() * sizeof(GemmProblem)));
    SH_CUDA_CHECK(dev_malloc(&d_obegin_, ob.size() * sizeof(int64_t)));
    SH_CUDA_CHECK(cudaMemcpy(d_out_, outp.data(), outp.size() * sizeof(GemmProblem), cudaMemcpyHostToDevice));
    SH_CUDA_CHECK(cudaMemcpy(d_obegin_, ob.data(), ob.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  if (n_red_) {
    SH_CUDA_CHECK(dev_malloc(&d_red_, redp.size() * sizeof(GemmProblem)));
    SH_CUDA_CHECK(dev_malloc(&d_rbegin_, rb.size() * sizeof(int64_t)));
    SH_CUDA_CHECK(dev_malloc(&d_woff_, wo.size() * sizeof(int64_t)));
    SH_CUDA_CHECK(dev_malloc(&d_nch_, nch.size() * sizeof(int32_t)));
    SH_CUDA_CHECK(dev_malloc(&ws_, wsz * sizeof(double)));
    SH_CUDA_CHECK(cudaMemcpy(d_red_, redp.data(), redp.size() * sizeof(GemmProblem), cudaMemcpyHostToDevice));
    SH_CUDA_CHECK(cudaMemcpy(d_rbegin_, rb.data(), rb.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    if (n_red_ > n_red4_) {  // CTA prefix of the M/N <= 8 problems, relative to their own launch
      std::vector<int64_t> rb8(rb.begin() + n_red4_, rb.end());
      for (auto& x : rb8) x -= n_red4_ctas_;
      SH_CUDA_CHECK(dev_malloc(&d_rbegin8_, rb8.size() * sizeof(int64_t)));
      SH_CUDA_CHECK(cudaMemcpy(d_rbegin8_, rb8.data(), rb8.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    }
    SH_CUDA_CHECK(cudaMemcpy(d_woff_, wo.data(), wo.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    SH_CUDA_CHECK(cudaMemcpy(d_nch_, nch.data(), nch.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  return SHAMPOO_OK;
}

template <typename T>
int ThinGemmBatch<T>::launch(cudaStream_t s, const int32_t* mask) const {
  if (n_r1_) {
    k_thin_rank1<T><<<(unsigned)n_r1_ctas_, 256, 0, s>>>(d_r1_, d_r1begin_, n_r1_, mask);
    SH_LAUNCH_CHECK();
  }
  if (n_out_) {
    k_thin_kout<T><<<(unsigned)n_out_items_, 256, 0, s>>>(d_out_, d_obegin_, n_out_, mask);
    SH_LAUNCH_CHECK();
  }
  if (n_red_) {
    // problems [0, n_red4_) have M, N <= 4 (CTAs [0, n_red4_ctas_)); the rest up to 8
    if (n_red4_) {
      k_thin_kred<T, 4><<<(unsigned)n_red4_ctas_, 256, 0, s>>>(d_red_, d_rbegin_, n_red4_, mask, d_woff_, ws_);
      SH_LAUNCH_CHECK();
    }
    if (n_red_ > n_red4_) {
      k_thin_kred<T, TMAX><<<(unsigned)(n_red_ctas_ - n_red4_ctas_), 256, 0, s>>>(
          d_red_ + n_red4_, d_rbegin8_, n_red_ - n_red4_, mask, d_woff_ + n_red4_, ws_);
      SH_LAUNCH_CHECK();
    }
    k_thin_kred_final<T><<<n_red_, 256, 0, s>>>(d_red_, n_red_, mask, d_woff_, d_nch_, ws_);
    SH_LAUNCH_CHECK();
  }
  return SHAMPOO_OK;
}

template <typename T>
double ThinGemmBatch<T>::flops() const {
  double f = 0;
  for (const auto& p : host) f += 2.0 * p.M * (double)p.N * p.K;
  return f;
}

template class ThinGemmBatch<float>;
template class ThinGemmBatch<double>;

}  // namespace shampoo
