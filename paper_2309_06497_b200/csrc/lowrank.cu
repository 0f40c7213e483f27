// Root inverse of structurally low-rank factors (see lowrank.cuh).
#include <algorithm>
#include <cmath>

#include "lowrank.cuh"
#include "rootinv.cuh"
#include "tcgen05.cuh"

namespace shampoo {

namespace {

constexpr int LR_ECH = 4096;  // elements per chunk of the elementwise kernels

struct LRDev {
  int32_t d, r;
  int64_t q_off, t_off, z_off;  // r x d arrays (Q rows, T = Q A, Z = M Q)
  int64_t b_off, xb_off;        // r x r arrays (B, f(B))
  int64_t x_off;                // d x d expansion
  const double* in;
  double* out;
  double f0;                    // f(0) = eps^(-eta/p) on the null space
  double idscale;               // identity fallback eps^(-eta/p) (or 1 if eps = 0)
  int32_t has_prev;
  int32_t bad;                  // set by the kernels: non-finite result
};

__device__ __forceinline__ int lr_find(const int32_t* __restrict__ begin, int n, int x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (begin[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Omega^T (r x d) Gaussian, counter-based (deterministic): written into the T slot (Y = Omega^T A -> Q).
__global__ void __launch_bounds__(256) k_lr_gauss(const LRDev* __restrict__ jobs, const int32_t* __restrict__ cbegin,
                                                  int njobs, double* __restrict__ ws) {
  const int j = lr_find(cbegin, njobs, blockIdx.x);
  const LRDev& J = jobs[j];
  const int64_t tot = (int64_t)J.r * J.d;
  const int64_t base = (int64_t)(blockIdx.x - cbegin[j]) * LR_ECH;
  for (int64_t e = base + threadIdx.x; e < base + LR_ECH && e < tot; e += blockDim.x) {
    const uint64_t key = ((uint64_t)j << 40) ^ (uint64_t)e;
    const double u1 = ((splitmix64(2 * key) >> 11) + 1) * 0x1.0p-53;  // (0, 1]
    const double u2 = (splitmix64(2 * key + 1) >> 11) * 0x1.0p-53;
    ws[J.t_off + e] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

// CGS2 on the r rows of Y (in place -> orthonormal Q rows), one CTA per factor.  A row whose norm
// collapses (Y rank deficient: rank(A) < r) is replaced by a unit vector and re-orthogonalised:
// the extra directions are null directions of A (B vanishes there), so f(A) is unchanged.
__global__ void __launch_bounds__(256) k_lr_cgs2(LRDev* jobs, double* __restrict__ ws) {
  extern __shared__ double h[];
  __shared__ double red[32];
  LRDev& J = jobs[blockIdx.x];
  const int d = J.d;
  double* Q = ws + J.q_off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = 0; j < J.r; ++j) {
    double* w = Q + (int64_t)j * d;
    double n0 = 0.0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) n0 = fma(w[i], w[i], n0);
    n0 = sqrt(block_sum<double, 256>(n0, red));
    for (int attempt = 0; attempt < 3; ++attempt) {
      for (int pass = 0; pass < 2; ++pass) {
        for (int k = warp; k < j; k += nw) {  // h_k = <q_k, w>
          const double* qk = Q + (int64_t)k * d;
          double s = 0.0;
          for (int i = lane; i < d; i += 32) s = fma(qk[i], w[i], s);
          s = warp_sum(s);
          if (lane == 0) h[k] = s;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < d; i += blockDim.x) {  // w -= sum_k h_k q_k
          double acc = w[i];
          for (int k = 0; k < j; ++k) acc = fma(-h[k], Q[(int64_t)k * d + i], acc);
          w[i] = acc;
        }
        __syncthreads();
      }
      double nrm = 0.0;
      for (int i = threadIdx.x; i < d; i += blockDim.x) nrm = fma(w[i], w[i], nrm);
      nrm = sqrt(block_sum<double, 256>(nrm, red));
      if (nrm > 1e-13 * n0 && nrm > 0.0 && isfinite(nrm)) {  // above the rounding floor of CGS2
        const double inv = 1.0 / nrm;
        for (int i = threadIdx.x; i < d; i += blockDim.x) w[i] *= inv;
        break;
      }
      // dependent row: a unit vector e_c, c cycling over the coordinates, then orthogonalise again
      const int c = (j * 7919 + attempt * 104729) % d;
      for (int i = threadIdx.x; i < d; i += blockDim.x) w[i] = (i == c) ? 1.0 : 0.0;
      n0 = 1.0;
      __syncthreads();
      if (attempt == 2 && threadIdx.x == 0) J.bad = 1;
    }
    __syncthreads();
  }
}

// B <- (B + B^T)/2 ; M = f(B) - f0 I is formed in place of f(B) later.
__global__ void k_lr_symb(const LRDev* __restrict__ jobs, double* __restrict__ ws) {
  const LRDev& J = jobs[blockIdx.x];
  double* B = ws + J.b_off;
  for (int e = threadIdx.x; e < J.r * J.r; e += blockDim.x) {
    const int i = e / J.r, k = e % J.r;
    if (i < k) {
      const double v = 0.5 * (B[e] + B[k * J.r + i]);
      B[e] = v;
      B[k * J.r + i] = v;
    }
  }
}

__global__ void k_lr_shift(const LRDev* __restrict__ jobs, double* __restrict__ ws) {
  const LRDev& J = jobs[blockIdx.x];
  double* M = ws + J.xb_off;
  for (int i = threadIdx.x; i < J.r; i += blockDim.x) M[i * J.r + i] -= J.f0;
}

// out = sym(X) + f0 I with the guard: non-finite (or a failed compressed solve) -> previous (left
// untouched) or eps^(-eta/p) I.
__global__ void __launch_bounds__(256) k_lr_check(LRDev* jobs, const int32_t* __restrict__ xbegin, int njobs,
                                                  const double* __restrict__ ws) {
  const int j = lr_find(xbegin, njobs, blockIdx.x);
  LRDev& J = jobs[j];
  const int64_t tot = (int64_t)J.d * J.d;
  const int64_t base = (int64_t)(blockIdx.x - xbegin[j]) * LR_ECH;
  int bad = 0;
  for (int64_t e = base + threadIdx.x; e < base + LR_ECH && e < tot; e += blockDim.x)
    if (!isfinite(ws[J.x_off + e])) bad = 1;
  if (__syncthreads_or(bad) && threadIdx.x == 0) J.bad = 1;
}

__global__ void __launch_bounds__(256) k_lr_finish(const LRDev* __restrict__ jobs, const int32_t* __restrict__ xbegin,
                                                   int njobs, const double* __restrict__ ws) {
  const int j = lr_find(xbegin, njobs, blockIdx.x);
  const LRDev& J = jobs[j];
  if (J.bad && J.has_prev) return;
  const int d = J.d;
  const int64_t tot = (int64_t)d * d;
  const int64_t base = (int64_t)(blockIdx.x - xbegin[j]) * LR_ECH;
  const double* X = ws + J.x_off;
  for (int64_t e = base + threadIdx.x; e < base + LR_ECH && e < tot; e += blockDim.x) {
    const int64_t i = e / d, k = e % d;
    double v;
    if (J.bad) v = (i == k) ? J.idscale : 0.0;
    else v = 0.5 * (X[e] + X[k * d + i]) + (i == k ? J.f0 : 0.0);
    J.out[e] = v;
  }
}

}  // namespace

int low_rank_root_inverse(const std::vector<LowRankJob>& jobs, double in_scale, double eta, double eps,
                          cudaStream_t s, int64_t* stats) {
  const int nj = (int)jobs.size();
  if (nj == 0) return SHAMPOO_OK;
  std::vector<LRDev> hj(nj);
  std::vector<int32_t> cbeg(nj), xbeg(nj);
  int64_t ws = 0;
  int32_t cch = 0, xch = 0;
  int rmax = 1;
  for (int j = 0; j < nj; ++j) {
    const LowRankJob& L = jobs[j];
    LRDev& D = hj[j];
    D.d = L.d;
    D.r = L.r;
    const int64_t rd = (int64_t)L.r * L.d;
    D.q_off = ws;
    ws += rd;
    D.t_off = ws;
    ws += rd;
    D.z_off = ws;
    ws += rd;
    D.b_off = ws;
    ws += (int64_t)L.r * L.r;
    D.xb_off = ws;
    ws += (int64_t)L.r * L.r;
    D.x_off = ws;
    ws += (int64_t)L.d * L.d;
    D.in = L.in;
    D.out = L.out;
    D.f0 = eps > 0.0 ? std::pow(eps, -eta / L.root_p) : 0.0;
    D.idscale = eps > 0.0 ? std::pow(eps, -eta / L.root_p) : 1.0;
    D.has_prev = L.has_prev;
    D.bad = 0;
    cbeg[j] = cch;
    cch += (int32_t)((rd + LR_ECH - 1) / LR_ECH);
    xbeg[j] = xch;
    xch += (int32_t)(((int64_t)L.d * L.d + LR_ECH - 1) / LR_ECH);
    rmax = std::max(rmax, L.r);
  }
  double* w = nullptr;
  LRDev* dj = nullptr;
  int32_t *dc = nullptr, *dx = nullptr;
  SH_CUDA_CHECK(cudaMallocAsync(&w, ws * sizeof(double), s));
  SH_CUDA_CHECK(cudaMallocAsync(&dj, nj * sizeof(LRDev), s));
  SH_CUDA_CHECK(cudaMallocAsync(&dc, nj * sizeof(int32_t), s));
  SH_CUDA_CHECK(cudaMallocAsync(&dx, nj * sizeof(int32_t), s));
  SH_CUDA_CHECK(cudaMemcpyAsync(dj, hj.data(), nj * sizeof(LRDev), cudaMemcpyHostToDevice, s));
  SH_CUDA_CHECK(cudaMemcpyAsync(dc, cbeg.data(), nj * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  SH_CUDA_CHECK(cudaMemcpyAsync(dx, xbeg.data(), nj * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  int rc = SHAMPOO_OK;
  {
    // Y = Omega^T A (Omega^T in the T slot) ; T = Q A ; B = T Q^T ; Z = M Q ; X = Z^T Q
    OzakiGemmBatch<double> gy, gt, gb, gz, gx;
    for (int j = 0; j < nj; ++j) {
      const LRDev& D = hj[j];
      const int r = D.r, d = D.d;
      gy.add(make_gemm(false, false, r, d, d, w + D.t_off, d, D.in, d, w + D.q_off, d, in_scale, 0.0));
      gt.add(make_gemm(false, false, r, d, d, w + D.q_off, d, D.in, d, w + D.t_off, d, in_scale, 0.0));
      gb.add(make_gemm(false, true, r, r, d, w + D.t_off, d, w + D.q_off, d, w + D.b_off, r, 1.0, 0.0));
      gz.add(make_gemm(false, false, r, d, r, w + D.xb_off, r, w + D.q_off, d, w + D.z_off, d, 1.0, 0.0));
      gx.add(make_gemm(true, false, d, d, r, w + D.z_off, d, w + D.q_off, d, w + D.x_off, d, 1.0, 0.0));
    }
    for (auto* b : {&gy, &gt, &gb, &gz, &gx})
      if ((rc = b->upload())) return rc;
    k_lr_gauss<<<cch, 256, 0, s>>>(dj, dc, nj, w);
    SH_LAUNCH_CHECK();
    if ((rc = gy.launch(s))) return rc;
    k_lr_cgs2<<<nj, 256, rmax * sizeof(double), s>>>(dj, w);
    SH_LAUNCH_CHECK();
    if ((rc = gt.launch(s))) return rc;
    if ((rc = gb.launch(s))) return rc;
    k_lr_symb<<<nj, 256, 0, s>>>(dj, w);
    SH_LAUNCH_CHECK();
    // f(B) on the r x r compressions (Jacobi path; B carries the null directions of Q exactly)
    RootInverseBatch rb;
    std::vector<int32_t> rn(nj), rp(nj), no_newton(nj, 0);
    for (int j = 0; j < nj; ++j) {
      rn[j] = hj[j].r;
      rp[j] = jobs[j].root_p;
    }
    if ((rc = rb.setup(rn, rp))) return rc;
    for (int j = 0; j < nj; ++j) rb.set_io(j, w + hj[j].b_off, false, w + hj[j].xb_off, false);
    int64_t bstats[4] = {0, 0, 0, 0};
    std::vector<int32_t> bstatus;
    if ((rc = rb.run(1.0, std::vector<int32_t>(nj, 0), eta, eps, SHAMPOO_SOLVER_EIGH, 1e-6, s, bstats, &bstatus,
                     nullptr, false, &no_newton)))
      return rc;
    std::vector<int32_t> failed(nj, 0);
    bool any_failed = false;
    for (int j = 0; j < nj; ++j) {
      failed[j] = bstatus[j] != kEigOk;
      any_failed |= failed[j] != 0;
    }
    if (any_failed) {
      for (int j = 0; j < nj; ++j) hj[j].bad = failed[j];
      SH_CUDA_CHECK(cudaMemcpyAsync(dj, hj.data(), nj * sizeof(LRDev), cudaMemcpyHostToDevice, s));
    }
    k_lr_shift<<<nj, 256, 0, s>>>(dj, w);
    SH_LAUNCH_CHECK();
    if ((rc = gz.launch(s))) return rc;
    if ((rc = gx.launch(s))) return rc;
    k_lr_check<<<xch, 256, 0, s>>>(dj, dx, nj, w);
    SH_LAUNCH_CHECK();
    k_lr_finish<<<xch, 256, 0, s>>>(dj, dx, nj, w);
    SH_LAUNCH_CHECK();
    SH_CUDA_CHECK(cudaMemcpyAsync(hj.data(), dj, nj * sizeof(LRDev), cudaMemcpyDeviceToHost, s));
    SH_CUDA_CHECK(cudaStreamSynchronize(s));
  }
  for (int j = 0; j < nj; ++j) {
    if (!hj[j].bad) ++stats[0];
    else if (hj[j].has_prev) ++stats[2];
    else ++stats[3];
  }
  SH_CUDA_CHECK(cudaFreeAsync(w, s));
  SH_CUDA_CHECK(cudaFreeAsync(dj, s));
  SH_CUDA_CHECK(cudaFreeAsync(dc, s));
  SH_CUDA_CHECK(cudaFreeAsync(dx, s));
  return rc;
}

}  // namespace shampoo
