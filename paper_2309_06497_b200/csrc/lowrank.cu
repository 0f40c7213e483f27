// Root inverse of structurally low-rank factors (see lowrank.cuh).
#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>

#include <cooperative_groups.h>

#include "lowrank.cuh"
#include "rootinv.cuh"
#include "tcgen05.cuh"

namespace shampoo {

namespace {

namespace cg = cooperative_groups;

constexpr int LR_ECH = 4096;  // elements per chunk of the elementwise kernels
constexpr int LR_BS = 64;     // rows per CGS2 block (inter-block projections on the tensor cores)
constexpr int LR_CL = 8;      // CTAs per factor in the shared-memory CGS2 (a thread-block cluster)
constexpr int LR_CW_MAX = 384;  // columns per CTA there (d <= 3072; larger factors: k_lr_cgs2)

struct LRDev {
  int32_t d, r;
  int64_t q_off, t_off, z_off;  // r x d arrays (Q rows, T = Q A, Z = M Q)
  int64_t b_off, xb_off;        // r x r arrays (B, f(B))
  int64_t x_off;                // d x d expansion
  int64_t h_off;                // LR_BS x r projection coefficients
  int64_t n0_off;               // r original row norms of Y
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
    const uint64_t key = ((uint64_t)J.d << 40) ^ (uint64_t)e;  // by size, not batch position (world-size invariance)
    const double u1 = ((splitmix64(2 * key) >> 11) + 1) * 0x1.0p-53;  // (0, 1]
    const double u2 = (splitmix64(2 * key + 1) >> 11) * 0x1.0p-53;
    ws[J.t_off + e] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

// Row norms of Y = Omega^T A before any projection (reference for the dependence test).
__global__ void __launch_bounds__(256) k_lr_rownorm(const LRDev* __restrict__ jobs, const double* __restrict__ ws,
                                                    double* __restrict__ y0n) {
  const LRDev& J = jobs[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= J.r) return;
  const double* w = ws + J.q_off + (int64_t)row * J.d;
  double n = 0.0;
  for (int i = lane; i < J.d; i += 32) n = fma(w[i], w[i], n);
  n = warp_sum(n);
  if (lane == 0) y0n[J.n0_off + row] = sqrt(n);
}

// Block CGS2, one CTA per factor: rows [LR_BS b, LR_BS b + LR_BS) of Y, already projected against
// the finished rows of earlier blocks (Ozaki GEMMs), orthonormalised against the block's own earlier
// rows.  A row whose norm collapses below 1e-13 of its original norm (Y numerically rank deficient)
// is replaced by a unit vector and re-orthogonalised inside the block; fix[j] then asks for one more
// inter-block projection + block pass (the unit vector is not yet orthogonal to earlier blocks).
// fix_pass: only jobs with fix[j] set run (and clear it).
__global__ void __launch_bounds__(256) k_lr_cgs2(LRDev* jobs, double* __restrict__ ws,
                                                 const double* __restrict__ y0n, int b,
                                                 const int32_t* __restrict__ fix_in, int32_t* __restrict__ fix_out) {
  __shared__ double h[LR_BS];
  __shared__ double red[32];
  LRDev& J = jobs[blockIdx.x];
  const int r0 = b * LR_BS, r1 = min(J.r, r0 + LR_BS);
  if (r0 >= J.r) return;
  const int fix_pass = fix_in != nullptr;
  if (fix_pass && !fix_in[blockIdx.x]) return;
  const int d = J.d;
  double* Q = ws + J.q_off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  bool replaced = false;
  for (int j = r0; j < r1; ++j) {
    double* w = Q + (int64_t)j * d;
    double n0 = fix_pass ? 1.0 : y0n[J.n0_off + j];
    for (int attempt = 0; attempt < 3; ++attempt) {
      for (int pass = 0; pass < 2; ++pass) {
        for (int k = r0 + warp; k < j; k += nw) {  // h_k = <q_k, w>
          const double* qk = Q + (int64_t)k * d;
          double s = 0.0;
          for (int i = lane; i < d; i += 32) s = fma(qk[i], w[i], s);
          s = warp_sum(s);
          if (lane == 0) h[k - r0] = s;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < d; i += blockDim.x) {  // w -= sum_k h_k q_k
          double acc = w[i];
          for (int k = r0; k < j; ++k) acc = fma(-h[k - r0], Q[(int64_t)k * d + i], acc);
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
      const int c = (j * 7919 + attempt * 104729 + fix_pass * 15485863) % d;
      for (int i = threadIdx.x; i < d; i += blockDim.x) w[i] = (i == c) ? 1.0 : 0.0;
      n0 = 1.0;
      replaced = true;
      __syncthreads();
      if (attempt == 2 && threadIdx.x == 0) J.bad = 1;
    }
    __syncthreads();
  }
  if (replaced && fix_out && threadIdx.x == 0) fix_out[blockIdx.x] = 1;
}

// The same block CGS2 with the block resident in shared memory: a cluster of LR_CL CTAs per factor,
// CTA c holding columns [c cw, (c + 1) cw) of the block's rows; every inner product is a partial sum
// per CTA, summed over the cluster through distributed shared memory in a fixed order (all CTAs get
// bit-identical coefficients).  One cluster barrier per reduction (partials double-buffered).
__global__ void __cluster_dims__(LR_CL, 1, 1) __launch_bounds__(256)
    k_lr_cgs2c(LRDev* jobs, double* __restrict__ ws, const double* __restrict__ y0n, int b,
               const int32_t* __restrict__ fix_in, int32_t* __restrict__ fix_out) {
  extern __shared__ double S[];  // [rows][cw]
  __shared__ double part[2][LR_BS];
  __shared__ double h[LR_BS];
  __shared__ double red[32];
  cg::cluster_group cl = cg::this_cluster();
  const int job = blockIdx.x / LR_CL;
  const int c = (int)cl.block_rank();
  LRDev& J = jobs[job];
  const int r0 = b * LR_BS;
  if (r0 >= J.r) return;                    // uniform over the cluster
  if (fix_in && !fix_in[job]) return;       // uniform over the cluster
  const int d = J.d, rows = min(LR_BS, J.r - r0);
  const int cw = (d + LR_CL - 1) / LR_CL;
  const int c0 = c * cw, ncol = max(0, min(d, c0 + cw) - c0);
  double* Q = ws + J.q_off;
  for (int e = threadIdx.x; e < rows * cw; e += blockDim.x) {
    const int rr = e / cw, i = e % cw;
    S[e] = i < ncol ? Q[(int64_t)(r0 + rr) * d + c0 + i] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int buf = 0;
  auto exchange = [&](int cnt) {  // h[0..cnt) = cluster sum of part[buf][0..cnt)
    cl.sync();
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
      double sum = 0.0;
      for (int q = 0; q < LR_CL; ++q) sum += cl.map_shared_rank(&part[buf][0], q)[k];
      h[k] = sum;
    }
    __syncthreads();
    buf ^= 1;
  };
  bool replaced = false;
  for (int jj = 0; jj < rows; ++jj) {
    double* w = S + jj * cw;
    double n0 = fix_in ? 1.0 : y0n[J.n0_off + r0 + jj];
    for (int attempt = 0; attempt < 3; ++attempt) {
      for (int pass = 0; pass < 2 && jj > 0; ++pass) {
        for (int k = warp; k < jj; k += 8) {
          double sdot = 0.0;
          for (int i = lane; i < ncol; i += 32) sdot = fma(S[k * cw + i], w[i], sdot);
          sdot = warp_sum(sdot);
          if (lane == 0) part[buf][k] = sdot;
        }
        exchange(jj);
        for (int i = threadIdx.x; i < ncol; i += blockDim.x) {
          double acc = w[i];
          for (int k = 0; k < jj; ++k) acc = fma(-h[k], S[k * cw + i], acc);
          w[i] = acc;
        }
        __syncthreads();
      }
      double nrm = 0.0;
      for (int i = threadIdx.x; i < ncol; i += blockDim.x) nrm = fma(w[i], w[i], nrm);
      nrm = block_sum<double, 256>(nrm, red);
      if (threadIdx.x == 0) part[buf][0] = nrm;
      exchange(1);
      nrm = sqrt(h[0]);
      if (nrm > 1e-13 * n0 && nrm > 0.0 && isfinite(nrm)) {
        const double inv = 1.0 / nrm;
        for (int i = threadIdx.x; i < ncol; i += blockDim.x) w[i] *= inv;
        __syncthreads();
        break;
      }
      const int cc = ((r0 + jj) * 7919 + attempt * 104729 + (fix_in ? 15485863 : 0)) % d;
      for (int i = threadIdx.x; i < ncol; i += blockDim.x) w[i] = (c0 + i == cc) ? 1.0 : 0.0;
      n0 = 1.0;
      replaced = true;
      __syncthreads();
      if (attempt == 2 && c == 0 && threadIdx.x == 0) J.bad = 1;
    }
  }
  for (int e = threadIdx.x; e < rows * cw; e += blockDim.x) {
    const int rr = e / cw, i = e % cw;
    if (i < ncol) Q[(int64_t)(r0 + rr) * d + c0 + i] = S[e];
  }
  if (replaced && fix_out && c == 0 && threadIdx.x == 0) fix_out[job] = 1;
  cl.sync();  // peers may still read this CTA's partials
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
  int64_t ws = 0, n0s = 0;
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
    D.h_off = ws;
    ws += (int64_t)LR_BS * L.r;
    D.n0_off = n0s;
    n0s += L.r;
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
  double *w = nullptr, *y0n = nullptr;
  LRDev* dj = nullptr;
  int32_t *dc = nullptr, *dx = nullptr, *fix = nullptr;
  // every exit path: wait for the queued work on s, then hand the workspaces back to the heap
  struct Release {
    cudaStream_t s;
    void* const* ptrs[6];
    ~Release() {
      cudaStreamSynchronize(s);
      for (void* const* p : ptrs)
        if (*p) dev_free(*p);
    }
  } release{s, {(void* const*)&w, (void* const*)&y0n, (void* const*)&dj, (void* const*)&dc, (void* const*)&dx,
                (void* const*)&fix}};
  SH_CUDA_CHECK(dev_malloc(&w, ws * sizeof(double)));
  SH_CUDA_CHECK(dev_malloc(&y0n, n0s * sizeof(double)));
  SH_CUDA_CHECK(dev_malloc(&dj, nj * sizeof(LRDev)));
  SH_CUDA_CHECK(dev_malloc(&dc, nj * sizeof(int32_t)));
  SH_CUDA_CHECK(dev_malloc(&dx, nj * sizeof(int32_t)));
  SH_CUDA_CHECK(dev_malloc(&fix, nj * sizeof(int32_t)));
  SH_CUDA_CHECK(cudaMemsetAsync(fix, 0, nj * sizeof(int32_t), s));
  SH_CUDA_CHECK(cudaMemcpyAsync(dj, hj.data(), nj * sizeof(LRDev), cudaMemcpyHostToDevice, s));
  SH_CUDA_CHECK(cudaMemcpyAsync(dc, cbeg.data(), nj * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  SH_CUDA_CHECK(cudaMemcpyAsync(dx, xbeg.data(), nj * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  int rc = SHAMPOO_OK;
  // SHAMPOO_LR_PROFILE=1: host-synchronised phase times (debug only)
  static const bool prof = [] {
    const char* e = std::getenv("SHAMPOO_LR_PROFILE");
    return e && std::atoi(e) != 0;
  }();
  auto t_last = std::chrono::steady_clock::now();
  std::string prof_line;
  auto mark = [&](const char* name) {
    if (!prof) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    char b[64];
    std::snprintf(b, sizeof b, " %s %.2f", name, std::chrono::duration<double, std::milli>(now - t_last).count());
    prof_line += b;
    t_last = now;
  };
  mark("alloc");
  {
    // Y = Omega^T A (Omega^T in the T slot) ; T = Q A ; B = T Q^T ; Z = M Q ; X = Z^T Q (symmetric:
    // lower tiles + mirror)
    OzakiGemmBatch<double> gy, gt, gb, gz, gx;
    const int nb = (rmax + LR_BS - 1) / LR_BS;
    std::vector<std::unique_ptr<OzakiGemmBatch<double>>> ph(nb), pu(nb);
    RootInverseBatch rb;
    // destroyed first: the batches above release their workspaces only after s has drained
    struct SyncOnExit {
      cudaStream_t s;
      ~SyncOnExit() { cudaStreamSynchronize(s); }
    } drain{s};
    for (int j = 0; j < nj; ++j) {
      const LRDev& D = hj[j];
      const int r = D.r, d = D.d;
      gy.add(make_gemm(false, false, r, d, d, w + D.t_off, d, D.in, d, w + D.q_off, d, in_scale, 0.0));
      gt.add(make_gemm(false, false, r, d, d, w + D.q_off, d, D.in, d, w + D.t_off, d, in_scale, 0.0));
      gb.add(make_gemm(false, true, r, r, d, w + D.t_off, d, w + D.q_off, d, w + D.b_off, r, 1.0, 0.0));
      gz.add(make_gemm(false, false, r, d, r, w + D.xb_off, r, w + D.q_off, d, w + D.z_off, d, 1.0, 0.0));
      GemmProblem px = make_gemm(true, false, d, d, r, w + D.z_off, d, w + D.q_off, d, w + D.x_off, d, 1.0, 0.0);
      px.flags |= kGemmSym;
      gx.add(px);
    }
    // block CGS2: block b's rows minus their projection on the rows of blocks < b, twice
    // (H = Y_b Q_<b^T ; Y_b -= H Q_<b), then the in-block pass; jobs whose block needed a
    // unit-vector replacement repeat both once (masked by fix[j])
    for (int b = 1; b < nb; ++b) {
      ph[b].reset(new OzakiGemmBatch<double>());
      pu[b].reset(new OzakiGemmBatch<double>());
      for (int j = 0; j < nj; ++j) {
        const LRDev& D = hj[j];
        const int r0 = b * LR_BS;
        if (r0 >= D.r) continue;
        const int rows = std::min(LR_BS, D.r - r0), d = D.d;
        double* Yb = w + D.q_off + (int64_t)r0 * d;
        GemmProblem g = make_gemm(false, true, rows, r0, d, Yb, d, w + D.q_off, d, w + D.h_off, D.r, 1.0, 0.0);
        g.flags |= kGemmMasked;
        g.mask_index = j;
        ph[b]->add(g);
        g = make_gemm(false, false, rows, d, r0, w + D.h_off, D.r, w + D.q_off, d, Yb, d, -1.0, 1.0);
        g.flags |= kGemmMasked;
        g.mask_index = j;
        pu[b]->add(g);
      }
    }
    for (auto* g : {&gy, &gt, &gb, &gz, &gx})
      if ((rc = g->upload())) return rc;
    for (int b = 1; b < nb; ++b)
      if ((rc = ph[b]->upload()) || (rc = pu[b]->upload())) return rc;
    mark("upload");
    k_lr_gauss<<<cch, 256, 0, s>>>(dj, dc, nj, w);
    SH_LAUNCH_CHECK();
    if ((rc = gy.launch(s))) return rc;
    k_lr_rownorm<<<dim3((rmax + 7) / 8, nj), 256, 0, s>>>(dj, w, y0n);
    SH_LAUNCH_CHECK();
    mark("sample");
    int dmax = 0;
    for (const auto& D : hj) dmax = std::max(dmax, D.d);
    const int cw = (dmax + LR_CL - 1) / LR_CL;
    const bool clustered = cw <= LR_CW_MAX;
    const size_t csmem = (size_t)LR_BS * cw * sizeof(double);
    if (clustered)
      SH_CUDA_CHECK(cudaFuncSetAttribute(k_lr_cgs2c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
    auto block_pass = [&](int b, const int32_t* fin, int32_t* fout) {
      if (clustered) k_lr_cgs2c<<<nj * LR_CL, 256, csmem, s>>>(dj, w, y0n, b, fin, fout);
      else k_lr_cgs2<<<nj, 256, 0, s>>>(dj, w, y0n, b, fin, fout);
    };
    for (int b = 0; b < nb; ++b) {
      if (b > 0)
        for (int pass = 0; pass < 2; ++pass)
          if ((rc = ph[b]->launch(s)) || (rc = pu[b]->launch(s))) return rc;
      block_pass(b, nullptr, b > 0 ? fix : nullptr);
      SH_LAUNCH_CHECK();
      if (b > 0) {
        if ((rc = ph[b]->launch(s, fix)) || (rc = pu[b]->launch(s, fix))) return rc;
        block_pass(b, fix, nullptr);
        SH_LAUNCH_CHECK();
        SH_CUDA_CHECK(cudaMemsetAsync(fix, 0, nj * sizeof(int32_t), s));
      }
    }
    mark("cgs2");
    if ((rc = gt.launch(s))) return rc;
    if ((rc = gb.launch(s))) return rc;
    k_lr_symb<<<nj, 256, 0, s>>>(dj, w);
    SH_LAUNCH_CHECK();
    // f(B) on the r x r compressions: B is the factor restricted to (a basis containing) its range,
    // full rank, so the Newton pre-pass applies (with its conditioning gate); Jacobi otherwise
    std::vector<int32_t> rn(nj), rp(nj), full(nj, 1);
    for (int j = 0; j < nj; ++j) {
      rn[j] = hj[j].r;
      rp[j] = jobs[j].root_p;
    }
    if ((rc = rb.setup(rn, rp))) return rc;
    mark("setupB");
    for (int j = 0; j < nj; ++j) rb.set_io(j, w + hj[j].b_off, false, w + hj[j].xb_off, false);
    int64_t bstats[4] = {0, 0, 0, 0};
    std::vector<int32_t> bstatus;
    if ((rc = rb.run(1.0, std::vector<int32_t>(nj, 0), eta, eps, SHAMPOO_SOLVER_EIGH, 1e-6, s, bstats, &bstatus,
                     nullptr, false, &full)))
      return rc;
    mark("solveB");
    std::vector<int32_t> failed(nj, 0);
    bool any_failed = false;
    for (int j = 0; j < nj; ++j) {
      failed[j] = bstatus[j] != kEigOk;
      any_failed |= failed[j] != 0;
    }
    if (any_failed) {
      SH_CUDA_CHECK(cudaMemcpyAsync(hj.data(), dj, nj * sizeof(LRDev), cudaMemcpyDeviceToHost, s));
      SH_CUDA_CHECK(cudaStreamSynchronize(s));
      for (int j = 0; j < nj; ++j) hj[j].bad |= failed[j];
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
    mark("expand");
  }
  if (prof) std::fprintf(stderr, "[lowrank] jobs %d rmax %d:%s ms\n", nj, rmax, prof_line.c_str());
  for (int j = 0; j < nj; ++j) {
    if (!hj[j].bad) ++stats[0];
    else if (hj[j].has_prev) ++stats[2];
    else ++stats[3];
  }
  return rc;
}

}  // namespace shampoo
