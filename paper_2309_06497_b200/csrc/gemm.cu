// Grouped strided GEMM / GEMV kernels (see gemm.cuh).
//
// FP64: 64x64x16 CTA tile, 4 warps, 32x32 warp tile of FP64 tensor-core MMAs
// (mma.sync.aligned.m16n8k4.row.col.f64 -> DMMA), k-major shared tiles with
// leading dim 68 (== 4 mod 16 doubles: conflict-free fragment loads).
// FP32: 64x64x16 tile, 256 threads, 4x4 FFMA micro-tiles (single-precision
// mode; the tcgen05 path replaces it for the statistics GEMM).
// Split-K: problems with K > kSplitChunk are cut into K chunks; each chunk
// writes a raw 64x64 partial into a workspace and k_split_reduce sums the
// chunks in a fixed order (deterministic) and applies the epilogue.
// Symmetric (SYRK) problems compute only tiles tm >= tn and write C[i][j] and
// C[j][i] from the same value, so factors stay exactly symmetric.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "gemm.cuh"

namespace shampoo {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int64_t kSplitChunk = 2048;

__device__ __forceinline__ int64_t ev(const Idx2& x, int32_t v) {
  if (x.div == 0x7fffffff) return (int64_t)v * x.lo;
  const uint32_t q = (uint32_t)v / (uint32_t)x.div;
  return (int64_t)q * x.hi + (int64_t)((uint32_t)v - q * (uint32_t)x.div) * x.lo;
}

__device__ __forceinline__ void tri_index(int64_t l, int& tm, int& tn) {
  int r = (int)((sqrt(8.0 * (double)l + 1.0) - 1.0) * 0.5);
  while ((int64_t)(r + 1) * (r + 2) / 2 <= l) ++r;
  while ((int64_t)r * (r + 1) / 2 > l) --r;
  tm = r;
  tn = (int)(l - (int64_t)r * (r + 1) / 2);
}

struct TileWork {
  int prob, tm, tn, split;
  int64_t tile;  // tile index within the problem
};

__device__ __forceinline__ TileWork locate(const GemmProblem* __restrict__ probs, const int64_t* __restrict__ begin,
                                           int nprob, int64_t item) {
  int lo = 0, hi = nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (begin[mid] <= item) lo = mid;
    else hi = mid - 1;
  }
  TileWork w;
  w.prob = lo;
  const GemmProblem& P = probs[lo];
  const int64_t l = item - begin[lo];
  w.split = (int)(l % P.ksplit);
  w.tile = l / P.ksplit;
  if (P.flags & kGemmSym) tri_index(w.tile, w.tm, w.tn);
  else {
    w.tm = (int)(w.tile / P.tiles_n);
    w.tn = (int)(w.tile % P.tiles_n);
  }
  return w;
}

// Epilogue for one output element; for SYM diagonal tiles only i >= j is written (mirrored).
template <typename T>
__device__ __forceinline__ void store_out(const GemmProblem& P, int tm, int tn, int gi, int gj, double acc) {
  if (gi >= P.M || gj >= P.N) return;
  const bool sym = (P.flags & kGemmSym) != 0;
  if (sym && tm == tn && gi < gj) return;
  T* __restrict__ C = static_cast<T*>(P.C);
  const int64_t at = ev(P.c_r, gi) + ev(P.c_c, gj);
  double v = P.alpha * acc;
  if (P.flags & kGemmReadC) v = fma(P.beta, (double)C[at], v);
  const T o = T(v);
  C[at] = o;
  if (sym && gi != gj) C[ev(P.c_r, gj) + ev(P.c_c, gi)] = o;
}

// ---------------------------------------------------------------- FP64 DMMA kernel


__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Multi-stage cp.async pipeline.  Per operand and problem one of three copy modes:
//   KVEC: k contiguous in global (and 16B aligned)  -> smem [row][k] (ld 20), 16-byte copies
//   RVEC: rows contiguous in global (and aligned)   -> smem [k][row] (ld 68/72), 16-byte copies
//   GEN : anything else (2-level or odd strides)    -> smem [k][row], element copies
// Both smem layouts give conflict-free MMA fragment reads (ld == 4 mod 16 doubles / 20 floats).
constexpr int STAGES = 3;
enum CopyMode : int { kGen = 0, kKvec = 1, kRvec = 2 };

template <typename T>
struct SmemTile {
  static constexpr int LDR = sizeof(T) == 8 ? 68 : 72;  // [k][row]
  static constexpr int LDK = 20;                         // [row][k]
  static constexpr int ELEMS = (BM * LDK > BK * LDR) ? BM * LDK : BK * LDR;
};

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

struct OperandCursor {
  int mode;
  int rows, r0;
  int64_t row_off;  // GEN / KVEC: ev(xr, r0 + my row)
  int row, k_lo;    // my slab row / first k
  bool row_ok;
};

template <typename T>
__device__ __forceinline__ int copy_mode(const void* base, const Idx2& xr, const Idx2& xk) {
  constexpr int V = 16 / sizeof(T);  // elements per 16 bytes
  const bool aligned = (reinterpret_cast<uintptr_t>(base) & 15) == 0;
  if (aligned && xk.div == 0x7fffffff && xk.lo == 1 && xr.div == 0x7fffffff && (xr.lo % V) == 0) return kKvec;
  if (aligned && xr.div == 0x7fffffff && xr.lo == 1 && xk.div == 0x7fffffff && (xk.lo % V) == 0) return kRvec;
  return kGen;
}

__device__ __forceinline__ OperandCursor make_cursor(int mode, const Idx2& xr, int rows, int r0) {
  OperandCursor c;
  const int tid = threadIdx.x;
  c.mode = mode;
  c.rows = rows;
  c.r0 = r0;
  if (mode == kKvec) {  // 2 threads per row, 8 consecutive k each
    c.row = tid >> 1;
    c.k_lo = (tid & 1) * 8;
  } else if (mode == kRvec) {  // 8 threads per k, 8 consecutive rows each
    c.row = (tid & 7) * 8;
    c.k_lo = tid >> 3;
  } else {
    c.row = tid & 63;
    c.k_lo = tid >> 6;
  }
  const int gr = r0 + c.row;
  c.row_ok = gr < rows;
  c.row_off = (c.row_ok && mode != kRvec) ? ev(xr, gr) : 0;
  return c;
}

template <typename T>
__device__ __forceinline__ void issue_slab(T* S, const T* __restrict__ X, const Idx2& xr, const Idx2& xk,
                                           const OperandCursor& c, int k0, int kend) {
  constexpr int V = 16 / sizeof(T);
  if (c.mode == kKvec) {
    constexpr int LD = SmemTile<T>::LDK;
#pragma unroll
    for (int e = 0; e < 8; e += V) {
      const int k = c.k_lo + e, gk = k0 + k;
      const int valid = c.row_ok ? max(0, min(V, kend - gk)) : 0;
      const T* src = valid ? X + c.row_off + gk : X;
      cp_async(S + c.row * LD + k, src, 16, valid * (int)sizeof(T));
    }
  } else if (c.mode == kRvec) {
    constexpr int LD = SmemTile<T>::LDR;
    const int gk = k0 + c.k_lo;
    const int64_t koff = (gk < kend) ? ev(xk, gk) : 0;
#pragma unroll
    for (int e = 0; e < 8; e += V) {
      const int gr = c.r0 + c.row + e;
      const int valid = (gk < kend) ? max(0, min(V, c.rows - gr)) : 0;
      const T* src = valid ? X + koff + ev(xr, gr) : X;
      cp_async(S + c.k_lo * LD + c.row + e, src, 16, valid * (int)sizeof(T));
    }
  } else {
    constexpr int LD = SmemTile<T>::LDR;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = c.k_lo + 2 * e, gk = k0 + k;
      const bool ok = c.row_ok && gk < kend;
      const T* src = ok ? X + c.row_off + ev(xk, gk) : X;
      cp_async(S + k * LD + c.row, src, (int)sizeof(T), ok ? (int)sizeof(T) : 0);
    }
  }
}


// T: storage type of A/B/C (float inputs are widened; accumulation is always FP64).
template <typename T>
__global__ void __launch_bounds__(128) gemm_f64_dmma(const GemmProblem* __restrict__ probs,
                                                     const int64_t* __restrict__ begin, int nprob,
                                                     const int32_t* __restrict__ mask, double* __restrict__ ws) {
  constexpr int TILE = SmemTile<T>::ELEMS;  // elements per operand per stage
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const TileWork w = locate(probs, begin, nprob, blockIdx.x);
  const GemmProblem& P = probs[w.prob];
  if ((P.flags & kGemmMasked) && mask && mask[P.mask_index] == 0) return;
  const int m0 = w.tm * BM, n0 = w.tn * BN;
  const int kbeg = w.split * P.kchunk;
  const int kend = min(P.K, kbeg + P.kchunk);
  const T* __restrict__ A = static_cast<const T*>(P.A);
  const T* __restrict__ B = static_cast<const T*>(P.B);
  const int amode = copy_mode<T>(P.A, P.a_r, P.a_k), bmode = copy_mode<T>(P.B, P.b_r, P.b_k);
  const OperandCursor ca = make_cursor(amode, P.a_r, P.M, m0);
  const OperandCursor cb = make_cursor(bmode, P.b_r, P.N, n0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int g = lane >> 2, tq = lane & 3;
  // fragment addressing: element (row, k) at row*rs + k*ks of the operand's smem tile
  const int a_rs = amode == kKvec ? SmemTile<T>::LDK : 1, a_ks = amode == kKvec ? 1 : SmemTile<T>::LDR;
  const int b_rs = bmode == kKvec ? SmemTile<T>::LDK : 1, b_ks = bmode == kKvec ? 1 : SmemTile<T>::LDR;
  const int a_base = (wm + g) * a_rs + tq * a_ks, b_base = (wn + g) * b_rs + tq * b_ks;

  double c[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) c[i][j][q] = 0.0;

  const int nk = (kend - kbeg + BK - 1) / BK;
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nk) {
      issue_slab<T>(sm + (2 * st) * TILE, A, P.a_r, P.a_k, ca, kbeg + st * BK, kend);
      issue_slab<T>(sm + (2 * st + 1) * TILE, B, P.b_r, P.b_k, cb, kbeg + st * BK, kend);
    }
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int cur = kt % STAGES;
    const T* As = sm + (2 * cur) * TILE;
    const T* Bs = sm + (2 * cur + 1) * TILE;
    {
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double a[2][2], b[4];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          a[i][0] = (double)As[a_base + (i * 16) * a_rs + kk * a_ks];
          a[i][1] = (double)As[a_base + (i * 16 + 8) * a_rs + kk * a_ks];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = (double)Bs[b_base + (j * 8) * b_rs + kk * b_ks];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_16x8x4(c[i][j], a[i][0], a[i][1], b[j]);
      }
    }
    const int nxt = kt + STAGES - 1;
    if (nxt < nk) {
      const int st = nxt % STAGES;
      issue_slab<T>(sm + (2 * st) * TILE, A, P.a_r, P.a_k, ca, kbeg + nxt * BK, kend);
      issue_slab<T>(sm + (2 * st + 1) * TILE, B, P.b_r, P.b_k, cb, kbeg + nxt * BK, kend);
    }
    cp_commit();
  }
  cp_wait<0>();
  if (P.ksplit > 1) {
    double* part = ws + P.ws_off + (w.tile * P.ksplit + w.split) * (BM * BN);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = wm + i * 16 + g + (q >> 1) * 8, cc = wn + j * 8 + 2 * tq + (q & 1);
          part[r * BN + cc] = c[i][j][q];
        }
    return;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = wm + i * 16 + g + (q >> 1) * 8, cc = wn + j * 8 + 2 * tq + (q & 1);
        store_out<T>(P, w.tm, w.tn, m0 + r, n0 + cc, c[i][j][q]);
      }
}

template <typename T>
constexpr int dmma_smem_bytes() {
  return STAGES * 2 * SmemTile<T>::ELEMS * (int)sizeof(T);
}

// ---------------------------------------------------------------- FP32 FFMA kernel

constexpr int PADF = 4;

template <typename T>
__device__ __forceinline__ void load_slab_f(const T* __restrict__ X, const Idx2& xr, const Idx2& xk, int rows,
                                            int kend, int r0, int k0, bool kfast, T (&v)[4]) {
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
    const int gr = r0 + r, gk = k0 + k;
    v[e] = (gr < rows && gk < kend) ? X[ev(xr, gr) + ev(xk, gk)] : T(0);
  }
}

template <typename T>
__device__ __forceinline__ void store_slab_f(T (*S)[BM + PADF], bool kfast, const T (&v)[4]) {
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

__global__ void __launch_bounds__(256) gemm_f32_ffma(const GemmProblem* __restrict__ probs,
                                                     const int64_t* __restrict__ begin, int nprob,
                                                     const int32_t* __restrict__ mask, double* __restrict__ ws) {
  __shared__ __align__(16) float As[2][BK][BM + PADF];
  __shared__ __align__(16) float Bs[2][BK][BN + PADF];
  const TileWork w = locate(probs, begin, nprob, blockIdx.x);
  const GemmProblem& P = probs[w.prob];
  if ((P.flags & kGemmMasked) && mask && mask[P.mask_index] == 0) return;
  const int m0 = w.tm * BM, n0 = w.tn * BN;
  const int kbeg = w.split * P.kchunk;
  const int kend = min(P.K, kbeg + P.kchunk);
  const float* __restrict__ A = static_cast<const float*>(P.A);
  const float* __restrict__ B = static_cast<const float*>(P.B);
  const bool akf = (P.a_k.lo == 1), bkf = (P.b_k.lo == 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ty = (warp >> 1) * 4 + (lane >> 3);
  const int tx = (warp & 1) * 8 + (lane & 7);
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  float ra[4], rb[4];
  const int nk = (kend - kbeg + BK - 1) / BK;
  load_slab_f<float>(A, P.a_r, P.a_k, P.M, kend, m0, kbeg, akf, ra);
  load_slab_f<float>(B, P.b_r, P.b_k, P.N, kend, n0, kbeg, bkf, rb);
  store_slab_f<float>(As[0], akf, ra);
  store_slab_f<float>(Bs[0], bkf, rb);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) {
      load_slab_f<float>(A, P.a_r, P.a_k, P.M, kend, m0, kbeg + (kt + 1) * BK, akf, ra);
      load_slab_f<float>(B, P.b_r, P.b_k, P.N, kend, n0, kbeg + (kt + 1) * BK, bkf, rb);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[cur][kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[cur][kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (kt + 1 < nk) {
      store_slab_f<float>(As[cur ^ 1], akf, ra);
      store_slab_f<float>(Bs[cur ^ 1], bkf, rb);
    }
    __syncthreads();
  }
  if (P.ksplit > 1) {
    double* part = ws + P.ws_off + (w.tile * P.ksplit + w.split) * (BM * BN);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) part[(ty * 4 + i) * BN + tx * 4 + j] = acc[i][j];
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) store_out<float>(P, w.tm, w.tn, m0 + ty * 4 + i, n0 + tx * 4 + j, acc[i][j]);
}

// Sum split-K partials in split order (fp64) and apply the epilogue; one CTA per split tile.
template <typename T>
__global__ void __launch_bounds__(256) k_split_reduce(const GemmProblem* __restrict__ probs,
                                                      const int64_t* __restrict__ rbegin,
                                                      const int32_t* __restrict__ rprob, int nred,
                                                      const int32_t* __restrict__ mask,
                                                      const double* __restrict__ ws) {
  int lo = 0, hi = nred - 1;
  const int64_t item = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (rbegin[mid] <= item) lo = mid;
    else hi = mid - 1;
  }
  const GemmProblem& P = probs[rprob[lo]];
  if ((P.flags & kGemmMasked) && mask && mask[P.mask_index] == 0) return;
  const int64_t tile = item - rbegin[lo];
  int tm, tn;
  if (P.flags & kGemmSym) tri_index(tile, tm, tn);
  else {
    tm = (int)(tile / P.tiles_n);
    tn = (int)(tile % P.tiles_n);
  }
  const double* part = ws + P.ws_off + tile * P.ksplit * (BM * BN);
  for (int e = threadIdx.x; e < BM * BN; e += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < P.ksplit; ++q) s += part[(int64_t)q * (BM * BN) + e];
    store_out<T>(P, tm, tn, tm * BM + e / BN, tn * BN + e % BN, s);
  }
}

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
GemmBatch<T>::~GemmBatch() {
  dev_free(d_prob_);
  dev_free(d_begin_);
  dev_free(d_rbegin_);
  dev_free(d_rprob_);
  dev_free(ws_);
}

template <typename T>
int GemmBatch<T>::upload() {
  dev_free(d_prob_);
  dev_free(d_begin_);
  dev_free(d_rbegin_);
  dev_free(d_rprob_);
  dev_free(ws_);
  d_prob_ = nullptr;
  d_begin_ = d_rbegin_ = nullptr;
  d_rprob_ = nullptr;
  ws_ = nullptr;
  total_items_ = total_red_ = 0;
  if (host.empty()) return SHAMPOO_OK;
  static bool attr = false;
  if (!attr) {
    SH_CUDA_CHECK(cudaFuncSetAttribute(gemm_f64_dmma<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       dmma_smem_bytes<double>()));
    SH_CUDA_CHECK(cudaFuncSetAttribute(gemm_f64_dmma<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       dmma_smem_bytes<float>()));
    attr = true;
  }
  std::vector<int64_t> begin(host.size()), rbegin;
  std::vector<int32_t> rprob;
  int64_t ws_elems = 0;
  for (size_t i = 0; i < host.size(); ++i) {
    GemmProblem& p = host[i];
    p.tiles_m = (p.M + BM - 1) / BM;
    p.tiles_n = (p.N + BN - 1) / BN;
    p.tiles = (p.flags & kGemmSym) ? (int64_t)p.tiles_m * (p.tiles_m + 1) / 2 : (int64_t)p.tiles_m * p.tiles_n;
    if (p.M == 0 || p.N == 0) p.tiles = 0;
    p.ksplit = (int32_t)std::max<int64_t>(1, (p.K + kSplitChunk - 1) / kSplitChunk);
    p.kchunk = (int32_t)(p.ksplit == 1 ? std::max(p.K, 1) : ((p.K + p.ksplit - 1) / p.ksplit + BK - 1) / BK * BK);
    p.ksplit = (int32_t)std::max<int64_t>(1, (p.K + p.kchunk - 1) / p.kchunk);
    p.ws_off = 0;
    if (p.ksplit > 1 && p.tiles > 0) {
      p.ws_off = ws_elems;
      ws_elems += p.tiles * p.ksplit * (int64_t)(BM * BN);
      rbegin.push_back(total_red_);
      rprob.push_back((int32_t)i);
      total_red_ += p.tiles;
    }
    begin[i] = total_items_;
    total_items_ += p.tiles * p.ksplit;
  }
  SH_CUDA_CHECK(dev_malloc(&d_prob_, host.size() * sizeof(GemmProblem)));
  SH_CUDA_CHECK(dev_malloc(&d_begin_, host.size() * sizeof(int64_t)));
  SH_CUDA_CHECK(cudaMemcpy(d_prob_, host.data(), host.size() * sizeof(GemmProblem), cudaMemcpyHostToDevice));
  SH_CUDA_CHECK(cudaMemcpy(d_begin_, begin.data(), begin.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  if (!rbegin.empty()) {
    SH_CUDA_CHECK(dev_malloc(&d_rbegin_, rbegin.size() * sizeof(int64_t)));
    SH_CUDA_CHECK(dev_malloc(&d_rprob_, rprob.size() * sizeof(int32_t)));
    SH_CUDA_CHECK(dev_malloc(&ws_, ws_elems * sizeof(double)));
    SH_CUDA_CHECK(cudaMemcpy(d_rbegin_, rbegin.data(), rbegin.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    SH_CUDA_CHECK(cudaMemcpy(d_rprob_, rprob.data(), rprob.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    nred_ = (int)rbegin.size();
  }
  return SHAMPOO_OK;
}

template <typename T>
int GemmBatch<T>::launch(cudaStream_t s, const int32_t* mask) const {
  if (total_items_ == 0) return SHAMPOO_OK;
  if (std::is_same<T, double>::value || fp64_accumulate)
    gemm_f64_dmma<T><<<(unsigned)total_items_, 128, dmma_smem_bytes<T>(), s>>>(d_prob_, d_begin_,
                                                                           (int)host.size(), mask, ws_);
  else
    gemm_f32_ffma<<<(unsigned)total_items_, 256, 0, s>>>(d_prob_, d_begin_, (int)host.size(), mask, ws_);
  SH_LAUNCH_CHECK();
  if (total_red_ > 0) {
    k_split_reduce<T><<<(unsigned)total_red_, 256, 0, s>>>(d_prob_, d_rbegin_, d_rprob_, nred_, mask, ws_);
    SH_LAUNCH_CHECK();
  }
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

template class GemmBatch<double>;
template class GemmBatch<float>;
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
