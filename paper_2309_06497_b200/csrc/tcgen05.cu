// Grouped Ozaki-split int8 GEMM on tcgen05 tensor cores (see tcgen05.cuh).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <atomic>
#include <map>
#include <mutex>
#include <tuple>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "tcgen05.cuh"

namespace shampoo {

namespace {

// CTA tile TM x TN, 32 int8 (= one MMA K) per pipeline stage.  TN = 64: the kernel is bound by the
// operand bytes each SM takes in per MMA (measured 49 GB/s per SM at TN = 32 for both S = 6 and 8);
// an A slice feeds twice the output columns per byte at TN = 64
constexpr int TM = 128, TN = 64, TKB = 32;
constexpr int SL_PER_MMA = 256 / TN;          // B slices stacked along N in one MMA (N <= 256)
constexpr int GEMM_THREADS_P = 320;           // warp 0 bulk copies, warp 1 MMA, warps 2-9 epilogue
constexpr int64_t kOzSplitStages = 256;       // 8192 k per split: int32 sums stay exact (< 2^31)
constexpr int PACK_UNITS = 256;               // pack threads per CTA (one unit = 16 k of one row)
constexpr int EXP_CHUNK = 64;                 // k per rowexp thread (strided rows)
constexpr int EXP_WARP_CHUNK = 2048;          // k per rowexp warp (contiguous rows)
constexpr int kExpFloor = -1100;              // exponent of an all-zero row (ldexp -> 0)

// Executed MMA work (bench evidence for the tensor-pipe roofline of phases whose problem sets are
// masked on the device, e.g. the root-inverse Newton iterations): one unit = one 32-wide k stage of
// one slice pair on a 128 x 32 tile, i.e. 2 * 128 * 32 * 32 int8 ops.  One atomic per tile.
__device__ unsigned long long g_oz_mma_units = 0;
// the same per step-phase tag (bench kernel-level roofline; slot kOzTags - 1 = untagged)
constexpr int kOzTags = 8;
__device__ unsigned long long g_oz_mma_units_tag[kOzTags] = {};

template <int S>
struct OzCfg {
  static constexpr int A_BYTES = (TM / 8) * S * 256;     // one stage of a 128-row tile, all slices
  static constexpr int B_BYTES = (TN / 8) * S * 256;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  // kind::i8: D s32 (bits 4-5 = 2), A/B signed int8 (bits 7-9, 10-12 = 1), K-major, M = 128; N (bits 17-22)
  // is set per instruction
  static constexpr uint32_t IDESC_BASE = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TM >> 4) << 24);
};

__device__ __forceinline__ int64_t evx(const Idx2& x, int64_t v) {
  if (x.div == 0x7fffffff) return v * x.lo;
  const uint32_t q = (uint32_t)v / (uint32_t)x.div;  // indices are < 2^31: 32-bit division
  return (int64_t)q * x.hi + (int64_t)((uint32_t)v - q * (uint32_t)x.div) * x.lo;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---- mbarrier / bulk copy (async proxy) ----
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
// Long waits (the epilogue warps wait out the whole mainloop): back off between polls so the
// spinning warps do not take issue slots (and the sync unit) from the producer / MMA lanes.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  uint32_t done = 0, ns = 32;
  for (;;) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(ns);
    ns = ns < 256 ? ns * 2 : 256;
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// TMA tile load of a 3-D box (tensor map in global memory) into shared memory.
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// ---- tcgen05 ----
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor, no swizzle, K-major: rows of 16 B inside an 8-row core
// matrix, the two K cores LBO apart, consecutive 8-row cores SBO apart.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
}

__device__ __forceinline__ void tc_mma_i8(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// tcgen05.ld without the wait (several loads in flight, one tcgen05.wait::ld for all of them);
// reg_fence16 after the wait keeps the consumers of the registers behind it
__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void reg_fence16(uint32_t* r) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]));
}

template <typename P>
__device__ __forceinline__ int find64(const int64_t* __restrict__ begin, int n, int64_t x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (begin[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// SYM problems: TM x TN tiles that touch the lower triangle, tn < (TM / TN)(tm + 1), row-major order.
__host__ __device__ __forceinline__ int64_t sym_tiles_before(int tm, int nt) {
  constexpr int R = TM / TN;
  int64_t c = 0;
  for (int t = 0; t < tm; ++t) c += (R * (t + 1) < nt) ? R * (t + 1) : nt;
  return c;
}
__device__ __forceinline__ void sym_decode(int64_t l, int nt, int& tm, int& tn) {
  constexpr int R = TM / TN;
  int t = 0;
  int64_t c = 0;
  for (;; ++t) {
    const int w = (R * (t + 1) < nt) ? R * (t + 1) : nt;
    if (l < c + w) break;
    c += w;
  }
  tm = t;
  tn = (int)(l - c);
}

// Epilogue for one element (same semantics as GemmBatch): SYM problems write i >= j and mirror
// every off-diagonal value, so factors stay exactly symmetric.
template <typename T>
__device__ __forceinline__ void oz_store(const GemmProblem& P, int gi, int gj, double acc) {
  if (gi >= P.M || gj >= P.N) return;
  const bool sym = (P.flags & kGemmSym) != 0;
  if (sym && gi < gj) return;
  T* __restrict__ C = static_cast<T*>(P.C);
  const int64_t at = evx(P.c_r, gi) + evx(P.c_c, gj);
  double v = P.alpha * acc;
  if (P.flags & kGemmReadC) v = fma(P.beta, (double)C[at], v);
  const T o = (T)v;
  C[at] = o;
  if (sym && gi != gj && !(P.flags & kGemmLowerOnly)) C[evx(P.c_r, gj) + evx(P.c_c, gi)] = o;
}

// Row exponents: e_r = max_k frexp-exponent(x_rk) (|x_rk| < 2^e_r).  Rows contiguous along k:
// a warp per (row, 2048-wide k chunk), lanes on consecutive k; otherwise a thread per
// (k chunk, row) with consecutive threads on consecutive rows (coalesced for column access).
__device__ __forceinline__ bool k_contig(const OzPackJob& J) { return J.k.div == 0x7fffffff && J.k.lo == 1; }

template <typename T>
__global__ void __launch_bounds__(256) k_oz_rowexp(const OzPackJob* __restrict__ jobs, const int64_t* __restrict__ ebegin,
                                                   int njobs, const int32_t* __restrict__ mask, int32_t* __restrict__ exps) {
  const int j = find64<OzPackJob>(ebegin, njobs, blockIdx.x);
  const OzPackJob J = jobs[j];  // by value: no reloads after the plane stores
  if (J.mask_index >= 0 && mask && !mask[J.mask_index]) return;
  const int64_t u = (int64_t)(blockIdx.x - ebegin[j]) * 256 + threadIdx.x;
  if (J.fexp != kNoFixedExp) {  // fixed exponent: one thread per row writes it
    if (u < J.rows) exps[J.exp + u] = J.fexp;
    return;
  }
  const T* __restrict__ src = static_cast<const T*>(J.src);
  double m = 0.0;
  int row;
  if (k_contig(J)) {
    const int64_t wu = u >> 5;
    const int lane = threadIdx.x & 31;
    const int nkc = (J.K + EXP_WARP_CHUNK - 1) / EXP_WARP_CHUNK;
    if (wu >= (int64_t)J.rows * nkc) return;  // whole warps exit together
    row = (int)(wu / nkc);
    const int k0 = (int)(wu % nkc) * EXP_WARP_CHUNK, k1 = min(J.K, k0 + EXP_WARP_CHUNK);
    const T* __restrict__ rp = src + evx(J.r, row);
    double m1 = 0.0, m2 = 0.0, m3 = 0.0;  // four independent chains: 4 loads in flight per lane
    int k = k0 + lane;
    for (; k + 96 < k1; k += 128) {
      m = fmax(m, fabs((double)rp[k]));
      m1 = fmax(m1, fabs((double)rp[k + 32]));
      m2 = fmax(m2, fabs((double)rp[k + 64]));
      m3 = fmax(m3, fabs((double)rp[k + 96]));
    }
    for (; k < k1; k += 32) m = fmax(m, fabs((double)rp[k]));
    m = fmax(fmax(m, m1), fmax(m2, m3));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane != 0) return;
  } else {
    if (u >= J.echunks) return;
    row = (int)(u % J.rows);
    const int k0 = (int)(u / J.rows) * EXP_CHUNK, k1 = min(J.K, k0 + EXP_CHUNK);
    const Idx2 kx = J.k;
    if (kx.div == 0x7fffffff) {
      const T* __restrict__ rp = src + evx(J.r, row) + (int64_t)k0 * kx.lo;
      for (int k = k0; k < k1; ++k, rp += kx.lo) m = fmax(m, fabs((double)*rp));
    } else {  // two-level k: one division, then carries
      int q = k0 / kx.div, r = k0 - q * kx.div;
      int64_t off = evx(J.r, row) + (int64_t)q * kx.hi + (int64_t)r * kx.lo;
      const int64_t wrap = kx.hi - (int64_t)kx.div * kx.lo;
      for (int k = k0; k < k1; ++k) {
        m = fmax(m, fabs((double)src[off]));
        off += kx.lo;
        if (++r == kx.div) {
          r = 0;
          off += wrap;
        }
      }
    }
  }
  if (m > 0.0) {
    int e;
    frexp(m, &e);
    atomicMax(exps + J.exp + row, e);
  }
}

// The S signed 7-bit slices of y = x 2^-e (|y| < 1): the digits of the fixed-point |y| in base 128
// with the sign of x, the last one rounded to nearest (ties away from zero) on the remaining bits
// and clamped to +-127 -- t = 128 y, q = trunc(t), y = t - q for the first S - 1 slices and
// q = round(t) for the last (the dropped remainder is rounded, not truncated: no bias in the
// factor sums), computed on the integer significand (no FP64 / conversion-pipe work).
// Y = floor(|x| 2^(63 - e)) < 2^63 is one variable right shift of the significand left-aligned
// at bit 63: digit k is bits [56 - 7k, 63 - 7k) of Y, the remainder the RB = 63 - 7S bits below.
// Split for packing: digits 0..S-2 as bit fields of `top`, the rounded last digit `last`.
template <int S>
__device__ __forceinline__ void ozaki_mag(double x, int e, unsigned long long& top, uint32_t& last) {
  constexpr int RB = 63 - 7 * S;
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const int bexp = (int)(bits >> 52) & 0x7ff;
  const unsigned long long M = (bits << 11) | ((unsigned long long)(bexp != 0) << 63);
  // |x| = (M >> 11) 2^(max(bexp,1) - 1075) < 2^e  =>  shift >= 1 for every nonzero x; an all-zero
  // row's floor exponent makes it negative (M = 0 there): clamp
  const int rs = min(max(1023 + e - max(bexp, 1), 0), 63);
  const unsigned long long Y = M >> rs;
  top = Y >> (RB + 7);
  const uint32_t l = (uint32_t)(Y >> RB) & 127u;
  const uint32_t up = (RB <= 32) ? (uint32_t)((uint32_t)Y & (uint32_t)((1ull << RB) - 1ull)) >= (1u << (RB - 1))
                                 : (Y & ((1ull << RB) - 1ull)) >= (1ull << (RB - 1));
  last = min(l + up, 127u);
}

// The 7-bit fields [7k, 7k + 7) of v, k < 4, into byte k (shifts on the FMA pipe as IMAD.SHL,
// masks on the ALU: the slicing kernels are ALU-bound).
__device__ __forceinline__ uint32_t spread4(uint32_t v) {
  return (v & 0x7fu) | ((v << 1) & 0x7f00u) | ((v << 2) & 0x7f0000u) | ((v << 3) & 0x7f000000u);
}
// 4 x 4 byte transpose: o[k] byte i = w[i] byte k.
__device__ __forceinline__ void transpose4(const uint32_t (&w)[4], uint32_t (&o)[4]) {
  const uint32_t alo = __byte_perm(w[0], w[1], 0x5140), ahi = __byte_perm(w[0], w[1], 0x7362);
  const uint32_t blo = __byte_perm(w[2], w[3], 0x5140), bhi = __byte_perm(w[2], w[3], 0x7362);
  o[0] = __byte_perm(alo, blo, 0x5410);
  o[1] = __byte_perm(alo, blo, 0x7632);
  o[2] = __byte_perm(ahi, bhi, 0x5410);
  o[3] = __byte_perm(ahi, bhi, 0x7632);
}

// Four consecutive elements -> S words of packed int8 slices (byte i = element i).  The S - 1
// truncated digits of an element sit in `top` 7 bits apart: groups of four are spread into the
// bytes of one word per element and byte-transposed across the four elements (8 PRMT per four
// slice words instead of 12, and no shift + mask per digit); a lone digit and the rounded last one
// are gathered directly.  Signs as a byte mask (PRMT sign replication of the high bytes), applied
// per byte: -d = (0x80 - d) ^ 0x80 for d in [0, 127], no borrow across bytes.
template <int S>
__device__ __forceinline__ void ozaki_pack4(const double (&x)[4], int e, uint32_t (&w)[S]) {
  constexpr int ND = S - 1;
  unsigned long long t[4];
  uint32_t l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) ozaki_mag<S>(x[i], e, t[i], l[i]);
  // prmt sign mode (selector nibble bit 3): result byte = the selected byte's sign bit replicated
  uint32_t h01, h23;
  asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(h01) : "r"(__double2hiint(x[0])), "r"(__double2hiint(x[1])));
  asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(h23) : "r"(__double2hiint(x[2])), "r"(__double2hiint(x[3])));
  const uint32_t msk = __byte_perm(h01, h23, 0x6420);  // byte i = 0xFF iff x[i] has its sign bit set
  uint32_t mag[S];
#pragma unroll
  for (int g = 0; 4 * g < ND; ++g) {  // digit sl = ND - 1 - 4 g - k is field k of t >> 28 g
    const int nd = ND - 4 * g < 4 ? ND - 4 * g : 4;
    if (nd == 1) {
      uint32_t b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) b[i] = (uint32_t)(t[i] >> (28 * g)) & 127u;
      mag[ND - 1 - 4 * g] =
          __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
    } else {
      uint32_t wv[4], o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) wv[i] = spread4((uint32_t)(t[i] >> (28 * g)));
      transpose4(wv, o);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < nd) mag[ND - 1 - 4 * g - k] = o[k];
    }
  }
  mag[S - 1] = __byte_perm(__byte_perm(l[0], l[1], 0x0040), __byte_perm(l[2], l[3], 0x0040), 0x5410);
#pragma unroll
  for (int sl = 0; sl < S; ++sl) {
    const uint32_t negw = (0x80808080u - mag[sl]) ^ 0x80808080u;
    w[sl] = (mag[sl] & ~msk) | (negw & msk);
  }
}

// 16 consecutive elements of one operand row (k0 .. k0+15, `valid` of them inside the row) as doubles:
// 16-byte vector loads when the run is complete and aligned (the common case), else scalar.
template <typename T>
__device__ __forceinline__ void load_run16(const T* __restrict__ rp, int valid, double (&xv)[16]) {
  if (valid >= 16 && (reinterpret_cast<uintptr_t>(rp) & 15u) == 0) {
    if constexpr (sizeof(T) == 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(rp) + i);
        xv[2 * i] = v.x;
        xv[2 * i + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(rp) + i);
        xv[4 * i] = v.x;
        xv[4 * i + 1] = v.y;
        xv[4 * i + 2] = v.z;
        xv[4 * i + 3] = v.w;
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) xv[i] = i < valid ? (double)rp[i] : 0.0;
}

// Operands -> int8 slice planes, slice-major per stage: byte offset
// ((stage * S + s) * rc + core) * 256 + kc * 128 + r8 * 16 holds row 8 core + r8,
// k = 32 stage + 16 kc .. +15 of slice s.  Unit u = ((stage * rc + core) * 2 + kc) * 8 + r8.
template <typename T, int S>
__global__ void __launch_bounds__(PACK_UNITS) k_oz_pack(const OzPackJob* __restrict__ jobs,
                                                        const int64_t* __restrict__ pbegin, int njobs,
                                                        const int32_t* __restrict__ mask,
                                                        const int32_t* __restrict__ exps, int8_t* __restrict__ arena) {
  const int j = find64<OzPackJob>(pbegin, njobs, blockIdx.x);
  const OzPackJob J = jobs[j];  // by value: no reloads after the plane stores
  if (J.mask_index >= 0 && mask && !mask[J.mask_index]) return;
  const int64_t u = (int64_t)(blockIdx.x - pbegin[j]) * PACK_UNITS + threadIdx.x;
  if (u >= J.units) return;
  const int r8 = (int)(u & 7), kc = (int)((u >> 3) & 1);
  const int64_t sc = u >> 4;  // stage * rc + core
  const int core = (int)(sc % J.rc), stage = (int)(sc / J.rc);
  const int row = core * 8 + r8;
  const int k0 = stage * TKB + kc * 16;
  uint32_t w[S][4];
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int q = 0; q < 4; ++q) w[s][q] = 0u;
  if (row < J.rows) {
    const T* __restrict__ src = static_cast<const T*>(J.src);
    const int64_t rb = evx(J.r, row);
    const int e = max(exps[J.exp + row], kExpFloor);
    const Idx2 kx = J.k;
    double xv[16];
    if (kx.div == 0x7fffffff && kx.lo == 1) {  // contiguous k: one 128-byte run
      load_run16<T>(src + rb + k0, J.K - k0, xv);
    } else if (kx.div == 0x7fffffff) {  // one stride along k: no per-element index map
      const T* rp = src + rb + (int64_t)k0 * kx.lo;
#pragma unroll
      for (int i = 0; i < 16; ++i) xv[i] = (k0 + i < J.K) ? (double)rp[(int64_t)i * kx.lo] : 0.0;
    } else {  // two-level k: one division, then the (q, r) digits advance by carries
      int q = k0 / kx.div, r = k0 - q * kx.div;
      int64_t off = rb + (int64_t)q * kx.hi + (int64_t)r * kx.lo;
      const int64_t wrap = kx.hi - (int64_t)kx.div * kx.lo;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        xv[i] = (k0 + i < J.K) ? (double)src[off] : 0.0;
        off += kx.lo;
        if (++r == kx.div) {
          r = 0;
          off += wrap;
        }
      }
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const double x4[4] = {xv[4 * g], xv[4 * g + 1], xv[4 * g + 2], xv[4 * g + 3]};
      uint32_t ws[S];
      ozaki_pack4<S>(x4, e, ws);
#pragma unroll
      for (int s = 0; s < S; ++s) w[s][g] = ws[s];
    }
  }
  int8_t* dst = arena + J.dst + ((int64_t)stage * S * J.rc + core) * 256 + kc * 128 + r8 * 16;
#pragma unroll
  for (int s = 0; s < S; ++s)
    *reinterpret_cast<uint4*>(dst + (int64_t)s * J.rc * 256) = make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
}

// Fused row exponents + slice planes: one CTA per PACK_CORES 8-row cores of an operand.  Phase 1
// reads the CTA's rows once for their maxima (warp per row along contiguous k; for strided k a
// thread per (row, k slice) with consecutive threads on consecutive rows -- coalesced column reads),
// phase 2 re-reads them (L2-resident: just touched) and writes the planes exactly like k_oz_pack.
// One DRAM pass over each operand instead of two (k_oz_rowexp + k_oz_pack), no exponent memset.
constexpr int PACK_CORES = 4;  // 32 rows per CTA

template <typename T, int S, bool XF>
__global__ void __launch_bounds__(256) k_oz_pack_rows(const OzPackJob* __restrict__ jobs,
                                                      const int64_t* __restrict__ cbegin, int njobs,
                                                      const int32_t* __restrict__ mask, int32_t* __restrict__ exps,
                                                      int8_t* __restrict__ arena) {
  __shared__ double rmax[8][PACK_CORES * 8 + 1];
  __shared__ int rexp[PACK_CORES * 8];
  const int j = find64<OzPackJob>(cbegin, njobs, blockIdx.x);
  const OzPackJob J = jobs[j];  // by value: no reloads after the plane stores
  if (J.mask_index >= 0 && mask && !mask[J.mask_index]) return;
  const int core0 = (int)(blockIdx.x - cbegin[j]) * PACK_CORES;
  const int ncores = min(PACK_CORES, J.rc - core0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const T* __restrict__ src = static_cast<const T*>(J.src);
  constexpr int R = PACK_CORES * 8;
  if (J.fexp != kNoFixedExp) {
    // fixed exponent (affine operands): no maxima pass
  } else if (k_contig(J)) {
    for (int rr = warp; rr < R; rr += 8) {  // warp per row, lanes along k
      const int row = core0 * 8 + rr;
      double m = 0.0, m1 = 0.0, m2 = 0.0, m3 = 0.0;
      if (rr < ncores * 8 && row < J.rows) {
        const T* __restrict__ rp = src + evx(J.r, row);
        int k = lane;
        for (; k + 96 < J.K; k += 128) {
          m = fmax(m, fabs((double)rp[k]));
          m1 = fmax(m1, fabs((double)rp[k + 32]));
          m2 = fmax(m2, fabs((double)rp[k + 64]));
          m3 = fmax(m3, fabs((double)rp[k + 96]));
        }
        for (; k < J.K; k += 32) m = fmax(m, fabs((double)rp[k]));
      }
      m = fmax(fmax(m, m1), fmax(m2, m3));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) rmax[0][rr] = m;
    }
  } else {  // thread (row = tid % 32, k slice = tid / 32): a warp reads 32 consecutive rows at one k
    const int rr = tid & 31, ksl = tid >> 5;
    const int row = core0 * 8 + rr;
    double m = 0.0;
    if (rr < ncores * 8 && row < J.rows) {
      const int64_t rb = evx(J.r, row);
      for (int k = ksl; k < J.K; k += 8) m = fmax(m, fabs((double)src[rb + evx(J.k, k)]));
    }
    rmax[ksl][rr] = m;
    __syncthreads();
    if (tid < R) {
      double q = rmax[0][tid];
#pragma unroll
      for (int t = 1; t < 8; ++t) q = fmax(q, rmax[t][tid]);
      rmax[0][tid] = q;
    }
  }
  __syncthreads();
  if (tid < ncores * 8) {
    const double m = rmax[0][tid];
    int e = kExpFloor;
    if (J.fexp != kNoFixedExp) e = J.fexp;
    else if (m > 0.0) frexp(m, &e);
    rexp[tid] = e;
    exps[J.exp + core0 * 8 + tid] = e;
  }
  __syncthreads();
  // phase 2: units (stage, core, kc, r8) of the CTA's cores; consecutive threads -> consecutive 16 B
  const int64_t nunits = (int64_t)J.ks * ncores * 16;
  for (int64_t u = tid; u < nunits; u += 256) {
    const int r8 = (int)(u & 7), kc = (int)((u >> 3) & 1);
    const int64_t sc = u >> 4;
    const int cl = (int)(sc % ncores), stage = (int)(sc / ncores);
    const int core = core0 + cl;
    const int row = core * 8 + r8;
    const int k0 = stage * TKB + kc * 16;
    uint32_t w[S][4];
#pragma unroll
    for (int s_ = 0; s_ < S; ++s_)
#pragma unroll
      for (int q = 0; q < 4; ++q) w[s_][q] = 0u;
    if (row < J.rows) {
      const int64_t rb = evx(J.r, row);
      const int e = rexp[cl * 8 + r8];
      const Idx2 kx = J.k;
      double xv[16];
      if (kx.div == 0x7fffffff && kx.lo == 1) {
        load_run16<T>(src + rb + k0, J.K - k0, xv);
      } else if (kx.div == 0x7fffffff) {
        const T* rp = src + rb + (int64_t)k0 * kx.lo;
#pragma unroll
        for (int i = 0; i < 16; ++i) xv[i] = (k0 + i < J.K) ? (double)rp[(int64_t)i * kx.lo] : 0.0;
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) xv[i] = (k0 + i < J.K) ? (double)src[rb + evx(kx, k0 + i)] : 0.0;
      }
      if constexpr (XF) {  // affine operand (Newton's T = ((p+1) I - M) / p), fixed exponent
#pragma unroll
        for (int i = 0; i < 16; ++i)
          xv[i] = (k0 + i < J.K) ? J.xa * xv[i] + (row == k0 + i ? J.xb : 0.0) : 0.0;
      }
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const double x4[4] = {xv[4 * g], xv[4 * g + 1], xv[4 * g + 2], xv[4 * g + 3]};
        uint32_t ws[S];
        ozaki_pack4<S>(x4, e, ws);
#pragma unroll
        for (int s_ = 0; s_ < S; ++s_) w[s_][g] = ws[s_];
      }
    }
    int8_t* dst = arena + J.dst + ((int64_t)stage * S * J.rc + core) * 256 + kc * 128 + r8 * 16;
#pragma unroll
    for (int s_ = 0; s_ < S; ++s_)
      *reinterpret_cast<uint4*>(dst + (int64_t)s_ * J.rc * 256) = make_uint4(w[s_][0], w[s_][1], w[s_][2], w[s_][3]);
  }
}

// Transposed operand pairs (OzDualJob).  The column operand's own path reads X down columns
// (strided, 8-byte loads) twice -- once for its maxima, once to pack; here both operands take one
// coalesced exponent pass and one pack pass whose 64 x 32 tile is staged in shared memory and read
// by rows (operand a) and by columns (operand b).  Bytes per element: 2 reads + 2 S plane bytes,
// against 4 reads + 2 S (two k_oz_rowexp + two k_oz_pack passes).
constexpr int DX_R = 64, DX_C = 64;  // exponent tile: a half warp per 16-column row segment
constexpr int DP_R = 64, DP_C = 32;  // pack tile: a = 8 cores x 1 stage, b = 4 cores x 2 stages

__device__ __forceinline__ bool dual_on(const OzDualJob& J, const int32_t* __restrict__ mask) {
  if (!mask) return true;
  return J.mask_a < 0 || J.mask_b < 0 || mask[J.mask_a] || mask[J.mask_b];
}

template <typename T>
__global__ void __launch_bounds__(256) k_oz_dual_exp(const OzDualJob* __restrict__ jobs,
                                                     const int64_t* __restrict__ tbegin, int njobs,
                                                     const int32_t* __restrict__ mask, int32_t* __restrict__ exps) {
  __shared__ double cmax[16][DX_C + 1];
  const int j = find64<OzDualJob>(tbegin, njobs, blockIdx.x);
  const OzDualJob& J = jobs[j];
  if (!dual_on(J, mask)) return;
  const int64_t t = blockIdx.x - tbegin[j];
  // job fields in registers and read-only global loads: all 16 loads issue back to back
  const int R = J.R, C = J.C;
  const int64_t ld = J.ld;
  const T* __restrict__ src = static_cast<const T*>(J.src);
  const int tcn = (C + DX_C - 1) / DX_C;
  const int tt = (int)t;
  const int r0 = (tt / tcn) * DX_R, c0 = (tt % tcn) * DX_C;
  const int cg = threadIdx.x & 15, rg = threadIdx.x >> 4;
  T x[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = r0 + rg + 16 * q;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = c0 + cg + 16 * i;
      x[q][i] = (r < R && c < C) ? __ldg(src + (int64_t)r * ld + c) : T(0);
    }
  }
  double v[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int i = 0; i < 4; ++i) v[q][i] = fabs((double)x[q][i]);
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // row maxima: the 16 lanes of a half warp share a row
    double m = fmax(fmax(v[q][0], v[q][1]), fmax(v[q][2], v[q][3]));
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    const int r = r0 + rg + 16 * q;
    if (cg == 0 && m > 0.0 && r < R) {
      int e;
      frexp(m, &e);
      atomicMax(exps + J.exp_a + r, e);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) cmax[rg][cg + 16 * i] = fmax(fmax(v[0][i], v[1][i]), fmax(v[2][i], v[3][i]));
  __syncthreads();
  if (threadIdx.x < DX_C) {  // column maxima over the 16 row groups
    double m = cmax[0][threadIdx.x];
#pragma unroll
    for (int g = 1; g < 16; ++g) m = fmax(m, cmax[g][threadIdx.x]);
    const int c = c0 + threadIdx.x;
    if (m > 0.0 && c < C) {
      int e;
      frexp(m, &e);
      atomicMax(exps + J.exp_b + c, e);
    }
  }
}

// One 16-element unit of slice planes from values already in registers (same bytes as k_oz_pack).
template <int S>
__device__ __forceinline__ void pack_unit16(const double (&xv)[16], int e, int8_t* __restrict__ dst, int64_t plane) {
  uint32_t w[S][4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const double x4[4] = {xv[4 * g], xv[4 * g + 1], xv[4 * g + 2], xv[4 * g + 3]};
    uint32_t ws[S];
    ozaki_pack4<S>(x4, e, ws);
#pragma unroll
    for (int s_ = 0; s_ < S; ++s_) w[s_][g] = ws[s_];
  }
#pragma unroll
  for (int s_ = 0; s_ < S; ++s_)
    *reinterpret_cast<uint4*>(dst + (int64_t)s_ * plane) = make_uint4(w[s_][0], w[s_][1], w[s_][2], w[s_][3]);
}

template <typename T, int S>
__global__ void __launch_bounds__(256) k_oz_pack_dual(const OzDualJob* __restrict__ jobs,
                                                      const int64_t* __restrict__ tbegin, int njobs,
                                                      const int32_t* __restrict__ mask,
                                                      const int32_t* __restrict__ exps, int8_t* __restrict__ arena) {
  __shared__ double tile[DP_R][DP_C + 1];  // +1: row and column reads both conflict-free
  const int j = find64<OzDualJob>(tbegin, njobs, blockIdx.x);
  const OzDualJob& J = jobs[j];
  if (!dual_on(J, mask)) return;
  const int64_t t = blockIdx.x - tbegin[j];
  const int R = J.R, C = J.C;
  const int64_t ld = J.ld;
  const T* __restrict__ src = static_cast<const T*>(J.src);
  const int tcn = (C + DP_C - 1) / DP_C;
  const int tt = (int)t;
  const int r0 = (tt / tcn) * DP_R, c0 = (tt % tcn) * DP_C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    const int c = c0 + lane;
    T x[DP_R / 8];
#pragma unroll
    for (int q = 0; q < DP_R / 8; ++q) {  // a warp per 32-wide row segment; all loads before the stores
      const int r = r0 + warp + 8 * q;
      x[q] = (r < R && c < C) ? __ldg(src + (int64_t)r * ld + c) : T(0);
    }
#pragma unroll
    for (int q = 0; q < DP_R / 8; ++q) tile[warp + 8 * q][lane] = (double)x[q];
  }
  __syncthreads();
  const int u = tid & 127, r8 = u & 7, kc = (u >> 3) & 1;
  double xv[16];
  if (tid < 128) {  // operand a (rows of X): core r0/8 + cl, stage c0/32
    const int cl = u >> 4, core = r0 / 8 + cl;
    if (core >= J.rc_a) return;
    const int lr = cl * 8 + r8;
#pragma unroll
    for (int i = 0; i < 16; ++i) xv[i] = tile[lr][kc * 16 + i];
    const int e = max(exps[J.exp_a + r0 + lr], kExpFloor);
    const int stage = c0 / TKB;
    pack_unit16<S>(xv, e, arena + J.dst_a + ((int64_t)stage * S * J.rc_a + core) * 256 + kc * 128 + r8 * 16,
                   (int64_t)J.rc_a * 256);
  } else {  // operand b (columns of X): core c0/8 + cl, stage r0/32 + st
    const int cl = (u >> 4) & 3, st = u >> 6;
    const int core = c0 / 8 + cl, stage = r0 / TKB + st;
    if (core >= J.rc_b || stage >= J.ks_b) return;
    const int lc = cl * 8 + r8;
#pragma unroll
    for (int i = 0; i < 16; ++i) xv[i] = tile[st * 32 + kc * 16 + i][lc];
    const int e = max(exps[J.exp_b + c0 + lc], kExpFloor);
    pack_unit16<S>(xv, e, arena + J.dst_b + ((int64_t)stage * S * J.rc_b + core) * 256 + kc * 128 + r8 * 16,
                   (int64_t)J.rc_b * 256);
  }
}

// 2^e for e in the normal range (exact).
__device__ __forceinline__ double pow2i(int e) {
  e = max(-1022, min(1023, e));
  return __longlong_as_double((long long)(e + 1023) << 52);
}

constexpr int LDE = TN + 1;  // staged epilogue tile leading dim (doubles)

template <int S>
struct OzPCfg {
  // TMEM: one accumulator set = S diagonals x TN columns; two sets (epilogue of tile i overlaps the
  // MMAs of tile i+1) when they fit the 512 columns, else one (the epilogue drains it first thing)
  static constexpr uint32_t ACC_COLS = S * TN;
  static constexpr int NBUF = 2 * ACC_COLS <= 512 ? 2 : 1;
  static constexpr uint32_t ALLOC = NBUF * ACC_COLS <= 256 ? 256 : 512;
  static_assert(ACC_COLS <= 512, "S x TN accumulator columns exceed TMEM");
  static constexpr int STAGE = OzCfg<S>::STAGE;
  static constexpr size_t TILE_BYTES = (size_t)TM * LDE * sizeof(double);
  static constexpr int STAGES_RAW = (int)((226 * 1024 - TILE_BYTES - 1024) / STAGE);
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE + TILE_BYTES + 1024;
};

struct OzItem {
  int pi, tm, tn, split, s0, nk;
  int64_t tile;
};

__device__ __forceinline__ bool oz_decode(const GemmProblem* __restrict__ probs, const OzProb* __restrict__ tps,
                                          const int64_t* __restrict__ begin, int nprob,
                                          const int32_t* __restrict__ mask, int64_t item, OzItem& it) {
  it.pi = find64<GemmProblem>(begin, nprob, item);
  const GemmProblem& P = probs[it.pi];
  if ((P.flags & kGemmMasked) && mask && !mask[P.mask_index]) return false;
  const OzProb& T_ = tps[it.pi];
  const int64_t l = item - begin[it.pi];
  it.split = (int)(l % T_.ksplit);
  it.tile = l / T_.ksplit;
  if (P.flags & kGemmSym) sym_decode(it.tile, T_.nt, it.tm, it.tn);
  else {
    it.tm = (int)(it.tile / T_.nt);
    it.tn = (int)(it.tile % T_.nt);
  }
  it.s0 = it.split * T_.kst;
  it.nk = min(T_.ks, it.s0 + T_.kst) - it.s0;
  return true;
}

template <typename T, int S>
__global__ void __launch_bounds__(GEMM_THREADS_P, 1) k_oz_gemm_p(const GemmProblem* __restrict__ probs,
                                                               const OzProb* __restrict__ tps,
                                                               const int64_t* __restrict__ begin, int nprob,
                                                               int64_t total_items, const int32_t* __restrict__ mask,
                                                               const int8_t* __restrict__ arena,
                                                               const int32_t* __restrict__ exps, double* __restrict__ ws,
                                                               const CUtensorMap* __restrict__ tmaps, int tag) {
  using Cfg = OzCfg<S>;
  using PC = OzPCfg<S>;
  extern __shared__ __align__(1024) uint8_t oz_smem[];
  __shared__ __align__(8) uint64_t full_bar[PC::STAGES][2], empty_bar[PC::STAGES], tfull[PC::NBUF],
      tempty[PC::NBUF];
  __shared__ uint32_t tmem_slot;
  __shared__ double col_scale[TN];
  __shared__ int64_t row_off[TM], col_off[TN], mrow_off[TN], mcol_off[TM];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // 1024-aligned base by pointer arithmetic on the __shared__ array (no integer round trip), so the
  // compiler keeps the shared address space: tileS accesses are LDS/STS, not generic loads and
  // stores that it must order against the epilogue's global stores (the store loop had serialised
  // on exactly that: 13 us per tile)
  uint8_t* sbase = oz_smem + ((1024u - (smem_u32(oz_smem) & 1023u)) & 1023u);
  double* tileS = reinterpret_cast<double*>(sbase + (size_t)PC::STAGES * PC::STAGE);

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < PC::STAGES; ++i) {
      mbar_init(&full_bar[i][0], 1);
      mbar_init(&full_bar[i][1], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int b = 0; b < PC::NBUF; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "n"(PC::ALLOC)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // producer
      uint32_t g = 0;
      OzItem it;
      for (int64_t item = blockIdx.x; item < total_items; item += gridDim.x) {
        if (!oz_decode(probs, tps, begin, nprob, mask, item, it)) continue;
        const OzProb& T_ = tps[it.pi];
        const int a_cores = min(TM / 8, T_.a_rc - it.tm * (TM / 8));
        const int b_cores = min(TN / 8, T_.b_rc - it.tn * (TN / 8));
        const int64_t a_plane = (int64_t)T_.a_rc * 256, b_plane = (int64_t)T_.b_rc * 256;
        const int8_t* a_src = arena + T_.a_pack + (int64_t)it.s0 * S * a_plane + (int64_t)it.tm * (TM / 8) * 256;
        const int8_t* b_src = arena + T_.b_pack + (int64_t)it.s0 * S * b_plane + (int64_t)it.tn * (TN / 8) * 256;
        const uint32_t a_bytes = (uint32_t)a_cores * 256, b_bytes = (uint32_t)b_cores * 256;
        for (int k = 0; k < it.nk; ++k, ++g) {
          const int st = (int)(g % PC::STAGES);
          const uint32_t use = g / PC::STAGES;
          if (g >= (uint32_t)PC::STAGES) mbar_wait(&empty_bar[st], (use & 1u) ^ 1u);
          uint8_t* sb = sbase + (size_t)st * PC::STAGE;
          constexpr int SH = (S + 1) / 2;
          if (tmaps) {
            const CUtensorMap* tm3 = tmaps + 3 * it.pi;
            const int z = (it.s0 + k) * S;
            mbar_expect_tx(&full_bar[st][0], (uint32_t)(S * (TN / 8) * 256 + SH * (TM / 8) * 256));
            mbar_expect_tx(&full_bar[st][1], (uint32_t)((S - SH) * (TM / 8) * 256));
            tma_load_3d(sb + Cfg::A_BYTES, tm3 + 2, 0, it.tn * (TN / 8), z, &full_bar[st][0]);
            tma_load_3d(sb, tm3 + 0, 0, it.tm * (TM / 8), z, &full_bar[st][0]);
            tma_load_3d(sb + SH * (TM / 8) * 256, tm3 + 1, 0, it.tm * (TM / 8), z + SH, &full_bar[st][1]);
            continue;
          }
          mbar_expect_tx(&full_bar[st][0], (uint32_t)S * b_bytes + (uint32_t)SH * a_bytes);
          mbar_expect_tx(&full_bar[st][1], (uint32_t)(S - SH) * a_bytes);
          const int8_t* as = a_src + (int64_t)k * S * a_plane;
          const int8_t* bs = b_src + (int64_t)k * S * b_plane;
#pragma unroll
          for (int q = 0; q < S; ++q) {
            bulk_g2s(sb + Cfg::A_BYTES + q * (TN / 8) * 256, bs + q * b_plane, b_bytes, &full_bar[st][0]);
            if (q < SH) bulk_g2s(sb + q * (TM / 8) * 256, as + q * a_plane, a_bytes, &full_bar[st][0]);
          }
#pragma unroll
          for (int q = SH; q < S; ++q) bulk_g2s(sb + q * (TM / 8) * 256, as + q * a_plane, a_bytes, &full_bar[st][1]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      uint32_t g = 0, tcount = 0;
      OzItem it;
      for (int64_t item = blockIdx.x; item < total_items; item += gridDim.x) {
        if (!oz_decode(probs, tps, begin, nprob, mask, item, it)) continue;
        const uint32_t b = tcount % PC::NBUF;
        mbar_wait(&tempty[b], ((tcount / PC::NBUF) & 1u) ^ 1u);  // the epilogue drained this buffer
        tc_fence_after();
        const uint32_t acc = tmem + b * PC::ACC_COLS;
        for (int k = 0; k < it.nk; ++k, ++g) {
          const int st = (int)(g % PC::STAGES);
          const uint32_t par = (g / PC::STAGES) & 1u;
          mbar_wait(&full_bar[st][0], par);
          tc_fence_after();
          const uint32_t sa_base = smem_u32(sbase + (size_t)st * PC::STAGE);
          const uint32_t sb_base = sa_base + Cfg::A_BYTES;
#pragma unroll
          for (int sa = 0; sa < S; ++sa) {
            if (sa == (S + 1) / 2) {
              mbar_wait(&full_bar[st][1], par);
              tc_fence_after();
            }
            const uint64_t ad = sdesc(sa_base + sa * (TM / 8) * 256, 128, 256);
#pragma unroll
            for (int sb0 = 0; sb0 < S - sa; sb0 += SL_PER_MMA) {
              const int nsl = min(SL_PER_MMA, S - sa - sb0);
              const uint64_t bd = sdesc(sb_base + sb0 * (TN / 8) * 256, 128, 256);
              const uint32_t idesc = Cfg::IDESC_BASE | ((uint32_t)(nsl * TN >> 3) << 17);
              tc_mma_i8(acc + (uint32_t)((sa + sb0) * TN), ad, bd, idesc, (k > 0 || sa > 0) ? 1u : 0u);
            }
          }
          tc_commit(&empty_bar[st]);
        }
        tc_commit(&tfull[b]);  // accumulators of this tile complete
        atomicAdd(&g_oz_mma_units, (unsigned long long)it.nk * (S * (S + 1) / 2));
        atomicAdd(&g_oz_mma_units_tag[tag], (unsigned long long)it.nk * (S * (S + 1) / 2));
        ++tcount;
      }
    }
  } else {
    // 8 epilogue warps: warp w drains TMEM lanes 32 (w % 4) .. +31, the two warpgroups split the columns
    const int et = threadIdx.x - 64;
    const int lg = warp & 3;
    const int rl = lg * 32 + lane;
    const int cbeg = (et >= 128) ? TN / 2 : 0;
    uint32_t tcount = 0;
    OzItem it;
    for (int64_t item = blockIdx.x; item < total_items; item += gridDim.x) {
      if (!oz_decode(probs, tps, begin, nprob, mask, item, it)) continue;
      const GemmProblem& P = probs[it.pi];
      const OzProb& T_ = tps[it.pi];
      const int tm = it.tm, tn = it.tn;
      asm volatile("bar.sync 1, 256;" ::: "memory");  // previous tile's readers of the smem arrays done
      if (et < TN) {
        const int gj = tn * TN + et;
        col_scale[et] = pow2i(exps[T_.b_exp + min(gj, T_.b_rc * 8 - 1)]);
        col_off[et] = evx(P.c_c, gj);
        mrow_off[et] = evx(P.c_r, gj);
      }
      if (et < TM) {
        const int gi = tm * TM + et;
        row_off[et] = evx(P.c_r, gi);
        mcol_off[et] = evx(P.c_c, gi);
      }
      if ((P.flags & kGemmReadC) && T_.ksplit == 1) {
        // beta C does not depend on the MMAs: pull this thread's half row of the C tile into L2 while
        // they run (small-K statistics tiles are otherwise bound by the epilogue's C round trips)
        const int gi = tm * TM + (et >> 1), gj = tn * TN + (et & 1) * (TN / 2);
        if (gi < P.M && gj < P.N) {
          const char* pc = reinterpret_cast<const char*>(static_cast<const T*>(P.C) + evx(P.c_r, gi) + evx(P.c_c, gj));
#pragma unroll
          for (int o = 0; o < (int)(TN / 2 * sizeof(T)); o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(pc + o));
        }
      }
      const uint32_t b = tcount % PC::NBUF;
      mbar_wait_sleep(&tfull[b], (tcount / PC::NBUF) & 1u);
      tc_fence_after();
      const uint32_t acc = tmem + b * PC::ACC_COLS;
      const double rscale = pow2i(exps[T_.a_exp + min(tm * TM + rl, T_.a_rc * 8 - 1)]);
      constexpr int H = (S + 1) / 2;
      for (int c0 = cbeg; c0 < cbeg + TN / 2; c0 += 16) {
        long long hi[16], lo[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) hi[q] = lo[q] = 0;
        if (it.nk > 0) {
          // two batches of diagonals (hi: d < H, lo: d >= H), each with its loads in flight together
          const uint32_t ta = acc + ((uint32_t)(lg * 32) << 16) + (uint32_t)c0;
          {
            uint32_t raw[H][16];
#pragma unroll
            for (int d = 0; d < H; ++d) tmem_ld16_async(ta + (uint32_t)(d * TN), raw[d]);
            tmem_wait_ld();
#pragma unroll
            for (int d = 0; d < H; ++d) {
              reg_fence16(raw[d]);
#pragma unroll
              for (int q = 0; q < 16; ++q) hi[q] += (long long)(int32_t)raw[d][q] << (7 * (H - 1 - d));
            }
          }
          if constexpr (S > H) {
            uint32_t raw[S - H][16];
#pragma unroll
            for (int d = H; d < S; ++d) tmem_ld16_async(ta + (uint32_t)(d * TN), raw[d - H]);
            tmem_wait_ld();
#pragma unroll
            for (int d = H; d < S; ++d) {
              reg_fence16(raw[d - H]);
#pragma unroll
              for (int q = 0; q < 16; ++q) lo[q] += (long long)(int32_t)raw[d - H][q] << (7 * (S - 1 - d));
            }
          }
        }
        const double whi = pow2i(-7 * (H + 1)), wlo = pow2i(-7 * (S + 1));
#pragma unroll
        for (int q = 0; q < 16; ++q)
          tileS[rl * LDE + c0 + q] = fma((double)hi[q], whi, (double)lo[q] * wlo) * rscale;
      }
      tc_fence_before();
      asm volatile("bar.sync 1, 256;" ::: "memory");  // all TMEM reads of buffer b done, tileS complete
      if (et == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[b])) : "memory");
      ++tcount;
      // problem fields in registers: C's stores could alias the problem table as far as the
      // compiler knows, which made it reload them after every store
      const int pflags = P.flags, PM = P.M, PN = P.N;
      const double palpha = P.alpha, pbeta = P.beta;
      const bool sym = (pflags & kGemmSym) != 0;
      if (T_.ksplit == 1) {
        T* __restrict__ C = static_cast<T*>(P.C);
        const bool readc = (pflags & kGemmReadC) != 0;
        const bool mirror = sym && !(pflags & kGemmLowerOnly);
        // thread et owns column c = et % TN of rows et / TN + 4 u: the column's scale and offset
        // are loaded once (the tensor core's operand reads keep shared memory busy while the
        // epilogue runs: fewer LDS per element)
        constexpr int RSTEP = 256 / TN, PER = 16;  // C values loaded per round trip (before any store)
        const int c = et % TN, rb = et / TN, gj = tn * TN + c;
        const double cs = palpha * col_scale[c];
        const int64_t coff = col_off[c];
        const bool cin = gj < PN;
        for (int r0 = rb; r0 < TM; r0 += PER * RSTEP) {
          double cv[PER];
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int r = r0 + u * RSTEP, gi = tm * TM + r;
            const bool live = cin && gi < PM && !(sym && gi < gj);
            cv[u] = (readc && live) ? (double)__ldcg(C + row_off[r] + coff) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int r = r0 + u * RSTEP, gi = tm * TM + r;
            if (!cin || gi >= PM || (sym && gi < gj)) continue;
            double val = tileS[r * LDE + c] * cs;
            if (readc) val = fma(pbeta, cv[u], val);
            if (mirror) tileS[r * LDE + c] = val;
            __stcg(C + row_off[r] + coff, (T)val);  // global stores (C is a generic pointer)
          }
        }
        if (mirror) {
          asm volatile("bar.sync 1, 256;" ::: "memory");
          for (int e = et; e < TM * TN; e += 256) {
            const int c = e / TM, r = e % TM;
            const int gi = tm * TM + r, gj = tn * TN + c;
            if (gi >= PM || gj >= PN || gi <= gj) continue;
            __stcg(C + mrow_off[c] + mcol_off[r], (T)tileS[r * LDE + c]);
          }
        }
      } else {
        double* dst = ws + T_.ws_off + (it.tile * T_.ksplit + it.split) * (int64_t)(TM * TN);
        for (int e = et; e < TM * TN; e += 256) {
          const int r = e / TN, c = e % TN;
          dst[e] = tileS[r * LDE + c] * col_scale[c];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(PC::ALLOC) : "memory");
  }
}

// Split-K: scaled partial tiles summed in split order in FP64, then the epilogue.
template <typename T>
__global__ void __launch_bounds__(256) k_oz_reduce(const GemmProblem* __restrict__ probs, const OzProb* __restrict__ tps,
                                                   const int64_t* __restrict__ rbegin, const int32_t* __restrict__ rprob,
                                                   int nred, const int32_t* __restrict__ mask,
                                                   const double* __restrict__ ws) {
  const int r = find64<int32_t>(rbegin, nred, blockIdx.x);
  const int pi = rprob[r];
  const GemmProblem P = probs[pi];  // by value: fields stay in registers across the stores to C
  if ((P.flags & kGemmMasked) && mask && !mask[P.mask_index]) return;
  const OzProb& T_ = tps[pi];
  const int64_t tile = blockIdx.x - rbegin[r];
  int tm, tn;
  if (P.flags & kGemmSym) sym_decode(tile, T_.nt, tm, tn);
  else {
    tm = (int)(tile / T_.nt);
    tn = (int)(tile % T_.nt);
  }
  const double* base = ws + T_.ws_off + tile * T_.ksplit * (int64_t)(TM * TN);
  for (int e = threadIdx.x; e < TM * TN; e += blockDim.x) {
    const int gi = tm * TM + e / TN, gj = tn * TN + e % TN;
    if (gi >= P.M || gj >= P.N) continue;
    double acc = 0.0;
    for (int sp = 0; sp < T_.ksplit; ++sp) acc += base[(int64_t)sp * TM * TN + e];
    oz_store<T>(P, gi, gj, acc);
  }
}

}  // namespace

namespace {
bool same_idx(const Idx2& a, const Idx2& b) { return a.div == b.div && a.hi == b.hi && a.lo == b.lo; }
bool same_operand(const GemmProblem& p) {
  const bool xa = (p.flags & kGemmXformA) != 0, xb = (p.flags & kGemmXformB) != 0;
  if (xa != xb || (xa && (p.a_xa != p.b_xa || p.a_xb != p.b_xb || p.a_fexp != p.b_fexp))) return false;
  return p.A == p.B && p.M == p.N && same_idx(p.a_r, p.b_r) && same_idx(p.a_k, p.b_k);
}
}  // namespace

// Runs BODY with `constexpr int S` = the batch's slice count (the instantiated set).
#define OZ_DISPATCH(SV, ...)                                 \
  switch (SV) {                                              \
    case 3: { constexpr int S = 3; __VA_ARGS__; } break;     \
    case 4: { constexpr int S = 4; __VA_ARGS__; } break;     \
    case 5: { constexpr int S = 5; __VA_ARGS__; } break;     \
    case 6: { constexpr int S = 6; __VA_ARGS__; } break;     \
    default: { constexpr int S = 8; __VA_ARGS__; } break;    \
  }

template <typename T>
int OzakiGemmBatch<T>::set_slices(int s) {
  if (s != 3 && s != 4 && s != 5 && s != 6 && s != 8) {
    set_error("Ozaki slice count must be one of 3, 4, 5, 6, 8");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  S_ = s;
  return SHAMPOO_OK;
}

template <typename T, int S>
static cudaError_t oz_set_smem_attrs() {
  static const cudaError_t e = [] {
    return cudaFuncSetAttribute(k_oz_gemm_p<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)OzPCfg<S>::SMEM);
  }();  // once per instantiation, thread-safe
  return e;
}

// Kernel-level timing of the GEMM launches (bench evidence): CUDA events around each k_oz_gemm_p
// launch on its stream, bucketed by the calling thread's step-phase tag (oz_set_tag).
thread_local int t_oz_tag = kOzTags - 1;
struct OzGemmTimer {
  std::atomic<bool> on{false};
  std::mutex mu;
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> pending;
  std::vector<cudaEvent_t> pool;
  void begin(cudaStream_t s, cudaEvent_t* a, cudaEvent_t* b) {
    {
      std::lock_guard<std::mutex> lk(mu);
      for (cudaEvent_t* e : {a, b}) {
        if (pool.empty()) {
          cudaEventCreate(e);
        } else {
          *e = pool.back();
          pool.pop_back();
        }
      }
    }
    cudaEventRecord(*a, s);
  }
  void end(cudaStream_t s, int tag, cudaEvent_t a, cudaEvent_t b) {
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> lk(mu);
    pending.emplace_back(tag, a, b);
  }
};
OzGemmTimer g_oz_timer;
int oz_tag() { return t_oz_tag; }

template <typename T>
OzakiGemmBatch<T>::~OzakiGemmBatch() {
  dev_free(d_prob_);
  dev_free(d_tp_);
  dev_free(d_begin_);
  for (auto& ps : sets_) {
    dev_free(ps.d_jobs);
    dev_free(ps.d_pbegin);
    dev_free(ps.d_ebegin);
    dev_free(ps.d_cbegin);
    dev_free(ps.d_dual);
    dev_free(ps.d_dxbegin);
    dev_free(ps.d_dpbegin);
  }
  dev_free(d_rbegin_);
  dev_free(d_rprob_);
  if (own_arena_) dev_free(arena_);
  dev_free(exps_);
  dev_free(ws_);
  dev_free(d_tmaps_);
}

inline bool k_contig_host(const OzPackJob& J) { return J.k.div == 0x7fffffff && J.k.lo == 1; }

// Moves every (rows of X, columns of X) job pair out of `jobs` into `dual`: a = rows (unit k
// stride, row stride ld >= K), b = columns (unit row stride, k stride ld) of the same source, both
// untransformed with computed exponents.
static void pair_transposed(std::vector<OzPackJob>& jobs, std::vector<OzDualJob>& dual) {
  auto plain = [](const OzPackJob& J) { return J.xa == 1.0 && J.xb == 0.0 && J.fexp == kNoFixedExp; };
  std::map<std::tuple<const void*, int64_t, int32_t, int32_t>, size_t> rows_of;  // (src, ld, R, C) -> a
  for (size_t i = 0; i < jobs.size(); ++i) {
    const OzPackJob& J = jobs[i];
    if (plain(J) && k_contig_host(J) && J.r.div == 0x7fffffff && J.r.lo >= J.K && J.rows > 0 && J.K > 0)
      rows_of.emplace(std::make_tuple(J.src, J.r.lo, J.rows, J.K), i);
  }
  std::vector<char> gone(jobs.size(), 0);
  for (size_t i = 0; i < jobs.size(); ++i) {
    const OzPackJob& B = jobs[i];
    if (!plain(B) || B.r.div != 0x7fffffff || B.r.lo != 1 || B.k.div != 0x7fffffff || B.k.lo < 2) continue;
    const auto it = rows_of.find(std::make_tuple(B.src, B.k.lo, B.K, B.rows));
    if (it == rows_of.end() || gone[it->second]) continue;
    const OzPackJob& A = jobs[it->second];
    OzDualJob D{};
    D.src = A.src;
    D.ld = A.r.lo;
    D.R = A.rows;
    D.C = A.K;
    D.mask_a = A.mask_index;
    D.mask_b = B.mask_index;
    D.rc_a = A.rc;
    D.rc_b = B.rc;
    D.ks_b = B.ks;
    D.dst_a = A.dst;
    D.dst_b = B.dst;
    D.exp_a = A.exp;
    D.exp_b = B.exp;
    dual.push_back(D);
    gone[it->second] = gone[i] = 1;
  }
  std::vector<OzPackJob> rest;
  for (size_t i = 0; i < jobs.size(); ++i)
    if (!gone[i]) rest.push_back(jobs[i]);
  jobs.swap(rest);
}

template <typename T>
int OzakiGemmBatch<T>::upload() {
  if (host.empty()) return SHAMPOO_OK;
  const int S = S_;
  {
    cudaError_t attr = cudaSuccess;
    OZ_DISPATCH(S, attr = oz_set_smem_attrs<T, S>());
    SH_CUDA_CHECK(attr);
  }
  std::vector<OzProb> tp(host.size());
  std::vector<int> a_set(host.size(), 0), b_set(host.size(), 0);
  std::vector<int64_t> begin(host.size()), rbegin, pbegin[2], ebegin[2], cbegin[2];
  std::vector<int32_t> rprob;
  std::vector<OzPackJob> jobs[2];
  int64_t arena = 0, wsz = 0, exp_count[2] = {0, 0};
  total_items_ = total_red_ = 0;
  mma_count_ = 0;
  for (auto& ps : sets_) ps = PackSet{};
  // exponent offsets are relative to the set; fixed up once both sets are sized
  // share_packs_: problems reading the same operand (same source, geometry, set) share one pack; the
  // first registered problem's mask governs it (the caller orders the problems so that it does)
  struct PackKey {
    int set;
    const void* src;
    int64_t r0, r1, r2, k0, k1, k2;
    int rows, K, ks;
    double xa, xb;
    int fexp;
    bool operator<(const PackKey& o) const {
      return std::tie(set, src, r0, r1, r2, k0, k1, k2, rows, K, ks, xa, xb, fexp) <
             std::tie(o.set, o.src, o.r0, o.r1, o.r2, o.k0, o.k1, o.k2, o.rows, o.K, o.ks, o.xa, o.xb, o.fexp);
    }
  };
  std::map<PackKey, std::tuple<int64_t, int32_t, int64_t>> packed;
  auto add_pack = [&](int set, const void* src, Idx2 r, Idx2 k, int rows, int K, int ks, int mask_index,
                      int64_t& off, int32_t& rc, int64_t& exp, double xa, double xb, int fexp) {
    const PackKey key{set, src, r.div, r.hi, r.lo, k.div, k.hi, k.lo, rows, K, ks, xa, xb, fexp};
    if (share_packs_) {
      const auto it = packed.find(key);
      if (it != packed.end()) {
        std::tie(off, rc, exp) = it->second;
        return;
      }
    }
    rc = std::max(1, (rows + 7) / 8);
    off = arena;
    arena += (int64_t)ks * rc * S * 256;
    exp = exp_count[set];
    exp_count[set] += rc * 8;
    OzPackJob J{};
    J.src = src;
    J.r = r;
    J.k = k;
    J.rows = rows;
    J.K = K;
    J.ks = ks;
    J.rc = rc;
    J.mask_index = mask_index;
    J.dst = off;
    J.exp = exp;
    J.units = (int64_t)ks * rc * 16;
    J.xa = xa;
    J.xb = xb;
    J.fexp = fexp;
    J.echunks = (k.div == 0x7fffffff && k.lo == 1)
                    ? (int64_t)rows * ((K + EXP_WARP_CHUNK - 1) / EXP_WARP_CHUNK) * 32  // threads (warps x 32)
                    : (int64_t)rows * ((K + EXP_CHUNK - 1) / EXP_CHUNK);
    jobs[set].push_back(J);
    if (share_packs_) packed[key] = std::make_tuple(off, rc, exp);
  };
  for (size_t i = 0; i < host.size(); ++i) {
    GemmProblem& p = host[i];
    OzProb& t = tp[i];
    t.mt = (p.M + TM - 1) / TM;
    t.nt = (p.N + TN - 1) / TN;
    t.ks = std::max(1, (p.K + TKB - 1) / TKB);
    t.ksplit = (int32_t)std::max<int64_t>(1, (t.ks + kOzSplitStages - 1) / kOzSplitStages);
    t.kst = (t.ks + t.ksplit - 1) / t.ksplit;
    t.ksplit = (t.ks + t.kst - 1) / t.kst;
    const bool sym = (p.flags & kGemmSym) != 0;
    // SYM output with A == B (a SYRK) shares one pack; SYM output of two distinct operands (products
    // of commuting symmetric matrices, e.g. the coupled-Newton iterates) packs both
    const bool share = sym && same_operand(p);
    if (p.M == 0 || p.N == 0) t.tiles = 0;
    else t.tiles = sym ? sym_tiles_before(t.mt, t.nt) : (int64_t)t.mt * t.nt;
    const int mi = (p.flags & kGemmMasked) ? p.mask_index : -1;
    const int aset = (p.flags & kGemmConstA) ? 1 : 0;
    const bool xfa = (p.flags & kGemmXformA) != 0, xfb = (p.flags & kGemmXformB) != 0;
    add_pack(aset, p.A, p.a_r, p.a_k, p.M, p.K, t.ks, mi, t.a_pack, t.a_rc, t.a_exp, xfa ? p.a_xa : 1.0,
             xfa ? p.a_xb : 0.0, xfa ? p.a_fexp : kNoFixedExp);
    a_set[i] = aset;
    if (share) {
      t.b_pack = t.a_pack;
      t.b_rc = t.a_rc;
      t.b_exp = t.a_exp;
    } else {
      const int bset = (p.flags & kGemmConstB) ? 1 : 0;
      add_pack(bset, p.B, p.b_r, p.b_k, p.N, p.K, t.ks, mi, t.b_pack, t.b_rc, t.b_exp, xfb ? p.b_xa : 1.0,
               xfb ? p.b_xb : 0.0, xfb ? p.b_fexp : kNoFixedExp);
      b_set[i] = bset;
    }
    t.ws_off = 0;
    if (t.ksplit > 1 && t.tiles > 0) {
      t.ws_off = wsz;
      wsz += t.tiles * t.ksplit * (int64_t)(TM * TN);
      rbegin.push_back(total_red_);
      rprob.push_back((int32_t)i);
      total_red_ += t.tiles;
    }
    begin[i] = total_items_;
    total_items_ += t.tiles * t.ksplit;
    mma_count_ += (double)t.tiles * t.ks * (S * (S + 1) / 2);
  }
  // exponent layout: set 0 first, then set 1
  sets_[0].exp_begin = 0;
  sets_[0].exp_elems = exp_count[0];
  sets_[1].exp_begin = exp_count[0];
  sets_[1].exp_elems = exp_count[1];
  for (size_t i = 0; i < host.size(); ++i) {
    if (a_set[i] == 1) tp[i].a_exp += exp_count[0];
    if ((host[i].flags & kGemmSym) && same_operand(host[i])) tp[i].b_exp = tp[i].a_exp;
    else if (b_set[i] == 1) tp[i].b_exp += exp_count[0];
  }
  for (int q = 0; q < 2; ++q)
    for (auto& J : jobs[q]) J.exp += sets_[q].exp_begin;
  // transposed operand pairs leave the per-operand job lists for the dual kernels
  std::vector<OzDualJob> dual[2];
  std::vector<int64_t> dxbegin[2], dpbegin[2];
  const char* dp_env = std::getenv("SHAMPOO_OZ_DUAL_PACK");
  if (!dp_env || std::atoi(dp_env) != 0)
    for (int q = 0; q < 2; ++q) pair_transposed(jobs[q], dual[q]);
  for (int q = 0; q < 2; ++q) {
    PackSet& ps = sets_[q];
    for (const OzPackJob& J : jobs[q]) {
      pbegin[q].push_back(ps.pack_ctas);
      ps.pack_ctas += (J.units + PACK_UNITS - 1) / PACK_UNITS;
      ebegin[q].push_back(ps.exp_ctas);
      ps.exp_ctas += std::max<int64_t>(1, (J.echunks + 255) / 256);
      cbegin[q].push_back(ps.core_ctas);
      ps.core_ctas += (J.rc + PACK_CORES - 1) / PACK_CORES;
      if (!k_contig_host(J)) ps.all_contig = false;
      if (J.xa != 1.0 || J.xb != 0.0) ps.has_xform = true;
    }
    for (const OzDualJob& D : dual[q]) {
      dxbegin[q].push_back(ps.dual_exp_ctas);
      ps.dual_exp_ctas += (int64_t)((D.R + DX_R - 1) / DX_R) * ((D.C + DX_C - 1) / DX_C);
      dpbegin[q].push_back(ps.dual_pack_ctas);
      ps.dual_pack_ctas += (int64_t)((D.R + DP_R - 1) / DP_R) * ((D.C + DP_C - 1) / DP_C);
    }
  }
  for (auto& ps : sets_) {
    ps.fused_ok = ps.all_contig && ps.core_ctas >= 2 * kNumSMs;
    if (ps.has_xform && !ps.all_contig) {
      set_error("affine operand packs need row-contiguous operands");
      return SHAMPOO_ERR_INVALID_ARGUMENT;
    }
  }
  nred_ = (int)rbegin.size();
  SH_CUDA_CHECK(dev_malloc(&d_prob_, host.size() * sizeof(GemmProblem)));
  SH_CUDA_CHECK(dev_malloc(&d_tp_, tp.size() * sizeof(OzProb)));
  SH_CUDA_CHECK(dev_malloc(&d_begin_, begin.size() * sizeof(int64_t)));
  if (ext_arena_ && arena <= ext_cap_ && sets_[1].pack_ctas == 0 && sets_[1].dual_pack_ctas == 0) {
    arena_ = ext_arena_;
    own_arena_ = false;
  } else {
    SH_CUDA_CHECK(dev_malloc(&arena_, std::max<int64_t>(arena, 256)));
    own_arena_ = true;
  }
  SH_CUDA_CHECK(dev_malloc(&exps_, std::max<int64_t>(exp_count[0] + exp_count[1], 1) * sizeof(int32_t)));
  SH_CUDA_CHECK(cudaMemcpy(d_prob_, host.data(), host.size() * sizeof(GemmProblem), cudaMemcpyHostToDevice));
  SH_CUDA_CHECK(cudaMemcpy(d_tp_, tp.data(), tp.size() * sizeof(OzProb), cudaMemcpyHostToDevice));
  SH_CUDA_CHECK(cudaMemcpy(d_begin_, begin.data(), begin.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  for (int q = 0; q < 2; ++q) {
    PackSet& ps = sets_[q];
    ps.njobs = (int)jobs[q].size();
    if (!ps.njobs) continue;
    SH_CUDA_CHECK(dev_malloc(&ps.d_jobs, jobs[q].size() * sizeof(OzPackJob)));
    SH_CUDA_CHECK(dev_malloc(&ps.d_pbegin, pbegin[q].size() * sizeof(int64_t)));
    SH_CUDA_CHECK(dev_malloc(&ps.d_ebegin, ebegin[q].size() * sizeof(int64_t)));
    SH_CUDA_CHECK(cudaMemcpy(ps.d_jobs, jobs[q].data(), jobs[q].size() * sizeof(OzPackJob), cudaMemcpyHostToDevice));
    SH_CUDA_CHECK(cudaMemcpy(ps.d_pbegin, pbegin[q].data(), pbegin[q].size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    SH_CUDA_CHECK(cudaMemcpy(ps.d_ebegin, ebegin[q].data(), ebegin[q].size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    SH_CUDA_CHECK(dev_malloc(&ps.d_cbegin, cbegin[q].size() * sizeof(int64_t)));
    SH_CUDA_CHECK(cudaMemcpy(ps.d_cbegin, cbegin[q].data(), cbegin[q].size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  for (int q = 0; q < 2; ++q) {
    PackSet& ps = sets_[q];
    ps.ndual = (int)dual[q].size();
    if (!ps.ndual) continue;
    SH_CUDA_CHECK(dev_malloc(&ps.d_dual, dual[q].size() * sizeof(OzDualJob)));
    SH_CUDA_CHECK(dev_malloc(&ps.d_dxbegin, dual[q].size() * sizeof(int64_t)));
    SH_CUDA_CHECK(dev_malloc(&ps.d_dpbegin, dual[q].size() * sizeof(int64_t)));
    SH_CUDA_CHECK(cudaMemcpy(ps.d_dual, dual[q].data(), dual[q].size() * sizeof(OzDualJob), cudaMemcpyHostToDevice));
    SH_CUDA_CHECK(cudaMemcpy(ps.d_dxbegin, dxbegin[q].data(), dxbegin[q].size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    SH_CUDA_CHECK(cudaMemcpy(ps.d_dpbegin, dpbegin[q].data(), dpbegin[q].size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  cached_valid_ = false;
  // TMA tensor maps of the packed operands: [S * ks slices-by-stage][rc cores][256 B core block]
  {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        fn = nullptr;
      cudaGetLastError();
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    std::vector<CUtensorMap> maps(3 * host.size());
    bool ok = encode != nullptr && std::getenv("SHAMPOO_OZ_NO_TMA") == nullptr;
    const int SH = (S + 1) / 2;
    auto make = [&](CUtensorMap* m, int64_t off, int rc, int ks, int cores, int slices) {
      const cuuint64_t dims[3] = {256, (cuuint64_t)rc, (cuuint64_t)S * ks};
      const cuuint64_t strides[2] = {256, (cuuint64_t)rc * 256};
      const cuuint32_t box[3] = {256, (cuuint32_t)cores, (cuuint32_t)slices};
      const cuuint32_t es[3] = {1, 1, 1};
      return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, arena_ + off, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    for (size_t i = 0; i < host.size() && ok; ++i) {
      const OzProb& t = tp[i];
      if (t.tiles == 0) continue;
      ok = make(&maps[3 * i + 0], t.a_pack, t.a_rc, t.ks, TM / 8, SH) &&
           make(&maps[3 * i + 1], t.a_pack, t.a_rc, t.ks, TM / 8, S - SH) &&
           make(&maps[3 * i + 2], t.b_pack, t.b_rc, t.ks, TN / 8, S);
    }
    if (ok) {
      SH_CUDA_CHECK(dev_malloc(&d_tmaps_, maps.size() * sizeof(CUtensorMap)));
      SH_CUDA_CHECK(cudaMemcpy(d_tmaps_, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
    }
  }
  if (nred_ > 0) {
    SH_CUDA_CHECK(dev_malloc(&ws_, wsz * sizeof(double)));
    SH_CUDA_CHECK(dev_malloc(&d_rbegin_, rbegin.size() * sizeof(int64_t)));
    SH_CUDA_CHECK(dev_malloc(&d_rprob_, rprob.size() * sizeof(int32_t)));
    SH_CUDA_CHECK(cudaMemcpy(d_rbegin_, rbegin.data(), rbegin.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    SH_CUDA_CHECK(cudaMemcpy(d_rprob_, rprob.data(), rprob.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  return SHAMPOO_OK;
}

template <typename T>
int OzakiGemmBatch<T>::launch_pack(const PackSet& ps, cudaStream_t s, const int32_t* mask) const {
  if (ps.ndual) {
    SH_CUDA_CHECK(cudaMemsetAsync(exps_ + ps.exp_begin, 0x80, ps.exp_elems * sizeof(int32_t), s));
    k_oz_dual_exp<T><<<(unsigned)ps.dual_exp_ctas, 256, 0, s>>>(ps.d_dual, ps.d_dxbegin, ps.ndual, mask, exps_);
    SH_LAUNCH_CHECK();
    OZ_DISPATCH(S_, (k_oz_pack_dual<T, S><<<(unsigned)ps.dual_pack_ctas, 256, 0, s>>>(ps.d_dual, ps.d_dpbegin,
                                                                                       ps.ndual, mask, exps_,
                                                                                       arena_)));
    SH_LAUNCH_CHECK();
  }
  if (!ps.njobs) return SHAMPOO_OK;
  // The fused single-pass kernel wins on row-contiguous operands with enough rows to fill the machine
  // (the root inverse's n x n iterates: 34.7 -> 27.0 ms of packing per steady-state refresh); operands
  // with strided k or few long rows (the mode-product B operands) keep the two-kernel path, whose
  // rowexp/pack grids scale with K (measured: fused 0.53 vs 0.30 ms on the plain step's packs).
  static const bool fused = [] {
    const char* e = std::getenv("SHAMPOO_OZ_FUSED_PACK");
    return e ? std::atoi(e) != 0 : true;  // 0: always the two-pass k_oz_rowexp + k_oz_pack (A/B)
  }();
  if (ps.has_xform) {  // affine operands are packed by the fused kernel only (its transform instantiation)
    OZ_DISPATCH(S_, (k_oz_pack_rows<T, S, true><<<(unsigned)ps.core_ctas, 256, 0, s>>>(ps.d_jobs, ps.d_cbegin,
                                                                                        ps.njobs, mask, exps_,
                                                                                        arena_)));
    SH_LAUNCH_CHECK();
    return SHAMPOO_OK;
  }
  if (fused && ps.fused_ok) {
    OZ_DISPATCH(S_, (k_oz_pack_rows<T, S, false><<<(unsigned)ps.core_ctas, 256, 0, s>>>(ps.d_jobs, ps.d_cbegin,
                                                                                         ps.njobs, mask, exps_,
                                                                                         arena_)));
    SH_LAUNCH_CHECK();
    return SHAMPOO_OK;
  }
  if (!ps.ndual)  // very negative (done above with the pairs)
    SH_CUDA_CHECK(cudaMemsetAsync(exps_ + ps.exp_begin, 0x80, ps.exp_elems * sizeof(int32_t), s));
  k_oz_rowexp<T><<<(unsigned)ps.exp_ctas, 256, 0, s>>>(ps.d_jobs, ps.d_ebegin, ps.njobs, mask, exps_);
  SH_LAUNCH_CHECK();
  OZ_DISPATCH(S_, k_oz_pack<T, S><<<(unsigned)ps.pack_ctas, PACK_UNITS, 0, s>>>(ps.d_jobs, ps.d_pbegin, ps.njobs,
                                                                                mask, exps_, arena_));
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

template <typename T>
int OzakiGemmBatch<T>::launch(cudaStream_t s, const int32_t* mask) const {
  if (total_items_ == 0) return SHAMPOO_OK;
  int rc;
  if (!cached_valid_) {
    if ((rc = launch_pack(sets_[1], s, mask))) return rc;
    cached_valid_ = true;
  }
  if ((rc = launch_pack(sets_[0], s, mask))) return rc;
  const unsigned grid = (unsigned)std::min<int64_t>(total_items_, kNumSMs);
  const int tag = oz_tag();
  cudaEvent_t ea = nullptr, eb = nullptr;
  if (g_oz_timer.on.load(std::memory_order_relaxed)) g_oz_timer.begin(s, &ea, &eb);
  OZ_DISPATCH(S_, k_oz_gemm_p<T, S><<<grid, GEMM_THREADS_P, OzPCfg<S>::SMEM, s>>>(
                      d_prob_, d_tp_, d_begin_, (int)host.size(), total_items_, mask, arena_, exps_, ws_,
                      static_cast<const CUtensorMap*>(d_tmaps_), tag));
  SH_LAUNCH_CHECK();
  if (ea) g_oz_timer.end(s, tag, ea, eb);
  if (total_red_ > 0) {
    k_oz_reduce<T><<<(unsigned)total_red_, 256, 0, s>>>(d_prob_, d_tp_, d_rbegin_, d_rprob_, nred_, mask, ws_);
    SH_LAUNCH_CHECK();
  }
  return SHAMPOO_OK;
}

template <typename T>
double OzakiGemmBatch<T>::flops() const {
  double f = 0;
  for (const auto& p : host) f += 2.0 * p.M * (double)p.N * p.K;
  return f;
}

template <typename T>
double OzakiGemmBatch<T>::int8_ops() const {
  return mma_count_ * 2.0 * TM * TN * TKB;
}

template class OzakiGemmBatch<float>;
template class OzakiGemmBatch<double>;

}  // namespace shampoo

// ---------------------------------------------------------------- C ABI utility

namespace shampoo {
int oz_set_tag(int tag) {
  const int prev = t_oz_tag;
  t_oz_tag = (tag >= 0 && tag < kOzTags - 1) ? tag : kOzTags - 1;
  return prev;
}
}  // namespace shampoo

extern "C" int shampoo_gemm_timing(int32_t enable, double* ms, double* int8_ops, int64_t* launches) {
  using namespace shampoo;
  std::lock_guard<std::mutex> lk(g_oz_timer.mu);
  if (ms || launches) {
    for (int q = 0; q < kOzTags; ++q) {
      if (ms) ms[q] = 0.0;
      if (launches) launches[q] = 0;
    }
    for (auto& p : g_oz_timer.pending) {
      float e = 0.f;
      SH_CUDA_CHECK(cudaEventSynchronize(std::get<2>(p)));
      SH_CUDA_CHECK(cudaEventElapsedTime(&e, std::get<1>(p), std::get<2>(p)));
      if (ms) ms[std::get<0>(p)] += e;
      if (launches) launches[std::get<0>(p)] += 1;
    }
  }
  for (auto& p : g_oz_timer.pending) {
    g_oz_timer.pool.push_back(std::get<1>(p));
    g_oz_timer.pool.push_back(std::get<2>(p));
  }
  g_oz_timer.pending.clear();
  unsigned long long units[kOzTags] = {};
  SH_CUDA_CHECK(cudaMemcpyFromSymbol(units, g_oz_mma_units_tag, sizeof(units)));
  if (int8_ops)
    for (int q = 0; q < kOzTags; ++q) int8_ops[q] = (double)units[q] * 2.0 * TM * TN * TKB;
  const unsigned long long zero[kOzTags] = {};
  SH_CUDA_CHECK(cudaMemcpyToSymbol(g_oz_mma_units_tag, zero, sizeof(zero)));
  g_oz_timer.on.store(enable != 0);
  return SHAMPOO_OK;
}

extern "C" int shampoo_tc_counter(int32_t reset, double* int8_ops) {
  using namespace shampoo;
  unsigned long long units = 0;
  SH_CUDA_CHECK(cudaMemcpyFromSymbol(&units, g_oz_mma_units, sizeof(units)));
  if (int8_ops) *int8_ops = (double)units * 2.0 * TM * TN * TKB;
  if (reset) {
    const unsigned long long zero = 0;
    SH_CUDA_CHECK(cudaMemcpyToSymbol(g_oz_mma_units, &zero, sizeof(zero)));
  }
  return SHAMPOO_OK;
}

extern "C" int shampoo_tc_gemm(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                               int32_t symmetric, double alpha, double beta, int32_t dtype, void* stream) {
  using namespace shampoo;
  if (M < 0 || N < 0 || K < 0 || (symmetric && (A != B || M != N)) ||
      (dtype != SHAMPOO_DTYPE_F32 && dtype != SHAMPOO_DTYPE_F64)) {
    set_error("tc_gemm: invalid arguments");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  GemmProblem p = make_gemm(false, true, M, N, K, A, K, B, K, C, N, alpha, beta);
  if (symmetric) p.flags |= kGemmSym;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc;
  if (dtype == SHAMPOO_DTYPE_F32) {
    OzakiGemmBatch<float> b;
    b.add(p);
    if ((rc = b.upload()) || (rc = b.launch(s))) return rc;
    SH_CUDA_CHECK(cudaStreamSynchronize(s));
  } else {
    OzakiGemmBatch<double> b;
    b.add(p);
    if ((rc = b.upload()) || (rc = b.launch(s))) return rc;
    SH_CUDA_CHECK(cudaStreamSynchronize(s));
  }
  return SHAMPOO_OK;
}
