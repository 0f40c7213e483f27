// HBM-bound elementwise kernels of the step.  One CTA per Chunk (<= kChunk
// elements of one block), block-contiguous state arrays, per-chunk partial
// sums reduced per block in a fixed order (deterministic norms).
//
// Reference semantics (optim.py:278-354, grafting.py:68-110):
//   prepare: g (+wd*w if L2) -> graft accumulator -> beta1 filter -> ||P_graft||^2
//   final:   p = ready ? (||P_graft||/||P_sh||) P_sh : P_graft ; + wd*w ; momentum/Nesterov
//   apply:   W -= lr * p  for every block, read back from the gather buffer
#include "elementwise.cuh"

namespace shampoo {

namespace {

constexpr int NT = 256;

template <typename T>
__device__ __forceinline__ T graft_dir(int32_t graft, T ge, T acc, double inv_bc2, double eps) {
  if (graft == SHAMPOO_GRAFT_SGD) return ge;
  return ge / (T(sqrt((double)acc * inv_bc2)) + T(eps));
}

__device__ __forceinline__ bool graft_summed(int32_t g) {
  return g == SHAMPOO_GRAFT_ADAGRAD || g == SHAMPOO_GRAFT_NORMALIZED_ADAGRAD;
}
__device__ __forceinline__ bool graft_normalized(int32_t g) {
  return g >= SHAMPOO_GRAFT_NORMALIZED_ADAGRAD;
}

__global__ void __launch_bounds__(NT) k_finite(const Chunk* __restrict__ chunks,
                                               const DevBlock* __restrict__ params,
                                               const void* const* __restrict__ grads, int32_t dtype,
                                               int32_t* flag, int32_t* go) {
  const Chunk c = chunks[blockIdx.x];
  const void* g = grads[params[c.block].param];
  int bad = 0;
  for (int64_t e = threadIdx.x; e < c.count; e += NT) {
    const double v = load_as<double>(g, c.start + e, dtype);
    if (!isfinite(v)) bad = 1;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) {
    atomicOr(flag, 1);
    if (go) *go = 0;  // deferred check: the step's state-writing kernels skip themselves
  }
}

// Step predication (deferred non-finite check): the state-writing kernels of a step return at once
// when the step's go word is 0; null = unconditional.
__device__ __forceinline__ bool skip_step(const int32_t* go) { return go != nullptr && *go == 0; }

template <typename T>
__global__ void __launch_bounds__(NT) k_prepare(int pass, const Chunk* __restrict__ chunks,
                                                const DevBlock* __restrict__ blocks,
                                                const void* const* __restrict__ grads,
                                                const void* const* __restrict__ params, StepScalars sc,
                                                ElemArenas ar) {
  __shared__ double red[32];
  if (skip_step(ar.go)) return;
  const Chunk c = chunks[blockIdx.x];
  const DevBlock& B = blocks[c.block];
  T* G = static_cast<T*>(ar.G) + B.vofs;
  T* GE = static_cast<T*>(ar.GE) + B.vofs;
  T* F = static_cast<T*>(ar.FILT) + B.vofs;
  T* GA = static_cast<T*>(ar.GA) + B.vofs;
  const void* gp = grads[B.param];
  const void* wp = params[B.param];
  const bool normalized = graft_normalized(sc.graft);
  double inv_norm = 1.0;
  if (pass == 1 && normalized) {
    const double n2 = ar.gnorm2[B.local];
    inv_norm = n2 > 0.0 ? 1.0 / sqrt(n2) : 1.0;
  }
  double acc = 0.0;
  // U elements per thread per iteration: every load of the batch is issued before the first store
  // (the state arrays may alias the caller's pointers as far as the compiler knows), same element
  // order as a plain strided loop, so the partial sums are unchanged
  constexpr int U = 4;
  for (int64_t e0 = threadIdx.x; e0 < c.count; e0 += U * NT) {
    T gq[U], aq[U], fq[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * NT;
      gq[u] = aq[u] = fq[u] = T(0);
      if (e >= c.count) continue;
      const int64_t j = c.start + e;
      if (pass == 0 || !normalized) {
        if (sc.gbuf) {  // reduced gradient: this block's slice of the gather-layout buffer
          gq[u] = T(sc.gscale * (double)static_cast<const T*>(ar.GBUF)[B.gofs + j]);
          if (sc.l2) gq[u] += T(sc.weight_decay) * load_as<T>(wp, block_to_param_offset(B, j), sc.pdtype);
        } else {
          const int64_t po = block_to_param_offset(B, j);
          gq[u] = load_as<T>(gp, po, sc.pdtype);
          if (sc.l2) gq[u] += T(sc.weight_decay) * load_as<T>(wp, po, sc.pdtype);
        }
      } else {
        gq[u] = G[j];
      }
      if (pass != 0 && sc.graft != SHAMPOO_GRAFT_SGD) aq[u] = GA[j];
      if (pass != 0 && sc.use_filter) fq[u] = F[j];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * NT;
      if (e >= c.count) continue;
      const int64_t j = c.start + e;
      const T g = gq[u];
      if (pass == 0 || !normalized) G[j] = g;
      if (pass == 0) {
        acc += (double)g * (double)g;
        continue;
      }
      T a = T(0);
      if (sc.graft != SHAMPOO_GRAFT_SGD) {
        const T gg = normalized ? T((double)g * inv_norm) : g;
        const T sq = gg * gg;
        a = aq[u];
        a = graft_summed(sc.graft) ? a + sq : T(sc.beta2g) * a + T(sc.one_minus_beta2g) * sq;
        GA[j] = a;
      }
      T ge = g;
      if (sc.use_filter) {
        const T f = T(sc.beta1) * fq[u] + T(sc.one_minus_beta1) * g;
        F[j] = f;
        ge = f * T(sc.inv_bc1);
        GE[j] = ge;
      }
      const T pg = graft_dir<T>(sc.graft, ge, a, sc.inv_bc2g, sc.graft_eps);
      acc += (double)pg * (double)pg;
    }
  }
  acc = block_sum<double, NT>(acc, red);
  if (threadIdx.x == 0) ar.part[blockIdx.x] = acc;
}

template <typename T>
__global__ void __launch_bounds__(NT) k_sumsq(const Chunk* __restrict__ chunks,
                                              const DevBlock* __restrict__ blocks,
                                              const T* __restrict__ X, double* part) {
  __shared__ double red[32];
  const Chunk c = chunks[blockIdx.x];
  const T* x = X + blocks[c.block].vofs + c.start;
  double acc = 0;
  for (int64_t e = threadIdx.x; e < c.count; e += NT) acc += (double)x[e] * (double)x[e];
  acc = block_sum<double, NT>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// one warp per block; fixed summation order over its chunks
__global__ void k_block_reduce(const int32_t* __restrict__ cb, const int32_t* __restrict__ cc, int nblocks,
                               const double* __restrict__ part, double* out) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= nblocks) return;
  const int lane = threadIdx.x & 31;
  double s = 0;
  for (int i = lane; i < cc[b]; i += 32) s += part[cb[b] + i];
  s = warp_sum(s);
  if (lane == 0) out[b] = s;
}

template <typename T, typename BT>
__global__ void __launch_bounds__(NT) k_final(const Chunk* __restrict__ chunks,
                                              const DevBlock* __restrict__ blocks,
                                              const void* const* __restrict__ params, StepScalars sc,
                                              ElemArenas ar) {
  if (skip_step(ar.go)) return;
  const Chunk c = chunks[blockIdx.x];
  const DevBlock& B = blocks[c.block];
  const T* G = static_cast<const T*>(sc.use_filter ? ar.GE : ar.G) + B.vofs;
  const T* GA = static_cast<const T*>(ar.GA) + B.vofs;
  const T* PS = static_cast<const T*>(ar.PS) + B.vofs;
  T* M = static_cast<T*>(ar.MOM) + B.vofs;
  BT* out = static_cast<BT*>(ar.BUF) + B.gofs;
  const void* wp = params[B.param];
  const bool use_ps = sc.precond && ((B.kind == SHAMPOO_BLOCK_SHAMPOO && ar.ready[B.local]) ||
                                     B.kind == SHAMPOO_BLOCK_ADAGRAD || B.kind == SHAMPOO_BLOCK_DIAGONAL);
  double ratio = 0.0;
  bool ps_zero = false;
  if (use_ps) {
    const double n2 = ar.ps2[B.local];
    ps_zero = (n2 == 0.0);
    if (!ps_zero) ratio = sqrt(ar.pg2[B.local]) / sqrt(n2);  // grafting.py:95-110
  }
  constexpr int U = 4;  // loads of U elements before their stores (see k_prepare)
  for (int64_t e0 = threadIdx.x; e0 < c.count; e0 += U * NT) {
    T pq[U], aq[U], wq[U], mq[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * NT;
      pq[u] = aq[u] = wq[u] = mq[u] = T(0);
      if (e >= c.count) continue;
      const int64_t j = c.start + e;
      if (use_ps && !ps_zero) {
        pq[u] = PS[j];
      } else {
        pq[u] = G[j];
        if (sc.graft != SHAMPOO_GRAFT_SGD) aq[u] = GA[j];
      }
      if (sc.decoupled) wq[u] = load_as<T>(wp, block_to_param_offset(B, j), sc.pdtype);
      if (sc.momentum > 0.0) mq[u] = M[j];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * NT;
      if (e >= c.count) continue;
      const int64_t j = c.start + e;
      T p = (use_ps && !ps_zero) ? T(ratio * (double)pq[u]) : graft_dir<T>(sc.graft, pq[u], aq[u], sc.inv_bc2g, sc.graft_eps);
      if (sc.decoupled) p += T(sc.weight_decay) * wq[u];
      if (sc.momentum > 0.0) {
        const T m = T(sc.momentum) * mq[u] + p;
        M[j] = m;
        p = sc.nesterov ? T(sc.momentum) * m + p : m;
      }
      out[j] = BT(p);
    }
  }
}

template <typename BT>
__global__ void __launch_bounds__(NT) k_apply(const Chunk* __restrict__ chunks,
                                              const DevBlock* __restrict__ blocks,
                                              void* const* __restrict__ params,
                                              const BT* __restrict__ buf, double lr, int32_t pdtype,
                                              const int32_t* __restrict__ go) {
  if (skip_step(go)) return;
  const Chunk c = chunks[blockIdx.x];
  const DevBlock& B = blocks[c.block];
  const BT* p = buf + B.gofs;
  void* wp = params[B.param];
  for (int64_t e = threadIdx.x; e < c.count; e += NT) {
    const int64_t j = c.start + e;
    const int64_t po = block_to_param_offset(B, j);
    const double step = __dmul_rn(lr, (double)p[j]);  // W -= lr * P (optim.py:354), no FMA contraction
    if (pdtype == SHAMPOO_DTYPE_F32) {
      float* w = static_cast<float*>(wp);
      w[po] = (float)__dsub_rn((double)w[po], step);
    } else {
      double* w = static_cast<double*>(wp);
      w[po] = __dsub_rn(w[po], step);
    }
  }
}

// multi-index component k of flat element e of a block
__device__ __forceinline__ int64_t mode_index(const DevBlock& b, int64_t e, int k) {
  int64_t inner = 1;
  for (int q = b.order - 1; q > k; --q) inner *= b.dims[q];
  return (e / inner) % b.dims[k];
}

// ADAGRAD: acc = acc + g^2 (or EMA); DIAGONAL: dsum[mode, i] += g^2 (precond.py:305-313, 355-364)
template <typename T>
__global__ void __launch_bounds__(NT) k_fb_update(const Chunk* __restrict__ chunks,
                                                  const DevBlock* __restrict__ blocks, ElemArenas ar,
                                                  FallbackArgs fa) {
  if (skip_step(ar.go)) return;
  const Chunk c = chunks[blockIdx.x];
  const DevBlock& B = blocks[c.block];
  const T* G = static_cast<const T*>(ar.G) + B.vofs;
  for (int64_t e = threadIdx.x; e < c.count; e += NT) {
    const int64_t j = c.start + e;
    const double g = (double)G[j];
    const double sq = g * g;
    if (B.kind == SHAMPOO_BLOCK_ADAGRAD) {
      T* acc = static_cast<T*>(fa.FB) + B.fofs;
      acc[j] = fa.ema ? T(fa.beta2 * (double)acc[j] + fa.one_minus_beta2 * (double)T(sq)) : T((double)acc[j] + (double)T(sq));
    } else {
      int64_t off = B.fofs;
      for (int k = 0; k < B.order; ++k) {
        atomicAdd(fa.dsum + off + mode_index(B, j, k), sq);
        off += B.dims[k];
      }
    }
  }
}

// DIAGONAL: diag = EMA(diag, dsum) ; dsum = 0 (one CTA per diagonal block)
template <typename T>
__global__ void __launch_bounds__(NT) k_fb_diag_ema(const DevBlock* __restrict__ blocks,
                                                    const int32_t* __restrict__ dblocks, FallbackArgs fa,
                                                    const int32_t* __restrict__ go) {
  if (skip_step(go)) return;
  const DevBlock& B = blocks[dblocks[blockIdx.x]];
  int64_t n = 0;
  for (int k = 0; k < B.order; ++k) n += B.dims[k];
  T* diag = static_cast<T*>(fa.FB) + B.fofs;
  for (int64_t e = threadIdx.x; e < n; e += NT) {
    const double sq = (double)T(fa.dsum[B.fofs + e]);  // cast like mode_square_sums(...).astype
    diag[e] = fa.ema ? T(fa.beta2 * (double)diag[e] + fa.one_minus_beta2 * sq) : T((double)diag[e] + sq);
    fa.dsum[B.fofs + e] = 0.0;
  }
}

// DIAGONAL: scale = (diag / corr + eps)^exponent (precond.py:384-395)
template <typename T>
__global__ void __launch_bounds__(NT) k_fb_scale(const DevBlock* __restrict__ blocks,
                                                 const int32_t* __restrict__ dblocks, FallbackArgs fa) {
  const DevBlock& B = blocks[dblocks[blockIdx.x]];
  int64_t n = 0;
  for (int k = 0; k < B.order; ++k) n += B.dims[k];
  const T* diag = static_cast<const T*>(fa.FB) + B.fofs;
  const double exponent = -fa.eta / (fa.root_override ? fa.root_override : 2 * B.order);  // precond.py:349,380
  for (int64_t e = threadIdx.x; e < n; e += NT)
    fa.dscale[B.fofs + e] = pow((double)diag[e] * fa.inv_corr + fa.epsilon, exponent);
}

// PS = fallback direction of g_eff (precond.py:315-320, 366-396)
template <typename T>
__global__ void __launch_bounds__(NT) k_fb_precondition(const Chunk* __restrict__ chunks,
                                                        const DevBlock* __restrict__ blocks, ElemArenas ar,
                                                        FallbackArgs fa, int use_filter) {
  const Chunk c = chunks[blockIdx.x];
  const DevBlock& B = blocks[c.block];
  const T* GE = static_cast<const T*>(use_filter ? ar.GE : ar.G) + B.vofs;
  T* PS = static_cast<T*>(ar.PS) + B.vofs;
  for (int64_t e = threadIdx.x; e < c.count; e += NT) {
    const int64_t j = c.start + e;
    const double g = (double)GE[j];
    double out;
    if (B.kind == SHAMPOO_BLOCK_ADAGRAD) {
      const double acc = (double)static_cast<const T*>(fa.FB)[B.fofs + j] * fa.inv_corr;
      out = g / (sqrt(acc) + fa.div_eps);
    } else {
      out = g;
      int64_t off = B.fofs;
      for (int k = 0; k < B.order; ++k) {
        out *= fa.dscale[off + mode_index(B, j, k)];
        off += B.dims[k];
      }
    }
    PS[j] = T(out);
  }
}

}  // namespace

template <typename T>
int launch_fallback_update(const Chunk* chunks, int nchunks, const DevBlock* blocks, const ElemArenas& ar,
                           const FallbackArgs& fa, const int32_t* dblocks, int ndiag, cudaStream_t s) {
  if (nchunks) {
    k_fb_update<T><<<nchunks, NT, 0, s>>>(chunks, blocks, ar, fa);
    SH_LAUNCH_CHECK();
  }
  if (ndiag) {
    k_fb_diag_ema<T><<<ndiag, NT, 0, s>>>(blocks, dblocks, fa, ar.go);
    SH_LAUNCH_CHECK();
  }
  return SHAMPOO_OK;
}

template <typename T>
int launch_fallback_precondition(const Chunk* chunks, int nchunks, const DevBlock* blocks, const ElemArenas& ar,
                                 const FallbackArgs& fa, const int32_t* dblocks, int ndiag, int use_filter,
                                 cudaStream_t s) {
  if (ndiag) {
    k_fb_scale<T><<<ndiag, NT, 0, s>>>(blocks, dblocks, fa);
    SH_LAUNCH_CHECK();
  }
  if (nchunks) {
    k_fb_precondition<T><<<nchunks, NT, 0, s>>>(chunks, blocks, ar, fa, use_filter);
    SH_LAUNCH_CHECK();
  }
  return SHAMPOO_OK;
}

template <typename T>
int launch_finite(const Chunk* chunks, int nchunks, const DevBlock* params, const void* const* grads,
                  int32_t dtype, int32_t* flag, int32_t* go, cudaStream_t s) {
  if (!nchunks) return SHAMPOO_OK;
  k_finite<<<nchunks, NT, 0, s>>>(chunks, params, grads, dtype, flag, go);
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

template <typename T>
int launch_prepare(int pass, const Chunk* chunks, int nchunks, const DevBlock* blocks,
                   const void* const* grads, const void* const* params, const StepScalars& sc,
                   const ElemArenas& ar, cudaStream_t s) {
  if (!nchunks) return SHAMPOO_OK;
  k_prepare<T><<<nchunks, NT, 0, s>>>(pass, chunks, blocks, grads, params, sc, ar);
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

template <typename T>
int launch_sumsq(const Chunk* chunks, int nchunks, const DevBlock* blocks, const void* X, double* part,
                 cudaStream_t s) {
  if (!nchunks) return SHAMPOO_OK;
  k_sumsq<T><<<nchunks, NT, 0, s>>>(chunks, blocks, static_cast<const T*>(X), part);
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

int launch_block_reduce(const int32_t* cb, const int32_t* cc, int nblocks, const double* part, double* out,
                        cudaStream_t s) {
  if (!nblocks) return SHAMPOO_OK;
  k_block_reduce<<<(nblocks + 7) / 8, 256, 0, s>>>(cb, cc, nblocks, part, out);
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

template <typename T>
int launch_final(const Chunk* chunks, int nchunks, const DevBlock* blocks, const void* const* params,
                 const StepScalars& sc, const ElemArenas& ar, cudaStream_t s) {
  if (!nchunks) return SHAMPOO_OK;
  if (sc.buf_f32) k_final<T, float><<<nchunks, NT, 0, s>>>(chunks, blocks, params, sc, ar);
  else k_final<T, T><<<nchunks, NT, 0, s>>>(chunks, blocks, params, sc, ar);
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

template <typename T>
int launch_apply(const Chunk* chunks, int nchunks, const DevBlock* blocks, void* const* params,
                 const void* buf, const StepScalars& sc, const int32_t* go, cudaStream_t s) {
  if (!nchunks) return SHAMPOO_OK;
  if (sc.buf_f32) k_apply<float><<<nchunks, NT, 0, s>>>(chunks, blocks, params, static_cast<const float*>(buf), sc.lr,
                                                        sc.pdtype, go);
  else k_apply<T><<<nchunks, NT, 0, s>>>(chunks, blocks, params, static_cast<const T*>(buf), sc.lr, sc.pdtype, go);
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

// Gradients (caller layout) -> gather-buffer layout: buf[gofs + j] for every block (all ranks pack
// every block; a reduce-scatter then leaves each owner the summed gradient of its blocks).
template <typename T>
__global__ void __launch_bounds__(NT) k_pack_grads(const Chunk* __restrict__ chunks, const DevBlock* __restrict__ blocks,
                                                   const void* const* __restrict__ grads, int32_t dtype,
                                                   T* __restrict__ buf) {
  const Chunk c = chunks[blockIdx.x];
  const DevBlock& B = blocks[c.block];
  const void* g = grads[B.param];
  for (int64_t e = threadIdx.x; e < c.count; e += NT) {
    const int64_t j = c.start + e;
    buf[B.gofs + j] = load_as<T>(g, block_to_param_offset(B, j), dtype);
  }
}

// Non-finite entries among the owned blocks' reduced gradients (device flag, no host sync).
template <typename T>
__global__ void __launch_bounds__(NT) k_region_finite(const Chunk* __restrict__ chunks,
                                                      const DevBlock* __restrict__ blocks,
                                                      const T* __restrict__ buf, int32_t* flag) {
  const Chunk c = chunks[blockIdx.x];
  const DevBlock& B = blocks[c.block];
  int bad = 0;
  for (int64_t e = threadIdx.x; e < c.count; e += NT)
    if (!isfinite((double)buf[B.gofs + c.start + e])) bad = 1;
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

template <typename T>
int launch_pack_grads(const Chunk* chunks, int nchunks, const DevBlock* blocks, const void* const* grads,
                      int32_t dtype, void* buf, cudaStream_t s) {
  if (!nchunks) return SHAMPOO_OK;
  k_pack_grads<T><<<nchunks, NT, 0, s>>>(chunks, blocks, grads, dtype, static_cast<T*>(buf));
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

template <typename T>
int launch_region_finite(const Chunk* chunks, int nchunks, const DevBlock* blocks, const void* buf, int32_t* flag,
                         cudaStream_t s) {
  if (!nchunks) return SHAMPOO_OK;
  k_region_finite<T><<<nchunks, NT, 0, s>>>(chunks, blocks, static_cast<const T*>(buf), flag);
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

// Small host<->device transfers of the step without the copy engines (a 4-byte cudaMemcpyAsync D2H
// queues behind any bulk D2H the caller has in flight on another stream -- e.g. a parameter
// read-back -- and stalls the step): the device writes host-mapped pinned memory / reads it.
__global__ void k_publish_flag(const int32_t* __restrict__ src, volatile int32_t* dst) {
  *dst = *src;
  __threadfence_system();
}

__global__ void __launch_bounds__(256) k_copy_ptrs(const volatile uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                                   int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

int launch_publish_flag(const int32_t* src, int32_t* mapped_dst, cudaStream_t s) {
  k_publish_flag<<<1, 1, 0, s>>>(src, mapped_dst);
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

int launch_copy_ptrs(const void* mapped_src, void* dst, int n, cudaStream_t s) {
  k_copy_ptrs<<<1, 256, 0, s>>>(static_cast<const volatile uint64_t*>(mapped_src), static_cast<uint64_t*>(dst), n);
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}

#define SH_INST(T)                                                                                   \
  template int launch_finite<T>(const Chunk*, int, const DevBlock*, const void* const*, int32_t,    \
                                int32_t*, int32_t*, cudaStream_t);                                             \
  template int launch_prepare<T>(int, const Chunk*, int, const DevBlock*, const void* const*,       \
                                 const void* const*, const StepScalars&, const ElemArenas&,         \
                                 cudaStream_t);                                                      \
  template int launch_sumsq<T>(const Chunk*, int, const DevBlock*, const void*, double*, cudaStream_t); \
  template int launch_final<T>(const Chunk*, int, const DevBlock*, const void* const*,              \
                               const StepScalars&, const ElemArenas&, cudaStream_t);                 \
  template int launch_apply<T>(const Chunk*, int, const DevBlock*, void* const*, const void*,        \
                               const StepScalars&, const int32_t*, cudaStream_t);                                    \
  template int launch_fallback_update<T>(const Chunk*, int, const DevBlock*, const ElemArenas&,      \
                                         const FallbackArgs&, const int32_t*, int, cudaStream_t);    \
  template int launch_fallback_precondition<T>(const Chunk*, int, const DevBlock*, const ElemArenas&, \
                                               const FallbackArgs&, const int32_t*, int, int, cudaStream_t); \
  template int launch_pack_grads<T>(const Chunk*, int, const DevBlock*, const void* const*, int32_t, void*, \
                                    cudaStream_t);                                                          \
  template int launch_region_finite<T>(const Chunk*, int, const DevBlock*, const void*, int32_t*, cudaStream_t);
SH_INST(double)
SH_INST(float)

}  // namespace shampoo
