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

// Two consecutive elements per access (8- or 16-byte vectors) on the contiguous-block fast paths.
template <typename T> struct Pair;
template <> struct Pair<double> { using V = double2; };
template <> struct Pair<float> { using V = float2; };
template <typename T>
__device__ __forceinline__ void ld2(const T* p, T& a, T& b) {
  const typename Pair<T>::V v = *reinterpret_cast<const typename Pair<T>::V*>(p);
  a = v.x;
  b = v.y;
}
template <typename T>
__device__ __forceinline__ void st2(T* p, T a, T b) {
  typename Pair<T>::V v;
  v.x = a;
  v.y = b;
  *reinterpret_cast<typename Pair<T>::V*>(p) = v;
}
template <typename T>
__device__ __forceinline__ void ld2_as(const void* p, int64_t i, int32_t dtype, T& a, T& b) {
  if (dtype == SHAMPOO_DTYPE_F32) {
    float x, y;
    ld2<float>(static_cast<const float*>(p) + i, x, y);
    a = T(x);
    b = T(y);
  } else {
    double x, y;
    ld2<double>(static_cast<const double*>(p) + i, x, y);
    a = T(x);
    b = T(y);
  }
}
__device__ __forceinline__ bool al(const void* p, int bytes) { return (reinterpret_cast<uintptr_t>(p) & (bytes - 1)) == 0; }
__device__ __forceinline__ int dsize(int32_t dtype) { return dtype == SHAMPOO_DTYPE_F32 ? 4 : 8; }

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
  const T* gb = sc.gbuf ? static_cast<const T*>(ar.GBUF) + B.gofs : nullptr;  // reduced gradients
  const bool normalized = graft_normalized(sc.graft);
  const bool fresh = pass == 0 || !normalized;  // g from the caller (else the pass-0 copy in G)
  const bool graft = pass != 0 && sc.graft != SHAMPOO_GRAFT_SGD;
  const bool filt = pass != 0 && sc.use_filter;
  double inv_norm = 1.0;
  if (pass == 1 && normalized) {
    const double n2 = ar.gnorm2[B.local];
    inv_norm = n2 > 0.0 ? 1.0 / sqrt(n2) : 1.0;
  }
  // Elements in pairs (2q, 2q+1), pair q on thread q % NT: one summation order whichever way the
  // pair is loaded -- 8/16-byte vectors when the block is one contiguous run and every array is
  // pair-aligned, else two scalar accesses -- so reduced-buffer and caller-gradient steps agree bitwise.
  const int64_t j0 = c.start;
  const bool contig = B.cbase >= 0;
  const int64_t p0 = contig ? B.cbase + c.start : 0;
  const int es = dsize(sc.pdtype);
  const bool vec = contig && al(G + j0, 2 * sizeof(T)) &&
                   (!fresh || (sc.gbuf ? al(gb + j0, 2 * sizeof(T)) : al(static_cast<const char*>(gp) + p0 * es, 2 * es))) &&
                   (!fresh || !sc.l2 || al(static_cast<const char*>(wp) + p0 * es, 2 * es)) &&
                   (!graft || al(GA + j0, 2 * sizeof(T))) && (!filt || (al(F + j0, 2 * sizeof(T)) && al(GE + j0, 2 * sizeof(T))));
  auto param_off = [&](int64_t j) { return contig ? B.cbase + j : block_to_param_offset(B, j); };
  // gradient of elements j, j + 1 (n = 2) or j (n = 1), scalar accesses
  auto load_g = [&](int64_t j, int n, T& g0, T& g1) {
    g1 = T(0);
    if (!fresh) {
      g0 = G[j];
      if (n == 2) g1 = G[j + 1];
      return;
    }
    if (sc.gbuf) {
      g0 = T(sc.gscale * (double)gb[j]);
      if (n == 2) g1 = T(sc.gscale * (double)gb[j + 1]);
    } else {
      g0 = load_as<T>(gp, param_off(j), sc.pdtype);
      if (n == 2) g1 = load_as<T>(gp, param_off(j + 1), sc.pdtype);
    }
    if (sc.l2) {
      g0 += T(sc.weight_decay) * load_as<T>(wp, param_off(j), sc.pdtype);
      if (n == 2) g1 += T(sc.weight_decay) * load_as<T>(wp, param_off(j + 1), sc.pdtype);
    }
  };
  double acc = 0.0;
  // the math of one pair (n = 2) or of the odd tail (n = 1), in element order
  auto pair_math = [&](int64_t j, int n, T (&g)[2], T (&a)[2], T (&f)[2], bool vstore) {
    auto stp = [&](T* arr, T x0, T x1) {
      if (vstore) st2<T>(arr + j, x0, x1);
      else {
        arr[j] = x0;
        if (n == 2) arr[j + 1] = x1;
      }
    };
    if (fresh) stp(G, g[0], g[1]);
    if (pass == 0) {
      for (int h = 0; h < n; ++h) acc += (double)g[h] * (double)g[h];
      return;
    }
    T ge[2] = {g[0], g[1]};
    if (graft) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const T gg = normalized ? T((double)g[h] * inv_norm) : g[h];
        const T sq = gg * gg;
        a[h] = graft_summed(sc.graft) ? a[h] + sq : T(sc.beta2g) * a[h] + T(sc.one_minus_beta2g) * sq;
      }
      stp(GA, a[0], a[1]);
    }
    if (filt) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        f[h] = T(sc.beta1) * f[h] + T(sc.one_minus_beta1) * g[h];
        ge[h] = f[h] * T(sc.inv_bc1);
      }
      stp(F, f[0], f[1]);
      stp(GE, ge[0], ge[1]);
    }
    for (int h = 0; h < n; ++h) {
      const T pg = graft_dir<T>(sc.graft, ge[h], a[h], sc.inv_bc2g, sc.graft_eps);
      acc += (double)pg * (double)pg;
    }
  };
  const int64_t npair = (c.count + 1) >> 1;
  constexpr int U2 = 2;  // pairs per thread per iteration: all loads of the batch before its stores
  if (vec) {
    const int64_t nfull = c.count >> 1;
    for (int64_t q0 = threadIdx.x; q0 < nfull; q0 += U2 * NT) {
      T g[U2][2], a[U2][2], f[U2][2];
#pragma unroll
      for (int u = 0; u < U2; ++u) {
        const int64_t q = q0 + (int64_t)u * NT;
        g[u][0] = g[u][1] = a[u][0] = a[u][1] = f[u][0] = f[u][1] = T(0);
        if (q >= nfull) continue;
        const int64_t j = j0 + 2 * q;
        if (!fresh) {
          ld2<T>(G + j, g[u][0], g[u][1]);
        } else {
          if (sc.gbuf) {
            ld2<T>(gb + j, g[u][0], g[u][1]);
            g[u][0] = T(sc.gscale * (double)g[u][0]);
            g[u][1] = T(sc.gscale * (double)g[u][1]);
          } else {
            ld2_as<T>(gp, p0 + 2 * q, sc.pdtype, g[u][0], g[u][1]);
          }
          if (sc.l2) {
            T w0, w1;
            ld2_as<T>(wp, p0 + 2 * q, sc.pdtype, w0, w1);
            g[u][0] += T(sc.weight_decay) * w0;
            g[u][1] += T(sc.weight_decay) * w1;
          }
        }
        if (graft) ld2<T>(GA + j, a[u][0], a[u][1]);
        if (filt) ld2<T>(F + j, f[u][0], f[u][1]);
      }
#pragma unroll
      for (int u = 0; u < U2; ++u) {  // pair_math inlined by hand (16-byte stores)
        const int64_t q = q0 + (int64_t)u * NT;
        if (q >= nfull) continue;
        const int64_t j = j0 + 2 * q;
        if (fresh) st2<T>(G + j, g[u][0], g[u][1]);
        if (pass == 0) {
          acc += (double)g[u][0] * (double)g[u][0];
          acc += (double)g[u][1] * (double)g[u][1];
          continue;
        }
        T ge0 = g[u][0], ge1 = g[u][1];
        if (graft) {
          const T g0 = normalized ? T((double)g[u][0] * inv_norm) : g[u][0];
          const T g1 = normalized ? T((double)g[u][1] * inv_norm) : g[u][1];
          const T s0 = g0 * g0, s1 = g1 * g1;
          if (graft_summed(sc.graft)) {
            a[u][0] += s0;
            a[u][1] += s1;
          } else {
            a[u][0] = T(sc.beta2g) * a[u][0] + T(sc.one_minus_beta2g) * s0;
            a[u][1] = T(sc.beta2g) * a[u][1] + T(sc.one_minus_beta2g) * s1;
          }
          st2<T>(GA + j, a[u][0], a[u][1]);
        }
        if (filt) {
          f[u][0] = T(sc.beta1) * f[u][0] + T(sc.one_minus_beta1) * g[u][0];
          f[u][1] = T(sc.beta1) * f[u][1] + T(sc.one_minus_beta1) * g[u][1];
          ge0 = f[u][0] * T(sc.inv_bc1);
          ge1 = f[u][1] * T(sc.inv_bc1);
          st2<T>(F + j, f[u][0], f[u][1]);
          st2<T>(GE + j, ge0, ge1);
        }
        const T pg0 = graft_dir<T>(sc.graft, ge0, a[u][0], sc.inv_bc2g, sc.graft_eps);
        const T pg1 = graft_dir<T>(sc.graft, ge1, a[u][1], sc.inv_bc2g, sc.graft_eps);
        acc += (double)pg0 * (double)pg0;
        acc += (double)pg1 * (double)pg1;
      }
    }
    // the odd tail is pair npair - 1: its thread's last pair, as in the scalar order below
    if ((c.count & 1) && threadIdx.x == (int)((npair - 1) % NT)) {
      const int64_t j = j0 + c.count - 1;
      T g[2], a[2] = {T(0), T(0)}, f[2] = {T(0), T(0)};
      load_g(j, 1, g[0], g[1]);
      if (graft) a[0] = GA[j];
      if (filt) f[0] = F[j];
      pair_math(j, 1, g, a, f, false);
    }
  } else {
    for (int64_t q0 = threadIdx.x; q0 < npair; q0 += U2 * NT) {
      T g[U2][2], a[U2][2], f[U2][2];
#pragma unroll
      for (int u = 0; u < U2; ++u) {
        const int64_t q = q0 + (int64_t)u * NT;
        g[u][0] = g[u][1] = a[u][0] = a[u][1] = f[u][0] = f[u][1] = T(0);
        if (q >= npair) continue;
        const int64_t j = j0 + 2 * q;
        const int n = (2 * q + 1 < c.count) ? 2 : 1;
        load_g(j, n, g[u][0], g[u][1]);
        if (graft) {
          a[u][0] = GA[j];
          if (n == 2) a[u][1] = GA[j + 1];
        }
        if (filt) {
          f[u][0] = F[j];
          if (n == 2) f[u][1] = F[j + 1];
        }
      }
#pragma unroll
      for (int u = 0; u < U2; ++u) {
        const int64_t q = q0 + (int64_t)u * NT;
        if (q < npair) pair_math(j0 + 2 * q, (2 * q + 1 < c.count) ? 2 : 1, g[u], a[u], f[u], false);
      }
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
  const bool from_ps = use_ps && !ps_zero;
  if (B.cbase >= 0) {  // contiguous block: two elements per access when every array is pair-aligned
    const int64_t j0 = c.start, p0 = B.cbase + c.start;
    const int pb = 2 * dsize(sc.pdtype);
    const bool graft = !from_ps && sc.graft != SHAMPOO_GRAFT_SGD;
    if (al(out + j0, 2 * sizeof(BT)) && (from_ps ? al(PS + j0, 2 * sizeof(T)) : al(G + j0, 2 * sizeof(T))) &&
        (!graft || al(GA + j0, 2 * sizeof(T))) && (sc.momentum <= 0.0 || al(M + j0, 2 * sizeof(T))) &&
        (!sc.decoupled || al(static_cast<const char*>(wp) + p0 * dsize(sc.pdtype), pb))) {
      const int64_t np2 = c.count >> 1;
      constexpr int U2 = 2;
      for (int64_t q0 = threadIdx.x; q0 < np2; q0 += U2 * NT) {
        T pv[U2][2], av[U2][2], wv[U2][2], mv[U2][2];
#pragma unroll
        for (int u = 0; u < U2; ++u) {
          const int64_t q = q0 + (int64_t)u * NT;
          pv[u][0] = pv[u][1] = av[u][0] = av[u][1] = wv[u][0] = wv[u][1] = mv[u][0] = mv[u][1] = T(0);
          if (q >= np2) continue;
          const int64_t j = j0 + 2 * q;
          if (from_ps) {
            ld2<T>(PS + j, pv[u][0], pv[u][1]);
          } else {
            ld2<T>(G + j, pv[u][0], pv[u][1]);
            if (graft) ld2<T>(GA + j, av[u][0], av[u][1]);
          }
          if (sc.decoupled) ld2_as<T>(wp, p0 + 2 * q, sc.pdtype, wv[u][0], wv[u][1]);
          if (sc.momentum > 0.0) ld2<T>(M + j, mv[u][0], mv[u][1]);
        }
#pragma unroll
        for (int u = 0; u < U2; ++u) {
          const int64_t q = q0 + (int64_t)u * NT;
          if (q >= np2) continue;
          const int64_t j = j0 + 2 * q;
          T r[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            T p = from_ps ? T(ratio * (double)pv[u][h]) : graft_dir<T>(sc.graft, pv[u][h], av[u][h], sc.inv_bc2g, sc.graft_eps);
            if (sc.decoupled) p += T(sc.weight_decay) * wv[u][h];
            if (sc.momentum > 0.0) {
              const T m = T(sc.momentum) * mv[u][h] + p;
              mv[u][h] = m;
              p = sc.nesterov ? T(sc.momentum) * m + p : m;
            }
            r[h] = p;
          }
          if (sc.momentum > 0.0) st2<T>(M + j, mv[u][0], mv[u][1]);
          st2<BT>(out + j, BT(r[0]), BT(r[1]));
        }
      }
      if (!(c.count & 1) || threadIdx.x != 0) return;
      // odd tail: the last element through the scalar loop below (thread 0 only)
      const int64_t j = j0 + c.count - 1;
      T p = from_ps ? T(ratio * (double)PS[j]) : graft_dir<T>(sc.graft, G[j], graft ? GA[j] : T(0), sc.inv_bc2g, sc.graft_eps);
      if (sc.decoupled) p += T(sc.weight_decay) * load_as<T>(wp, p0 + c.count - 1, sc.pdtype);
      if (sc.momentum > 0.0) {
        const T m = T(sc.momentum) * M[j] + p;
        M[j] = m;
        p = sc.nesterov ? T(sc.momentum) * m + p : m;
      }
      out[j] = BT(p);
      return;
    }
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
  if (B.cbase >= 0) {  // contiguous block: two elements per access when pair-aligned
    const int64_t j0 = c.start, p0 = B.cbase + c.start;
    const int es = dsize(pdtype);
    if (al(p + j0, 2 * sizeof(BT)) && al(static_cast<char*>(wp) + p0 * es, 2 * es)) {
      const int64_t np2 = c.count >> 1;
#pragma unroll 4
      for (int64_t q = threadIdx.x; q < np2; q += NT) {
        BT d0, d1;
        ld2<BT>(p + j0 + 2 * q, d0, d1);
        const double s0 = __dmul_rn(lr, (double)d0), s1 = __dmul_rn(lr, (double)d1);
        if (pdtype == SHAMPOO_DTYPE_F32) {
          float* w = static_cast<float*>(wp) + p0 + 2 * q;
          float w0, w1;
          ld2<float>(w, w0, w1);
          st2<float>(w, (float)__dsub_rn((double)w0, s0), (float)__dsub_rn((double)w1, s1));
        } else {
          double* w = static_cast<double*>(wp) + p0 + 2 * q;
          double w0, w1;
          ld2<double>(w, w0, w1);
          st2<double>(w, __dsub_rn(w0, s0), __dsub_rn(w1, s1));
        }
      }
      if ((c.count & 1) && threadIdx.x == 0) {
        const int64_t j = j0 + c.count - 1, po = p0 + c.count - 1;
        const double step = __dmul_rn(lr, (double)p[j]);
        if (pdtype == SHAMPOO_DTYPE_F32) {
          float* w = static_cast<float*>(wp);
          w[po] = (float)__dsub_rn((double)w[po], step);
        } else {
          double* w = static_cast<double*>(wp);
          w[po] = __dsub_rn(w[po], step);
        }
      }
      return;
    }
  }
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

// Lower -> upper triangle of every factor (the statistics write lower triangles only; run before
// anything reads full factors).  CTA per 32 x 32 tile (ti >= tj) of one factor; off-diagonal tiles
// are transposed through shared memory, diagonal tiles mirrored in place.
template <typename T>
__global__ void __launch_bounds__(256) k_symmetrize(const SymJob* __restrict__ jobs, const int64_t* __restrict__ tbegin,
                                                    int njobs, T* __restrict__ F) {
  __shared__ T tile[32][33];
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tbegin[mid] <= (int64_t)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const SymJob J = jobs[lo];
  const int64_t l = blockIdx.x - tbegin[lo];
  int ti = (int)((sqrt(8.0 * (double)l + 1.0) - 1.0) * 0.5);
  while ((int64_t)(ti + 1) * (ti + 2) / 2 <= l) ++ti;
  while ((int64_t)ti * (ti + 1) / 2 > l) --ti;
  const int tj = (int)(l - (int64_t)ti * (ti + 1) / 2);
  const int n = J.d;
  T* C = F + J.off;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int i = ti * 32 + r, j = tj * 32 + tx;
    tile[r][tx] = (i < n && j < n && i >= j) ? C[(int64_t)i * n + j] : T(0);
  }
  __syncthreads();
#pragma unroll
  for (int r = ty; r < 32; r += 8) {  // element (tj*32 + r, ti*32 + tx) = (ti*32 + tx, tj*32 + r)
    const int i2 = tj * 32 + r, j2 = ti * 32 + tx;
    if (i2 < n && j2 < n && j2 > i2) C[(int64_t)i2 * n + j2] = tile[tx][r];
  }
}

template <typename T>
int launch_symmetrize(const SymJob* jobs, const int64_t* tbegin, int njobs, int64_t ntiles, void* F, cudaStream_t s) {
  if (!njobs || !ntiles) return SHAMPOO_OK;
  k_symmetrize<T><<<(unsigned)ntiles, 256, 0, s>>>(jobs, tbegin, njobs, static_cast<T*>(F));
  SH_LAUNCH_CHECK();
  return SHAMPOO_OK;
}
template int launch_symmetrize<double>(const SymJob*, const int64_t*, int, int64_t, void*, cudaStream_t);
template int launch_symmetrize<float>(const SymJob*, const int64_t*, int, int64_t, void*, cudaStream_t);

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
