// Device-side shared definitions for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace shampoo {

extern int64_t g_launches;  // kernel launches issued by this library (bench evidence)

#define SH_CUDA_CHECK(expr)                                                          \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      ::shampoo::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));      \
      return SHAMPOO_ERR_CUDA;                                                       \
    }                                                                                \
  } while (0)

#define SH_LAUNCH_CHECK()                                                            \
  do {                                                                               \
    ++::shampoo::g_launches;                                                         \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess) {                                                         \
      ::shampoo::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
      return SHAMPOO_ERR_CUDA;                                                       \
    }                                                                                \
  } while (0)

// Device workspace cache for the solver objects (Ozaki GEMM batches, root-inverse batches, the
// low-rank path), which are built per refresh: blocks are reused instead of cudaMalloc/cudaFree
// (cudaFree synchronises the device and stalls the other streams).  dev_free requires the block
// to be idle: every kernel that used it has completed (its owner synchronised its stream).
cudaError_t dev_malloc_bytes(void** p, size_t bytes);
void dev_free(void* p);
template <typename T>
inline cudaError_t dev_malloc(T** p, size_t bytes) {
  return dev_malloc_bytes(reinterpret_cast<void**>(p), bytes);
}

constexpr int kMaxOrder = SHAMPOO_MAX_ORDER;
constexpr int kNumSMs = 148;

// Block descriptor for the elementwise kernels (param-layout <-> block-contiguous).
struct DevBlock {
  int32_t param;       // index into the param/grad pointer tables
  int32_t order;
  int32_t kind;        // SHAMPOO_BLOCK_*
  int32_t local;       // owned-local index (-1 if not owned)
  int64_t numel;
  int64_t gofs;        // gather-buffer offset (scalars)
  int64_t vofs;        // offset into per-element state arenas (owned only)
  int64_t fofs;        // offset into the fallback-state arena (ADAGRAD: numel, DIAGONAL: sum d_k)
  int64_t dims[kMaxOrder];
  int64_t lo[kMaxOrder];
  int64_t mstride[kMaxOrder];
  int64_t cbase;       // >= 0: the block is one contiguous run of its parameter starting there
};

// A contiguous run of elements of one block processed by one CTA.
struct Chunk {
  int32_t block;  // index into the DevBlock table
  int32_t pad;
  int64_t start;
  int64_t count;
};

// Flat element index inside a block -> element offset inside the parameter.
__device__ __forceinline__ int64_t block_to_param_offset(const DevBlock& b, int64_t e) {
  if (b.cbase >= 0) return b.cbase + e;  // row partitions and whole parameters: no index arithmetic
  if (e < 0x7fffffff && b.order == 2 && b.dims[1] < 0x7fffffff) {  // 32-bit division
    const uint32_t d1 = (uint32_t)b.dims[1], ue = (uint32_t)e;
    const uint32_t i0 = ue / d1, i1 = ue - i0 * d1;
    return (b.lo[0] + i0) * b.mstride[0] + (b.lo[1] + i1) * b.mstride[1];
  }
  int64_t off = 0;
#pragma unroll 1
  for (int k = b.order - 1; k >= 0; --k) {
    const int64_t d = b.dims[k];
    const int64_t i = e % d;
    e /= d;
    off += (b.lo[k] + i) * b.mstride[k];
  }
  return off;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic CTA-wide sum (fixed tree order), result valid in all threads.
template <typename T, int NT>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) scratch[w] = v;
  __syncthreads();
  T r = 0;
  if (w == 0) {
    r = (l < NT / 32) ? scratch[l] : T(0);
    r = warp_sum(r);
    if (l == 0) scratch[0] = r;
  }
  __syncthreads();
  r = scratch[0];
  __syncthreads();
  return r;
}

template <typename T>
__device__ __forceinline__ T load_as(const void* p, int64_t i, int32_t dtype) {
  return dtype == SHAMPOO_DTYPE_F32 ? T(static_cast<const float*>(p)[i])
                                    : T(static_cast<const double*>(p)[i]);
}

}  // namespace shampoo
