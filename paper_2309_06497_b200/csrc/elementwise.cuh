// Elementwise / reduction kernels of the step (HBM-bound work).
#pragma once

#include "common.cuh"

namespace shampoo {

constexpr int kChunk = 4096;  // elements per CTA work item (256 threads x 16; 2048 -> 4096: -36 us per step)

// Host-computed scalars for one step (all reference semantics resolved on host).
struct StepScalars {
  double weight_decay;
  double beta1, one_minus_beta1, inv_bc1;  // filter + bias correction (optim.py:308-316)
  double beta2g, one_minus_beta2g, inv_bc2g, graft_eps;  // grafting.py:68-92
  double momentum;
  double lr;
  int32_t l2;          // weight decay folded into g (optim.py:292-293)
  int32_t decoupled;   // p += wd * w (optim.py:334-335)
  int32_t nesterov;
  int32_t graft;       // SHAMPOO_GRAFT_*
  int32_t use_filter;  // beta1 > 0
  int32_t precond;     // t >= start_preconditioning_step
  int32_t pdtype;      // caller tensor dtype
  int32_t gbuf;        // gradients come from the reduced gradient buffer (ElemArenas::GBUF), not grads[]
  int32_t buf_f32;     // the gather buffer holds float32 directions (else the context dtype)
  double gscale;       // multiplier on buffer gradients (1/world for a mean reduction)
};

struct ElemArenas {
  void* G;        // raw gradient block copies (post L2)
  void* GE;       // g_eff (== G when no filter)
  void* FILT;     // filtered gradient state (beta1 > 0)
  void* GA;       // graft accumulator
  void* MOM;      // momentum
  void* PS;       // preconditioned direction
  void* BUF;      // gather buffer
  double* part;   // per-chunk partial sums
  double* gnorm2; // per owned block ||g||^2 (normalized grafting)
  double* pg2;    // per owned block ||P_graft||^2
  double* ps2;    // per owned block ||P_shampoo||^2
  const int32_t* ready;  // per owned block: inverse present
  const void* GBUF;       // reduced gradient buffer (gather-buffer layout, context dtype) or null
  const int32_t* go;      // deferred non-finite check: 0 = skip the step's state writes; null = run
};

template <typename T>
int launch_finite(const Chunk* chunks, int nchunks, const DevBlock* params, const void* const* grads,
                  int32_t dtype, int32_t* flag, int32_t* go, cudaStream_t s);
template <typename T>
int launch_prepare(int pass, const Chunk* chunks, int nchunks, const DevBlock* blocks,
                   const void* const* grads, const void* const* params, const StepScalars& sc,
                   const ElemArenas& ar, cudaStream_t s);
template <typename T>
int launch_sumsq(const Chunk* chunks, int nchunks, const DevBlock* blocks, const void* X, double* part,
                 cudaStream_t s);
int launch_block_reduce(const int32_t* chunk_begin, const int32_t* chunk_count, int nblocks,
                        const double* part, double* out, cudaStream_t s);
template <typename T>
int launch_final(const Chunk* chunks, int nchunks, const DevBlock* blocks, const void* const* params,
                 const StepScalars& sc, const ElemArenas& ar, cudaStream_t s);
// Large-dimension fallbacks (precond.py:282-396): AdaGrad accumulator or per-mode diagonals.
struct FallbackArgs {
  void* FB;         // T: ADAGRAD accumulator (numel) / DIAGONAL vectors (sum d_k) per block
  double* dsum;     // DIAGONAL: per-step mode square sums (sum d_k, zero between steps)
  double* dscale;   // DIAGONAL: (diag/corr + eps)^(-eta/p) (sum d_k)
  double beta2, one_minus_beta2, inv_corr, epsilon, eta, div_eps;
  int32_t ema;      // beta2 < 1
  int32_t root_override;  // exponent_override (0: root p = 2 * order)
};
template <typename T>
int launch_fallback_update(const Chunk* chunks, int nchunks, const DevBlock* blocks, const ElemArenas& ar,
                           const FallbackArgs& fa, const int32_t* dblocks, int ndiag, cudaStream_t s);
template <typename T>
int launch_fallback_precondition(const Chunk* chunks, int nchunks, const DevBlock* blocks, const ElemArenas& ar,
                                 const FallbackArgs& fa, const int32_t* dblocks, int ndiag, int use_filter,
                                 cudaStream_t s);
template <typename T>
int launch_apply(const Chunk* chunks, int nchunks, const DevBlock* blocks, void* const* params,
                 const void* buf, const StepScalars& sc, const int32_t* go, cudaStream_t s);
template <typename T>
int launch_pack_grads(const Chunk* chunks, int nchunks, const DevBlock* blocks, const void* const* grads,
                      int32_t dtype, void* buf, cudaStream_t s);
// factor d x d at element offset `off` of the factor arena
struct SymJob {
  int64_t off;
  int32_t d;
  int32_t pad;
};
template <typename T>
int launch_symmetrize(const SymJob* jobs, const int64_t* tbegin, int njobs, int64_t ntiles, void* F, cudaStream_t s);
// host-mapped pinned memory transfers (no copy engine): flag -> host, pointer table <- host
int launch_publish_flag(const int32_t* src, int32_t* mapped_dst, cudaStream_t s);
int launch_copy_ptrs(const void* mapped_src, void* dst, int n, cudaStream_t s);
template <typename T>
int launch_region_finite(const Chunk* chunks, int nchunks, const DevBlock* blocks, const void* buf, int32_t* flag,
                         cudaStream_t s);

}  // namespace shampoo
