/*
 * shampoo_b200.h -- C ABI of the B200-native Distributed Shampoo optimizer step.
 *
 * The reference (minishampoo, pure numpy) has no FFI; its boundary is the Python
 * class interface.  Every entry point below replaces one reference interface,
 * cited as file:line relative to /root/reference/pkg/src/minishampoo:
 *
 *   shampoo_merge_dims          precond.py:56-77     merge_dims
 *   shampoo_plan_create         precond.py:99-158    block_partition / plan_parameter
 *                               dist.py:232-243      enumerate_blocks
 *                               dist.py:133-183      greedy_assign / buffer_size
 *   shampoo_plan_block          dist.py:68-86        BlockRegion / GlobalBlock
 *   shampoo_ctx_create          optim.py:189-265     Shampoo.__init__ / _build_block (owned only)
 *   shampoo_check_finite        optim.py:362-366     non-finite gradient guard (dist.py:344-348)
 *   shampoo_stats_update        optim.py:291-299     L2 WD + ShampooBlockState.update + GraftState.update
 *                               precond.py:232-242, grafting.py:68-83
 *   shampoo_root_inverse        precond.py:244-267   maybe_refresh -> matfun.py:240-293 guarded_root_inverse
 *   shampoo_precondition_graft  optim.py:301-344     filter, graft direction, precondition, rescale,
 *                                                    decoupled WD, momentum -> gather-buffer region
 *                               dist.py:275-280      WorkerSim.fill_region
 *   shampoo_apply               optim.py:346-354     apply_directions (all blocks, from the gather buffer)
 *                               dist.py:282-290      WorkerSim.apply_gathered
 *   shampoo_state_*             optim.py:387-460     state_tree / load_state_tree (device views)
 *   shampoo_batched_root_inverse matfun.py:139-222   root_inverse_eigh / root_inverse_newton (batched)
 *
 * Conventions: all pointers to tensors are DEVICE pointers unless named host_*;
 * `stream` is a cudaStream_t passed as void*; every compute call is
 * stream-ordered and asynchronous unless documented otherwise.  One context
 * per rank; a context is not thread-safe.  Return value: SHAMPOO_OK (0) or a
 * negative error code; shampoo_last_error() gives a message.
 */
#ifndef SHAMPOO_B200_H_
#define SHAMPOO_B200_H_

#include <stdint.h>

#if defined(__GNUC__)
#define SHAMPOO_API __attribute__((visibility("default")))
#else
#define SHAMPOO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (reference exception -> code) */
#define SHAMPOO_OK 0
#define SHAMPOO_ERR_INVALID_ARGUMENT (-1)   /* ValueError (config / shapes)            */
#define SHAMPOO_ERR_INVALID_GROUP    (-2)   /* dist.InvalidGroupSizeError              */
#define SHAMPOO_ERR_NONFINITE_GRAD   (-3)   /* optim.NonFiniteGradientError (no state touched) */
#define SHAMPOO_ERR_CUDA             (-4)   /* CUDA runtime failure                    */
#define SHAMPOO_ERR_OUT_OF_MEMORY    (-5)
#define SHAMPOO_ERR_SHAPE            (-6)   /* gradient shape/count mismatch           */
#define SHAMPOO_ERR_UNSUPPORTED      (-7)   /* feature not built for this configuration */

/* ---- enums (values mirror the reference enums' order) */
#define SHAMPOO_METHOD_BLOCKING 0  /* precond.LargeDimMethod */
#define SHAMPOO_METHOD_ADAGRAD  1
#define SHAMPOO_METHOD_DIAGONAL 2

#define SHAMPOO_GRAFT_SGD 0        /* grafting.GraftKind */
#define SHAMPOO_GRAFT_ADAGRAD 1
#define SHAMPOO_GRAFT_RMSPROP 2
#define SHAMPOO_GRAFT_ADAM 3
#define SHAMPOO_GRAFT_NORMALIZED_ADAGRAD 4
#define SHAMPOO_GRAFT_NORMALIZED_RMSPROP 5
#define SHAMPOO_GRAFT_NORMALIZED_ADAM 6

#define SHAMPOO_SOLVER_EIGH 0      /* matfun.Solver */
#define SHAMPOO_SOLVER_NEWTON 1

#define SHAMPOO_PRECISION_DOUBLE 0 /* ShampooConfig.precision */
#define SHAMPOO_PRECISION_SINGLE 1

#define SHAMPOO_DTYPE_F32 0        /* element type of caller tensors */
#define SHAMPOO_DTYPE_F64 1
#define SHAMPOO_GATHER_STATE 0     /* shampoo_config.gather_dtype */
#define SHAMPOO_GATHER_F32 1

#define SHAMPOO_BLOCK_SHAMPOO 0    /* BlockSlot.kind */
#define SHAMPOO_BLOCK_GRAFT_ONLY 1
#define SHAMPOO_BLOCK_ADAGRAD 2
#define SHAMPOO_BLOCK_DIAGONAL 3

#define SHAMPOO_MAX_ORDER 8

typedef struct shampoo_plan shampoo_plan;
typedef struct shampoo_ctx shampoo_ctx;

/* One global block (dist.GlobalBlock + dist.BlockRegion, offsets in SCALARS). */
typedef struct {
  int32_t block_id;
  int32_t param_index;
  int32_t block_index;
  int32_t order;
  int32_t owner_rank;      /* group rank */
  int32_t kind;            /* SHAMPOO_BLOCK_* */
  int64_t var_count;
  int64_t gather_offset;   /* absolute scalar offset in the group gather buffer */
  int64_t lo[SHAMPOO_MAX_ORDER];
  int64_t hi[SHAMPOO_MAX_ORDER];
} shampoo_block_info;

/* Flat mirror of ShampooConfig (optim.py:53-84). */
typedef struct {
  double lr;
  double beta1, beta2;
  double epsilon;
  double momentum;
  int32_t use_nesterov;
  double weight_decay;
  int32_t use_decoupled_weight_decay;
  int32_t use_bias_correction;
  int64_t max_preconditioner_dim;
  int64_t precondition_frequency;
  double start_preconditioning_step;   /* may be +inf */
  int32_t exponent_override;
  double exponent_multiplier;
  int32_t grafting;                    /* SHAMPOO_GRAFT_* */
  double grafting_epsilon;
  double grafting_beta2;
  int32_t large_dim_method;            /* SHAMPOO_METHOD_* */
  int32_t solver;                      /* SHAMPOO_SOLVER_* */
  double newton_tolerance;
  int32_t precision;                   /* SHAMPOO_PRECISION_* */
  /* search-direction gather buffer: SHAMPOO_GATHER_STATE (0) = the precision's dtype,
   * SHAMPOO_GATHER_F32 (1) = float32 (for float32 parameters: the update W -= lr * p lands in
   * float32 anyway, and the all-gather moves half the bytes).  Not a reference field: the
   * reference's f64 wire scalar (dist.py:48-50) is a simulation detail. */
  int32_t gather_dtype;
} shampoo_config;

/* Counters of matfun.GuardStats (matfun.py:98-105). */
typedef struct {
  int64_t primary;
  int64_t double_retry;
  int64_t fallback_previous;
  int64_t fallback_identity;
} shampoo_guard_stats;

SHAMPOO_API const char* shampoo_last_error(void);
SHAMPOO_API const char* shampoo_version(void);

/* ---- planning (host only; bit-exact with the reference) */
SHAMPOO_API int shampoo_merge_dims(const int64_t* shape, int32_t ndim, int64_t max_dim,
                       int64_t* out_shape, int32_t* out_ndim);
SHAMPOO_API int shampoo_plan_create(const int64_t* shapes_flat, const int32_t* ndims, int32_t nparams,
                        int64_t max_dim, int32_t large_dim_method, int32_t world_size,
                        int32_t group_size, shampoo_plan** out);
SHAMPOO_API void shampoo_plan_destroy(shampoo_plan* plan);
SHAMPOO_API int32_t shampoo_plan_num_blocks(const shampoo_plan* plan);
SHAMPOO_API int32_t shampoo_plan_num_params(const shampoo_plan* plan);
SHAMPOO_API int shampoo_plan_block(const shampoo_plan* plan, int32_t block_id, shampoo_block_info* out);
/* merged shape + effective method of one parameter */
SHAMPOO_API int shampoo_plan_param(const shampoo_plan* plan, int32_t param, int64_t* merged_shape,
                       int32_t* merged_ndim, int32_t* method);
/* per group rank var-count totals (greedy counters); out has group_size entries */
SHAMPOO_API int shampoo_plan_counters(const shampoo_plan* plan, int64_t* out);
SHAMPOO_API int64_t shampoo_plan_max_payload(const shampoo_plan* plan);   /* scalars */
SHAMPOO_API int32_t shampoo_plan_group_size(const shampoo_plan* plan);
SHAMPOO_API int32_t shampoo_plan_world_size(const shampoo_plan* plan);

/* ---- optimizer context: device state for the blocks owned by `rank` */
SHAMPOO_API int shampoo_ctx_create(const shampoo_plan* plan, const shampoo_config* cfg, int32_t rank,
                       int32_t device, shampoo_ctx** out);
SHAMPOO_API void shampoo_ctx_destroy(shampoo_ctx* ctx);
SHAMPOO_API int64_t shampoo_ctx_device_bytes(const shampoo_ctx* ctx);

/* Non-finite check over ALL gradients (every rank checks everything so ranks
 * agree).  Synchronises `stream`; returns SHAMPOO_ERR_NONFINITE_GRAD if any
 * entry is NaN/Inf.  grads: host array of nparams device pointers. */
SHAMPOO_API int shampoo_check_finite(shampoo_ctx* ctx, const void* const* grads, int32_t dtype, void* stream);

/* The same guard without the host synchronisation (optim.py:362-366 semantics, raised one call
 * late): the check writes a device go word that predicates every state-writing kernel of step t
 * (graft accumulators, filter, factor statistics, momentum, gather-buffer directions, parameter
 * update), so a non-finite step leaves the device state untouched.  A refresh step (t >= start,
 * t % frequency == 0) is checked eagerly instead (*deferred = 0, identical to
 * shampoo_check_finite).  With *deferred = 1 the caller must call shampoo_check_finite_resolve
 * before the next check; it returns SHAMPOO_ERR_NONFINITE_GRAD (and *aborted = 1) if step t was
 * skipped, having restored the context's host-side step counters. */
SHAMPOO_API int shampoo_check_finite_deferred(shampoo_ctx* ctx, const void* const* grads, int32_t dtype,
                                              int64_t t, int32_t* deferred, void* stream);
SHAMPOO_API int shampoo_check_finite_resolve(shampoo_ctx* ctx, int32_t* aborted);

/* Step t phase 1: gather owned gradient blocks (+ L2 weight decay), graft
 * accumulator update, Kronecker factor statistics (EMA or sum). */
SHAMPOO_API int shampoo_stats_update(shampoo_ctx* ctx, const void* const* grads, const void* const* params,
                         int32_t dtype, int64_t t, void* stream);
/* Step t phase 2: if t >= start and t % frequency == 0, guarded root inverse of
 * every owned factor (eigh or coupled Newton).  Synchronises `stream` (one
 * small readback per solver sweep). Returns 1 in *refreshed if it ran. */
/* Step phase 3 on several ranks (dist.py:350-359 WorkerSim exchange): in-place NCCL all-gather of the
 * direction gather buffer within this rank's replica group, on `stream`.  nccl_comm: the group's
 * ncclComm_t (ranks ordered by group rank, as the plan's owner ranks).  NCCL is resolved at run time
 * (the libnccl.so.2 already loaded in the process, else the system one); the buffer holds float32
 * when the parameters are float32 (gather_dtype) or the state is single precision, else float64. */
SHAMPOO_API int shampoo_allgather(shampoo_ctx* ctx, void* nccl_comm, void* stream);

/* ---- gradient reduction to block owners (replaces the DDP all-reduce the reference
 * does not model, dist.py:332-356): every rank packs its LOCAL gradients into the gather-buffer layout
 * (gbuf: group_size * max_payload scalars of the context dtype, block b at its gather offset), the
 * caller reduce-scatters gbuf within the group (+ all-reduces the owned region across replica
 * groups), checks non-finite entries of the owned blocks (device flag, to be max-reduced across
 * ranks) and runs the stats phase from the reduced buffer, scaled by gscale (1/world for a mean). */
SHAMPOO_API int shampoo_pack_gradients(shampoo_ctx* ctx, const void* const* grads, int32_t dtype, void* gbuf,
                                       void* stream);
SHAMPOO_API int shampoo_reduced_nonfinite(shampoo_ctx* ctx, const void* gbuf, int32_t* device_flag, void* stream);
SHAMPOO_API int shampoo_stats_update_reduced(shampoo_ctx* ctx, const void* gbuf, double gscale,
                                             const void* const* params, int32_t dtype, int64_t t, void* stream);
SHAMPOO_API int shampoo_root_inverse(shampoo_ctx* ctx, int64_t t, int32_t* refreshed, void* stream);
/* Step t phase 3: directions of owned blocks -> this rank's gather-buffer region. */
SHAMPOO_API int shampoo_precondition_graft(shampoo_ctx* ctx, const void* const* params, int32_t dtype,
                               int64_t t, void* stream);
/* Step t phase 4 (after the all-gather): W -= lr * P for every block. */
SHAMPOO_API int shampoo_apply(shampoo_ctx* ctx, void* const* params, int32_t dtype, double lr, void* stream);

/* Gather buffer owned by the context: group_size * max_payload scalars of
 * *dtype (F64 for precision=double, F32 for single).  Rank k's region starts
 * at k * max_payload scalars. */
SHAMPOO_API void* shampoo_gather_buffer(shampoo_ctx* ctx, int64_t* scalars, int32_t* dtype);

SHAMPOO_API int shampoo_guard_stats_get(shampoo_ctx* ctx, shampoo_guard_stats* out);
SHAMPOO_API int shampoo_guard_stats_set(shampoo_ctx* ctx, const shampoo_guard_stats* in);
/* Phase timing with CUDA events on the launching stream (off by default).
 * Phases: 0 stats (gather+graft+factor GEMM), 1 root inverse, 2 precondition GEMMs + norms,
 * 3 graft/momentum/direction, 4 apply.  shampoo_timing_get synchronises and returns the
 * accumulated milliseconds per phase (5 entries) and per-phase counts, then resets. */
#define SHAMPOO_NUM_PHASES 5
SHAMPOO_API int shampoo_timing_enable(shampoo_ctx* ctx, int32_t enable);
SHAMPOO_API int shampoo_timing_get(shampoo_ctx* ctx, double* ms, int64_t* counts);
/* algorithmic work of one plain step for the owned blocks: flops of the factor GEMMs,
 * flops of the preconditioner GEMMs, sum n^3 over owned factors (root-inverse work) */
SHAMPOO_API int shampoo_work(shampoo_ctx* ctx, double* stats_flops, double* precond_flops, double* sum_n3);
/* the tensor-core (tcgen05 int8, Ozaki) share of the two GEMM phases: executed int8 ops per step
 * (2 * 128 * N * 32 per MMA instruction) and the algorithmic FP64 flops they carry */
SHAMPOO_API int shampoo_work_tc(shampoo_ctx* ctx, double* stats_int8_ops, double* precond_int8_ops,
                                double* stats_tc_flops, double* precond_tc_flops);
/* number of kernel launches issued by this library since load (bench evidence) */
SHAMPOO_API int64_t shampoo_launch_count(void);
/* int8 tensor-core ops executed by the tcgen05 GEMM engine since load (or the last reset), counted
 * on the device per output tile (masked-out problems are not counted).  Synchronises the device. */
SHAMPOO_API int shampoo_tc_counter(int32_t reset, double* int8_ops);
/* Kernel-level timing of the tensor-core GEMM launches (bench evidence): with enable = 1 every
 * k_oz_gemm_p launch is bracketed by CUDA events on its stream and its executed int8 ops are counted,
 * both per step phase (the SHAMPOO_NUM_PHASES indices; slot 7 = outside a phase).  Each call returns
 * (8 entries each, any may be null) the milliseconds, int8 ops and launches accumulated since the
 * previous call, resets them, and sets the enable state. */
SHAMPOO_API int shampoo_gemm_timing(int32_t enable, double* ms, double* int8_ops, int64_t* launches);

/* ---- state export/import: device views into the context's arena.
 * name: "factor","inv_factor","graft_accumulator","filtered_grad","momentum",
 * "accumulator" (ADAGRAD fallback block), "diag" (DIAGONAL fallback block, per mode).
 * For factors, `mode` selects k.  Returns NULL if absent (not owned / not used).
 * *numel and *dtype describe the view; views stay valid until ctx destroy. */
SHAMPOO_API void* shampoo_state_view(shampoo_ctx* ctx, int32_t block_id, const char* name, int32_t mode,
                         int64_t* numel, int32_t* dtype);
/* per-block scalars: step (factor updates), last_inverse_step, ready (inverse present) */
SHAMPOO_API int shampoo_state_scalars_get(shampoo_ctx* ctx, int32_t block_id, int64_t* step,
                              int64_t* last_inverse_step, int32_t* ready);
SHAMPOO_API int shampoo_state_scalars_set(shampoo_ctx* ctx, int32_t block_id, int64_t step,
                              int64_t last_inverse_step, int32_t ready);
/* graft step counter shared by all owned blocks (GraftState.step) */
SHAMPOO_API int shampoo_graft_step_get(shampoo_ctx* ctx, int64_t* step);
SHAMPOO_API int shampoo_graft_step_set(shampoo_ctx* ctx, int64_t step);

/* ---- batched root inverse on caller matrices (config 5 sweep, matfun parity)
 * mats: host array of `count` device pointers to n_i x n_i row-major float64
 * matrices (symmetric).  outs: host array of device pointers receiving
 * A^(-eta/p).  status (host, count entries): 0 ok, 1 non-finite input,
 * 2 no convergence, 3 epsilon-zero singular, 4 non-finite result.
 * iters (host, optional): sweeps (eigh) or iterations (Newton).  Synchronous. */
SHAMPOO_API int shampoo_batched_root_inverse(const double* const* mats, double* const* outs,
                                 const int32_t* n, int32_t count, int32_t root_p,
                                 double exponent_multiplier, double epsilon, int32_t solver,
                                 double newton_tolerance, int32_t* status, int32_t* iters,
                                 void* stream);

/* ---- tensor-core GEMM utility: C (M x N) = alpha * A B^T + beta * C on tcgen05.mma kind::i8 with
 * Ozaki operand splitting (per-row power-of-two scaling, 7-bit int8 slices, exact int32
 * accumulation in TMEM, slice diagonals combined in FP64): 8 slices for dtype F64 (operand
 * truncation 2^-56 of each row's maximum), 5 for F32 (2^-35).  A (M x K), B (N x K), C row-major
 * device buffers of `dtype`.  symmetric != 0 requires A == B, M == N: tiles on/below the diagonal
 * are computed and mirrored (exactly symmetric C).  This engine runs the factor statistics and the
 * mode products of the optimizer step (precond.py:161-174).  Synchronous. */
SHAMPOO_API int shampoo_tc_gemm(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                                int32_t symmetric, double alpha, double beta, int32_t dtype, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SHAMPOO_B200_H_ */
