// Optimizer context and the C ABI entry points (include/shampoo_b200.h).
//
// A context owns the device state of the blocks assigned to one rank
// (optim.py:205-210 "owned" restriction), laid out in one HBM arena:
//   per-element arrays in owned-block order (G, g_eff, filter, graft acc,
//   momentum, P_sh, two mode-chain temporaries), Kronecker factors and their
//   inverses (sum_k d_k^2 per block), the group gather buffer
//   (group_size x max_payload scalars, dist.py:179-183) and solver workspaces.
// Each step phase is a handful of grouped launches over device-side block and
// chunk tables, independent of the number of blocks.
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: phase ranges for nsys / ncu --nvtx (no-ops untraced)

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>

#include "elementwise.cuh"
#include "gemm.cuh"
#include "tcgen05.cuh"
#include "thin.cuh"
#include "lowrank.cuh"
#include "rootinv.cuh"

namespace shampoo {

int64_t g_launches = 0;

namespace {

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// factors of structural rank r <= d - kLowRankGap take the low-rank path (range compression, lowrank.cuh):
// their null space makes the full-size Newton pre-pass inapplicable, the compressed r x r factor is full rank
constexpr int kLowRankGap = 8;
constexpr int kRootGroups = 2;  // measured: 2 -> 1234 ms, 4 -> 1221 ms per t=50 refresh (ResNet-50)

struct EngineBase {
  virtual ~EngineBase() = default;
  virtual void inverses_changed() = 0;  // cached tensor-core packs of the inverse factors are stale
};

template <typename T>
struct Engine : EngineBase {
  // tcgen05 int8 tensor cores, Ozaki split (exact accumulation; 8 slices for double, 5 for single)
  OzakiGemmBatch<T> stats;             // factor EMA updates, all owned blocks x modes
  // plain steps: the statistics and the first mode product in ONE launch -- for order-2 blocks the
  // Gram of G's columns and the product L^(-1/4) G read the same operand, packed once.  Mask word 0
  // = the step's go word (statistics), 1 + l = inverse of owned block l present (mode product)
  OzakiGemmBatch<T> stats_prec;
  bool merged = false;
  OzakiGemmBatch<T> prec[kMaxOrder];   // mode-k products, k = 0..order-1 (order >= 2)
  // problems too thin for a 128 x 64 tensor-core tile (rank-1 factor updates of vector blocks,
  // 3 x 3 / 7 x 7 kernel modes): HBM-bound CUDA-core kernels, exact products, FP64 sums
  ThinGemmBatch<T> stats_thin;
  ThinGemmBatch<T> prec_thin[kMaxOrder];
  GemvBatch<T> prec1;                  // order-1 blocks: P = X g
  void inverses_changed() override {
    for (auto& b : prec) b.invalidate_cached();
    stats_prec.invalidate_cached();
  }
};

// Event pairs per phase; elapsed times are collected lazily in shampoo_timing_get.
struct PhaseTimer {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending[SHAMPOO_NUM_PHASES];
  std::vector<cudaEvent_t> pool;
  double ms[SHAMPOO_NUM_PHASES] = {0, 0, 0, 0, 0};
  int64_t count[SHAMPOO_NUM_PHASES] = {0, 0, 0, 0, 0};
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  ~PhaseTimer() {
    for (auto& v : pending)
      for (auto& p : v) {
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
      }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

struct PhaseScope {
  PhaseTimer* t;
  int phase;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  int prev_tag;
  PhaseScope(PhaseTimer* t_, int p, cudaStream_t s_) : t(t_), phase(p), s(s_), prev_tag(oz_set_tag(p)) {
    static const char* const kNames[SHAMPOO_NUM_PHASES] = {"shampoo.stats", "shampoo.root_inverse",
                                                            "shampoo.precondition", "shampoo.graft_momentum",
                                                            "shampoo.apply"};
    nvtxRangePushA(kNames[p]);
    if (t->on) {
      a = t->get();
      cudaEventRecord(a, s);
    }
  }
  ~PhaseScope() {
    nvtxRangePop();
    oz_set_tag(prev_tag);
    if (t->on) {
      cudaEvent_t b = t->get();
      cudaEventRecord(b, s);
      t->pending[phase].push_back({a, b});
    }
  }
};

}  // namespace
}  // namespace shampoo

using namespace shampoo;

struct shampoo_ctx {
  shampoo_plan plan;
  shampoo_config cfg{};
  int32_t rank = 0, grank = 0, device = 0;
  bool f32 = false;
  bool buf_f32 = false;  // float32 gather buffer (cfg.gather_dtype)
  bool low_rank = true;  // low-rank root-inverse path (SHAMPOO_EIG_LOWRANK=0 disables)
  size_t esz = 8;
  int32_t nparams = 0;
  // owned blocks
  std::vector<int32_t> owned;       // global ids, ascending
  std::vector<int32_t> local_of;    // global id -> local or -1
  std::vector<int64_t> vofs;        // per owned: element offset in per-element arenas
  std::vector<int64_t> fac_off;     // per owned: element offset of factor 0 in FACT/INV
  std::vector<int64_t> step;        // per owned: ShampooBlockState.step
  std::vector<int64_t> last_inv;    // per owned: last_inverse_step
  std::vector<int32_t> ready_h;     // per owned: inverse present
  int64_t graft_step = 0;           // GraftState.step (identical for all owned blocks)
  int64_t n_elem = 0, n_fac = 0, n_fb = 0;
  bool any_order3 = false;
  std::vector<int64_t> fb_off;      // per owned: offset into FB (fallback blocks)
  void* FB = nullptr;               // fallback state (T)
  double *dsum = nullptr, *dscale = nullptr;
  Chunk* d_fb_chunks = nullptr;
  int n_fb_chunks = 0;
  int32_t* d_diag_blocks = nullptr;
  int n_diag = 0;
  // arena
  char* arena = nullptr;
  size_t arena_bytes = 0;
  void *G = nullptr, *GE = nullptr, *FILT = nullptr, *GA = nullptr, *MOM = nullptr, *PS = nullptr;
  void *T1 = nullptr, *T2 = nullptr, *FACT = nullptr, *INV = nullptr, *BUF = nullptr;
  double *part = nullptr, *gnorm2 = nullptr, *pg2 = nullptr, *ps2 = nullptr;
  int32_t* d_ready = nullptr;      // = d_gomask + 1
  int32_t* d_gomask = nullptr;     // [go word | ready per owned block]
  bool prec0_done = false;         // this step's first mode products ran with the statistics
  // the statistics write lower triangles only; k_symmetrize restores the upper ones before a refresh
  // or an export reads full factors
  SymJob* d_sym_jobs = nullptr;
  int64_t* d_sym_tbegin = nullptr;
  int n_sym_jobs = 0;
  int64_t n_sym_tiles = 0;
  bool fact_lower = false;
  int32_t *d_cb = nullptr, *d_cc = nullptr;
  // tables
  DevBlock* d_blocks = nullptr;
  DevBlock* d_params = nullptr;
  Chunk *d_owned_chunks = nullptr, *d_all_chunks = nullptr, *d_param_chunks = nullptr;
  int n_owned_chunks = 0, n_all_chunks = 0, n_param_chunks = 0;
  void** d_ptrs = nullptr;  // [grads | params]
  int32_t* d_flag = nullptr;
  int32_t* h_flag = nullptr;        // host-mapped pinned (written by k_publish_flag)
  int32_t* h_flag_dev = nullptr;    // its device alias
  // pointer-table uploads: host mirror of d_ptrs (uploads only on change) and a ring of host-mapped
  // staging slots read by k_copy_ptrs (a slot is reused once its copy kernel has run)
  std::vector<const void*> ptr_mirror;
  static constexpr int kPtrRing = 16;
  void** h_ptr_ring = nullptr;
  void** h_ptr_ring_dev = nullptr;
  cudaEvent_t ptr_ev[kPtrRing] = {};
  bool ptr_ev_used[kPtrRing] = {};
  int ptr_slot = 0;
  // deferred non-finite check (shampoo_check_finite_deferred): the step's state-writing kernels are
  // predicated on the device word d_go (= 1 - non-finite); the host reads the flag one call later
  int32_t* d_go = nullptr;
  bool go_armed = false;            // the step in flight is predicated on d_go
  bool deferred_pending = false;    // a deferred check awaits shampoo_check_finite_resolve
  cudaEvent_t ev_check = nullptr;   // after the deferred check's flag read-back
  int64_t saved_graft_step = 0;     // host counters before the predicated step (restored if it aborted)
  std::vector<int64_t> saved_step;
  std::unique_ptr<EngineBase> engine;
  // root-inverse jobs in kRootGroups load-balanced groups solved concurrently on their own streams
  // (host thread per group): one group's latency-bound sub-solves overlap another's DMMA rounds
  RootInverseBatch rinv[kRootGroups];
  std::vector<int32_t> job_block[kRootGroups];  // root-inverse job -> owned local block
  cudaStream_t side[kRootGroups] = {};          // side[0] unused (group 0 runs on the caller's stream)
  cudaEvent_t ev_fork = nullptr, ev_join[kRootGroups] = {};
  // plain steps: the statistics GEMMs run on side[1] concurrently with precondition/graft/apply
  // (they read only G; the factors they write are read again only at the next refresh)
  cudaEvent_t ev_prep = nullptr, ev_stats = nullptr;
  bool stats_pending = false;
  cudaStream_t lr_stream = nullptr;  // the low-rank path, concurrent with the two root-inverse groups
  cudaEvent_t ev_lr = nullptr;
  int64_t guard[4] = {0, 0, 0, 0};
  PhaseTimer timer;

  ~shampoo_ctx() {
    engine.reset();
    cudaFree(arena);
    cudaFree(d_blocks);
    cudaFree(d_params);
    cudaFree(d_owned_chunks);
    cudaFree(d_all_chunks);
    cudaFree(d_param_chunks);
    cudaFree(d_fb_chunks);
    cudaFree(d_diag_blocks);
    cudaFree(d_ptrs);
    cudaFree(d_sym_jobs);
    cudaFree(d_sym_tbegin);
    cudaFreeHost(h_flag);
    cudaFreeHost(h_ptr_ring);
    for (auto& e : ptr_ev)
      if (e) cudaEventDestroy(e);
    for (int g = 1; g < kRootGroups; ++g) {
      if (side[g]) cudaStreamDestroy(side[g]);
      if (ev_join[g]) cudaEventDestroy(ev_join[g]);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_prep) cudaEventDestroy(ev_prep);
    if (ev_lr) cudaEventDestroy(ev_lr);
    if (lr_stream) cudaStreamDestroy(lr_stream);
    if (ev_stats) cudaEventDestroy(ev_stats);
    if (ev_check) cudaEventDestroy(ev_check);
  }
  template <typename T>
  Engine<T>& eng() { return *static_cast<Engine<T>*>(engine.get()); }
};

namespace {

int upload_ptrs(shampoo_ctx* c, const void* const* grads, const void* const* params, cudaStream_t s) {
  // d_ptrs = [grads | params]; a null half keeps its previous entries.  Uploaded only when the
  // table changed (a training loop passes the same p.grad / parameter tensors every step), through
  // a host-mapped staging slot and a one-CTA copy kernel: no copy-engine transfer in the step
  bool changed = false;
  for (int i = 0; i < c->nparams; ++i) {
    if (grads && c->ptr_mirror[i] != grads[i]) {
      c->ptr_mirror[i] = grads[i];
      changed = true;
    }
    if (params && c->ptr_mirror[c->nparams + i] != params[i]) {
      c->ptr_mirror[c->nparams + i] = params[i];
      changed = true;
    }
  }
  if (!changed) return SHAMPOO_OK;
  const int slot = c->ptr_slot;
  c->ptr_slot = (c->ptr_slot + 1) % shampoo_ctx::kPtrRing;
  if (c->ptr_ev_used[slot]) SH_CUDA_CHECK(cudaEventSynchronize(c->ptr_ev[slot]));  // its last copy has run
  const size_t n = 2 * (size_t)c->nparams;
  std::memcpy(c->h_ptr_ring + slot * n, c->ptr_mirror.data(), n * sizeof(void*));
  int rc = launch_copy_ptrs(c->h_ptr_ring_dev + slot * n, c->d_ptrs, (int)n, s);
  if (rc) return rc;
  SH_CUDA_CHECK(cudaEventRecord(c->ptr_ev[slot], s));
  c->ptr_ev_used[slot] = true;
  return SHAMPOO_OK;
}

StepScalars make_scalars(const shampoo_ctx* c, int64_t t, int32_t dtype, int64_t graft_step) {
  const shampoo_config& k = c->cfg;
  StepScalars sc{};
  sc.weight_decay = k.weight_decay;
  sc.l2 = k.weight_decay > 0.0 && !k.use_decoupled_weight_decay;
  sc.decoupled = k.weight_decay > 0.0 && k.use_decoupled_weight_decay;
  sc.beta1 = k.beta1;
  sc.one_minus_beta1 = 1.0 - k.beta1;
  sc.use_filter = k.beta1 > 0.0;
  sc.inv_bc1 = (sc.use_filter && k.use_bias_correction) ? 1.0 / (1.0 - std::pow(k.beta1, (double)(t + 1))) : 1.0;
  sc.graft = k.grafting;
  sc.beta2g = k.grafting_beta2;
  sc.one_minus_beta2g = 1.0 - k.grafting_beta2;
  const bool debias = (k.grafting == SHAMPOO_GRAFT_ADAM || k.grafting == SHAMPOO_GRAFT_NORMALIZED_ADAM);
  sc.inv_bc2g = (debias && k.use_bias_correction && graft_step > 0)
                    ? 1.0 / (1.0 - std::pow(k.grafting_beta2, (double)graft_step))
                    : 1.0;
  sc.graft_eps = k.grafting_epsilon;
  sc.momentum = k.momentum;
  sc.nesterov = k.use_nesterov;
  sc.precond = (double)t >= k.start_preconditioning_step;
  sc.pdtype = dtype;
  sc.lr = k.lr;
  sc.buf_f32 = c->buf_f32;
  return sc;
}

FallbackArgs fallback_args(const shampoo_ctx* c, int64_t t) {
  const shampoo_config& k = c->cfg;
  FallbackArgs fa{};
  fa.FB = c->FB;
  fa.dsum = c->dsum;
  fa.dscale = c->dscale;
  fa.beta2 = k.beta2;
  fa.one_minus_beta2 = 1.0 - k.beta2;
  fa.ema = k.beta2 < 1.0;
  // precond.py:318-319, 384-386: correction from the global step t, not the state step
  fa.inv_corr = (k.use_bias_correction && k.beta2 < 1.0) ? 1.0 / (1.0 - std::pow(k.beta2, (double)(t + 1))) : 1.0;
  fa.epsilon = k.epsilon;
  fa.eta = k.exponent_multiplier;
  fa.div_eps = k.grafting_epsilon;  // AdaGradFallbackState division_epsilon (optim.py:241)
  fa.root_override = k.exponent_override;
  return fa;
}

ElemArenas arenas(shampoo_ctx* c) {
  ElemArenas a{};
  a.G = c->G;
  a.GE = c->cfg.beta1 > 0.0 ? c->GE : c->G;
  a.FILT = c->FILT;
  a.GA = c->GA;
  a.MOM = c->MOM;
  a.PS = c->PS;
  a.BUF = c->BUF;
  a.part = c->part;
  a.gnorm2 = c->gnorm2;
  a.pg2 = c->pg2;
  a.ps2 = c->ps2;
  a.ready = c->d_ready;
  a.go = c->go_armed ? c->d_go : nullptr;
  return a;
}

// A problem too thin for the 128 x 64 tensor-core tiles.
bool thin(const GemmProblem& p) { return ThinGemmBatch_accepts(p); }

template <typename T>
int build_engine(shampoo_ctx* c) {
  auto* e = new Engine<T>();
  c->engine.reset(e);
  const shampoo_config& k = c->cfg;
  const double alpha = k.beta2 == 1.0 ? 1.0 : 1.0 - k.beta2;  // precond.py:237-241
  const double beta = k.beta2 == 1.0 ? 1.0 : k.beta2;
  T* G = static_cast<T*>(c->G);
  T* GE = static_cast<T*>(k.beta1 > 0.0 ? c->GE : c->G);
  T* FACT = static_cast<T*>(c->FACT);
  T* INV = static_cast<T*>(c->INV);
  T* PS = static_cast<T*>(c->PS);
  T* tmp[2] = {static_cast<T*>(c->T1), static_cast<T*>(c->T2)};
  {
    // Slices of the mode-product operands (SHAMPOO_PREC_SLICES overrides).  The directions need 1e-3
    // (north_star), not FP64: measured against S = 8 and the oracle (scripts/slices_probe.py,
    // tests/test_gpu_parity.py): at the steady state S = 4/5/6 are 1.2e-6/1.3e-8/1.1e-10 from S = 8; on
    // the rank-deficient early steps at eps = 1e-12 (inverse factors ~eps^(-1/4) on the null space,
    // heavy cancellation) S = 4 reaches 9e-4 and S = 5 moves the parameters by 4e-6 (S = 8: < 1e-7),
    // so double keeps 2^-42 operand truncation (S = 6; 21 instead of 36 products).  The factor
    // statistics feed the root inverse and keep the FP64-class default.
    const char* ev = std::getenv("SHAMPOO_PREC_SLICES");
    const int ps = ev ? std::atoi(ev) : (sizeof(T) == 8 ? 6 : OzakiGemmBatch<T>::kDefaultSlices);
    for (auto& b : e->prec) {
      const int rc = b.set_slices(ps);
      if (rc) return rc;
    }
    // Statistics slices (SHAMPOO_STATS_SLICES overrides): 6 for double, operand truncation 2^-42 of the
    // row maximum.  Measured against S = 8 over a ResNet-50 run (scripts/stats_slices_probe.py,
    // profiles/r2_stats_slices.log): factors 3.3e-12 relative, inverses 8e-13 once full rank, directions
    // <= 1e-5 at the rank-1 t = 0 factors (eps = 1e-12 amplifies the null space) and 3e-7 at the steady
    // state; every reference/oracle parity test passes unchanged.  S = 5 reaches 1e-3 on early
    // directions, so 6 it is.  The ingress-bound GEMM runs 21 instead of 36 products per MAC.
    const char* es = std::getenv("SHAMPOO_STATS_SLICES");
    const int ss = es ? std::atoi(es) : (sizeof(T) == 8 ? 6 : OzakiGemmBatch<T>::kDefaultSlices);
    {
      const int rc = e->stats.set_slices(ss);
      if (rc) return rc;
    }
  }
  std::vector<GemmProblem> prec0;  // first mode products, for the merged plain-step launch
  for (size_t l = 0; l < c->owned.size(); ++l) {
    const BlockPlan& b = c->plan.blocks[c->owned[l]];
    if (b.kind != SHAMPOO_BLOCK_SHAMPOO) continue;
    const std::vector<int64_t> d = b.dims();
    const int order = b.order;
    int64_t off = c->fac_off[l];
    for (int m = 0; m < order; ++m) {
      int64_t outer = 1, inner = 1;
      for (int q = 0; q < m; ++q) outer *= d[q];
      for (int q = m + 1; q < order; ++q) inner *= d[q];
      {
        GemmProblem g = make_mode_gram(G + c->vofs[l], outer, d[m], inner, FACT + off, alpha, beta);
        g.flags |= kGemmMasked | kGemmLowerOnly;  // predicated on the step's go word (deferred check)
        g.mask_index = 0;
        if (thin(g)) e->stats_thin.add(g);
        else e->stats.add(g);
      }
      if (order == 1) {
        GemvProblem gp{};
        gp.n = (int32_t)d[0];
        gp.mask_index = (int32_t)l;
        gp.X = INV + off;
        gp.x = GE + c->vofs[l];
        gp.y = PS + c->vofs[l];
        gp.alpha = 1.0;
        e->prec1.add(gp);
      } else {
        const T* in = (m == 0) ? GE + c->vofs[l] : tmp[(m - 1) & 1] + c->vofs[l];
        T* out = (m == order - 1) ? PS + c->vofs[l] : tmp[m & 1] + c->vofs[l];
        GemmProblem p = make_mode_product(INV + off, in, out, outer, d[m], inner, 1.0);
        p.flags |= kGemmMasked;
        p.mask_index = (int32_t)l;
        if (thin(p)) e->prec_thin[m].add(p);
        else e->prec[m].add(p);
        if (m == 0 && !thin(p)) {
          p.mask_index = 1 + (int32_t)l;  // d_gomask layout
          prec0.push_back(p);
        }
      }
      off += d[m] * d[m];
    }
  }
  // merged plain-step launch: statistics first (their masks govern the shared packs: a skipped step
  // skips them, and its mode products are discarded with it), then the first mode products
  e->merged = !e->stats.empty() && !prec0.empty() && e->stats.slices() == e->prec[0].slices();
  if (e->merged) {
    for (const GemmProblem& g : e->stats.host) e->stats_prec.add(g);
    for (const GemmProblem& g : prec0) e->stats_prec.add(g);
    e->stats_prec.set_share_packs(true);
    int rc = e->stats_prec.set_slices(e->stats.slices());
    if (rc) return rc;
    if ((rc = e->stats_prec.upload())) return rc;
  }
  int rc = e->stats.upload();
  if (rc) return rc;
  if ((rc = e->stats_thin.upload())) return rc;
  for (int m = 0; m < kMaxOrder; ++m) {
    if ((rc = e->prec[m].upload())) return rc;
    if ((rc = e->prec_thin[m].upload())) return rc;
  }
  return e->prec1.upload();
}

template <typename T>
int precondition_impl(shampoo_ctx* c, cudaStream_t s) {
  Engine<T>& e = c->eng<T>();
  int rc;
  if ((rc = e.prec1.launch(s, c->d_ready))) return rc;
  for (int m = 0; m < kMaxOrder; ++m) {
    if (!(m == 0 && c->prec0_done) && (rc = e.prec[m].launch(s, c->d_ready))) return rc;
    if ((rc = e.prec_thin[m].launch(s, c->d_ready))) return rc;
  }
  c->prec0_done = false;
  if ((rc = launch_sumsq<T>(c->d_owned_chunks, c->n_owned_chunks, c->d_blocks, c->PS, c->part, s))) return rc;
  return launch_block_reduce(c->d_cb, c->d_cc, (int)c->owned.size(), c->part, c->ps2, s);
}

int check_cfg(const shampoo_config* k) {
  // optim.py:86-126 validation (host mirror also validates; this guards the C ABI)
  auto bad = [](const char* m) {
    set_error(m);
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  };
  if (!(k->beta1 >= 0.0 && k->beta1 < 1.0)) return bad("betas[0] must lie in [0, 1)");
  if (!(k->beta2 > 0.0 && k->beta2 <= 1.0)) return bad("betas[1] must lie in (0, 1]");
  if (!(k->grafting_beta2 > 0.0 && k->grafting_beta2 <= 1.0)) return bad("grafting_beta2 must lie in (0, 1]");
  if (!(k->lr > 0.0)) return bad("lr must be positive");
  if (k->epsilon < 0.0) return bad("epsilon must be non-negative");
  if (k->momentum < 0.0 || k->momentum >= 1.0) return bad("momentum must lie in [0, 1)");
  if (k->weight_decay < 0.0) return bad("weight_decay must be non-negative");
  if (k->max_preconditioner_dim < 1) return bad("max_preconditioner_dim must be at least 1");
  if (k->precondition_frequency < 1) return bad("precondition_frequency must be at least 1");
  if (k->start_preconditioning_step < 0) return bad("start_preconditioning_step must be non-negative");
  if (k->exponent_override < 0) return bad("exponent_override must be a non-negative integer");
  if (!(k->exponent_multiplier > 0.0)) return bad("exponent_multiplier must be positive");
  if (!(k->grafting_epsilon > 0.0)) return bad("grafting_epsilon must be positive");
  if (k->grafting < 0 || k->grafting > 6) return bad("unknown grafting kind");
  if (k->solver == SHAMPOO_SOLVER_NEWTON && k->exponent_multiplier != 1.0)
    return bad("the coupled Newton solver supports exponent_multiplier=1 only");
  if (k->gather_dtype != SHAMPOO_GATHER_STATE && k->gather_dtype != SHAMPOO_GATHER_F32)
    return bad("gather_dtype must be SHAMPOO_GATHER_STATE or SHAMPOO_GATHER_F32");
  return SHAMPOO_OK;
}

}  // namespace

extern "C" {

const char* shampoo_version(void) { return "paper_2309_06497_b200 0.1 (sm_100a)"; }
int64_t shampoo_launch_count(void) { return g_launches; }

int shampoo_ctx_create(const shampoo_plan* plan, const shampoo_config* cfg, int32_t rank, int32_t device,
                       shampoo_ctx** out) {
  *out = nullptr;
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (rank < 0 || rank >= plan->world) {
    set_error("rank out of range");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  SH_CUDA_CHECK(cudaSetDevice(device));
  std::unique_ptr<shampoo_ctx> c(new shampoo_ctx());
  c->plan = *plan;
  c->cfg = *cfg;
  c->rank = rank;
  c->grank = rank % plan->group;
  c->device = device;
  c->f32 = cfg->precision == SHAMPOO_PRECISION_SINGLE;
  c->buf_f32 = c->f32 || cfg->gather_dtype == SHAMPOO_GATHER_F32;
  c->esz = c->f32 ? 4 : 8;
  c->nparams = (int32_t)plan->params.size();
  const int nb = (int)plan->blocks.size();
  c->local_of.assign(nb, -1);
  for (int i = 0; i < nb; ++i) {
    const BlockPlan& b = plan->blocks[i];
    if (b.owner != c->grank) continue;
    c->local_of[i] = (int32_t)c->owned.size();
    c->fb_off.push_back(c->n_fb);
    if (b.kind == SHAMPOO_BLOCK_ADAGRAD) c->n_fb += b.var_count;
    if (b.kind == SHAMPOO_BLOCK_DIAGONAL)
      for (int64_t d : b.dims()) c->n_fb += d;
    c->owned.push_back(i);
    c->vofs.push_back(c->n_elem);
    c->n_elem += b.var_count;
    c->fac_off.push_back(c->n_fac);
    if (b.kind == SHAMPOO_BLOCK_SHAMPOO) {
      for (int64_t d : b.dims()) c->n_fac += d * d;
      if (b.order >= 3) c->any_order3 = true;
    }
  }
  const size_t no = c->owned.size();
  c->step.assign(no, 0);
  c->last_inv.assign(no, -1);
  c->ready_h.assign(no, 0);
  // chunk tables
  std::vector<Chunk> oc, ac, pc;
  std::vector<int32_t> cb(no), cc(no);
  for (size_t l = 0; l < no; ++l) {
    const BlockPlan& b = plan->blocks[c->owned[l]];
    cb[l] = (int32_t)oc.size();
    for (int64_t s = 0; s < b.var_count; s += kChunk) oc.push_back(Chunk{b.block_id, 0, s, std::min<int64_t>(kChunk, b.var_count - s)});
    cc[l] = (int32_t)oc.size() - cb[l];
  }
  for (int i = 0; i < nb; ++i) {
    const BlockPlan& b = plan->blocks[i];
    for (int64_t s = 0; s < b.var_count; s += kChunk) ac.push_back(Chunk{i, 0, s, std::min<int64_t>(kChunk, b.var_count - s)});
  }
  std::vector<Chunk> fc;
  std::vector<int32_t> dblk;
  for (size_t l = 0; l < no; ++l) {
    const BlockPlan& b = plan->blocks[c->owned[l]];
    if (b.kind != SHAMPOO_BLOCK_ADAGRAD && b.kind != SHAMPOO_BLOCK_DIAGONAL) continue;
    for (int64_t s = 0; s < b.var_count; s += kChunk)
      fc.push_back(Chunk{b.block_id, 0, s, std::min<int64_t>(kChunk, b.var_count - s)});
    if (b.kind == SHAMPOO_BLOCK_DIAGONAL) dblk.push_back(b.block_id);
  }
  c->n_fb_chunks = (int)fc.size();
  c->n_diag = (int)dblk.size();
  std::vector<DevBlock> db(nb), dp(c->nparams);
  for (int i = 0; i < nb; ++i) {
    const BlockPlan& b = plan->blocks[i];
    const ParamPlan& pp = plan->params[b.param];
    DevBlock& d = db[i];
    std::memset(&d, 0, sizeof(d));
    d.param = b.param;
    d.order = b.order;
    d.kind = b.kind;
    d.local = c->local_of[i];
    d.numel = b.var_count;
    d.gofs = b.gather_offset;
    d.vofs = d.local >= 0 ? c->vofs[d.local] : 0;
    d.fofs = d.local >= 0 ? c->fb_off[d.local] : 0;
    for (int k = 0; k < b.order; ++k) {
      d.dims[k] = b.hi[k] - b.lo[k];
      d.lo[k] = b.lo[k];
      d.mstride[k] = pp.mstride[k];
    }
    bool contig = b.order > 0 && d.mstride[b.order - 1] == 1;
    for (int k = 0; k + 1 < b.order && contig; ++k) contig = d.mstride[k] == d.dims[k + 1] * d.mstride[k + 1];
    for (int k = 1; k < b.order && contig; ++k) contig = d.lo[k] == 0;
    d.cbase = -1;
    if (contig) {
      d.cbase = 0;
      for (int k = 0; k < b.order; ++k) d.cbase += d.lo[k] * d.mstride[k];
    }
  }
  for (int p = 0; p < c->nparams; ++p) {
    std::memset(&dp[p], 0, sizeof(DevBlock));
    dp[p].param = p;
    dp[p].cbase = -1;
    const int64_t n = plan->params[p].numel;
    for (int64_t s = 0; s < n; s += kChunk) pc.push_back(Chunk{p, 0, s, std::min<int64_t>(kChunk, n - s)});
  }
  c->n_owned_chunks = (int)oc.size();
  c->n_all_chunks = (int)ac.size();
  c->n_param_chunks = (int)pc.size();
  // arena layout
  const size_t E = (size_t)c->n_elem, es = c->esz;
  const bool filt = cfg->beta1 > 0.0, graft = cfg->grafting != SHAMPOO_GRAFT_SGD, mom = cfg->momentum > 0.0;
  const size_t buf_elems = (size_t)plan->group * plan->max_payload;
  struct Sl {
    void** p;
    size_t bytes;
  };
  std::vector<Sl> slots = {
      {&c->G, E * es},
      {&c->GE, filt ? E * es : 0},
      {&c->FILT, filt ? E * es : 0},
      {&c->GA, graft ? E * es : 0},
      {&c->MOM, mom ? E * es : 0},
      {&c->PS, E * es},
      {&c->T1, E * es},
      {&c->T2, c->any_order3 ? E * es : 0},
      {&c->FACT, (size_t)c->n_fac * es},
      {&c->INV, (size_t)c->n_fac * es},
      {&c->BUF, std::max<size_t>(buf_elems, 1) * (c->buf_f32 ? 4 : es)},
      {(void**)&c->part, std::max<size_t>(oc.size(), 1) * 8},
      {(void**)&c->gnorm2, std::max<size_t>(no, 1) * 8},
      {(void**)&c->pg2, std::max<size_t>(no, 1) * 8},
      {(void**)&c->ps2, std::max<size_t>(no, 1) * 8},
      {(void**)&c->d_gomask, (1 + std::max<size_t>(no, 1)) * 4},
      {(void**)&c->d_cb, std::max<size_t>(no, 1) * 4},
      {(void**)&c->d_cc, std::max<size_t>(no, 1) * 4},
      {(void**)&c->d_flag, 16},
      {&c->FB, (size_t)c->n_fb * es},
      {(void**)&c->dsum, (size_t)c->n_fb * 8},
      {(void**)&c->dscale, (size_t)c->n_fb * 8},
  };
  size_t total = 0;
  for (auto& s : slots) total += align_up(s.bytes);
  cudaError_t err = cudaMalloc(&c->arena, total);
  if (err != cudaSuccess) {
    set_error(std::string("arena allocation of ") + std::to_string(total) + " bytes: " + cudaGetErrorString(err));
    return SHAMPOO_ERR_OUT_OF_MEMORY;
  }
  c->arena_bytes = total;
  SH_CUDA_CHECK(cudaMemset(c->arena, 0, total));
  size_t at = 0;
  for (auto& s : slots) {
    *s.p = s.bytes ? (void*)(c->arena + at) : nullptr;
    at += align_up(s.bytes);
  }
  c->d_go = c->d_gomask;  // 1 outside a predicated step (the merged statistics launch reads it)
  c->d_ready = c->d_gomask + 1;
  {
    const int32_t one = 1;
    SH_CUDA_CHECK(cudaMemcpy(c->d_go, &one, sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  {
    std::vector<SymJob> sj;
    std::vector<int64_t> tb;
    for (size_t l = 0; l < c->owned.size(); ++l) {
      const BlockPlan& b = plan->blocks[c->owned[l]];
      if (b.kind != SHAMPOO_BLOCK_SHAMPOO) continue;
      int64_t off = c->fac_off[l];
      for (int64_t d : b.dims()) {
        sj.push_back(SymJob{off, (int32_t)d, 0});
        tb.push_back(c->n_sym_tiles);
        const int64_t t = (d + 31) / 32;
        c->n_sym_tiles += t * (t + 1) / 2;
        off += d * d;
      }
    }
    c->n_sym_jobs = (int)sj.size();
    SH_CUDA_CHECK(cudaMalloc(&c->d_sym_jobs, std::max<size_t>(sj.size(), 1) * sizeof(SymJob)));
    SH_CUDA_CHECK(cudaMalloc(&c->d_sym_tbegin, std::max<size_t>(tb.size(), 1) * sizeof(int64_t)));
    if (!sj.empty()) {
      SH_CUDA_CHECK(cudaMemcpy(c->d_sym_jobs, sj.data(), sj.size() * sizeof(SymJob), cudaMemcpyHostToDevice));
      SH_CUDA_CHECK(cudaMemcpy(c->d_sym_tbegin, tb.data(), tb.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    }
  }
  SH_CUDA_CHECK(cudaMalloc(&c->d_blocks, std::max(nb, 1) * sizeof(DevBlock)));
  SH_CUDA_CHECK(cudaMalloc(&c->d_params, std::max(c->nparams, 1) * sizeof(DevBlock)));
  SH_CUDA_CHECK(cudaMalloc(&c->d_owned_chunks, std::max<size_t>(oc.size(), 1) * sizeof(Chunk)));
  SH_CUDA_CHECK(cudaMalloc(&c->d_all_chunks, std::max<size_t>(ac.size(), 1) * sizeof(Chunk)));
  SH_CUDA_CHECK(cudaMalloc(&c->d_param_chunks, std::max<size_t>(pc.size(), 1) * sizeof(Chunk)));
  SH_CUDA_CHECK(cudaMalloc(&c->d_ptrs, std::max(2 * c->nparams, 1) * sizeof(void*)));
  SH_CUDA_CHECK(cudaMalloc(&c->d_fb_chunks, std::max<size_t>(fc.size(), 1) * sizeof(Chunk)));
  SH_CUDA_CHECK(cudaMalloc(&c->d_diag_blocks, std::max<size_t>(dblk.size(), 1) * sizeof(int32_t)));
  if (!fc.empty())
    SH_CUDA_CHECK(cudaMemcpy(c->d_fb_chunks, fc.data(), fc.size() * sizeof(Chunk), cudaMemcpyHostToDevice));
  if (!dblk.empty())
    SH_CUDA_CHECK(cudaMemcpy(c->d_diag_blocks, dblk.data(), dblk.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  SH_CUDA_CHECK(cudaHostAlloc(&c->h_flag, 16, cudaHostAllocMapped));
  SH_CUDA_CHECK(cudaHostGetDevicePointer((void**)&c->h_flag_dev, c->h_flag, 0));
  SH_CUDA_CHECK(cudaHostAlloc(&c->h_ptr_ring, (size_t)shampoo_ctx::kPtrRing * 2 * std::max(c->nparams, 1) * sizeof(void*),
                              cudaHostAllocMapped));
  SH_CUDA_CHECK(cudaHostGetDevicePointer((void**)&c->h_ptr_ring_dev, c->h_ptr_ring, 0));
  for (auto& e : c->ptr_ev) SH_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  c->ptr_mirror.assign(2 * (size_t)c->nparams, nullptr);
  SH_CUDA_CHECK(cudaMemcpy(c->d_blocks, db.data(), nb * sizeof(DevBlock), cudaMemcpyHostToDevice));
  SH_CUDA_CHECK(cudaMemcpy(c->d_params, dp.data(), c->nparams * sizeof(DevBlock), cudaMemcpyHostToDevice));
  SH_CUDA_CHECK(cudaMemcpy(c->d_owned_chunks, oc.data(), oc.size() * sizeof(Chunk), cudaMemcpyHostToDevice));
  SH_CUDA_CHECK(cudaMemcpy(c->d_all_chunks, ac.data(), ac.size() * sizeof(Chunk), cudaMemcpyHostToDevice));
  SH_CUDA_CHECK(cudaMemcpy(c->d_param_chunks, pc.data(), pc.size() * sizeof(Chunk), cudaMemcpyHostToDevice));
  SH_CUDA_CHECK(cudaMemcpy(c->d_cb, cb.data(), no * sizeof(int32_t), cudaMemcpyHostToDevice));
  SH_CUDA_CHECK(cudaMemcpy(c->d_cc, cc.data(), no * sizeof(int32_t), cudaMemcpyHostToDevice));
  rc = c->f32 ? build_engine<float>(c.get()) : build_engine<double>(c.get());
  if (rc) return rc;
  // root-inverse jobs: every (owned shampoo block, mode), split into two groups by LPT on n^3
  struct JobDesc {
    int32_t n, p, l;
    int64_t off;
  };
  std::vector<JobDesc> all;
  for (size_t l = 0; l < no; ++l) {
    const BlockPlan& b = plan->blocks[c->owned[l]];
    if (b.kind != SHAMPOO_BLOCK_SHAMPOO) continue;
    const int p = cfg->exponent_override ? cfg->exponent_override : 2 * b.order;  // precond.py:217
    int64_t off = c->fac_off[l];
    for (int64_t d : b.dims()) {
      all.push_back({(int32_t)d, p, (int32_t)l, off});
      off += d * d;
    }
  }
  std::vector<size_t> order(all.size());
  for (size_t q = 0; q < order.size(); ++q) order[q] = q;
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return all[a].n > all[b].n; });
  std::vector<JobDesc> grp[kRootGroups];
  double load[kRootGroups] = {};
  for (size_t q : order) {
    const int g = (int)(std::min_element(load, load + kRootGroups) - load);
    grp[g].push_back(all[q]);
    load[g] += (double)all[q].n * all[q].n * all[q].n;
  }
  for (int g = 0; g < kRootGroups; ++g) {
    std::vector<int32_t> jn, jp;
    for (const auto& J : grp[g]) {
      jn.push_back(J.n);
      jp.push_back(J.p);
      c->job_block[g].push_back(J.l);
    }
    if ((rc = c->rinv[g].setup(jn, jp))) return rc;
    for (size_t q = 0; q < grp[g].size(); ++q) {
      char* f = static_cast<char*>(c->FACT) + grp[g][q].off * c->esz;
      char* x = static_cast<char*>(c->INV) + grp[g][q].off * c->esz;
      c->rinv[g].set_io((int)q, f, c->f32, x, c->f32);
    }
  }
  SH_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  SH_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_prep, cudaEventDisableTiming));
  SH_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_lr, cudaEventDisableTiming));
  SH_CUDA_CHECK(cudaStreamCreateWithFlags(&c->lr_stream, cudaStreamNonBlocking));
  SH_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_stats, cudaEventDisableTiming));
  SH_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_check, cudaEventDisableTiming));
  {
    const char* lr = std::getenv("SHAMPOO_EIG_LOWRANK");
    c->low_rank = lr ? std::atoi(lr) != 0 : true;
  }
  for (int g = 1; g < kRootGroups; ++g) {
    SH_CUDA_CHECK(cudaStreamCreateWithFlags(&c->side[g], cudaStreamNonBlocking));
    SH_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_join[g], cudaEventDisableTiming));
  }
  SH_CUDA_CHECK(cudaDeviceSynchronize());
  *out = c.release();
  return SHAMPOO_OK;
}

void shampoo_ctx_destroy(shampoo_ctx* ctx) {
  cudaDeviceSynchronize();  // the solver workspaces return to the device cache idle (dev_free)
  delete ctx;
}

int64_t shampoo_ctx_device_bytes(const shampoo_ctx* ctx) { return (int64_t)ctx->arena_bytes; }

int shampoo_check_finite(shampoo_ctx* c, const void* const* grads, int32_t dtype, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc = upload_ptrs(c, grads, nullptr, s);
  if (rc) return rc;
  SH_CUDA_CHECK(cudaMemsetAsync(c->d_flag, 0, sizeof(int32_t), s));
  if ((rc = launch_finite<double>(c->d_param_chunks, c->n_param_chunks, c->d_params,
                                  (const void* const*)c->d_ptrs, dtype, c->d_flag, nullptr, s)))
    return rc;
  if ((rc = launch_publish_flag(c->d_flag, c->h_flag_dev, s))) return rc;
  SH_CUDA_CHECK(cudaStreamSynchronize(s));
  if (*(volatile int32_t*)c->h_flag) {
    set_error("gradient contains non-finite entries; step aborted");
    return SHAMPOO_ERR_NONFINITE_GRAD;
  }
  return SHAMPOO_OK;
}

namespace {
bool refresh_step(const shampoo_ctx* c, int64_t t) {
  const shampoo_config& k = c->cfg;
  if ((double)t < k.start_preconditioning_step || t % k.precondition_frequency != 0) return false;
  for (const auto& r : c->rinv)
    if (r.jobs()) return true;
  return false;
}
}  // namespace

int shampoo_check_finite_deferred(shampoo_ctx* c, const void* const* grads, int32_t dtype, int64_t t,
                                  int32_t* deferred, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (deferred) *deferred = 0;
  if (c->deferred_pending) {
    set_error("check_finite_deferred: the previous deferred check was not resolved");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  // a refresh step's root inverse rewrites the inverses from host-side decisions: checked eagerly
  if (refresh_step(c, t)) return shampoo_check_finite(c, grads, dtype, stream);
  int rc = upload_ptrs(c, grads, nullptr, s);
  if (rc) return rc;
  static const int32_t kOne = 1;
  SH_CUDA_CHECK(cudaMemsetAsync(c->d_flag, 0, sizeof(int32_t), s));
  SH_CUDA_CHECK(cudaMemcpyAsync(c->d_go, &kOne, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  if ((rc = launch_finite<double>(c->d_param_chunks, c->n_param_chunks, c->d_params,
                                  (const void* const*)c->d_ptrs, dtype, c->d_flag, c->d_go, s)))
    return rc;
  if ((rc = launch_publish_flag(c->d_flag, c->h_flag_dev, s))) return rc;
  SH_CUDA_CHECK(cudaEventRecord(c->ev_check, s));
  c->saved_graft_step = c->graft_step;
  c->saved_step = c->step;
  c->go_armed = true;
  c->deferred_pending = true;
  if (deferred) *deferred = 1;
  return SHAMPOO_OK;
}

int shampoo_check_finite_resolve(shampoo_ctx* c, int32_t* aborted) {
  if (aborted) *aborted = 0;
  if (!c->deferred_pending) return SHAMPOO_OK;
  c->deferred_pending = false;
  SH_CUDA_CHECK(cudaEventSynchronize(c->ev_check));
  if (!*(volatile int32_t*)c->h_flag) return SHAMPOO_OK;
  // the predicated step wrote no device state; undo its host-side counters and re-arm the go word
  c->graft_step = c->saved_graft_step;
  c->step = c->saved_step;
  {
    const int32_t one = 1;
    SH_CUDA_CHECK(cudaMemcpy(c->d_go, &one, sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  if (aborted) *aborted = 1;
  set_error("gradient contains non-finite entries; step aborted (deferred check)");
  return SHAMPOO_ERR_NONFINITE_GRAD;
}

namespace {
// Orders the caller's stream after the statistics launched on side[1] (before anything that reads
// the factors or overwrites G, and at the end of every step).
int join_stats(shampoo_ctx* c, cudaStream_t s) {
  if (!c->stats_pending) return SHAMPOO_OK;
  SH_CUDA_CHECK(cudaStreamWaitEvent(s, c->ev_stats, 0));
  c->stats_pending = false;
  return SHAMPOO_OK;
}

// Restore the upper triangles of the factors (stream-ordered on s after the statistics).
int symmetrize_factors(shampoo_ctx* c, cudaStream_t s) {
  if (!c->fact_lower) return SHAMPOO_OK;
  int rc = join_stats(c, s);
  if (rc) return rc;
  rc = c->f32 ? launch_symmetrize<float>(c->d_sym_jobs, c->d_sym_tbegin, c->n_sym_jobs, c->n_sym_tiles, c->FACT, s)
              : launch_symmetrize<double>(c->d_sym_jobs, c->d_sym_tbegin, c->n_sym_jobs, c->n_sym_tiles, c->FACT, s);
  if (rc) return rc;
  c->fact_lower = false;
  return SHAMPOO_OK;
}

// The stats phase; gradients from the caller's tensors (grads) or from a reduced gather-layout
// buffer (gbuf, context dtype, scaled by gscale).
int stats_update_impl(shampoo_ctx* c, const void* const* grads, const void* gbuf, double gscale,
                      const void* const* params, int32_t dtype, int64_t t, cudaStream_t s) {
  int rc = join_stats(c, s);
  if (rc) return rc;
  rc = upload_ptrs(c, grads, params, s);
  if (rc) return rc;
  const int64_t gstep = c->graft_step + 1;  // GraftState.update increments first (grafting.py:71)
  StepScalars sc = make_scalars(c, t, dtype, gstep);
  ElemArenas ar = arenas(c);
  if (gbuf) {
    sc.gbuf = 1;
    sc.gscale = gscale;
    ar.GBUF = gbuf;
  }
  const void* const* gp = (const void* const*)c->d_ptrs;
  const void* const* pp = (const void* const*)(c->d_ptrs + c->nparams);
  const int no = (int)c->owned.size();
  const bool normalized = c->cfg.grafting >= SHAMPOO_GRAFT_NORMALIZED_ADAGRAD;
  PhaseScope scope(&c->timer, 0, s);
  if (normalized) {
    rc = c->f32 ? launch_prepare<float>(0, c->d_owned_chunks, c->n_owned_chunks, c->d_blocks, gp, pp, sc, ar, s)
                : launch_prepare<double>(0, c->d_owned_chunks, c->n_owned_chunks, c->d_blocks, gp, pp, sc, ar, s);
    if (rc) return rc;
    if ((rc = launch_block_reduce(c->d_cb, c->d_cc, no, c->part, c->gnorm2, s))) return rc;
  }
  rc = c->f32 ? launch_prepare<float>(1, c->d_owned_chunks, c->n_owned_chunks, c->d_blocks, gp, pp, sc, ar, s)
              : launch_prepare<double>(1, c->d_owned_chunks, c->n_owned_chunks, c->d_blocks, gp, pp, sc, ar, s);
  if (rc) return rc;
  if ((rc = launch_block_reduce(c->d_cb, c->d_cc, no, c->part, c->pg2, s))) return rc;
  // concurrent statistics (not under per-phase timing, where phases must not overlap)
  const bool concurrent = !c->timer.on && c->side[1] != nullptr;
  cudaStream_t ss = s;
  if (concurrent) {
    SH_CUDA_CHECK(cudaEventRecord(c->ev_prep, s));
    SH_CUDA_CHECK(cudaStreamWaitEvent(c->side[1], c->ev_prep, 0));
    ss = c->side[1];
  }
  // statistics problems are masked on word 0 of the go pointer (deferred check; null: unconditional)
  const int32_t* go = c->go_armed ? c->d_go : nullptr;
  const bool merged = c->f32 ? c->eng<float>().merged : c->eng<double>().merged;
  c->prec0_done = merged && sc.precond && !refresh_step(c, t);
  if (c->prec0_done) {
    // plain step: statistics + first mode products in one launch on the caller's stream (shared packs)
    rc = c->f32 ? c->eng<float>().stats_prec.launch(s, c->d_gomask) : c->eng<double>().stats_prec.launch(s, c->d_gomask);
    ss = s;
  } else {
    rc = c->f32 ? c->eng<float>().stats.launch(ss, go) : c->eng<double>().stats.launch(ss, go);
  }
  if (rc) return rc;
  rc = c->f32 ? c->eng<float>().stats_thin.launch(ss, go) : c->eng<double>().stats_thin.launch(ss, go);
  if (rc) return rc;
  if (concurrent && ss != s) {
    SH_CUDA_CHECK(cudaEventRecord(c->ev_stats, ss));
    c->stats_pending = true;
  }
  if (c->n_fb_chunks) {
    const FallbackArgs fa = fallback_args(c, t);
    rc = c->f32 ? launch_fallback_update<float>(c->d_fb_chunks, c->n_fb_chunks, c->d_blocks, ar, fa,
                                                 c->d_diag_blocks, c->n_diag, s)
                : launch_fallback_update<double>(c->d_fb_chunks, c->n_fb_chunks, c->d_blocks, ar, fa,
                                                  c->d_diag_blocks, c->n_diag, s);
    if (rc) return rc;
  }
  c->fact_lower = true;  // the statistics GEMMs wrote lower triangles
  c->graft_step = gstep;
  for (size_t l = 0; l < c->owned.size(); ++l)
    if (c->plan.blocks[c->owned[l]].kind != SHAMPOO_BLOCK_GRAFT_ONLY) ++c->step[l];
  return SHAMPOO_OK;
}
}  // namespace

int shampoo_stats_update(shampoo_ctx* c, const void* const* grads, const void* const* params, int32_t dtype,
                         int64_t t, void* stream) {
  return stats_update_impl(c, grads, nullptr, 1.0, params, dtype, t, static_cast<cudaStream_t>(stream));
}

int shampoo_stats_update_reduced(shampoo_ctx* c, const void* gbuf, double gscale, const void* const* params,
                                 int32_t dtype, int64_t t, void* stream) {
  if (!gbuf) {
    set_error("stats_update_reduced: null gradient buffer");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  return stats_update_impl(c, nullptr, gbuf, gscale, params, dtype, t, static_cast<cudaStream_t>(stream));
}

int shampoo_pack_gradients(shampoo_ctx* c, const void* const* grads, int32_t dtype, void* gbuf, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc = upload_ptrs(c, grads, nullptr, s);
  if (rc) return rc;
  const void* const* gp = (const void* const*)c->d_ptrs;
  return c->f32 ? launch_pack_grads<float>(c->d_all_chunks, c->n_all_chunks, c->d_blocks, gp, dtype, gbuf, s)
                : launch_pack_grads<double>(c->d_all_chunks, c->n_all_chunks, c->d_blocks, gp, dtype, gbuf, s);
}

int shampoo_reduced_nonfinite(shampoo_ctx* c, const void* gbuf, int32_t* d_flag, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SH_CUDA_CHECK(cudaMemsetAsync(d_flag, 0, sizeof(int32_t), s));
  return c->f32 ? launch_region_finite<float>(c->d_owned_chunks, c->n_owned_chunks, c->d_blocks, gbuf, d_flag, s)
                : launch_region_finite<double>(c->d_owned_chunks, c->n_owned_chunks, c->d_blocks, gbuf, d_flag, s);
}

int shampoo_root_inverse(shampoo_ctx* c, int64_t t, int32_t* refreshed, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (refreshed) *refreshed = 0;
  const shampoo_config& k = c->cfg;
  if ((double)t < k.start_preconditioning_step || t % k.precondition_frequency != 0) return SHAMPOO_OK;
  size_t njobs = 0;
  for (const auto& r : c->rinv) njobs += r.jobs();
  if (njobs == 0) return SHAMPOO_OK;
  const double corr = (k.use_bias_correction && k.beta2 < 1.0) ? 1.0 - std::pow(k.beta2, (double)(t + 1)) : 1.0;
  {
    const int rj = symmetrize_factors(c, s);  // the refresh reads this step's full factors
    if (rj) return rj;
  }
  PhaseScope scope(&c->timer, 1, s);
  std::vector<int32_t> has_prev[kRootGroups], full_rank[kRootGroups], low_rank[kRootGroups];
  std::vector<LowRankJob> lr_jobs;
  for (int g = 0; g < kRootGroups; ++g) {
    has_prev[g].resize(c->rinv[g].jobs());
    full_rank[g].resize(c->rinv[g].jobs());
    low_rank[g].assign(c->rinv[g].jobs(), 0);
    for (size_t j = 0; j < has_prev[g].size(); ++j) {
      const int l = c->job_block[g][j];
      has_prev[g][j] = c->ready_h[l];
      // structural rank of the factor: `step` accumulated Gram terms of rank numel/d each; only a
      // possibly full-rank factor is worth the Newton pre-pass of the eigh path, and a factor of
      // small rank r is solved through its r x r compression (lowrank.cuh)
      const int64_t d = c->rinv[g].job_n((int)j);
      const int64_t numel = c->plan.blocks[c->owned[l]].var_count;
      const int64_t rank = (int64_t)c->step[l] * (numel / std::max<int64_t>(d, 1));
      full_rank[g][j] = rank >= d ? 1 : 0;
      if (k.solver == SHAMPOO_SOLVER_EIGH && k.epsilon > 0.0 && !c->f32 && d >= 16 &&
          rank + kLowRankGap <= d && c->low_rank) {
        low_rank[g][j] = 1;
        LowRankJob L{};
        L.d = (int32_t)d;
        L.r = (int32_t)std::max<int64_t>(rank, 1);
        L.root_p = c->rinv[g].job_p((int)j);
        L.has_prev = c->ready_h[l];
        L.in = static_cast<const double*>(c->rinv[g].job_in((int)j));
        L.out = static_cast<double*>(c->rinv[g].job_out((int)j));
        lr_jobs.push_back(L);
      }
    }
  }
  // group g > 0 on side stream g, the low-rank jobs on lr_stream (each after everything already
  // queued on s, each driven by its own host thread), group 0 on s; the groups skip the low-rank jobs
  SH_CUDA_CHECK(cudaEventRecord(c->ev_fork, s));
  int64_t lstats[4] = {0, 0, 0, 0};
  int lrc = SHAMPOO_OK;
  std::string lerr;
  int64_t gstats[kRootGroups][4] = {};
  int grc[kRootGroups] = {};
  std::string gerr[kRootGroups];
  auto solve = [&](int g, cudaStream_t st) {
    oz_set_tag(1);  // root-inverse phase (worker threads too)
    if (c->rinv[g].jobs() == 0) return;
    grc[g] = c->rinv[g].run(1.0 / corr, has_prev[g], k.exponent_multiplier, k.epsilon, k.solver, k.newton_tolerance,
                            st, gstats[g], nullptr, nullptr, /*allow_warm=*/true, &full_rank[g], &low_rank[g]);
    if (grc[g]) gerr[g] = shampoo_last_error();
  };
  std::thread lr_thread;
  std::vector<std::thread> threads;
  struct JoinAll {  // every early return below still joins the worker threads
    std::thread& a;
    std::vector<std::thread>& b;
    ~JoinAll() {
      if (a.joinable()) a.join();
      for (auto& t : b)
        if (t.joinable()) t.join();
    }
  } join_all{lr_thread, threads};
  if (!lr_jobs.empty()) {
    SH_CUDA_CHECK(cudaStreamWaitEvent(c->lr_stream, c->ev_fork, 0));
    lr_thread = std::thread([&] {
      oz_set_tag(1);
      lrc = low_rank_root_inverse(lr_jobs, 1.0 / corr, k.exponent_multiplier, k.epsilon, c->lr_stream, lstats);
      if (lrc) lerr = shampoo_last_error();
    });
  }
  for (int g = 1; g < kRootGroups; ++g) {
    SH_CUDA_CHECK(cudaStreamWaitEvent(c->side[g], c->ev_fork, 0));
    threads.emplace_back(solve, g, c->side[g]);
  }
  solve(0, s);
  for (auto& th : threads)
    if (th.joinable()) th.join();
  if (lr_thread.joinable()) {
    lr_thread.join();
    SH_CUDA_CHECK(cudaEventRecord(c->ev_lr, c->lr_stream));
    SH_CUDA_CHECK(cudaStreamWaitEvent(s, c->ev_lr, 0));
    if (lrc) {
      set_error(lerr);
      return lrc;
    }
    for (int q = 0; q < 4; ++q) c->guard[q] += lstats[q];
  }
  for (int g = 1; g < kRootGroups; ++g) {
    SH_CUDA_CHECK(cudaEventRecord(c->ev_join[g], c->side[g]));
    SH_CUDA_CHECK(cudaStreamWaitEvent(s, c->ev_join[g], 0));
  }
  for (int g = 0; g < kRootGroups; ++g)
    if (grc[g]) {
      set_error(gerr[g]);
      return grc[g];
    }
  for (int g = 0; g < kRootGroups; ++g)
    for (int q = 0; q < 4; ++q) c->guard[q] += gstats[g][q];
  for (size_t l = 0; l < c->owned.size(); ++l) {
    if (c->plan.blocks[c->owned[l]].kind != SHAMPOO_BLOCK_SHAMPOO) continue;
    c->ready_h[l] = 1;
    c->last_inv[l] = t;
  }
  SH_CUDA_CHECK(cudaMemcpyAsync(c->d_ready, c->ready_h.data(), c->ready_h.size() * sizeof(int32_t),
                                cudaMemcpyHostToDevice, s));
  c->engine->inverses_changed();
  if (refreshed) *refreshed = 1;
  return SHAMPOO_OK;
}

int shampoo_precondition_graft(shampoo_ctx* c, const void* const* params, int32_t dtype, int64_t t,
                               void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc = upload_ptrs(c, nullptr, params, s);
  if (rc) return rc;
  const StepScalars sc = make_scalars(c, t, dtype, c->graft_step);
  if (sc.precond) {
    PhaseScope scope(&c->timer, 2, s);
    if (c->n_fb_chunks) {  // fallback directions into PS before the norms
      const FallbackArgs fa = fallback_args(c, t);
      const ElemArenas ar = arenas(c);
      rc = c->f32 ? launch_fallback_precondition<float>(c->d_fb_chunks, c->n_fb_chunks, c->d_blocks, ar, fa,
                                                        c->d_diag_blocks, c->n_diag, sc.use_filter, s)
                  : launch_fallback_precondition<double>(c->d_fb_chunks, c->n_fb_chunks, c->d_blocks, ar, fa,
                                                         c->d_diag_blocks, c->n_diag, sc.use_filter, s);
      if (rc) return rc;
    }
    rc = c->f32 ? precondition_impl<float>(c, s) : precondition_impl<double>(c, s);
    if (rc) return rc;
  }
  const void* const* pp = (const void* const*)(c->d_ptrs + c->nparams);
  PhaseScope scope(&c->timer, 3, s);
  return c->f32 ? launch_final<float>(c->d_owned_chunks, c->n_owned_chunks, c->d_blocks, pp, sc, arenas(c), s)
                : launch_final<double>(c->d_owned_chunks, c->n_owned_chunks, c->d_blocks, pp, sc, arenas(c), s);
}

int shampoo_apply(shampoo_ctx* c, void* const* params, int32_t dtype, double lr, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc = upload_ptrs(c, nullptr, (const void* const*)params, s);
  if (rc) return rc;
  StepScalars sc{};
  sc.lr = lr;
  sc.pdtype = dtype;
  sc.buf_f32 = c->buf_f32;
  void* const* pp = (void* const*)(c->d_ptrs + c->nparams);
  {
    PhaseScope scope(&c->timer, 4, s);
    const int32_t* go = c->go_armed ? c->d_go : nullptr;
    rc = c->f32 ? launch_apply<float>(c->d_all_chunks, c->n_all_chunks, c->d_blocks, pp, c->BUF, sc, go, s)
                : launch_apply<double>(c->d_all_chunks, c->n_all_chunks, c->d_blocks, pp, c->BUF, sc, go, s);
  }
  c->go_armed = false;  // the predicated step ends here
  if (rc) return rc;
  return join_stats(c, s);  // the step ends with everything it launched ordered before the caller's stream
}

// NCCL, resolved at run time: the library already in the process (PyTorch's) or the system one, so
// this library does not link a second NCCL next to the caller's.
namespace {
typedef int (*nccl_allgather_fn)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef const char* (*nccl_errstr_fn)(int);
struct NcclApi {
  nccl_allgather_fn allgather = nullptr;
  nccl_errstr_fn errstr = nullptr;
  std::string error;
};
const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      a.error = std::string("libnccl.so.2 not found: ") + dlerror();
      return a;
    }
    a.allgather = reinterpret_cast<nccl_allgather_fn>(dlsym(h, "ncclAllGather"));
    a.errstr = reinterpret_cast<nccl_errstr_fn>(dlsym(h, "ncclGetErrorString"));
    if (!a.allgather) a.error = "ncclAllGather not exported by libnccl.so.2";
    return a;
  }();
  return api;
}
}  // namespace

int shampoo_allgather(shampoo_ctx* c, void* nccl_comm, void* stream) {
  if (!nccl_comm) {
    set_error("allgather: null communicator");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  const NcclApi& api = nccl_api();
  if (!api.allgather) {
    set_error("allgather: " + api.error);
    return SHAMPOO_ERR_CUDA;
  }
  const int64_t count = c->plan.max_payload;
  if (count == 0) return SHAMPOO_OK;
  const bool f32 = c->buf_f32 || c->f32;
  const size_t es = f32 ? 4 : 8;
  char* buf = static_cast<char*>(c->BUF);
  // in place: this rank's region is already at group_rank * max_payload of the group buffer
  const int r = api.allgather(buf + (size_t)c->grank * count * es, buf, (size_t)count, f32 ? 7 : 8, nccl_comm,
                              static_cast<cudaStream_t>(stream));
  if (r != 0) {
    set_error(std::string("ncclAllGather: ") + (api.errstr ? api.errstr(r) : std::to_string(r)));
    return SHAMPOO_ERR_CUDA;
  }
  return SHAMPOO_OK;
}

int shampoo_timing_enable(shampoo_ctx* c, int32_t enable) {
  c->timer.on = enable != 0;
  return SHAMPOO_OK;
}

int shampoo_timing_get(shampoo_ctx* c, double* ms, int64_t* counts) {
  for (int p = 0; p < SHAMPOO_NUM_PHASES; ++p) {
    for (auto& ev : c->timer.pending[p]) {
      SH_CUDA_CHECK(cudaEventSynchronize(ev.second));
      float e = 0.f;
      SH_CUDA_CHECK(cudaEventElapsedTime(&e, ev.first, ev.second));
      c->timer.ms[p] += e;
      c->timer.count[p] += 1;
      c->timer.pool.push_back(ev.first);
      c->timer.pool.push_back(ev.second);
    }
    c->timer.pending[p].clear();
    if (ms) ms[p] = c->timer.ms[p];
    if (counts) counts[p] = c->timer.count[p];
    c->timer.ms[p] = 0;
    c->timer.count[p] = 0;
  }
  return SHAMPOO_OK;
}

int shampoo_work(shampoo_ctx* c, double* stats_flops, double* precond_flops, double* sum_n3) {
  if (c->f32) {
    *stats_flops = c->eng<float>().stats.flops() + c->eng<float>().stats_thin.flops();
    double f = 0;
    for (int m = 0; m < kMaxOrder; ++m) f += c->eng<float>().prec[m].flops() + c->eng<float>().prec_thin[m].flops();
    *precond_flops = f;
  } else {
    *stats_flops = c->eng<double>().stats.flops() + c->eng<double>().stats_thin.flops();
    double f = 0;
    for (int m = 0; m < kMaxOrder; ++m) f += c->eng<double>().prec[m].flops() + c->eng<double>().prec_thin[m].flops();
    *precond_flops = f;
  }
  // order-1 matvecs: 2 n^2 each
  for (size_t l = 0; l < c->owned.size(); ++l) {
    const BlockPlan& b = c->plan.blocks[c->owned[l]];
    if (b.kind == SHAMPOO_BLOCK_SHAMPOO && b.order == 1) *precond_flops += 2.0 * b.var_count * b.var_count;
  }
  *sum_n3 = 0;
  for (const auto& r : c->rinv) *sum_n3 += r.work_n3();
  return SHAMPOO_OK;
}

int shampoo_work_tc(shampoo_ctx* c, double* stats_int8_ops, double* precond_int8_ops, double* stats_tc_flops,
                    double* precond_tc_flops) {
  double so = 0, po = 0, sf = 0, pf = 0;
  auto acc = [&](auto& e) {
    so = e.stats.int8_ops();
    sf = e.stats.flops();
    for (int m = 0; m < kMaxOrder; ++m) {
      po += e.prec[m].int8_ops();
      pf += e.prec[m].flops();
    }
  };
  if (c->f32) acc(c->eng<float>());
  else acc(c->eng<double>());
  if (stats_int8_ops) *stats_int8_ops = so;
  if (precond_int8_ops) *precond_int8_ops = po;
  if (stats_tc_flops) *stats_tc_flops = sf;
  if (precond_tc_flops) *precond_tc_flops = pf;
  return SHAMPOO_OK;
}

void* shampoo_gather_buffer(shampoo_ctx* c, int64_t* scalars, int32_t* dtype) {
  if (scalars) *scalars = (int64_t)c->plan.group * c->plan.max_payload;
  if (dtype) *dtype = c->buf_f32 ? SHAMPOO_DTYPE_F32 : SHAMPOO_DTYPE_F64;
  return c->BUF;
}

int shampoo_guard_stats_get(shampoo_ctx* c, shampoo_guard_stats* out) {
  out->primary = c->guard[0];
  out->double_retry = c->guard[1];
  out->fallback_previous = c->guard[2];
  out->fallback_identity = c->guard[3];
  return SHAMPOO_OK;
}

int shampoo_guard_stats_set(shampoo_ctx* c, const shampoo_guard_stats* in) {
  c->guard[0] = in->primary;
  c->guard[1] = in->double_retry;
  c->guard[2] = in->fallback_previous;
  c->guard[3] = in->fallback_identity;
  return SHAMPOO_OK;
}

void* shampoo_state_view(shampoo_ctx* c, int32_t block_id, const char* name, int32_t mode, int64_t* numel,
                         int32_t* dtype) {
  if (block_id < 0 || block_id >= (int32_t)c->local_of.size()) return nullptr;
  const int l = c->local_of[block_id];
  if (l < 0) return nullptr;
  const BlockPlan& b = c->plan.blocks[block_id];
  if (dtype) *dtype = c->f32 ? SHAMPOO_DTYPE_F32 : SHAMPOO_DTYPE_F64;
  const std::string n(name);
  char* base = nullptr;
  if (n == "factor" || n == "inv_factor") {
    if (b.kind != SHAMPOO_BLOCK_SHAMPOO || mode < 0 || mode >= b.order) return nullptr;
    int64_t off = c->fac_off[l];
    const auto d = b.dims();
    for (int m = 0; m < mode; ++m) off += d[m] * d[m];
    if (numel) *numel = d[mode] * d[mode];
    if (n == "inv_factor" && c->engine) c->engine->inverses_changed();  // the caller may write through it
    if (n == "factor" && c->fact_lower) {  // exports read full factors (the caller synchronised before)
      if (symmetrize_factors(c, 0) || cudaStreamSynchronize(0) != cudaSuccess) return nullptr;
    }
    base = static_cast<char*>(n == "factor" ? c->FACT : c->INV);
    return base + off * c->esz;
  }
  if (n == "accumulator" && b.kind == SHAMPOO_BLOCK_ADAGRAD) {
    if (numel) *numel = b.var_count;
    return static_cast<char*>(c->FB) + c->fb_off[l] * c->esz;
  }
  if (n == "diag" && b.kind == SHAMPOO_BLOCK_DIAGONAL) {
    const auto d = b.dims();
    if (mode < 0 || mode >= b.order) return nullptr;
    int64_t off = c->fb_off[l];
    for (int m = 0; m < mode; ++m) off += d[m];
    if (numel) *numel = d[mode];
    return static_cast<char*>(c->FB) + off * c->esz;
  }
  void* arr = nullptr;
  if (n == "graft_accumulator") arr = c->GA;
  else if (n == "filtered_grad") arr = c->FILT;
  else if (n == "momentum") arr = c->MOM;
  if (!arr) return nullptr;
  if (numel) *numel = b.var_count;
  return static_cast<char*>(arr) + c->vofs[l] * c->esz;
}

int shampoo_state_scalars_get(shampoo_ctx* c, int32_t block_id, int64_t* step, int64_t* last_inverse_step,
                              int32_t* ready) {
  if (block_id < 0 || block_id >= (int32_t)c->local_of.size() || c->local_of[block_id] < 0) {
    set_error("block not owned by this context");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  const int l = c->local_of[block_id];
  *step = c->step[l];
  *last_inverse_step = c->last_inv[l];
  *ready = c->ready_h[l];
  return SHAMPOO_OK;
}

int shampoo_state_scalars_set(shampoo_ctx* c, int32_t block_id, int64_t step, int64_t last_inverse_step,
                              int32_t ready) {
  if (block_id < 0 || block_id >= (int32_t)c->local_of.size() || c->local_of[block_id] < 0) {
    set_error("block not owned by this context");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  const int l = c->local_of[block_id];
  c->step[l] = step;
  c->last_inv[l] = last_inverse_step;
  c->ready_h[l] = ready;
  SH_CUDA_CHECK(cudaMemcpy(c->d_ready, c->ready_h.data(), c->ready_h.size() * sizeof(int32_t),
                           cudaMemcpyHostToDevice));
  if (c->engine) c->engine->inverses_changed();
  return SHAMPOO_OK;
}

int shampoo_graft_step_get(shampoo_ctx* c, int64_t* step) {
  *step = c->graft_step;
  return SHAMPOO_OK;
}

int shampoo_graft_step_set(shampoo_ctx* c, int64_t step) {
  c->graft_step = step;
  return SHAMPOO_OK;
}

int shampoo_batched_root_inverse(const double* const* mats, double* const* outs, const int32_t* n, int32_t count,
                                 int32_t root_p, double exponent_multiplier, double epsilon, int32_t solver,
                                 double newton_tolerance, int32_t* status, int32_t* iters, void* stream) {
  if (root_p < 1 || !(exponent_multiplier > 0.0) || epsilon < 0.0) {
    set_error("invalid root-inverse request");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  if (solver == SHAMPOO_SOLVER_NEWTON && exponent_multiplier != 1.0) {
    set_error("the coupled Newton solver computes plain p-th root inverses; exponent_multiplier must be 1");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RootInverseBatch rb;
  std::vector<int32_t> nv(n, n + count), pv(count, root_p);
  int rc = rb.setup(nv, pv);
  if (rc) return rc;
  for (int j = 0; j < count; ++j) rb.set_io(j, mats[j], false, outs[j], false);
  int64_t stats[4] = {0, 0, 0, 0};
  std::vector<int32_t> st, it;
  rc = rb.run(1.0, {}, exponent_multiplier, epsilon, solver, newton_tolerance, s, stats, &st, &it);
  if (rc) return rc;
  for (int j = 0; j < count; ++j) {
    if (status) status[j] = st[j];
    if (iters) iters[j] = it[j];
  }
  return SHAMPOO_OK;
}

}  // extern "C"
