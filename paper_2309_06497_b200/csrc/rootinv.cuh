// Batched guarded root inverse X = A^(-eta/p) of symmetric PSD matrices.
//
// Follows matfun.py:139-157 (eigh path: shift-clamp w - min(w_min,0) + eps,
// X = Q diag(w^(-eta/p)) Q^T) and matfun.py:164-222 (coupled Newton), wrapped
// in the retry guard of matfun.py:240-293.  All arithmetic is FP64 (the
// reference default precision): the eigen path is a parallel two-sided block
// Jacobi solver; the Newton path uses the grouped DGEMM.
#pragma once

#include <memory>
#include <vector>

#include "gemm.cuh"
#include "tcgen05.cuh"

namespace shampoo {

enum EigStatus : int32_t {
  kEigOk = 0,
  kEigNonFiniteInput = 1,
  kEigNoConvergence = 2,
  kEigEpsZeroSingular = 3,
  kEigNonFiniteResult = 4,
  kEigSkipped = 5,  // solved elsewhere (low-rank path): untouched by this batch
};

// One matrix of a batch.
struct RootJob {
  int32_t n;         // true size
  int32_t np;        // padded size (n<=64: n rounded to even; else multiple of 64)
  int32_t m;         // 32-row blocks (np/32) for big jobs, 0 for small
  int32_t root_p;
  int64_t ws_off;    // A workspace offset (np*np)
  int64_t v_off;     // V workspace offset (np*np)
  int64_t u_off;     // pair-slot offset (big jobs)
  int64_t w_off;     // vector workspace offset (np)
  int64_t x_off;     // n x n offset: scaled input A0, later the result X
  const void* in;    // n x n input (row-major)
  void* out;         // n x n output (row-major)
  int32_t in_f32, out_f32;
  int32_t has_prev;  // output already holds a previous inverse
  int32_t warm;      // start Jacobi from the eigenvectors kept in V (previous refresh)
  double in_scale;   // multiply input by this (1/bias-correction)
  double idscale;    // identity-fallback scale eps^(-eta/p) (or 1)
};

// Mutable per-job solver state (device).
struct RootState {
  int32_t active, round, sweep, rotated;
  int32_t status, result;  // result: 0 primary, 2 previous, 3 identity
  double norm2;            // ||A||_F^2
  double tol_abs;
  double tol_null;
  double trace;            // tr(A)
  int32_t nonfinite, capped;  // capped: sweep cap reached (result still used)
  int32_t via_newton;         // eigh job solved by the coupled-Newton pre-pass (no eigenvectors kept)
};

// Coupled-Newton job; per job scratch at nx + off: X0, X1, M0, M1, T, Pa, Pb, Xbest (8 n^2).
struct NewtonJob {
  int32_t n, p;
  int64_t off;
  double best;
  int32_t iters, converged;
  int32_t cap;  // hybrid pre-pass: iteration cap (conditioning gate, kHybridNewtonKappa)
  int32_t fin;  // hybrid pre-pass: residual small enough that one more X <- X T is final
  int32_t tpack;  // T = ((p+1) I - M) / p is packed straight from M (affine pack, fixed exponent): no FP64 T
  int32_t pad_;
  double lam;   // hybrid pre-pass: power-iteration estimate of lambda_max(A) (scales X0, M0)
  double scale; // hybrid pre-pass: spectrum scaling applied at the start of the next iteration
  double vit;   // hybrid pre-pass: iterations counted for the conditioning gate (scaled ones count more)
  double ub;    // hybrid pre-pass: guaranteed upper bound on lambda_max(A + eps I) (k_newton_ub)
};

class RootInverseBatch {
 public:
  RootInverseBatch() = default;
  RootInverseBatch(const RootInverseBatch&) = delete;
  RootInverseBatch& operator=(const RootInverseBatch&) = delete;
  ~RootInverseBatch();
  // sizes/root_p per job; allocates workspaces; jobs' in/out filled by set_io.
  int setup(const std::vector<int32_t>& n, const std::vector<int32_t>& root_p);
  void set_io(int j, const void* in, bool in_f32, void* out, bool out_f32);
  // Run on all jobs. scale: input multiplier; has_prev per job (host).
  // eigh with eta = 1: jobs with n > 64 (and newton_hint[j] != 0 if given: the factor can be full
  // rank) first try the coupled-Newton iteration to an FP64-level residual within a fixed budget --
  // the same matrix function (lambda + eps)^(-1/p) when lambda_min >= 0 -- and only the
  // non-converged ones run the Jacobi rounds.
  // stats[4] accumulates GuardStats branches; host_status receives per-job status.
  // allow_warm: start from eigenvectors of the previous successful run of the same job.
  int run(double in_scale, const std::vector<int32_t>& has_prev, double eta, double eps,
          int32_t solver, double newton_tol, cudaStream_t s, int64_t* stats,
          std::vector<int32_t>* host_status, std::vector<int32_t>* host_iters, bool allow_warm = false,
          const std::vector<int32_t>* newton_hint = nullptr, const std::vector<int32_t>* skip = nullptr);
  int64_t sweeps_total() const { return sweeps_total_; }
  size_t jobs() const { return host_.size(); }
  int32_t job_n(int j) const { return host_[j].n; }
  int32_t job_p(int j) const { return host_[j].root_p; }
  const void* job_in(int j) const { return host_[j].in; }
  void* job_out(int j) const { return host_[j].out; }
  double work_n3() const;  // sum n^3

 private:
  int run_eigh(double eta, double eps, cudaStream_t s, std::vector<int32_t>* iters);
  int run_newton(double eps, double tol, cudaStream_t s, std::vector<int32_t>* iters);
  int build_newton();
  int newton_phase(double eps, double tol, int budget, const int32_t* cand, bool hybrid, cudaStream_t s);
  int prepare_warm(cudaStream_t s);
  int build_warm_gemms();
  std::vector<RootJob> host_;
  RootJob* d_jobs_ = nullptr;
  RootState* d_state_ = nullptr;
  double* ws_ = nullptr;   // A workspaces
  double* vs_ = nullptr;   // V workspaces
  double* us_ = nullptr;   // pair slots
  double* wv_ = nullptr;   // vectors
  double* nx_ = nullptr;   // Newton scratch (8 x n^2 per job)
  double* xs_ = nullptr;   // n x n per job: scaled input A0, then X
  double* ts_ = nullptr;   // np x np per job: warm-start temporary
  int32_t* d_warm_ = nullptr;
  std::vector<int32_t> vec_valid_;  // V holds eigenvectors of the last successful solve
  int64_t x_elems_ = 0, sweeps_total_ = 0;
  OzakiGemmBatch<double> rr_, warm1_, warm2_;  // big n^3 GEMMs on tcgen05 (Ozaki, FP64-class)
  bool cross_only_ = true;  // SHAMPOO_EIG_CROSS=0: full inner sweeps in every outer round
  int32_t* d_pair_begin_ = nullptr;
  int32_t* d_item_begin_ = nullptr;
  int32_t* d_elem_begin_ = nullptr;
  int32_t* d_col_begin_ = nullptr;
  int32_t* d_count_ = nullptr;
  int32_t h_count_[4] = {0, 0, 0, 0};  // pageable: the D2H read is a sync point anyway (no pinned
                                       // alloc per batch: cudaMallocHost/cudaFreeHost stall the device)
  int64_t* d_stats_ = nullptr;
  int32_t total_pairs_ = 0, total_items_ = 0, total_elem_chunks_ = 0, total_col_chunks_ = 0;
  int64_t ws_elems_ = 0, u_elems_ = 0, w_elems_ = 0, n2_elems_ = 0;
  std::vector<int64_t> n2_off_;
  bool has_big_ = false;
  // coupled Newton (solver NEWTON, and the eigh pre-pass for well-conditioned factors): persistent
  // tcgen05 Ozaki GEMM sets X_nxt = X T, T^p (binary powering), M_nxt = T^p M
  NewtonJob* d_newton_ = nullptr;
  unsigned long long* d_resbits_ = nullptr;  // per job max row sum of |M - I| (bit pattern)
  int32_t* d_improved_ = nullptr;
  int32_t* d_mask2_ = nullptr;
  double* d_part_ = nullptr;    // per element-chunk partial sums (lambda_max bound)  // Newton: jobs that still need T^p and M (not in their final step)
  int8_t* pack_arena_ = nullptr;  // one pack space for all of this batch's Ozaki GEMM sets (sequential)
  int64_t pack_cap_ = 0;
  bool newton_built_ = false;
  OzakiGemmBatch<double> newton_x_[2], newton_m_[2];
  OzakiGemmBatch<double> newton_sq_;  // (A + eps I)^2 for the guaranteed lambda_max bound (hybrid pre-pass)
  std::vector<std::unique_ptr<OzakiGemmBatch<double>>> newton_pow_;
  int32_t* d_cand_ = nullptr;  // eigh jobs tried with the Newton pre-pass
  bool hybrid_ = true;          // SHAMPOO_EIG_NEWTON=0 disables the pre-pass
  bool ub_on_ = true;           // SHAMPOO_NEWTON_UB=0 (diagnostics): no guaranteed lambda_max bound
  bool scale_on_ = true;        // SHAMPOO_NEWTON_SCALE=0 disables the scaled pre-pass steps (read at setup)
  // reconstruction X = Y Y^T for all jobs (into xs_)
  OzakiGemmBatch<double> recon_;
  bool recon_ready_ = false;
};

}  // namespace shampoo
