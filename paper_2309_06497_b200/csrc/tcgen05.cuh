// Grouped GEMM on the 5th-generation tensor cores (sm_100a tcgen05.mma kind::i8) with
// exact integer accumulation: Ozaki-style operand splitting.
//
// Why integers: Shampoo's factors feed an inverse 4th/6th root whose small
// eigenvalues amplify any bias in the statistics.  fp32 tensor-core accumulation
// (3xTF32 / bf16x3) rounds toward zero at every MMA step; over K = 4096 that is a
// coherent ~3e-5 relative bias -- measured here: 4e-5 factor error and 1.4e-2
// direction error against the reference at eps = 1e-6 on ResNet-50 blocks.
// int8 x int8 products summed in int32 are exact, so the only error left is the
// operand truncation, which is controlled by the number of slices.
//
// Scheme (per operand row r, e_r = frexp exponent of max_k |x_rk|):
//   x_rk = 2^e_r * sum_{s=0}^{S-1} q_rks 2^(-7(s+1)) + O(2^(e_r - 7S)),  q in [-127, 127]
//   C_ij = 2^(e_i + f_j) * sum_{d=0}^{S-1} 2^(-7(d+2)) * acc_d[i][j],
//   acc_d = sum over slice pairs (s, t), s + t = d, of the exact int32 dot products.
// Pairs with s + t >= S are dropped (below the truncation error).  Slice counts: 6 for the plain
// steps of precision "double" (statistics and mode products, 2^-42 of the row maximum), 8 for the
// root-inverse iterates (FP64 class: the Newton errors scale with 2^-7S), 5 for "single" (2^-35).
// Used for the factor statistics (precond.py:161-165, 232-242), the mode products
// (precond.py:168-174) and the root-inverse GEMMs (matfun.py:164-222).
//
// Pipeline per launch (one launch set covers every block of a phase):
//   k_oz_rowexp     per-row exponents (atomicMax of frexp exponents);
//   k_oz_pack       operands -> int8 slice planes in the canonical no-swizzle K-major UMMA layout,
//                   [stage][slice][8-row core][2 K cores][8 rows][16 B] (branch-free integer slicing,
//                   16-byte operand loads); k_oz_pack_rows fuses both passes for row-contiguous sets
//                   and applies affine operand maps (Newton's T = ((p+1) I - M) / p, fixed exponent);
//                   problems of one launch that read the same operand share one pack;
//   k_oz_gemm_p     persistent, one CTA per SM over (problem, 128x64 tile, K split) items: warp 0
//                   issues TMA (cp.async.bulk.tensor) boxes into a 3-5 stage mbarrier ring, warp 1
//                   owns TMEM and issues tcgen05.mma (one elected thread): A slice sa against the B
//                   slices 0..S-1-sa stacked along N (<= 4 per instruction), so output block sb lands
//                   in the TMEM accumulator of diagonal d = sa + sb; warps 2-9 drain TMEM with
//                   tcgen05.ld, combine the diagonals in FP64 and store through a shared-memory tile
//                   (coalesced; alpha, beta*C, SYRK mirror or lower triangle only, split-K partials).
//                   Accumulators double-buffered when 2 x S x 64 columns fit TMEM (S <= 4);
//   k_oz_reduce     split-K partials summed in FP64 in a fixed order (deterministic).
#pragma once

#include <vector>

#include "gemm.cuh"

namespace shampoo {

struct OzProb {
  int32_t mt, nt;       // 128-row tiles along M, 64-row tiles along N
  int32_t ks;           // 32-wide K stages
  int32_t ksplit;       // K splits (exact int32 accumulation bound)
  int32_t kst;          // stages per split
  int32_t pad;
  int64_t tiles;        // output tiles (SYM: tiles on or below the diagonal)
  int64_t a_pack, b_pack;   // byte offsets of the packed operands
  int32_t a_rc, b_rc;       // 8-row cores per stage and slice of each operand (rows padded to 8)
  int64_t a_exp, b_exp;     // row-exponent offsets (int32 units)
  int64_t ws_off;           // split-K partials (doubles)
};

struct OzPackJob {
  const void* src;
  Idx2 r, k;
  int32_t rows, K;
  int32_t ks, rc;        // stages, 8-row cores (padded rows / 8)
  int32_t mask_index;    // -1: unmasked
  int32_t pad;
  int64_t dst;           // byte offset of the packed planes
  int64_t exp;           // row-exponent offset
  int64_t units;         // pack threads: rc * 8 * ks * 2 (row, stage, K core)
  int64_t echunks;       // rowexp threads (contiguous rows: 32 per 2048-wide chunk; else 1 per 64)
  double xa, xb;         // packed value = xa * src + xb * (row == k); identity: 1, 0
  int32_t fexp;          // kNoFixedExp, or the fixed row exponent (no row-maximum pass)
  int32_t pad2;
};
constexpr int32_t kNoFixedExp = 0x7fffffff;

// A source matrix X (R x C, row stride ld, unit column stride) that is an operand both by rows
// (k along a row: job a) and by columns (k down a column: job b) -- an order-2 block's two
// statistics, or a mode-0 statistic and the first mode product's B operand.  Packed by one
// exponent pass and one tile-transposing pack pass instead of two of each.
struct OzDualJob {
  const void* src;
  int64_t ld;
  int32_t R, C;
  int32_t mask_a, mask_b;  // -1: unmasked; the pair runs if either is on
  int32_t rc_a, rc_b;      // 8-row cores of the row (a) and column (b) operands
  int32_t ks_b, pad;       // stages of b (a's stage never exceeds its ks)
  int64_t dst_a, dst_b;    // byte offsets of the two plane sets
  int64_t exp_a, exp_b;    // exponent offsets (R rows, C columns)
};

// Step-phase tag of the calling host thread for the GEMM kernel timer / counters (returns the
// previous tag; out-of-range = untagged).
int oz_set_tag(int tag);

template <typename T>
class OzakiGemmBatch {
 public:
  // slices per operand: 8 for double (FP64 class), 5 for single; set_slices() before upload() trades
  // accuracy (operand truncation 2^-7S of the row maximum) for S(S+1)/2 int8 products per MAC
  static constexpr int kDefaultSlices = sizeof(T) == 8 ? 8 : 5;
  static constexpr int kMaxSlices = 8;
  std::vector<GemmProblem> host;
  int set_slices(int s);     // 3..8 (supported: 3, 4, 5, 6, 8); SHAMPOO_ERR_INVALID_ARGUMENT otherwise
  int slices() const { return S_; }
  OzakiGemmBatch() = default;
  OzakiGemmBatch(const OzakiGemmBatch&) = delete;
  OzakiGemmBatch& operator=(const OzakiGemmBatch&) = delete;
  ~OzakiGemmBatch();
  void add(const GemmProblem& p) { host.push_back(p); }
  bool empty() const { return host.empty(); }
  int upload();
  int launch(cudaStream_t s, const int32_t* mask = nullptr) const;
  // operands flagged kGemmConstA/B (inverse factors: they change once per refresh) are packed
  // on the first launch after upload() or invalidate_cached() only
  void invalidate_cached() { cached_valid_ = false; }
  // Pack space shared with other batches that are only ever launched one after another on one
  // stream (no cached operands): used by upload() when large enough, never freed here.
  void set_external_arena(int8_t* p, int64_t cap) {
    ext_arena_ = p;
    ext_cap_ = cap;
  }
  // before upload(): problems that read the same operand (source, geometry) share one pack; the
  // first such problem's mask decides whether the pack runs
  void set_share_packs(bool on) { share_packs_ = on; }
  double flops() const;      // algorithmic 2*M*N*K (SYM counted as full)
  double int8_ops() const;   // executed tensor-core int8 ops

 private:
  struct PackSet {           // operands packed together (row exponents + slice planes)
    OzPackJob* d_jobs = nullptr;
    int64_t* d_pbegin = nullptr;   // pack CTA prefix per job
    int64_t* d_ebegin = nullptr;   // rowexp CTA prefix per job
    int64_t* d_cbegin = nullptr;   // fused pack CTA prefix per job (PACK_CORES cores per CTA)
    int64_t exp_begin = 0, exp_elems = 0, pack_ctas = 0, exp_ctas = 0, core_ctas = 0;
    bool all_contig = true, fused_ok = false;  // fused single-pass pack: contiguous rows, >= 2 CTAs per SM
    bool has_xform = false;                    // affine operands: always the fused kernel's transform variant
    int njobs = 0;
    OzDualJob* d_dual = nullptr;   // transposed operand pairs (k_oz_dual_exp + k_oz_pack_dual)
    int64_t* d_dxbegin = nullptr;  // exponent-tile CTA prefix per pair
    int64_t* d_dpbegin = nullptr;  // pack-tile CTA prefix per pair
    int64_t dual_exp_ctas = 0, dual_pack_ctas = 0;
    int ndual = 0;
  };
  int launch_pack(const PackSet& ps, cudaStream_t s, const int32_t* mask) const;
  GemmProblem* d_prob_ = nullptr;
  OzProb* d_tp_ = nullptr;
  int64_t* d_begin_ = nullptr;     // item prefix per problem
  PackSet sets_[2];                // [0] every launch, [1] cached (const) operands
  mutable bool cached_valid_ = false;
  int64_t* d_rbegin_ = nullptr;    // reduce tile prefix
  int32_t* d_rprob_ = nullptr;
  int8_t* arena_ = nullptr;        // packed slice planes
  bool own_arena_ = true;
  int8_t* ext_arena_ = nullptr;
  int64_t ext_cap_ = 0;
  int32_t* exps_ = nullptr;        // row exponents
  double* ws_ = nullptr;           // split-K partial tiles
  void* d_tmaps_ = nullptr;        // per problem 3 TMA tensor maps (A first/second slice half, B)
  int64_t total_items_ = 0, total_red_ = 0;
  int nred_ = 0;
  double mma_count_ = 0;
  int S_ = kDefaultSlices;
  bool share_packs_ = false;
};

}  // namespace shampoo
