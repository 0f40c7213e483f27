// Host-side planner: merge -> block partition -> global enumeration -> greedy
// (LPT) rank assignment -> padded gather-buffer layout.  Integer work only,
// bit-exact with the reference:
//   merge_dims          precond.py:56-77
//   block_partition     precond.py:99-111 (row-major, itertools.product order)
//   method selection    precond.py:114-120, plan_parameter precond.py:138-158
//   enumerate_blocks    dist.py:232-243 (param-major, block-minor ids)
//   greedy_assign       dist.py:133-176 (sort (-count, id); argmin (counter, rank))
//   layout              dist.py:157-164 (rank region = k * max_payload, ascending ids)
// Offsets are in scalars (the reference's byte offsets / 8, dist.py:48-50).
#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>

#include "internal.h"

namespace shampoo {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

static int merge(const int64_t* shape, int32_t ndim, int64_t max_dim, std::vector<int64_t>& out) {
  if (max_dim < 1) {
    set_error("max_dim must be at least 1");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  out.clear();
  int64_t acc = 1;
  for (int32_t i = 0; i < ndim; ++i) {
    const int64_t d = shape[i];
    if (d < 1) {
      set_error("dimensions must be positive");
      return SHAMPOO_ERR_INVALID_ARGUMENT;
    }
    // fold when the running product is trivial, the dim is trivial, or it still fits
    if (acc == 1 || d == 1 || acc * d <= max_dim) {
      acc *= d;
    } else {
      out.push_back(acc);
      acc = d;
    }
  }
  if (acc > 1 || out.empty()) out.push_back(acc);
  return SHAMPOO_OK;
}

}  // namespace shampoo

using namespace shampoo;

extern "C" {

const char* shampoo_last_error(void) { return g_last_error.c_str(); }

int shampoo_merge_dims(const int64_t* shape, int32_t ndim, int64_t max_dim, int64_t* out_shape,
                       int32_t* out_ndim) {
  std::vector<int64_t> m;
  int rc = merge(shape, ndim, max_dim, m);
  if (rc) return rc;
  for (size_t i = 0; i < m.size(); ++i) out_shape[i] = m[i];
  *out_ndim = (int32_t)m.size();
  return SHAMPOO_OK;
}

int shampoo_plan_create(const int64_t* shapes_flat, const int32_t* ndims, int32_t nparams,
                        int64_t max_dim, int32_t large_dim_method, int32_t world_size,
                        int32_t group_size, shampoo_plan** out) {
  *out = nullptr;
  if (world_size < 1 || group_size < 1 || world_size % group_size != 0) {
    set_error("group size " + std::to_string(group_size) + " must divide world size " +
              std::to_string(world_size));
    return SHAMPOO_ERR_INVALID_GROUP;
  }
  if (large_dim_method < 0 || large_dim_method > 2) {
    set_error("unknown large_dim_method");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  auto* plan = new shampoo_plan();
  plan->max_dim = max_dim;
  plan->world = world_size;
  plan->group = group_size;
  const int64_t* cursor = shapes_flat;
  for (int32_t p = 0; p < nparams; ++p) {
    ParamPlan pp;
    pp.shape.assign(cursor, cursor + ndims[p]);
    cursor += ndims[p];
    int rc = merge(pp.shape.data(), ndims[p], max_dim, pp.merged);
    if (rc) {
      delete plan;
      return rc;
    }
    pp.mstride.assign(pp.merged.size(), 1);
    for (int k = (int)pp.merged.size() - 2; k >= 0; --k) pp.mstride[k] = pp.mstride[k + 1] * pp.merged[k + 1];
    pp.numel = 1;
    for (int64_t d : pp.merged) pp.numel *= d;
    bool fits = std::all_of(pp.merged.begin(), pp.merged.end(), [&](int64_t d) { return d <= max_dim; });
    pp.method = fits ? SHAMPOO_METHOD_BLOCKING : large_dim_method;
    if ((int)pp.merged.size() > SHAMPOO_MAX_ORDER) {
      set_error("merged tensor order exceeds SHAMPOO_MAX_ORDER");
      delete plan;
      return SHAMPOO_ERR_UNSUPPORTED;
    }
    // blocks: cartesian product of per-dim cuts, last dim fastest
    const int order = (int)pp.merged.size();
    std::vector<int64_t> ncut(order), idx(order, 0);
    int64_t nblocks = 1;
    for (int k = 0; k < order; ++k) {
      ncut[k] = pp.method == SHAMPOO_METHOD_BLOCKING ? (pp.merged[k] + max_dim - 1) / max_dim : 1;
      nblocks *= ncut[k];
    }
    for (int64_t b = 0; b < nblocks; ++b) {
      BlockPlan bp;
      bp.block_id = (int32_t)plan->blocks.size();
      bp.param = p;
      bp.bindex = (int32_t)b;
      bp.order = order;
      bp.lo.resize(order);
      bp.hi.resize(order);
      bp.var_count = 1;
      bool all_one = true;
      for (int k = 0; k < order; ++k) {
        if (pp.method == SHAMPOO_METHOD_BLOCKING) {
          bp.lo[k] = idx[k] * max_dim;
          bp.hi[k] = std::min(bp.lo[k] + max_dim, pp.merged[k]);
        } else {
          bp.lo[k] = 0;
          bp.hi[k] = pp.merged[k];
        }
        bp.var_count *= bp.hi[k] - bp.lo[k];
        all_one &= (bp.hi[k] - bp.lo[k]) == 1;
      }
      // optim.py:220-255 block kind
      if (all_one) bp.kind = SHAMPOO_BLOCK_GRAFT_ONLY;
      else if (pp.method == SHAMPOO_METHOD_BLOCKING) bp.kind = SHAMPOO_BLOCK_SHAMPOO;
      else if (pp.method == SHAMPOO_METHOD_ADAGRAD) bp.kind = SHAMPOO_BLOCK_ADAGRAD;
      else bp.kind = SHAMPOO_BLOCK_DIAGONAL;
      plan->blocks.push_back(bp);
      for (int k = order - 1; k >= 0; --k) {  // odometer, row-major
        if (++idx[k] < ncut[k]) break;
        idx[k] = 0;
      }
    }
    plan->params.push_back(std::move(pp));
  }
  // greedy LPT over the group (dist.py:150-156)
  const int32_t G = group_size;
  const int32_t nb = (int32_t)plan->blocks.size();
  std::vector<int32_t> order(nb);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    const int64_t ca = plan->blocks[a].var_count, cb = plan->blocks[b].var_count;
    if (ca != cb) return ca > cb;
    return a < b;
  });
  plan->counters.assign(G, 0);
  for (int32_t i : order) {
    int32_t best = 0;
    for (int32_t k = 1; k < G; ++k)
      if (plan->counters[k] < plan->counters[best]) best = k;  // ties -> lowest rank
    plan->blocks[i].owner = best;
    plan->counters[best] += plan->blocks[i].var_count;
  }
  plan->max_payload = nb ? *std::max_element(plan->counters.begin(), plan->counters.end()) : 0;
  for (int32_t k = 0; k < G; ++k) {  // dist.py:159-164
    int64_t at = (int64_t)k * plan->max_payload;
    for (int32_t i = 0; i < nb; ++i) {
      if (plan->blocks[i].owner != k) continue;
      plan->blocks[i].gather_offset = at;
      at += plan->blocks[i].var_count;
    }
  }
  *out = plan;
  return SHAMPOO_OK;
}

void shampoo_plan_destroy(shampoo_plan* plan) { delete plan; }
int32_t shampoo_plan_num_blocks(const shampoo_plan* plan) { return (int32_t)plan->blocks.size(); }
int32_t shampoo_plan_num_params(const shampoo_plan* plan) { return (int32_t)plan->params.size(); }
int64_t shampoo_plan_max_payload(const shampoo_plan* plan) { return plan->max_payload; }
int32_t shampoo_plan_group_size(const shampoo_plan* plan) { return plan->group; }
int32_t shampoo_plan_world_size(const shampoo_plan* plan) { return plan->world; }

int shampoo_plan_block(const shampoo_plan* plan, int32_t id, shampoo_block_info* out) {
  if (id < 0 || id >= (int32_t)plan->blocks.size()) {
    set_error("block id out of range");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  const BlockPlan& b = plan->blocks[id];
  std::memset(out, 0, sizeof(*out));
  out->block_id = b.block_id;
  out->param_index = b.param;
  out->block_index = b.bindex;
  out->order = b.order;
  out->owner_rank = b.owner;
  out->kind = b.kind;
  out->var_count = b.var_count;
  out->gather_offset = b.gather_offset;
  for (int k = 0; k < b.order; ++k) {
    out->lo[k] = b.lo[k];
    out->hi[k] = b.hi[k];
  }
  return SHAMPOO_OK;
}

int shampoo_plan_param(const shampoo_plan* plan, int32_t p, int64_t* merged, int32_t* ndim,
                       int32_t* method) {
  if (p < 0 || p >= (int32_t)plan->params.size()) {
    set_error("param index out of range");
    return SHAMPOO_ERR_INVALID_ARGUMENT;
  }
  const ParamPlan& pp = plan->params[p];
  for (size_t k = 0; k < pp.merged.size(); ++k) merged[k] = pp.merged[k];
  *ndim = (int32_t)pp.merged.size();
  *method = pp.method;
  return SHAMPOO_OK;
}

int shampoo_plan_counters(const shampoo_plan* plan, int64_t* out) {
  for (size_t k = 0; k < plan->counters.size(); ++k) out[k] = plan->counters[k];
  return SHAMPOO_OK;
}

}  // extern "C"
