// Internal declarations shared by the host-side translation units.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/shampoo_b200.h"

namespace shampoo {

void set_error(const std::string& msg);

struct ParamPlan {
  std::vector<int64_t> shape;    // original shape
  std::vector<int64_t> merged;   // merge_dims result
  std::vector<int64_t> mstride;  // row-major strides of `merged` (elements)
  int32_t method = SHAMPOO_METHOD_BLOCKING;
  int64_t numel = 1;
};

struct BlockPlan {
  int32_t block_id = 0, param = 0, bindex = 0, order = 0, owner = 0, kind = 0;
  int64_t var_count = 0;
  int64_t gather_offset = 0;  // scalars, absolute (rank region base included)
  std::vector<int64_t> lo, hi;
  std::vector<int64_t> dims() const {
    std::vector<int64_t> d(lo.size());
    for (size_t k = 0; k < lo.size(); ++k) d[k] = hi[k] - lo[k];
    return d;
  }
};

}  // namespace shampoo

struct shampoo_plan {
  int64_t max_dim = 0;
  int32_t world = 1, group = 1;
  std::vector<shampoo::ParamPlan> params;
  std::vector<shampoo::BlockPlan> blocks;
  std::vector<int64_t> counters;  // per group rank
  int64_t max_payload = 0;        // scalars
};
