// (e) Row-shard helpers of the multi-GPU path.
// Host code: the shard plan is a binary search over rowPtr, the extraction a
// single pass over the shard's nonzeros.
#include "guard.h"
#include <algorithm>
#include <string>

#include "pspmm.h"

namespace pspmm {
void set_error(const std::string &msg);
}

extern "C" pspmm_status pspmm_shard_plan(int64_t n, const int32_t *h_rowptr, int32_t P,
                                         int32_t align, int64_t *bounds) {
  return pspmm::guarded("shard_plan", [&]() -> pspmm_status {
    if (n < 1 || !h_rowptr || P < 1 || align < 1 || !bounds) {
      pspmm::set_error("shard_plan: bad arguments");
      return PSPMM_ERR_INVALID_ARG;
    }
    const int64_t nnz = h_rowptr[n];
    bounds[0] = 0;
    for (int32_t g = 1; g < P; ++g) {
      // target = ceil(g nnz / P); first row r with rowPtr[r] >= target
      const int64_t target = (g * nnz + P - 1) / P;
      const int32_t *it = std::lower_bound(h_rowptr, h_rowptr + n + 1, (int64_t)target,
                                           [](int32_t a, int64_t t) { return (int64_t)a < t; });
      int64_t r = it - h_rowptr;
      r = ((r + align - 1) / align) * align;
      if (r > n) r = n;
      if (r < bounds[g - 1]) r = bounds[g - 1];
      bounds[g] = r;
    }
    bounds[P] = n;
    return PSPMM_OK;
  });
}

extern "C" pspmm_status pspmm_shard_extract(int64_t n, const int32_t *h_rowptr,
                                            const int32_t *h_colidx, const float *h_val,
                                            int32_t P, const int64_t *bounds, int32_t r,
                                            int32_t *h_lrowptr, int32_t *h_lcolidx,
                                            float *h_lval, int64_t *n_max_out) {
  return pspmm::guarded("shard_extract", [&]() -> pspmm_status {
    if (n < 1 || !h_rowptr || P < 1 || !bounds || r < 0 || r >= P || !h_lrowptr) {
      pspmm::set_error("shard_extract: bad arguments");
      return PSPMM_ERR_INVALID_ARG;
    }
    if (bounds[0] != 0 || bounds[P] != n) {
      pspmm::set_error("shard_extract: bounds must start at 0 and end at n");
      return PSPMM_ERR_INVALID_ARG;
    }
    int64_t n_max = 0;
    for (int32_t g = 0; g < P; ++g) {
      if (bounds[g + 1] < bounds[g]) {
        pspmm::set_error("shard_extract: bounds not non-decreasing");
        return PSPMM_ERR_INVALID_ARG;
      }
      n_max = std::max<int64_t>(n_max, bounds[g + 1] - bounds[g]);
    }
    if (n_max * (int64_t)P >= INT32_MAX) {
      pspmm::set_error("shard_extract: gathered B exceeds int32 row indexing");
      return PSPMM_ERR_UNSUPPORTED;
    }
    if (n_max_out) *n_max_out = n_max;
    const int64_t lo = bounds[r], hi = bounds[r + 1];
    const int64_t base = h_rowptr[lo];
    if ((h_rowptr[hi] > base) && (!h_colidx || !h_lcolidx)) {
      pspmm::set_error("shard_extract: null column arrays");
      return PSPMM_ERR_INVALID_ARG;
    }
    for (int64_t i = lo; i <= hi; ++i) h_lrowptr[i - lo] = (int32_t)(h_rowptr[i] - base);
    for (int64_t p = base; p < h_rowptr[hi]; ++p) {
      const int64_t c = h_colidx[p];
      // owner = last g with bounds[g] <= c (skips empty shards)
      const int64_t owner = (std::upper_bound(bounds, bounds + P + 1, c) - bounds) - 1;
      h_lcolidx[p - base] = (int32_t)(owner * n_max + (c - bounds[owner]));
      if (h_lval && h_val) h_lval[p - base] = h_val[p];
    }
    return PSPMM_OK;
  });
}
