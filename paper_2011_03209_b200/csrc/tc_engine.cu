// tc_engine.cu — tcgen05 candidate engine (placeholder until implemented).
#include <vector>

#include "dbscan.cuh"

namespace bm {

bool tc_supported(int64_t d) { (void)d; return false; }

int tc_build_adjacency(const double*, int64_t, const ElemTables&, int64_t, int64_t, double,
                       uint32_t*, const uint8_t*, const std::vector<int32_t>&, int64_t*,
                       cudaStream_t) {
  set_error("tensor-core engine not built");
  return BM_ERR_INTERNAL;
}

}  // namespace bm
