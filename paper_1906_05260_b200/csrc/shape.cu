// Bundle shape matching (apply_shape_match / fit_similarity / extract_rotation,
// bundling.cpp:50-133), applied after every shape_match_period-th sweep (solver.cpp:336-338).
//
// One warp per group (shape.cuh). The reference applies groups sequentially; groups are
// disjoint in vertices but may share a frame (vertices m-1 and m map to element m-1), so the
// host schedules groups into dependency levels (host_model.cpp) and each level is one launch:
// within a level no two groups touch the same frame, across levels the reference's order is kept.
#include "shape.cuh"

namespace vdev {

namespace {

constexpr int kWarpsPerBlock = 4;

__global__ void k_shape_level(World w, Groups g, double* __restrict__ X, int gbeg, int gend, int pdl) {
  if (pdl) {
    pdl_wait();
    pdl_trigger();
  }
  const int gi = gbeg + (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (gi >= gend) return;
  shape_group(w, g, X, w.xrec, g.level_groups[gi], threadIdx.x & 31);
}

}  // namespace

void launch_shape_match(const World& w, const Groups& g, double* X, const int* level_off_host, bool pdl, cudaStream_t st) {
  for (int l = 0; l < g.levels; ++l) {
    const int gb = level_off_host[l], ge = level_off_host[l + 1];
    const int ng = ge - gb;
    if (ng <= 0) continue;
    const int blocks = (ng + kWarpsPerBlock - 1) / kWarpsPerBlock;
    launch_kernel(k_shape_level, blocks, 32 * kWarpsPerBlock, 0, st, pdl, w, g, X, gb, ge, pdl ? 1 : 0);
  }
}

}  // namespace vdev
