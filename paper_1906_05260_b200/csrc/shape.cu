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

__global__ void k_shape_level(World w, Groups g, double* __restrict__ X, int gbeg, int gend, int pdl, double* fits) {
  if (pdl) {
    pdl_wait();
    pdl_trigger();
  }
  __shared__ double scratch[kWarpsPerBlock][kShapeScratch];  // exact path's ordered sums
  const int gi = gbeg + (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (gi >= gend) return;
  const int grp = g.level_groups[gi];
  shape_group(w, g, X, w.xrec, grp, threadIdx.x & 31, nullptr, nullptr, fits ? fits + 14ll * grp : nullptr,
              g.exact ? scratch[threadIdx.x >> 5] : nullptr);
}

// Standalone extract_rotation (bundling.h:42-43): one thread per problem.
__global__ void k_extract_rotation(long long n, const double* __restrict__ B, const double* __restrict__ guess,
                                   int max_iterations, double tol2, double* __restrict__ out) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    vm::M3 m;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) m.m[a][b] = B[9 * i + 3 * a + b];
    const double* gq = guess + 4 * i;
    const vm::Q4 q = extract_rotation(m, vm::Q4{gq[0], gq[1], gq[2], gq[3]}, nullptr, max_iterations, tol2);
    out[4 * i] = q.w;
    out[4 * i + 1] = q.x;
    out[4 * i + 2] = q.y;
    out[4 * i + 3] = q.z;
  }
}

}  // namespace

void launch_extract_rotation(long long n, const double* B, const double* guess, int max_iterations, double tolerance,
                             double* out, cudaStream_t st) {
  if (n <= 0) return;
  const long long b = (n + 127) / 128;
  k_extract_rotation<<<static_cast<unsigned>(b > 148 * 32 ? 148 * 32 : b), 128, 0, st>>>(n, B, guess, max_iterations,
                                                                                        tolerance * tolerance, out);
}

void launch_shape_match(const World& w, const Groups& g, double* X, const int* level_off_host, bool pdl, cudaStream_t st,
                        double* fits) {
  for (int l = 0; l < g.levels; ++l) {
    const int gb = level_off_host[l], ge = level_off_host[l + 1];
    const int ng = ge - gb;
    if (ng <= 0) continue;
    const int blocks = (ng + kWarpsPerBlock - 1) / kWarpsPerBlock;
    launch_kernel(k_shape_level, blocks, 32 * kWarpsPerBlock, 0, st, pdl, w, g, X, gb, ge, pdl ? 1 : 0, fits);
  }
}

}  // namespace vdev
