// GPU implementations of the fine-grained collision entry points of include/vrod_capi.h.
#pragma once

#include <cstdint>

#include "../../include/vrod_capi.h"

namespace vhost {

void gpu_pill_project(long long n, const double* x, const vrod_pill* pills, double* t, double* d, uint8_t* deg);
void gpu_deepest(long long n, const vrod_pill* a, const vrod_pill* b, int iters, const double* warm, double* alpha,
                 double* beta, double* dist);
long long gpu_broad_phase(long long n, const vrod_pill* pills, long long cap, int32_t* pairs);
long long gpu_find_contacts(long long n, const vrod_pill* pills, long long npairs, const int32_t* pairs, int iters,
                            long long nwarm, const uint64_t* wkeys, const double* walpha, long long cap, int32_t* pa,
                            int32_t* pb, double* alpha, double* beta, double* dist);

// extract_rotation (bundling.h:42-43) on the GPU: n problems, covariance row-major 9 each.
void gpu_extract_rotation(long long n, const double* B, const double* guess, int max_iterations, double tolerance,
                          double* out);

}  // namespace vhost
