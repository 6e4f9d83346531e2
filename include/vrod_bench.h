/*
 * Benchmark / profiling extensions of the product library (not part of the reference API).
 * Used by bench.py to time the device-resident step and to attribute device time to kernel
 * categories for the roofline; exported only by libvrod_b200.so.
 */
#ifndef VROD_BENCH_H
#define VROD_BENCH_H

#include <stdint.h>

#include "vrod_capi.h"

#ifdef __cplusplus
extern "C" {
#endif

enum vrod_kernel_category {
  VROD_CAT_PREDICT = 0,   /* animate + predict + lambda reset */
  VROD_CAT_COLLIDE = 1,   /* pills, hash grid, candidates, narrow phase, compaction, half-planes */
  VROD_CAT_EXT_SETUP = 2, /* slot -> external block incidence */
  VROD_CAT_EXT_SOLVE = 3, /* soft pins / contacts / half-planes, per sweep */
  VROD_CAT_ROD_SWEEP = 4, /* fused elastic stencil + gather + apply, per sweep */
  VROD_CAT_SHAPE = 5,     /* shape matching levels */
  VROD_CAT_REPORT = 6,    /* finalize + residual norms + penetration */
  VROD_CAT_ITERATE = 7,   /* persistent kernel: the whole iteration loop (ext + rod sweeps + shape) */
  VROD_CAT_COUNT = 8
};

/* Replays `steps` steps of the captured graph, each bracketed by CUDA events on the solver's
 * stream; before every step an untimed memset of `flush_bytes` evicts L2. Writes the summed
 * device milliseconds and the kernel launches per step (kernel nodes of the graph). */
int vrod_bench_run(vrod_solver* solver, int32_t steps, int64_t flush_bytes, double* device_ms,
                   int64_t* kernels_per_step);
/* Runs `steps` steps with direct launches and event pairs around each kernel category;
 * ms[VROD_CAT_COUNT] = summed device ms, launches[VROD_CAT_COUNT] = bracket counts. */
int vrod_bench_kernel_times(vrod_solver* solver, int32_t steps, double* ms, int64_t* launches);
/* Debug: phase timestamps (globaltimer ns) of CTA 0 in the last persistent iteration kernel,
 * when the solver was created with VROD_TRACE=1 (else count = 0). */
int vrod_bench_trace(vrod_solver* solver, int32_t capacity, int64_t* out, int32_t* count);
/* Skinning throughput: `iterations` per-frame deformations (pill transforms of the solver's live
 * state + deform_mesh, all on the solver's stream, result left on the device), bracketed by CUDA
 * events. Writes the summed device milliseconds and, if non-NULL, the milliseconds of the deform
 * kernel alone (events around it). */
int vrod_bench_skin_deform(vrod_skin* skin, vrod_solver* solver, int32_t iterations, double* device_ms,
                           double* deform_ms);
/* Contacts and candidates of the last step (capacity diagnostics). */
int vrod_bench_last_counts(vrod_solver* solver, int64_t* max_candidates, int64_t* max_contacts);

#ifdef __cplusplus
}
#endif

#endif /* VROD_BENCH_H */
