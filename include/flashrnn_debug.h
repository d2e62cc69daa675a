/*
 * flashrnn_debug.h -- developer instrumentation for libflashrnn.so (not part of
 * the drop-in boundary).
 *
 * frnn_debug_profile: when a device buffer is registered, the persistent
 *   kernels record clock64() phase stamps for the first `steps` steps of every
 *   CTA: buf[(cta * steps + step) * 8 + phase].  Pass NULL to disable.
 * frnn_debug_timing / frnn_debug_kernel_ms: CUDA-event timing of each kernel
 *   class on its launch stream -- [0] forward recurrence, [1] backward
 *   recurrence, [2] dR/db reduction -- summed in ms with launch counts.
 * frnn_debug_launches: total kernels the library has launched since load.
 */
#ifndef FLASHRNN_DEBUG_H_
#define FLASHRNN_DEBUG_H_
#include <stddef.h>

#include "flashrnn.h"
#ifdef __cplusplus
extern "C" {
#endif
FRNN_API int frnn_debug_profile(void* device_buffer, int32_t steps);
FRNN_API int frnn_debug_timing(int32_t enable);
FRNN_API int frnn_debug_kernel_ms(double* ms3, int64_t* count3);
FRNN_API int frnn_debug_launches(int64_t* count);
/* 1: the cluster-resident kernels run their synchronisation skeleton only (h
 * all-gather / partial exchange, TMEM drains, barriers; no MMAs, no cell math):
 * the per-step floor of the sequential dependency.  Results are
 * meaningless while enabled. */
FRNN_API int frnn_debug_skeleton(int32_t enable);
/* The planner's tiling CSP (algo FRNN_ALGO_FUSED = cluster-resident kernels,
 * FRNN_ALGO_ALTERNATING) for a shape, in the text form of flashrnn_csp.h. */
FRNN_API int frnn_debug_plan_csp(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass,
                                 int32_t algo, char* out, size_t out_bytes);
/* The cluster tiling the planner launches for a pass: out10 = {algo, cluster,
 * UPC, CL, MBT, MS, SSM, KBP, R1, R2} (zeros past `cluster` when not clustered). */
FRNN_API int frnn_debug_cluster_shape(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass,
                                      int32_t* out10);
/* The internal plan of a pass as 16 fields {algo, rows_per_cta, batch_tile,
 * units_per_cta, ctas_per_group, groups, grid, threads, smem_bytes, tmem_cols,
 * k_split, cluster, ka, stages, ffma, workspace_bytes}, and the residual check
 * (frnn_plan_check) of an arbitrary such plan -- tests corrupt a field and
 * expect a violation. */
FRNN_API int frnn_debug_plan_fields(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass,
                                    const frnn_options* opts, int64_t* fields16);
FRNN_API int frnn_debug_plan_residuals(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t pass,
                                       const int64_t* fields16, char* out, size_t out_bytes);
/* The placement half of frnn_dist_gather (flashrnn_dist.h) for a `world`-rank
 * layout, from a caller-filled staging buffer [world][blk] (what ncclAllGather
 * would deliver) into the full tensor k (0 states, 1 gates, 2 dx, 3 ds0, 4 dR,
 * 5 dbias); *blk_out = blk (elements).  NULL stage/full: just report blk. */
FRNN_API int frnn_debug_dist_place(const frnn_cell* cell, frnn_shape shape, int32_t dtype, int32_t world, int32_t k,
                                   const void* stage, void* full, size_t* blk_out, void* stream);
#ifdef __cplusplus
}
#endif
#endif
