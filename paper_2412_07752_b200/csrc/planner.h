// planner.h -- B200 tiling solver interface (ConstrINT-style integer CSP; see
// planner.cpp and DESIGN.md section 5).
#pragma once
#include <string>
#include <vector>

#include "kernels.h"

namespace frnn {

// Hardware limits the constraints are built from (queried from the device,
// B200 defaults when none is present).
struct DeviceLimits {
  int sm_count = 148;
  int smem_optin = 232448;        // max dynamic shared memory per CTA (bytes)
  int regs_per_sm = 65536;        // 32-bit registers
  int tmem_cols = 512;            // TMEM columns (x 128 lanes x 32 bit) per SM
  int max_threads = 1024;
  int cluster_max = 16;            // non-portable thread-block cluster size
  int umma_m = 128;               // tcgen05 kind::f16 M with cta_group::1
  int umma_k = 16;                // tcgen05 kind::f16 K per instruction
};
const DeviceLimits& device_limits();

// Fills *out for the pass (0 fwd, 1 bwd).  algo_request is an frnn_algo.
// Returns an frnn_status; *why explains infeasibility.
int solve_plan(const Problem& p, int pass, int algo_request, const DeviceLimits& lim, Plan* out,
               std::string* why);

// The tiling CSP of a kernel family (FRNN_ALGO_FUSED: cluster-resident kernels,
// FRNN_ALGO_ALTERNATING) in the text form of include/flashrnn_csp.h.
// Workspace bytes the kernels of `pl` carve up for problem `p` (recomputed from
// the plan's fields, so a persisted plan never carries a stale size).
size_t plan_workspace(const Problem& p, int pass, const Plan& pl);

std::string plan_csp_text(const Problem& p, int pass, int algo, const DeviceLimits& lim);

// Re-check of a solved plan against every constraint its kernel family relies
// on (the counterpart of rnnkit::plan::plan_residuals, planner.cpp:349-402):
// human-readable violations, empty when every residual is zero.  The derived
// geometry (shared memory, TMEM columns, threads, grid, workspace) is
// recomputed from the plan's choices and must equal the plan's values.
std::vector<std::string> plan_residuals(const Problem& p, int pass, const Plan& pl, const DeviceLimits& lim);

// Bytes moved per time step by a plan (the counterpart of hbm_traffic_per_step,
// planner.cpp:233-243), by where they travel:
//   io: the compulsory per-step HBM traffic of the trace and the inputs /
//       gradients (x or the trace in, gates / states or dx out, the fp32
//       carries of the alternating path);
//   exchange: the per-step all-gather of h (forward) or the partial sums of
//       R^T dg (backward) between CTAs -- through DSMEM / multicast inside a
//       cluster, through L2 between clusters or CTAs of the L2-flag kernels;
//   r_stream: R (R^T) re-read every step from L2 by the alternating path (0
//       when R is resident on chip).
struct PlanTraffic {
  double io, exchange_onchip, exchange_l2, r_stream;
};
PlanTraffic plan_traffic(const Problem& p, int pass, const Plan& pl);

}  // namespace frnn
