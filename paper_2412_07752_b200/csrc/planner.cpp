// planner.cpp -- tiling solver for the B200 kernels.
//
// First version: explicit enumeration over the (small) candidate domains with
// the same constraints the CSP formulation uses (TMEM columns, SMEM bytes,
// co-residency, tcgen05 shape rules).  Replaced by the propagating CSP solver
// in csp.cpp.
#include "planner.h"

#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "../../include/flashrnn.h"

namespace frnn {

const DeviceLimits& device_limits() {
  static DeviceLimits lim;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaDeviceProp prop{};
    if (cudaGetDevice(&dev) == cudaSuccess && cudaGetDeviceProperties(&prop, dev) == cudaSuccess) {
      lim.sm_count = prop.multiProcessorCount;
      lim.smem_optin = (int)prop.sharedMemPerBlockOptin;
      lim.regs_per_sm = prop.regsPerMultiprocessor;
      lim.max_threads = prop.maxThreadsPerBlock;
    } else {
      cudaGetLastError();
    }
  });
  return lim;
}

static int ngp_of(int NG) { return NG <= 1 ? 1 : NG <= 2 ? 2 : 4; }

static bool plan_fused(const Problem& p, int pass, const DeviceLimits& lim, Plan* out, std::string* why) {
  const int NGP = ngp_of(p.NG);
  const int N = 16;
  if (p.DH % 8) {
    *why = "fused: head_dim must be a multiple of 8 (16-byte h chunks)";
    return false;
  }
  const int K = (int)align_up(p.DH, 32);
  const int NBT = (p.B + N - 1) / N;
  if ((int)fused_tmem_cols(p, N, pass == 1) > lim.tmem_cols) {
    *why = pass == 0 ? "fused forward: R slice + accumulators exceed TMEM"
                     : "fused backward: R^T slice + accumulators exceed TMEM";
    return false;
  }
  const size_t smem = pass == 0 ? (size_t)N * K * 2 + 128 * (N + 1) * 4 + 16 : (size_t)N * 128 * 2 + 16;
  if ((int)smem > lim.smem_optin) {
    *why = "fused: shared memory";
    return false;
  }
  // Largest units-per-CTA that divides DH (fewest CTAs to synchronise).
  int best = 0;
  for (int upc = 128 / NGP; upc >= 1; --upc)
    if (p.DH % upc == 0) {
      best = upc;
      break;
    }
  const int CPG = p.DH / best;
  const int grid = p.NH * NBT * CPG;
  if (grid > lim.sm_count) {
    *why = "fused: grid of " + std::to_string(grid) + " CTAs exceeds co-residency";
    return false;
  }
  Plan& pl = *out;
  pl = Plan{};
  pl.algo = FRNN_ALGO_FUSED;
  pl.rows_per_cta = best * NGP;
  pl.batch_tile = N;
  pl.units_per_cta = best;
  pl.ctas_per_group = CPG;
  pl.groups = p.NH * NBT;
  pl.grid = grid;
  pl.threads = 128;
  pl.smem_bytes = (int)smem;
  pl.tmem_cols = (int)fused_tmem_cols(p, N, pass == 1);
  pl.k_split = 1;
  pl.ws_bytes = pass == 0 ? fused_forward_ws(p, pl) : fused_backward_ws(p, pl);
  return true;
}

// Cluster-resident fused kernels (fused_cluster.cu): largest units-per-CTA
// (fewest CTAs in the cluster) whose slice fits TMEM (<=128 rows) + one M=64
// SMEM block, with cluster size <= 16 and SMEM/TMEM within the device limits.
static bool plan_cluster(const Problem& p, int pass, const DeviceLimits& lim, Plan* out, std::string* why) {
  const int NGP = ngp_of(p.NG);
  const int N = 16;
  if (p.DH % 16 || p.DH > 960) {
    *why = "cluster: head_dim must be a multiple of 16 and <= 960";
    return false;
  }
  for (int upc : {48, 32, 16, 8}) {
    if (p.DH % upc) continue;
    const int rows = upc * NGP, CL = p.DH / upc;
    if (rows > 192 || CL > 16) continue;
    ClusterShape cf = cluster_shape(p, upc, N, false), cb = cluster_shape(p, upc, N, true);
    if (!cluster_ept_supported(cf.EPT)) continue;
    const ClusterShape& cs = pass == 0 ? cf : cb;
    if ((int)cs.tmem_cols > lim.tmem_cols || (int)cs.smem > lim.smem_optin) continue;
    if (pass == 1 && cb.MBT < 1) continue;
    Plan& pl = *out;
    pl = Plan{};
    pl.algo = FRNN_ALGO_FUSED;
    pl.cluster = CL;
    pl.rows_per_cta = rows;
    pl.batch_tile = N;
    pl.units_per_cta = upc;
    pl.ctas_per_group = CL;
    pl.groups = cs.groups;
    pl.grid = cs.groups * CL;
    pl.threads = cs.threads;
    pl.smem_bytes = (int)cs.smem;
    pl.tmem_cols = (int)cs.tmem_cols;
    pl.k_split = 1;
    pl.ws_bytes = pass == 0 ? cluster_forward_ws(p, pl) : cluster_backward_ws(p, pl);
    return true;
  }
  *why = "cluster: no units-per-CTA fits (cluster <= 16, rows <= 192)";
  return false;
}

static bool plan_simt(const Problem& p, int pass, const DeviceLimits& lim, Plan* out, std::string* why) {
  const size_t smem = simt_smem_bytes(p, pass == 1);
  if ((int)smem > lim.smem_optin) {
    *why = "simt: R block does not fit in shared memory";
    return false;
  }
  Plan& pl = *out;
  pl = Plan{};
  pl.algo = FRNN_ALGO_SIMT;
  pl.rows_per_cta = p.NG * p.DH;
  pl.batch_tile = 8;
  pl.units_per_cta = p.DH;
  pl.ctas_per_group = 1;
  pl.groups = p.NH * ((p.B + 7) / 8);
  pl.grid = pl.groups;
  pl.threads = 256;
  pl.smem_bytes = (int)smem;
  pl.k_split = 1;
  pl.ws_bytes = pass == 0 ? 0
                          : align_up(sizeof(float) * (size_t)p.T * p.NG * p.B * p.D, 256) + param_grads_ws(p);
  return true;
}

int solve_plan(const Problem& p, int pass, int algo, const DeviceLimits& lim, Plan* out, std::string* why) {
  if (!p.bf16) {
    if (algo != FRNN_ALGO_AUTO && algo != FRNN_ALGO_SIMT) {
      *why = "fp32 mode runs on the SIMT (FFMA) kernels only";
      return FRNN_EUNSUPPORTED;
    }
    return plan_simt(p, pass, lim, out, why) ? FRNN_OK : FRNN_EINFEASIBLE;
  }
  if (algo == FRNN_ALGO_SIMT) {
    *why = "bf16 mode has no SIMT path";
    return FRNN_EUNSUPPORTED;
  }
  if (algo == FRNN_ALGO_AUTO || algo == FRNN_ALGO_FUSED) {
    if (!getenv("FRNN_NO_CLUSTER") && plan_cluster(p, pass, lim, out, why)) return FRNN_OK;
    if (plan_fused(p, pass, lim, out, why)) return FRNN_OK;
    if (algo == FRNN_ALGO_FUSED) return FRNN_EINFEASIBLE;
  }
  std::string alt_why;
  if (!alt_supported(p, &alt_why)) {
    *why = why->empty() ? alt_why : *why + "; " + alt_why;
    return FRNN_EINFEASIBLE;
  }
  const AltShape sh = alt_shape(p, pass == 1, lim.sm_count);
  if ((int)sh.smem > lim.smem_optin) {
    *why = "alternating path: shared memory";
    return FRNN_EINFEASIBLE;
  }
  Plan& pl = *out;
  pl = Plan{};
  pl.algo = FRNN_ALGO_ALTERNATING;
  pl.rows_per_cta = 128;
  pl.batch_tile = sh.N;
  pl.units_per_cta = pass == 0 ? sh.UPT : 128 / sh.KS;
  pl.ctas_per_group = sh.KS;
  pl.groups = sh.tiles * p.NH * sh.NBT;
  pl.grid = sh.grid;
  pl.threads = 256;
  pl.smem_bytes = (int)sh.smem;
  pl.tmem_cols = (int)sh.tmem_cols;
  pl.k_split = sh.KS;
  pl.cluster = sh.KS > 1 ? sh.KS : 0;
  pl.ws_bytes = pass == 0 ? alt_forward_ws(p, pl) : alt_backward_ws(p, pl);
  return FRNN_OK;
}

}  // namespace frnn
