// planner.cpp -- the B200 tiling solver: integer CSPs in the ConstrINT style
// (reference planner.cpp:100-313), solved by csp.cpp.
//
// The reference encodes an Ampere/Hopper fused kernel (13 E/W/B/L variables
// per axis, register/SRAM footprints).  The B200 kernels have different
// resources, so each kernel family gets its own formulation over B200 limits
// queried from the device: SMEM opt-in bytes, TMEM columns (512 x 128 lanes x
// 32 bit per SM), thread-block cluster size (16 non-portable), SM count
// (co-residency), tcgen05 shapes (M = 128 TMEM block + M = 64 SMEM block,
// N = 16-wide batch tiles, K = 16) and TMA box/stage sizes.  As in the
// reference, a heuristic order + value preference picks among feasible
// tilings (planner.cpp:203-228: minimise the synchronising / accumulating
// blocks first), and the reference's missing compiler-feedback loop
// is closed: the chosen kernel's register count and
// spill bytes (cudaFuncGetAttributes) are checked and, if the launch would not
// fit, a tighter thread constraint is added and the CSP re-solved.
#include "planner.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <optional>

#include "../../include/flashrnn.h"
#include "csp.h"

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

namespace {

using csp::Domain;
using csp::Int;
using csp::Pref;
using csp::Rel;

int ngp_of(int NG) { return NG <= 1 ? 1 : NG <= 2 ? 2 : 4; }

// Readable constraint building on top of csp::Problem (node handles).
struct Builder {
  csp::Problem p;
  std::map<std::string, int> var_of;
  struct E {
    Builder* b;
    int n;
    E operator+(E o) const { return {b, b->p.add(n, o.n)}; }
    E operator*(E o) const { return {b, b->p.mul(n, o.n)}; }
    E operator+(Int c) const { return *this + b->k(c); }
    E operator*(Int c) const { return *this * b->k(c); }
  };
  E var(const std::string& id, Domain d) {
    const int v = p.add_var(id, std::move(d));
    var_of[id] = v;
    return {this, p.leaf(v)};
  }
  E k(Int c) { return {this, p.constant(c)}; }
  void le(E a, E b) { p.require(Rel::Le, a.n, b.n); }
  void le(E a, Int c) { le(a, k(c)); }
  void le(Int c, E b) { le(k(c), b); }
  void eq(E a, E b) { p.require(Rel::Eq, a.n, b.n); }
  void eq(E a, Int c) { eq(a, k(c)); }
  void divides(Int c, E b) { p.require(Rel::Div, k(c).n, b.n); }
  void prefer(const std::string& id, Pref pr) { p.prefer(var_of.at(id), pr); }
};

// ---------------------------------------------------------------------------
// Cluster-resident fused kernels (fused_cluster.cu).  Per group (head x batch
// tile of 16 rows) one cluster of CL CTAs; CTA p owns UPC hidden units and all
// NG gates of them: rows = NGP*UPC gate rows, R1 of them as the TMEM A operand
// (M=128 block), R2 = rows - R1 in SMEM (M=64 block, allocated as 64 rows).
// `thread_cap`: feedback bound on threads per CTA (0 = none).
Builder cluster_csp(const Problem& p, int pass, const DeviceLimits& lim, int thread_cap) {
  Builder b;
  const int NGP = ngp_of(p.NG), N = 16, DH = p.DH;
  const int MB = (DH + 127) / 128;
  const int nbt_max = (p.B + N - 1) / N;
  auto UPC = b.var("UPC", Domain::grid(8, std::max(8, std::min(DH, 128)), 8));
  auto CL = b.var("CL", Domain::span(1, lim.cluster_max));
  auto NB = b.var("NB", Domain::span(1, nbt_max));
  auto R1 = b.var("R1", Domain::span(1, lim.umma_m));
  auto R2P = b.var("R2P1", Domain::span(1, 65));        // R2 + 1
  auto A2P = b.var("A2P1", Domain::set({1, 65}));        // SMEM block rows + 1 (0 or 64)
  b.eq(UPC * CL, DH);                                    // every unit owned once
  b.divides(16, b.k(DH));                                // 16-byte h chunks, K multiple of 16
  b.le(p.B, NB * N);                                     // batch tiles cover B
  b.eq(UPC * NGP + 1, R1 + R2P);                         // rows = R1 (TMEM) + R2 (SMEM)
  b.le(R2P, A2P);                                        // SMEM block present iff R2 > 0
  b.le(UPC * (N / 2), thread_cap > 0 ? std::min(384, thread_cap) : 384);  // one unit pair per thread
  b.le(CL * NB * p.NH, lim.sm_count);                    // all clusters co-resident
  if (pass == 0) {
    // SMEM: double-buffered h tile [N x DH], SMEM A block, fp32 accumulator
    // staging [N][rows+1], own h slice, barriers (fused_cluster.cu cluster_shape)
    // (the accumulator staging pitch is rows + 4 per 32 rows, rounded to 4 words: <= 9/8 rows + 4)
    b.le(A2P * (DH * 2) + UPC * (N * NGP * 4 + N * NGP / 2 + N * 2) + (4 * N * DH + N * 16 + 64),
         lim.smem_optin + DH * 2);
    // TMEM: R slice as bf16 pairs (DH/2 columns, 32-aligned) + two N-wide accumulators
    b.le(b.k(((DH / 2 + 31) / 32) * 32 + 2 * N), lim.tmem_cols);
  } else {
    // Backward: R_p^T as MBT 128-column blocks in TMEM and MS 128-column blocks
    // in SMEM, K = rows padded to 16 (KBH = K/2 TMEM columns per block)
    auto MBT = b.var("MBT", Domain::span(1, MB));
    auto MS1 = b.var("MS1", Domain::span(1, 17));  // MS + 1 (domains are positive)
    auto KBH = b.var("KBH", Domain::grid(8, 128, 8));
    b.le(UPC * NGP, KBH * 2);
    b.le(KBH * 2, UPC * NGP + 15);
    b.le(b.k(DH + 128), MBT * 128 + MS1 * 128);                 // the blocks cover DH columns
    b.le(MBT + MS1, b.k(MB + 1));                               // MBT + MS = MB
    b.le(MBT * KBH + (MBT + MS1) * N, b.k(lim.tmem_cols + N));  // A blocks + accumulators
    // SMEM: MS blocks [128 x K] + partial receive [CL][N][UPC] fp32 + dg tile + db scratch
    b.le(MS1 * KBH * 512 + KBH * (N * 4) + CL * UPC * (N * 4) + UPC * (p.NG * N * 4) + 192,
         b.k(lim.smem_optin) + KBH * 512);
  }
  // Heuristic (planner.cpp:203-228 in spirit): fewest CTAs synchronising per
  // step, fewest batch tiles, fill TMEM before SMEM, most R^T in TMEM.
  b.prefer("CL", Pref::Smallest);
  b.prefer("NB", Pref::Smallest);
  b.prefer("R1", Pref::Largest);
  if (pass == 1) {
    b.prefer("MBT", Pref::Largest);
    b.prefer("MS1", Pref::Smallest);
    b.prefer("KBH", Pref::Smallest);
  }
  b.prefer("A2P1", Pref::Smallest);
  return b;
}

// ---------------------------------------------------------------------------
// Alternating path (alternating.cu): per-step TMA-streamed GEMM.  Batch tile N
// (MMA N) x NB tiles, K atoms per stage KA, ring depth ST, backward cluster
// K-split KS; one wave of CTAs.
Builder alt_csp(const Problem& p, int pass, const DeviceLimits& lim) {
  Builder b;
  const int DH = p.DH;
  int nrec = 0;
  for (int j = 0; j < p.NG; ++j) nrec += p.rec[j];
  const int ring = getenv("FRNN_ALT_SMEM_KB") ? atoi(getenv("FRNN_ALT_SMEM_KB")) * 1024 : 200 * 1024;
  auto N = b.var("N", Domain::grid(16, 128, 16));
  auto NB = b.var("NB", Domain::span(1, (p.B + 15) / 16));
  const int ka_max = getenv("FRNN_ALT_KA_MAX") ? std::max(1, atoi(getenv("FRNN_ALT_KA_MAX"))) : 4;  // experiments
  auto KA = b.var("KA", Domain::span(1, ka_max));
  auto KPG = b.var("KPG", Domain::span(1, std::max(1, DH / 64)));
  auto ST = b.var("ST", Domain::span(2, 8));
  b.le(p.B, N * NB);
  b.eq(KA * KPG * 64, DH);                                        // whole 64-wide K atoms
  b.le(ST * KA * (int)kAltAStage + ST * KA * N * 128 + 2048, ring);  // stage ring
  if (pass == 0) {
    const int UPT = p.NG == 1 ? 128 : 32;
    b.le(N * 512 + (512 + 2048), lim.smem_optin);                 // epilogue [128][N+1] fp32
    b.le(NB * ((DH + UPT - 1) / UPT * p.NH), std::max(lim.sm_count, (DH + UPT - 1) / UPT * p.NH));
    b.prefer("NB", Pref::Smallest);
  } else {
    const int ks_cap = getenv("FRNN_ALT_KS") ? std::max(1, atoi(getenv("FRNN_ALT_KS"))) : kAltMaxKS;  // experiments
    auto KS = b.var("KS", Domain::span(1, std::min(ks_cap, kAltMaxKS)));
    b.le(KS, KPG * std::max(1, nrec));                            // every rank has K blocks
    if (nrec == 0) b.eq(KS, 1);
    b.le(N * 528 + 2048, lim.smem_optin);                         // epilogue [N][132] fp32
    // one wave that leaves a third of the SMs free: the next step's CTAs (PDL) become
    // resident and prefetch R while this step drains (measured at H=3072: 96 CTAs
    // 27 us/step, 144 CTAs 42 us/step -- profiles/r01_alt_ks_sweep_c5.txt)
    b.le(KS * NB * ((DH + 127) / 128 * p.NH), std::max(lim.sm_count * 2 / 3, (DH + 127) / 128 * p.NH));
    b.prefer("NB", Pref::Smallest);
    b.prefer("KS", Pref::Largest);  // spread the per-step R^T stream over the SMs
  }
  b.prefer("N", Pref::Smallest);
  b.prefer("KA", Pref::Largest);
  b.prefer("ST", Pref::Largest);
  return b;
}

std::optional<std::map<std::string, Int>> run(const Builder& b) {
  const auto sol = csp::solve(b.p);
  if (!sol) return std::nullopt;
  return sol->values;
}

bool plan_cluster(const Problem& p, int pass, const DeviceLimits& lim, Plan* out, std::string* why) {
  if (getenv("FRNN_NO_CLUSTER")) {
    *why = "cluster kernels disabled (FRNN_NO_CLUSTER)";
    return false;
  }
  int cap = 0;
  for (int round = 0; round < 3; ++round) {
    const auto sol = run(cluster_csp(p, pass, lim, cap));
    if (!sol) {
      *why = "cluster: no tiling satisfies the B200 TMEM/SMEM/cluster constraints";
      return false;
    }
    const int upc = (int)sol->at("UPC"), CL = (int)sol->at("CL");
    const ClusterShape cs = cluster_shape(p, upc, 16, pass == 1);
    if (!cluster_ept_supported(cs.EPT) || (pass == 1 && cs.MBT < 1)) {
      *why = "cluster: solver/launcher geometry mismatch";
      return false;
    }
    // Compiler feedback: the launch must fit the register file without spills.
    int regs = 0, local = 0, maxt = 0;
    if (cluster_kernel_attrs(p.variant, pass == 1, &regs, &local, &maxt) &&
        ((long long)regs * cs.threads > lim.regs_per_sm || cs.threads > maxt)) {
      cap = std::min(maxt, (int)(lim.regs_per_sm / std::max(1, regs))) / 128 * 128;
      if (cap < 128) {
        *why = "cluster: kernel register use leaves no feasible block size";
        return false;
      }
      continue;
    }
    Plan& pl = *out;
    pl = Plan{};
    pl.algo = FRNN_ALGO_FUSED;
    pl.cluster = CL;
    pl.rows_per_cta = upc * ngp_of(p.NG);
    pl.batch_tile = 16;
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
  *why = "cluster: compiler feedback did not converge";
  return false;
}

// Heads whose R does not fit one cluster (4-gate DH > 768): the group's
// units over NCL clusters of CL CTAs (fused_cluster.cu, NCL > 1) -- R stays
// resident in TMEM + SMEM, h slices cross clusters through L2 with release
// flags.  Fewest clusters first (every extra cluster is another L2 round trip
// per step), then the largest cluster; all NCL * groups clusters must be
// co-resident (the kernel spins on the other clusters' flags).
bool plan_multicluster(const Problem& p, int pass, const DeviceLimits& lim, Plan* out, std::string* why) {
  if (getenv("FRNN_NO_MULTICLUSTER")) {
    *why = "multi-cluster kernels disabled (FRNN_NO_MULTICLUSTER)";
    return false;
  }
  const int NGP = ngp_of(p.NG), N = 16;
  // Backward (4-gate cells, bf16 column-pair exchange; partials for other clusters'
  // owners through L2): faster than the alternating backward with two clusters on
  // the tilings with a compile-time MMA issue instance (H=896 7.2-7.3 vs 8.6, H=1024
  // 7.5-7.6 vs 8.2 us/step); with three clusters box-dependent (H=1152 8.8-9.8 vs
  // 9.1), with the generic issue loop slower (H=1024 8.8) -- so by default only
  // two-cluster instance tilings; FRNN_MC_BWD=1 any tiling, =0 none.
  const char* mcb = getenv("FRNN_MC_BWD");
  const int mc_bwd = mcb ? atoi(mcb) : -1;
  if (pass == 1 && (NGP != 4 || mc_bwd == 0)) {
    *why = "multi-cluster backward: 4-gate cells (FRNN_MC_BWD=0 disables it)";
    return false;
  }
  for (int ncl = 2; ncl <= 9; ++ncl)
    for (int CL = lim.cluster_max; CL >= 2; --CL) {
      if (p.DH % (ncl * CL)) continue;
      const int upc = p.DH / (ncl * CL);
      // (UPC % 8: a slice is whole 8-wide K core-matrix columns of the h tile)
      if (upc % 8 || upc * NGP > 128 || upc / 2 * N > 384) continue;
      if ((CL * upc) % 16) continue;  // whole 16-wide K steps per cluster
      const ClusterShape cs = cluster_shape(p, upc, N, pass == 1, ncl);
      if ((int)cs.smem > lim.smem_optin || (int)cs.tmem_cols > lim.tmem_cols || !cluster_ept_supported(cs.EPT))
        continue;
      if (pass == 0 && ((cs.K - cs.Ks) % 16 || cs.Ks % 16)) continue;
      if (pass == 1 && (cs.MBT < 1 || cs.dsm != 2 || !cs.pbf16 || cs.pvec != 2)) continue;
      if (pass == 1 && mc_bwd < 0 && (ncl > 2 || !cluster_mc_bwd_instance(cs))) continue;
      const int active = cluster_max_active(p, cs, pass == 1);
      if (active > 0 && active < ncl * cs.groups) continue;  // (no device: assume co-resident)
      if (active == 0 && ncl * cs.groups * CL > lim.sm_count) continue;
      Plan& pl = *out;
      pl = Plan{};
      pl.algo = FRNN_ALGO_FUSED;
      pl.cluster = CL;
      pl.rows_per_cta = upc * NGP;
      pl.batch_tile = N;
      pl.units_per_cta = upc;
      pl.ctas_per_group = ncl * CL;
      pl.groups = cs.groups;
      pl.grid = cs.groups * ncl * CL;
      pl.threads = cs.threads;
      pl.smem_bytes = (int)cs.smem;
      pl.tmem_cols = (int)cs.tmem_cols;
      pl.k_split = 1;
      pl.ws_bytes = pass == 0 ? cluster_forward_ws(p, pl) : cluster_backward_ws(p, pl);
      return true;
    }
  *why = "multi-cluster: no NCL x CL x UPC split of the head fits";
  return false;
}

bool plan_alt(const Problem& p, int pass, const DeviceLimits& lim, Plan* out, std::string* why) {
  if (!alt_supported(p, why)) return false;
  const auto sol = run(alt_csp(p, pass, lim));
  if (!sol) {
    *why = "alternating path: no tiling satisfies the B200 constraints";
    return false;
  }
  const int N = (int)sol->at("N"), KA = (int)sol->at("KA"), ST = (int)sol->at("ST");
  const int KS = pass == 1 ? (int)sol->at("KS") : 1;
  const AltShape sh = alt_shape(p, pass == 1, N, KS, KA, ST);
  if ((int)sh.smem > lim.smem_optin) {
    *why = "alternating path: shared memory";
    return false;
  }
  Plan& pl = *out;
  pl = Plan{};
  pl.algo = FRNN_ALGO_ALTERNATING;
  pl.rows_per_cta = 128;
  pl.batch_tile = N;
  pl.units_per_cta = pass == 0 ? sh.UPT : 128 / KS;
  pl.ctas_per_group = KS;
  pl.groups = sh.tiles * p.NH * sh.NBT;
  pl.grid = sh.grid;
  pl.threads = 256;
  pl.smem_bytes = (int)sh.smem;
  pl.tmem_cols = (int)sh.tmem_cols;
  pl.k_split = KS;
  pl.cluster = KS > 1 ? KS : 0;
  pl.ka = KA;
  pl.stages = ST;
  pl.ws_bytes = pass == 0 ? alt_forward_ws(p, pl) : alt_backward_ws(p, pl);
  return true;
}

// L2-flag fused kernels (fused_bf16.cu): the measured baseline of the cluster
// design, used when no cluster shape fits.  Largest units-per-CTA that divides
// DH with the grid co-resident.
bool plan_fused(const Problem& p, int pass, const DeviceLimits& lim, Plan* out, std::string* why) {
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
  // The L2-flag kernels' tiling CSP: UPC units per CTA (all NGP gates of each:
  // at most one 128-lane TMEM block of rows), CPG CTAs per group with
  // UPC x CPG = DH, every group's CTAs co-resident (cooperative launch);
  // heuristic: fewest CTAs synchronising per step (largest UPC).
  Builder b;
  auto vU = b.var("UPC", Domain::span(1, std::max(1, 128 / NGP)));
  auto vC = b.var("CPG", Domain::span(1, std::max(1, p.DH)));
  b.eq(vU * vC, p.DH);
  b.le(vC * (p.NH * NBT), lim.sm_count);
  b.prefer("UPC", Pref::Largest);
  const auto sol = run(b);
  if (!sol) {
    *why = "fused: no UPC x CPG split of the head with the grid co-resident";
    return false;
  }
  const int best = (int)sol->at("UPC"), CPG = (int)sol->at("CPG");
  const int grid = p.NH * NBT * CPG;
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

bool plan_simt(const Problem& p, int pass, const DeviceLimits& lim, Plan* out, std::string* why) {
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

// FFMA step kernels (alt_fp32.cu): 32 gate rows / 32 state columns x 16 batch
// rows per CTA, R streamed through shared memory every step.
void plan_ffma(const Problem& p, int pass, Plan* out) {
  Plan& pl = *out;
  pl = Plan{};
  pl.algo = FRNN_ALGO_ALTERNATING;
  pl.ffma = 1;
  pl.rows_per_cta = 32;
  pl.batch_tile = 16;
  pl.units_per_cta = pass == 0 ? 32 / (p.NG == 1 ? 1 : 4) : 32;
  pl.ctas_per_group = 1;
  pl.groups = ((p.DH + pl.units_per_cta - 1) / pl.units_per_cta) * p.NH * ((p.B + 15) / 16);
  pl.grid = pl.groups;
  pl.threads = 256;
  pl.k_split = 1;
  pl.ws_bytes = pass == 0 ? alt32_forward_ws(p) : alt32_backward_ws(p);
}

}  // namespace

size_t plan_workspace(const Problem& p, int pass, const Plan& pl) {
  switch (pl.algo) {
    case FRNN_ALGO_SIMT: {
      Plan q{};
      std::string why;
      plan_simt(p, pass, device_limits(), &q, &why);
      return q.ws_bytes;
    }
    case FRNN_ALGO_FUSED:
      if (pl.cluster) return pass == 0 ? cluster_forward_ws(p, pl) : cluster_backward_ws(p, pl);
      return pass == 0 ? fused_forward_ws(p, pl) : fused_backward_ws(p, pl);
    default:
      if (pl.ffma) return pass == 0 ? alt32_forward_ws(p) : alt32_backward_ws(p);
      return pass == 0 ? alt_forward_ws(p, pl) : alt_backward_ws(p, pl);
  }
}

std::vector<std::string> plan_residuals(const Problem& p, int pass, const Plan& pl, const DeviceLimits& lim) {
  std::vector<std::string> out;
  auto fail = [&out](const std::string& m) { out.push_back(m); };
  auto eq = [&](long long a, long long b, const char* what) {
    if (a != b) fail(std::string(what) + ": plan " + std::to_string(a) + ", recomputed " + std::to_string(b));
  };
  const bool bwd = pass == 1;
  const int NGP = ngp_of(p.NG), N = pl.batch_tile;
  if (pl.threads < 32 || pl.threads % 32 || pl.threads > lim.max_threads) fail("threads not a warp multiple within the block limit");
  if (pl.smem_bytes > lim.smem_optin) fail("shared memory exceeds the opt-in limit");
  if (pl.tmem_cols > lim.tmem_cols) fail("TMEM columns exceed the SM's 512");
  if (pl.tmem_cols && (pl.tmem_cols < 32 || (pl.tmem_cols & (pl.tmem_cols - 1)))) fail("TMEM allocation not a power of two >= 32");
  if (pl.grid != pl.groups * pl.ctas_per_group) fail("grid != groups x CTAs per group");
  eq((long long)pl.ws_bytes, (long long)plan_workspace(p, pass, pl), "workspace bytes");
  if (pl.algo == FRNN_ALGO_FUSED && pl.cluster > 0) {  // cluster-resident (one or several clusters)
    const int CL = pl.cluster, UPC = pl.units_per_cta;
    if (pl.ctas_per_group % CL) {
      fail("CTAs per group not a multiple of the cluster");
      return out;
    }
    const int ncl = pl.ctas_per_group / CL;
    if (CL > lim.cluster_max) fail("cluster larger than the device's non-portable maximum");
    if ((long long)UPC * pl.ctas_per_group != p.DH) fail("units per CTA x CTAs per group != head dim");
    eq(pl.rows_per_cta, UPC * NGP, "rows per CTA");
    eq(pl.groups, p.NH * ((p.B + N - 1) / N), "groups (heads x batch tiles)");
    if (UPC % 2 || UPC / 2 * N > 384) fail("one unit pair per thread needs UPC even and UPC/2 x N <= 384");
    const ClusterShape cs = cluster_shape(p, UPC, N, bwd, ncl);
    eq(pl.smem_bytes, (long long)cs.smem, "shared memory");
    eq(pl.tmem_cols, cs.tmem_cols, "TMEM columns");
    eq(pl.threads, cs.threads, "threads");
    if (!cluster_ept_supported(cs.EPT)) fail("element ownership unsupported");
    if (!bwd) {
      if (ncl == 1 && (cs.R1 > 128 || cs.R2 > 64)) fail("rows exceed the TMEM (128) + SMEM (64) blocks");
      if (ncl > 1 && (cs.R2 != 0 || UPC % 8 || (CL * UPC) % 16)) fail("multi-cluster slice geometry");
      if ((cs.K - cs.Ks) % 16 || cs.Ks % 16) fail("K split not in whole 16-wide steps");
    } else {
      if (cs.MBT < 1) fail("no R^T column block in TMEM");
      if (std::max(cs.MBT, cs.MS) > 16) fail("more than 16 block pairs");
      if (ncl > 1 && (NGP != 4 || cs.dsm != 2 || !cs.pbf16 || cs.pvec != 2)) fail("multi-cluster backward exchange");
    }
    const int active = cluster_max_active(p, cs, bwd && ncl > 1);
    if (ncl > 1 && active > 0 && active < ncl * pl.groups) fail("clusters of a group not co-resident");
    if (ncl > 1 && active == 0 && pl.grid > lim.sm_count) fail("grid exceeds the SM count");
    int regs = 0, local = 0, maxt = 0;
    if (ncl == 1 && cluster_kernel_attrs(p.variant, bwd, &regs, &local, &maxt) &&
        (long long)regs * pl.threads > lim.regs_per_sm)
      fail("registers x threads exceed the register file");
  } else if (pl.algo == FRNN_ALGO_FUSED) {  // L2-flag fused kernels
    if ((long long)pl.units_per_cta * pl.ctas_per_group != p.DH) fail("units per CTA x CTAs per group != head dim");
    eq(pl.tmem_cols, fused_tmem_cols(p, N, bwd), "TMEM columns");
    if (pl.grid > lim.sm_count) fail("cooperative grid exceeds the SM count");
  } else if (pl.algo == FRNN_ALGO_ALTERNATING && !pl.ffma) {
    std::string why;
    if (!alt_supported(p, &why)) fail(why);
    const AltShape sh = alt_shape(p, bwd, N, pl.k_split, pl.ka, pl.stages);
    eq(pl.smem_bytes, (long long)sh.smem, "shared memory");
    eq(pl.tmem_cols, sh.tmem_cols, "TMEM columns");
    eq(pl.grid, sh.grid, "grid");
    if ((size_t)sh.stages * sh.stage_bytes > sh.region) fail("stage ring exceeds its region");
    if ((long long)sh.ka * sh.kpg * 64 != p.DH) fail("K atoms x atoms per gate != head dim");
    if (p.B > N * sh.NBT) fail("batch tiles do not cover the batch");
  } else if (pl.algo == FRNN_ALGO_SIMT) {
    eq(pl.smem_bytes, (long long)simt_smem_bytes(p, bwd), "shared memory");
  }
  return out;
}

PlanTraffic plan_traffic(const Problem& p, int pass, const Plan& pl) {
  PlanTraffic t{};
  const double e = p.bf16 ? 2 : 4, B = p.B, D = p.D, NS = p.NS, NG = p.NG, DH = p.DH, NH = p.NH;
  int nin = 0, nrec = 0;
  for (int j = 0; j < p.NG; ++j) {
    nin += p.inp[j];
    nrec += p.rec[j];
  }
  const bool alt = pl.algo == FRNN_ALGO_ALTERNATING;
  const double N = pl.batch_tile > 0 ? pl.batch_tile : 16, nbt = std::ceil(B / N);
  if (pass == 0) {  // engine.hpp:170-201: x_t in, gates_t and states_{t+1} out
    t.io = B * nin * D * e + B * NG * D * e + B * NS * D * e;
    if (alt) t.io += 2 * NS * B * D * 4;  // fp32 carry in and out
    const double h = B * D * e;           // the h_t all-gather source
    if (pl.algo == FRNN_ALGO_FUSED && pl.cluster > 0) {
      const int ncl = std::max(1, pl.ctas_per_group / pl.cluster);
      t.exchange_l2 = h + h * (ncl - 1) / ncl;  // slices staged in L2, the other clusters' slices imported
      t.exchange_onchip = h * pl.cluster;       // multicast delivery into every CTA of a cluster
    } else if (pl.algo == FRNN_ALGO_FUSED) {
      t.exchange_l2 = h + h * pl.ctas_per_group;  // every CTA of a group re-reads all of h
    } else if (alt) {
      const double tiles = std::ceil(DH * (p.NG == 1 ? 1.0 : 4.0) / 128.0);
      t.exchange_l2 = h * tiles;                  // every unit tile streams h
      t.r_stream = nrec * DH * DH * NH * e;
    }
  } else {  // engine.hpp:257-336: the trace in, dh in, dx out
    t.io = B * (NS + NG) * D * e + B * NG * D * e;
    if (alt) t.io += 2 * NS * B * D * 4;
    const double part = B * D * 4;  // one fp32 R^T.dg partial per CTA source and column
    if (pl.algo == FRNN_ALGO_FUSED && pl.cluster > 0) {
      const int ncl = std::max(1, pl.ctas_per_group / pl.cluster);
      const double pb = p.NG == 4 ? 2 : 4;  // bf16-pair partials for 4-gate cells
      t.exchange_onchip = B * D * pb * pl.cluster;                     // every source pushes every column
      t.exchange_l2 = ncl > 1 ? B * D * pb * pl.cluster * (ncl - 1) : 0;  // columns owned by other clusters
    } else if (pl.algo == FRNN_ALGO_FUSED) {
      t.exchange_l2 = 2 * part * pl.ctas_per_group;
    } else if (alt) {
      t.exchange_onchip = part * pl.k_split;  // split-K partials through DSMEM
      t.exchange_l2 = B * nrec * D * e * std::ceil(DH / 128.0);  // dg streamed by every column tile
      t.r_stream = nrec * DH * DH * NH * e;
    }
    (void)nbt;
  }
  return t;
}

std::string plan_csp_text(const Problem& p, int pass, int algo, const DeviceLimits& lim) {
  if (algo == FRNN_ALGO_ALTERNATING) return csp::format(alt_csp(p, pass, lim).p);
  return csp::format(cluster_csp(p, pass, lim, 0).p);
}

int solve_plan(const Problem& p, int pass, int algo, const DeviceLimits& lim, Plan* out, std::string* why) {
  if (!p.bf16) {  // fp32 parity mode: FFMA kernels (no fp32 tensor-core path meets rel 1e-5)
    if (algo == FRNN_ALGO_FUSED) {
      *why = "fp32 mode runs on the FFMA kernels (simt or alternating)";
      return FRNN_EUNSUPPORTED;
    }
    if (algo != FRNN_ALGO_ALTERNATING && plan_simt(p, pass, lim, out, why)) return FRNN_OK;
    if (algo == FRNN_ALGO_SIMT) return FRNN_EINFEASIBLE;
    plan_ffma(p, pass, out);
    return FRNN_OK;
  }

  if (algo == FRNN_ALGO_SIMT) {
    *why = "bf16 mode has no SIMT path";
    return FRNN_EUNSUPPORTED;
  }
  std::string w1, w2, w3;
  if (algo == FRNN_ALGO_AUTO || algo == FRNN_ALGO_FUSED) {
    if (plan_cluster(p, pass, lim, out, &w1)) return FRNN_OK;
    std::string w4;
    if (plan_multicluster(p, pass, lim, out, &w4)) return FRNN_OK;
    if (plan_fused(p, pass, lim, out, &w2)) return FRNN_OK;
    if (algo == FRNN_ALGO_FUSED) {
      *why = w1 + "; " + w2;
      return FRNN_EINFEASIBLE;
    }
  }
  if (plan_alt(p, pass, lim, out, &w3)) return FRNN_OK;
  if (algo == FRNN_ALGO_AUTO || algo == FRNN_ALGO_ALTERNATING) {
    // no tensor-core tiling for this head dim (not a multiple of 8 / of 64):
    // bf16 storage on the FFMA step kernels
    plan_ffma(p, pass, out);
    return FRNN_OK;
  }
  *why = w3;
  return FRNN_EINFEASIBLE;
}

}  // namespace frnn
