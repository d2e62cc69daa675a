// kernels.h -- internal launch interface between the C-ABI layer (abi.cpp) and
// the CUDA translation units.  Not installed; the public surface is flashrnn.h.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <string>

namespace frnn {

// Everything a pass needs, device pointers only.  Element type is given by
// `bf16` (true: __nv_bfloat16, false: float).
struct Problem {
  int variant, NS, NG;
  bool rec[4], inp[4];
  int T, B, NH, DH, D;
  bool bf16;
  // forward
  const void *R, *bias, *x, *s0;
  void *states, *gates;
  // backward
  const void *cstates, *cgates, *dsf, *dh;
  int clip_mode;
  float clip_mag;
  void *dx, *dbias, *dR, *ds0;
};

// Tiling chosen by the planner for one pass.
struct Plan {
  int algo;            // frnn_algo
  int rows_per_cta;    // tcgen05 M (128) or SIMT rows
  int batch_tile;      // N
  int units_per_cta;   // hidden units owned per CTA
  int ctas_per_group;  // CTAs synchronising per step
  int groups;          // heads x batch tiles
  int grid, threads, smem_bytes, tmem_cols, k_split;
  int cluster;         // >0: cluster-resident fused kernels with this cluster size
  int ka, stages;      // alternating path: K atoms per pipeline stage, ring depth
  int ffma;            // alternating path on the FFMA step kernels (alt_fp32.cu)
  size_t ws_bytes;
  double solve_us;
};

// C-ABI error string (abi.cpp), shared by every exported entry point.
int set_error(int code, const std::string& msg);
void clear_error();

// Workspace carve-up helpers.
__host__ __device__ inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// ---- SIMT fp32 path (simt_fp32.cu) ----
size_t simt_smem_bytes(const Problem& p, bool backward);
cudaError_t simt_forward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s);
cudaError_t simt_backward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s);

// ---- fused tcgen05 bf16 path (fused_bf16.cu) ----
cudaError_t fused_forward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s);
cudaError_t fused_backward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s);
size_t fused_forward_ws(const Problem& p, const Plan& pl);
uint32_t fused_tmem_cols(const Problem& p, int N, bool backward);
size_t fused_backward_ws(const Problem& p, const Plan& pl);

// ---- cluster-resident fused path (fused_cluster.cu) ----
constexpr int kSmemOptin = 232448;  // B200 max dynamic shared memory per CTA (opt-in)
struct ClusterShape {
  int UPC, CL, R1, R2, K, KBP, MB, MBT, EPT, groups, threads;
  int MS, SSM;  // backward: SMEM-A column blocks and their M (64 | 128)
  int dsm;  // backward partial exchange: 0 global + TMA bulk load, 1 DSMEM v4 [cu][n], 2 DSMEM rows [n][cu]
  int pbf16, pvec;  // backward: bf16-pair partials; their receive layout (2 = [n][cu/2] column pairs)
  uint32_t acc1, acc2, tmem_cols, slice;
  size_t smem, ws;
  int NCL;  // clusters per group (> 1: h slices / partials cross clusters through L2 with release counters)
  int Ks;   // forward: K columns of the R rows held in SMEM (M=128 SS) when K/2 + accumulators exceed TMEM
  int m64;  // forward, multi-cluster: rows <= 64 -- both halves of the K split as M=64 MMAs
};
// ncl > 1: the group's DH units are split over ncl clusters of
// DH / (UPC * ncl) CTAs each.
ClusterShape cluster_shape(const Problem& p, int UPC, int N, bool backward, int ncl = 1);
// Clusters of `CL` CTAs of the multi-cluster kernel that can be co-resident (0 without a device).
int cluster_max_active(const Problem& p, const ClusterShape& cs, bool backward);
bool cluster_ept_supported(int ept);
// The multi-cluster backward tiling has a compile-time MMA issue instance (fused_cluster.cu).
bool cluster_mc_bwd_instance(const ClusterShape& cs);
cudaError_t cluster_forward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s);
cudaError_t cluster_backward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s);
size_t cluster_forward_ws(const Problem& p, const Plan& pl);
size_t cluster_backward_ws(const Problem& p, const Plan& pl);
// Registers per thread / local (spill) bytes of the cluster kernel the plan
// would launch (compiler feedback for the planner); false without a device.
bool cluster_kernel_attrs(int variant, bool backward, int* regs, int* local_bytes, int* max_threads);

// ---- alternating path (alternating.cu) ----
struct AltShape {
  int N, NBT;            // batch tile (MMA N) and batch tiles
  int UPT;               // forward: hidden units per CTA (128 / NG gate rows each)
  int tiles;             // forward: unit tiles; backward: 128-column tiles
  int numk;              // K blocks (of 64) per CTA
  int KS, KT, kpg, nrec; // backward: cluster K split, K blocks, blocks per gate, R-gates
  int recg[4];
  int stages, grid, ka;  // ka: 64-wide K atoms per stage
  uint32_t stage_bytes, a_bytes, region, tmem_cols;
  size_t smem;
};
AltShape alt_shape(const Problem& p, bool backward, int N, int KS, int ka, int stages);
constexpr uint32_t kAltAStage = 128 * 64 * 2;  // A bytes per K atom (128 rows x 64 bf16)
constexpr int kAltMaxKS = 8;
bool alt_supported(const Problem& p, std::string* why);
cudaError_t alt_forward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s);
cudaError_t alt_backward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s);
size_t alt_forward_ws(const Problem& p, const Plan& pl);
size_t alt_backward_ws(const Problem& p, const Plan& pl);

// ---- fp32 mode beyond shared-memory R (alt_fp32.cu) ----
cudaError_t alt32_forward(const Problem& p, void* ws, cudaStream_t s);
cudaError_t alt32_backward(const Problem& p, void* ws, cudaStream_t s);
size_t alt32_forward_ws(const Problem& p);
size_t alt32_backward_ws(const Problem& p);

// ---- parameter gradients dR / db (param_grads.cu) ----
// dg element (t, b, j, e) lives at dg[t*ts + b*bs + j*js + e].
struct DgView {
  const void* ptr;
  long long ts, bs, js;
};
cudaError_t param_grads(const Problem& p, DgView dg, void* ws, cudaStream_t s);
size_t param_grads_ws(const Problem& p);

// ---- tcgen05 dR GEMM (dr_gemm.cu) ----
bool dr_gemm_supported(const Problem& p);
cudaError_t dr_gemm(const Problem& p, const void* dg_dx_layout, cudaStream_t s);
// db[i] = sum over batch tiles (fixed order) of acc[tile * n + i]
cudaError_t db_convert(const float* acc, void* db, int n, int tiles, cudaStream_t s);

// ---- input projection x = u W^T (wx_gemm.cu) ----
cudaError_t wx_gemm(const void* W, const void* u, void* x, long long M, int N, int K, cudaStream_t s);

// ---- utilities (util.cu) ----
// Sets *flag (device int) to 1 if any of the n elements is non-finite.
cudaError_t check_finite(const void* ptr, size_t n, bool bf16, int* flag, cudaStream_t s);

int sm_count();

// Counts every kernel this library launches (frnn_debug_launches).
void note_launch(int n = 1);

// ---- optional per-kernel-class event timing (ktimer.cpp) ----
enum KernelClass { KT_FWD = 0, KT_BWD = 1, KT_PARAM = 2, KT_N = 3 };
void kt_begin(int cls, cudaStream_t s);
void kt_end(int cls, cudaStream_t s);

}  // namespace frnn
