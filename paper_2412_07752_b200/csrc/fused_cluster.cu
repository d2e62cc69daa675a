// fused_cluster.cu -- cluster-resident persistent recurrence kernels (bf16):
// K1c forward (engine.hpp:170-201) and K2c backward (engine.hpp:257-336).
//
// One thread-block cluster per group (head x batch tile of N=16 rows); CL CTAs
// per cluster, each owning UPC hidden units and all NG gates of them
// (row = u*NGP + g), so the cell update is CTA-local.  R stays on-chip for
// all T steps: rows [0,R1) in TMEM (A operand of tcgen05.mma kind::f16 'TS'),
// rows [R1,R1+R2) (R2 <= 64) in SMEM (an M=64 'SS' MMA).  For H=768, NG=4:
// CL=16, UPC=48, R1=128, R2=64 -- 4.7 MB of R spread over 16 SMs.
//
// Per forward step the only inter-CTA traffic is h: each CTA writes its
// [UPC x N] bf16 slice (already in the MMA's K-major core-matrix layout) to a
// global staging buffer and ONE thread issues a TMA multicast that drops it
// into every CTA's double-buffered B tile, completing bytes on each CTA's
// mbarrier.  No flag polling through L2: a CTA's MMA for step t+1 starts when
// its mbarrier has counted all CL slices.  (All-gather of 24 KB in a 16-CTA
// cluster: ~890 cycles measured, vs ~5-6k for release/acquire flags + loads;
// profiles/r01_allgather_microbench.txt.)
//
// Per backward step each CTA computes the partial R_p^T dg_p for all DH state
// columns (A = R_p^T resident: MBT 128-column blocks in TMEM, MS in SMEM), one
// tcgen05.commit per block pair; as each block completes, its drain lanes push
// the partials straight into the owner CTA's shared memory (st.async with
// mbarrier complete_tx, DSMEM), as bf16 column pairs for 4-gate cells (fp32
// otherwise); the owner sums the CL sources in a fixed order (deterministic),
// clips (engine.hpp:300-303) and applies the Jacobian -- whose coefficients
// were formed under the previous step's MMAs for long MMA windows
// (cells.cuh coef/apply).  FRNN_XCHG=0 keeps the round-1 global-staging
// exchange (stores + TMA bulk load) for A/B.
//
// Element work: NT = up to 384 threads (3 warps per scheduler, so ALU/MUFU
// latencies overlap); each thread owns a PAIR of adjacent units of one batch
// row (own_pair: eight consecutive threads take eight consecutive rows, so
// the dg-tile / h-slice stores are bank-conflict free), trace/x/dx traffic is
// bf16x2.  MMAs are issued by warp 0 as straight-line PTX blocks (sm100.cuh
// mma8_* / mma12_*, issue_bwd_fixed for every tiling the planner reaches).
// Backward instances: L = 0 generic (all A/B switches), 1 the H=768 4-gate
// layout, 2 / 3 lean (default exchange only; 3 also without split coefficients),
// 4 multi-cluster.
//
// Multi-cluster (NCL > 1, heads beyond one cluster; forward instance MC = 1,
// backward L = 4): the group's units over NCL clusters.  Forward: each CTA's
// block of <= 128 rows is split along K between TMEM and an SMEM tile (M=128,
// or M=64 for blocks of <= 64 rows) with two accumulators; the own cluster's h
// slices arrive by the multicast above, the other clusters' slices are imported
// through L2 (per-slice step counters released by each writer CTA, polled by
// lanes of warp 1, TMA multicast into the own cluster).  Backward: partials for
// owners in the own cluster by DSMEM as above, for other clusters' owners stored
// to L2 and pulled by TMA after the source's release counter.  Launched as
// cooperative cluster grids (every cluster resident or the launch fails).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "cells.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace frnn {

extern long long* g_prof_buf;
extern int g_prof_steps;
int g_skeleton = 0;  // frnn_debug_skeleton

namespace {

using bf16 = __nv_bfloat16;
using namespace sm100;

constexpr int MAXT = 384;


struct CArgs {
  Problem p;
  int UPC, CL, NBT;
  int R1, R2;      // forward: rows in the TMEM block / the SMEM (M=64) block
  int K;           // forward contraction = DH (multiple of 16)
  int KBP;         // backward contraction = UPC*NGP padded to 16
  int MB, MBT;     // backward: 128-column blocks of DH / how many have A in TMEM
  int MS, SSM;     // backward: SMEM-A column blocks of SSM (64 | 128) columns
  uint32_t tmem_cols, acc1, acc2;
  uint32_t slice;  // forward: bytes of one CTA's h slice
  bf16* xstage;    // forward staging [groups][2][CL][slice]
  float* pstage;   // backward staging [groups][2][CL dest][CL src][N][UPC]
  bf16* dgw;
  float* dbacc;    // [NBT][NG][D]
  long long* prof;
  int prof_steps;
  int dsm;         // backward partial exchange: 1 = DSMEM st.async pushes, 0 = global + TMA bulk load
  int pbf16;       // dsm 2: push the partials as bf16 pairs (half the exchange bytes and pushes)
  int xpf;         // forward: L2 prefetch of x two steps ahead (FRNN_XPF)
  int kcompact;    // backward: GRU K rows without the n gate (gru_compact)
  int waitmode;    // MMA-completion waits of non-issuing warps: 0 test_wait spin, 1 try_wait (FRNN_WAITMODE)
  int itab;        // backward: compile-time issue instances for the planner's tilings (FRNN_ISSUE_TABLE=0: loop)
  int csplit;      // backward: Jacobian coefficients under the previous MMA window (FRNN_COEFSPLIT)
  int map;         // element ownership (own_pair): 1 = row-fastest groups of 8, 0 = unit-fastest
  int hdirect;     // forward: cell threads write h straight to the global staging slice (FRNN_HDIRECT)
  int rot;         // backward column rotation per CTA (FRNN_ROT=1; A/B knob, off: no gain measured)
  int nodx, noload;  // debug (FRNN_DBG_NODX / FRNN_DBG_NOLOAD): skip the backward's dx stores / trace loads
  int noxchg;      // debug (FRNN_DBG_NOXCHG): backward without the partial exchange (results garbage)
  int dxearly;     // store dx inside the MMA window (after the Jacobian) -- A/B knob FRNN_DXEARLY
  int absu;        // absorb: CL == 16 unrolled (all loads first) -- A/B knob FRNN_ABSU
  int pvec;        // pbf16: [cu/2][n/2][2] layout, two 16-byte pushes per lane (push_pair_cols);
                   //        0 = [n/2][cu] layout, N/2 4-byte pushes per lane
  int NCL;         // forward: clusters per group; > 1: slices of other clusters imported through L2
  int Ks;          // forward: K columns of the R rows in SMEM (M=128 SS, second accumulator)
  int m64;         // forward (MC): rows <= 64 -- TMEM half M=128 (lanes 64.. zero), SMEM half an M=64 tile
  uint32_t* xflags;  // forward, NCL > 1: [groups][NCL*CL] step counters of the published slices
  int mcfence, mcpoll;  // NCL > 1: full fence before the flag release; relaxed polling (A/B knobs)
  int mcwarp, mclocal;  // NCL > 1: the importing warp; own cluster's K range issued first (A/B knobs)
  int mcrelw;           // NCL > 1: the importing warp (not thread 0) releases the slice flag
  int mcdbg;            // debug (FRNN_MC_DBG bits: 1 no remote loads, 2 no remote stores, 4 no flag waits)
  uint32_t* bflags;     // backward, NCL > 1: [groups][NCL*CL] publish counters of the partials
                        // (the partials for other clusters' owners go to pstage, [grp][2][dest][src][N][PW] words)
  int skeleton;    // 1: synchronisation skeleton only -- no MMAs, no cell math (the sequential-
                   //    dependency floor of SURVEY 8d; frnn_debug_skeleton, results are garbage)
};

#define FRNN_PROF_AT(slot, step, thr)                                      \
  if (a.prof && threadIdx.x == (thr) && (step) < a.prof_steps)             \
    a.prof[((size_t)blockIdx.x * a.prof_steps + (step)) * 8 + (slot)] = clock64();
#define FRNN_PROF(slot, step) FRNN_PROF_AT(slot, step, 0)

__device__ __forceinline__ float bf(const bf16* p, size_t i) { return __bfloat162float(p[i]); }
__host__ __device__ constexpr int xs_row(int r) { return r + 4 * (r >> 5); }
__host__ __device__ constexpr int xs_pitch(int rows) { return (xs_row(rows - 1) + 1 + 3) & ~3; }
__device__ __forceinline__ float lo16(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float hi16(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t ld2(const bf16* p, size_t i) { return *reinterpret_cast<const uint32_t*>(p + i); }
__device__ __forceinline__ void st2(bf16* p, size_t i, float lo, float hi) {
  *reinterpret_cast<uint32_t*>(p + i) = pack_bf16(lo, hi);
}

// Element ownership: thread tid owns the unit pair (u, u+1) of batch row b.
// Eight consecutive threads take eight consecutive rows b of the same pair, so
// their 16-byte (backward dg) / 4-byte (forward h) stores into a K-major tile
// land in the eight distinct 16-byte rows of one core matrix: no bank conflicts.
// (Trace/x loads of a warp then touch 8 rows x 16 B -- off the critical path.)
// map 0 (round 1): consecutive threads take consecutive unit pairs of one row
// (coalesced trace / x / dx rows, but 8-way conflicted 16-byte dg-tile stores).
__device__ __forceinline__ void own_pair(int tid, int NP, int& u, int& b, int map = 1) {
  if (map) {
    u = 2 * ((tid >> 3) % NP);
    b = (tid & 7) + 8 * (tid / (8 * NP));
  } else {
    u = 2 * (tid % NP);
    b = tid / NP;
  }
}

// Backward partial exchange, bf16 pairs.  The receive block of source CTA `me`
// in the owner's recv buffer is laid out [cu/2][n/2][2] (32-bit words: the bf16
// pair (n, n+1) of column cu at word ((cu/2)*(N/2) + n/2)*2 + (cu&1)), so that
//  * a drain lane (one column cu, N accumulator rows in v) and its neighbour
//    lane (column cu^1) swap half their packed words with 4 shuffles and each
//    push 32 contiguous bytes -- two st.async.v4 instead of N/2 scalar pushes;
//  * the owner thread of units (u, u+1), batch row b, reads one 8-byte word
//    pair per source, and 8 threads (b = 0..7) read 32 contiguous bytes.
// Whole warp (the shuffles); `ok` guards the push (lanes pair up: cu even on
// even lanes, UPC even).
template <int N>
__device__ __forceinline__ void push_pair_cols(const float* v, int lane, bool ok, int cu, uint32_t rb_me,
                                               uint32_t q, uint32_t mbr) {
  static_assert(N == 16, "bf16-pair exchange layout assumes N = 16");
  uint32_t w[8], o[8];
#pragma unroll
  for (int n2 = 0; n2 < 8; ++n2) w[n2] = pack_bf16(v[2 * n2], v[2 * n2 + 1]);
  const bool odd = lane & 1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t got = __shfl_xor_sync(0xffffffffu, odd ? w[i] : w[4 + i], 1);
    o[2 * i] = odd ? got : w[i];
    o[2 * i + 1] = odd ? w[4 + i] : got;
  }
  if (ok) {
    const uint32_t dst = mapa_shared(rb_me + (uint32_t)(((cu >> 1) * 16 + (odd ? 8 : 0)) * 4), q);
    st_async_v4_b32(dst, o[0], o[1], o[2], o[3], mbr);
    st_async_v4_b32(dst + 16, o[4], o[5], o[6], o[7], mbr);
  }
}

// pvec 2: receive block [n][PW] of 32-bit words, word (n, cu/2) = bf16 pair
// (column cu even, cu+1) of batch row n; PW = UPC/2 rounded up to 4 mod 8 so
// that 8 owner threads (rows b..b+7, same unit pair) hit 8 distinct bank
// groups.  A drain lane and its neighbour (columns cu, cu^1) swap 8 values so
// the even lane holds rows 0..N/2-1 of the column pair and the odd lane rows
// N/2..N-1; each pushes N/2 words.  The owner reads ONE word per source (no
// half-used words: half the shared-memory traffic of the [n/2][cu] layout).
__host__ __device__ constexpr int pair_pitch(int upc) { return ((upc / 2 + 3) / 8) * 8 + 4; }
template <int N>
__device__ __forceinline__ void push_col_pairs(const float* v, int lane, bool ok, int cu, int PW, uint32_t rb_me,
                                               uint32_t q, uint32_t mbr) {
  constexpr int H = N / 2;
  const bool odd = lane & 1;
  uint32_t w[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const float got = __shfl_xor_sync(0xffffffffu, odd ? v[i] : v[H + i], 1);
    w[i] = odd ? pack_bf16(got, v[H + i]) : pack_bf16(v[i], got);
  }
  if (ok) {
    const uint32_t dst = mapa_shared(rb_me + (uint32_t)(((odd ? H : 0) * PW + (cu >> 1)) * 4), q);
#pragma unroll
    for (int i = 0; i < H; ++i) st_async_b32(dst + (uint32_t)(i * PW * 4), __uint_as_float(w[i]), mbr);
  }
}

// push_col_pairs for the multi-cluster backward: the same shuffle, then each lane
// pushes to its owner's shared memory (`local`: owner in this cluster) or stores
// the words to the owner's global staging block `gdst` ([n][PW] words).
template <int N>
__device__ __forceinline__ void push_col_pairs_mc(const float* v, int lane, bool ok, bool local, int cu, int PW,
                                                  uint32_t rb_me, uint32_t q, uint32_t mbr, uint32_t* gdst) {
  constexpr int H = N / 2;
  const bool odd = lane & 1;
  uint32_t w[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const float got = __shfl_xor_sync(0xffffffffu, odd ? v[i] : v[H + i], 1);
    w[i] = odd ? pack_bf16(got, v[H + i]) : pack_bf16(v[i], got);
  }
  if (ok && local) {
    const uint32_t dst = mapa_shared(rb_me + (uint32_t)(((odd ? H : 0) * PW + (cu >> 1)) * 4), q);
#pragma unroll
    for (int i = 0; i < H; ++i) st_async_b32(dst + (uint32_t)(i * PW * 4), __uint_as_float(w[i]), mbr);
  } else if (ok) {
    uint32_t* g = gdst + (odd ? H : 0) * PW + (cu >> 1);
#pragma unroll
    for (int i = 0; i < H; ++i) g[i * PW] = w[i];
  }
}

// K-major, no-swizzle operand tile with `rows` rows: core matrix (k/8, r/8).
__device__ __forceinline__ uint32_t kmaj(int r, int k, int rows) {
  return (uint32_t)(((k >> 3) * (rows >> 3) + (r >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

// Forward MMA issue for K = 16*NK known at compile time (TMEM-A M=128 block
// interleaved with the SMEM-A M=64 block), out of line like issue_bwd_fixed.
template <int NK>
__device__ __noinline__ void issue_fwd_fixed(uint32_t d1, uint32_t ta, uint32_t d2, uint64_t a2, uint64_t bd,
                                             uint32_t id1, uint32_t id2) {
  constexpr uint64_t a2k = (2 * 64 * 16) >> 4, bk = (2 * 16 * 16) >> 4;
#pragma unroll
  for (int k = 0; k + 8 <= NK; k += 8)
    mma8_ts_ss(d1, ta + 8u * k, d2, a2 + k * a2k, a2k, bd + k * bk, bk, id1, id2, k > 0);
}

// ------------------------------------------------------------ forward ----
// MC = 1: the multi-cluster / K-split instance (NCL > 1 or Ks > 0); MC = 0 keeps
// the single-cluster code free of those branches (its register allocation and
// scheduling are what the headline numbers were measured with).
template <int V, int N, int MC>
__global__ void __launch_bounds__(MAXT, 1) cl_fwd_kernel(CArgs a) {
  using C = Cell<V>;
  constexpr int NS = C::NS, NG = C::NG, NGP = C::NGP;
  using M = Math<true>;
  const Problem& p = a.p;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31, NT = blockDim.x;
  const uint32_t me = cluster_ctarank();
  const int NCL = MC ? a.NCL : 1, Ks = MC ? a.Ks : 0;
  const int NSL = a.CL * NCL;                             // h slices per group
  const int grp = blockIdx.x / NSL;
  const int cl = MC ? (blockIdx.x / a.CL) % NCL : 0;      // this CTA's cluster within the group
  const int gq = MC ? cl * a.CL + (int)me : (int)me;      // this CTA's slice (unit block) within the group
  const int hd = grp / a.NBT, b0 = (grp % a.NBT) * N;
  const int nb = min(N, p.B - b0);
  const int unit0 = gq * a.UPC;
  const int DH = p.DH, D = p.D, B = p.B, K = a.K, T = p.T, Kt = a.K - Ks;
  // xs[b][row'] with row' = row + 4*(row/32): a pad of 4 words per 32 rows makes
  // both the TMEM drain (consecutive rows) and the pointwise float4 reads (8
  // consecutive rows per thread) bank-conflict free.
  const int ROWS = a.R1 + a.R2, XP = xs_pitch(ROWS);
  const bf16* R = static_cast<const bf16*>(p.R);
  const bf16* bias = static_cast<const bf16*>(p.bias);
  const bf16* x = static_cast<const bf16*>(p.x);
  const bf16* s0 = static_cast<const bf16*>(p.s0);
  bf16* states = static_cast<bf16*>(p.states);
  bf16* gates = static_cast<bf16*>(p.gates);

  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* hB0 = smem;                       // [N x K] K-major (step parity 0)
  uint8_t* hB1 = hB0 + N * K * 2;            // (step parity 1)
  uint8_t* A2 = hB1 + N * K * 2;             // [64 x K] K-major, rows R1..R1+R2 (or [128 x Ks]: K split)
  float* xs = reinterpret_cast<float*>(A2 + (a.R2 ? 64 * K * 2 : (MC && a.m64 ? 64 : 128) * Ks * 2));  // [N][ROWS+1]
  uint8_t* hs = reinterpret_cast<uint8_t*>(xs + N * XP);               // my h slice
  uint64_t* bars = reinterpret_cast<uint64_t*>(hs + ((a.slice + 15) & ~15u));  // mma, x0, x1
  // bars: MMA done, h(t) parity 0/1 (own cluster's slices), MC: other clusters' slices parity 0/1
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(bars + (MC ? 5 : 3));

  if (w == 0) tmem_alloc(tbase_s, a.tmem_cols);
  if (tid == 0) {
    for (int i = 0; i < (MC ? 5 : 3); ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 2 * N * K * 2 / 16; i += NT) reinterpret_cast<uint4*>(hB0)[i] = make_uint4(0, 0, 0, 0);
  if (a.R2) {  // R rows R1.. -> SMEM, K-major M=64 tile
    for (int i = tid; i < 64 * (K / 8); i += NT) {
      const int m = i % 64, kc = i / 64, r = a.R1 + m, u = r / NGP, g = r % NGP;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (m < a.R2 && g < NG && p.rec[g])
        v = *reinterpret_cast<const uint4*>(R + ((size_t)(hd * NG + g) * DH + unit0 + u) * DH + kc * 8);
      *reinterpret_cast<uint4*>(A2 + kmaj(m, kc * 8, 64)) = v;
    }
  }
  // K-step placement of the split block (MC).  Issue order: the own cluster's
  // steps [k0, k0+span) first, then the other clusters' steps ("remote", natural
  // order).  With mclocal each group is split between TMEM and SMEM in the
  // block's TS:SS ratio, so that both halves overlap their two operand paths:
  // TMEM positions [0, tsL) = local steps k0.., [tsL, nts) = remote steps 0..;
  // SMEM positions [0, ssL) = the rest of the local steps, then the rest of the
  // remote ones.  Without mclocal: TMEM = steps [0, nts), SMEM = [nts, nk).
  const int nkS = K / 16, ntsS = Kt / 16, nssS = Ks / 16;
  // (1: two clusters only -- with more, the remote part dominates and arrives piecemeal:
  //  H=1152 4.03 -> 4.55, H=1408 4.69 -> 5.77 us/step; 2: always)
  const bool loc = MC && NCL > 1 && (a.mclocal == 2 || (a.mclocal == 1 && NCL == 2));
  const int spanS = loc ? a.CL * a.UPC / 16 : nkS, k0S = loc ? cl * spanS : 0;
  const int tsL = loc ? max(max(0, spanS - nssS), min(min(spanS, ntsS), (spanS * ntsS + nkS / 2) / nkS)) : ntsS;
  const int ssL = spanS - tsL, tsR = ntsS - tsL;
  auto rstep = [&](int i) { return i < k0S ? i : i + spanS; };
  auto tpos_k = [&](int j) { return j < tsL ? k0S + j : rstep(j - tsL); };
  auto spos_k = [&](int j) { return j < ssL ? k0S + tsL + j : rstep(tsR + j - ssL); };
  const bool m64 = MC && a.m64;
  const int MR = m64 ? 64 : 128;  // rows of the split block's MMAs
  if (Ks) {  // the SMEM part of rows 0..R1-1 -> SMEM, K-major M=MR tile (positions: spos_k)
    for (int i = tid; i < MR * (Ks / 8); i += NT) {
      const int m = i % MR, kc = i / MR, u = m / NGP, g = m % NGP;
      const int kel = spos_k((kc * 8) >> 4) * 16 + ((kc * 8) & 15);
      uint4 v = make_uint4(0, 0, 0, 0);
      if (m < a.R1 && g < NG && p.rec[g])
        v = *reinterpret_cast<const uint4*>(R + ((size_t)(hd * NG + g) * DH + unit0 + u) * DH + kel);
      *reinterpret_cast<uint4*>(A2 + kmaj(m, kc * 8, MR)) = v;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, *tbase_s, 0);
  if (w < 4) {  // R rows 0..R1-1 -> TMEM: lane = row, columns = bf16 pairs along K
    const int row = 32 * w + l, u = row / NGP, g = row % NGP;
    const bool valid = row < a.R1 && g < NG && p.rec[g];
    const bf16* src = R + ((size_t)(hd * NG + (valid ? g : 0)) * DH + unit0 + (valid ? u : 0)) * DH;
    for (int c0 = 0; c0 < Kt / 2; c0 += 16) {
      uint32_t v[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = 2 * c0 + 8 * q;
        const int kel = MC ? tpos_k(k >> 4) * 16 + (k & 15) : k;  // (TMEM position k holds K element kel)
        uint4 r4 = make_uint4(0, 0, 0, 0);
        if (valid && k < DH && k < Kt) r4 = *reinterpret_cast<const uint4*>(src + kel);
        v[4 * q] = r4.x;
        v[4 * q + 1] = r4.y;
        v[4 * q + 2] = r4.z;
        v[4 * q + 3] = r4.w;
      }
      tmem_st16(tbase + ((uint32_t)(32 * w) << 16) + c0, v);
    }
    tmem_st_wait();
  }
  // ---- element ownership: one pair (u, u+1) of one batch row b per thread
  const int NP = a.UPC / 2;
  const bool own = tid < NP * N;
  int u, b;
  own_pair(tid, NP, u, b, a.map);
  const bool valid = own && b < nb;
  const int e = hd * DH + unit0 + u;
  const size_t so = (size_t)(b0 + b) * D + e;       // offset in [.][B][D] tensors
  const size_t xo = (size_t)(b0 + b) * NG * D + e;  // offset in [.][B][NG][D] tensors
  const size_t sstep = (size_t)NS * B * D, gstep = (size_t)NG * B * D;
  float st[NS][2], bj[NG][2];
  uint32_t xr[NG], xn[NG];
  float gsave[NG][2], nsave[NS][2];  // step t-1 outputs, stored while MMA(t) runs
#pragma unroll
  for (int j = 0; j < NG; ++j) {
    bj[j][0] = own ? bf(bias, (size_t)j * D + e) : 0.f;
    bj[j][1] = own ? bf(bias, (size_t)j * D + e + 1) : 0.f;
    xr[j] = xn[j] = 0;
    gsave[j][0] = gsave[j][1] = 0.f;
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) nsave[s][0] = nsave[s][1] = 0.f;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const uint32_t v = valid ? ld2(s0, (size_t)s * B * D + so) : 0u;
    st[s][0] = lo16(v);
    st[s][1] = hi16(v);
    if (valid) *reinterpret_cast<uint32_t*>(states + (size_t)s * B * D + so) = v;  // states[0] = s0
  }
  if (valid && T > 0) {
#pragma unroll
    for (int j = 0; j < NG; ++j)
      if (p.inp[j]) xr[j] = ld2(x, xo + (size_t)j * D);
  }
  // h_0 tile straight from s0 into hB0
  for (int i = tid; i < nb * (K / 8); i += NT) {
    const int bb = i % nb, kc = i / nb;
    *reinterpret_cast<uint4*>(hB0 + kmaj(bb, kc * 8, N)) =
        *reinterpret_cast<const uint4*>(s0 + (size_t)(b0 + bb) * D + hd * DH + kc * 8);
  }
  fence_proxy_async_smem();
  if (tid == 0) {  // step 1's h
    mbar_arrive_expect_tx(&bars[2], (uint32_t)a.CL * a.slice);
    if (NCL > 1) mbar_arrive_expect_tx(&bars[4], (uint32_t)(NCL - 1) * a.CL * a.slice);
  }
  __syncthreads();
  cluster_sync_all();  // all barriers initialised + armed before any multicast

  const uint32_t idesc1 = idesc_bf16(128, N), idesc2 = idesc_bf16(64, N);
  constexpr uint32_t LBO = N * 16, SBO = 128;
  const uint16_t mask = (uint16_t)((1u << a.CL) - 1u);
  for (int t = 0; t < T; ++t) {
    const int buf = t & 1;
    FRNN_PROF(0, t);
    if (w == 0) {
      if (t > 0) mbar_wait_cluster(&bars[1 + buf], ((t - 1) >> 1) & 1);
      FRNN_PROF(1, t);
      tc_fence_after();
      const uint64_t bd = sdesc_kmajor(smem_u32(buf ? hB1 : hB0), LBO, SBO);
      if (MC) {  // (skeleton mode: the barrier waits still run, only the MMAs are skipped)
        // One M=128 block, K split TMEM | SMEM.  The own cluster's K range first
        // (its slices arrive by multicast ~1 k cycles after publishing), then the
        // other clusters' slices once their L2 imports have landed.
        const uint64_t a2 = sdesc_kmajor(smem_u32(A2), MR * 16, 128), a2k = (uint64_t)(2 * MR * 16) >> 4,
                       bk = (2 * LBO) >> 4;
        const uint32_t d1 = tbase + a.acc1, d2 = tbase + a.acc2;
        const uint32_t ids = m64 ? idesc2 : idesc1;  // the SMEM half: M=64 tile for blocks of <= 64 rows
        if (!loc) {  // TMEM steps [0, nts), SMEM steps [nts, nk), after every slice arrived
          if (NCL > 1 && t > 0) mbar_wait_cluster(&bars[3 + buf], ((t - 1) >> 1) & 1);
          tc_fence_after();
          if (!a.skeleton)
            mma_chain_ksplit(d1, tbase, bd, ntsS, 0, d2, a2, a2k, bd + (uint64_t)ntsS * bk, nssS, 0, bk, idesc1, ids);
        } else {
          // own cluster's steps: TMEM positions [0, tsL), SMEM positions [0, ssL)
          if (!a.skeleton)
            mma_chain_ksplit(d1, tbase, bd + (uint64_t)k0S * bk, tsL, 0, d2, a2, a2k, bd + (uint64_t)(k0S + tsL) * bk,
                             ssL, 0, bk, idesc1, ids);
          if (t > 0) mbar_wait_cluster(&bars[3 + buf], ((t - 1) >> 1) & 1);
          tc_fence_after();
          // remote steps r(i) = i (< k0) | i + span, TMEM i in [0, tsR), SMEM i in [tsR, nR): each
          // stream in two contiguous pieces (before / after the own range)
          const int nR = nkS - spanS;
          const int ta_ = min(tsR, k0S), tb_ = tsR - ta_;
          const int sa_ = max(0, k0S - tsR), sb0 = max(tsR, k0S), sb_ = nR - sb0;
          if (!a.skeleton) {
            mma_chain_ksplit(d1, tbase + 8u * tsL, bd, ta_, tsL > 0, d2, a2 + (uint64_t)ssL * a2k, a2k,
                             bd + (uint64_t)tsR * bk, sa_, ssL > 0, bk, idesc1, ids);
            mma_chain_ksplit(d1, tbase + 8u * (tsL + ta_), bd + (uint64_t)(ta_ + spanS) * bk, tb_, tsL + ta_ > 0, d2,
                             a2 + (uint64_t)(ssL + sa_) * a2k, a2k, bd + (uint64_t)(sb0 + spanS) * bk, sb_,
                             ssL + sa_ > 0, bk, idesc1, ids);
          }
        }
      } else if (a.skeleton) {
      } else if (a.R2 && K == 768) {  // H=768 per head: 6 blocks of 8 K-steps, spelled out
        const uint64_t a2 = sdesc_kmajor(smem_u32(A2), 64 * 16, 128);
        constexpr uint64_t a2k = (2 * 64 * 16) >> 4, bk = (2 * LBO) >> 4;
        const uint32_t d1 = tbase + a.acc1, d2 = tbase + a.acc2;
        mma8_ts_ss(d1, tbase, d2, a2, a2k, bd, bk, idesc1, idesc2, 0);
        mma8_ts_ss(d1, tbase + 64, d2, a2 + 8 * a2k, a2k, bd + 8 * bk, bk, idesc1, idesc2, 1);
        mma8_ts_ss(d1, tbase + 128, d2, a2 + 16 * a2k, a2k, bd + 16 * bk, bk, idesc1, idesc2, 1);
        mma8_ts_ss(d1, tbase + 192, d2, a2 + 24 * a2k, a2k, bd + 24 * bk, bk, idesc1, idesc2, 1);
        mma8_ts_ss(d1, tbase + 256, d2, a2 + 32 * a2k, a2k, bd + 32 * bk, bk, idesc1, idesc2, 1);
        mma8_ts_ss(d1, tbase + 320, d2, a2 + 40 * a2k, a2k, bd + 40 * bk, bk, idesc1, idesc2, 1);
      } else if (N == 16 && a.R2 && K == 640) {
        issue_fwd_fixed<40>(tbase + a.acc1, tbase, tbase + a.acc2, sdesc_kmajor(smem_u32(A2), 64 * 16, 128), bd, idesc1,
                            idesc2);
      } else if (N == 16 && a.R2 && K == 512) {
        issue_fwd_fixed<32>(tbase + a.acc1, tbase, tbase + a.acc2, sdesc_kmajor(smem_u32(A2), 64 * 16, 128), bd, idesc1,
                            idesc2);
      } else if (a.R2 && K == 192) {  // DH=192 per head (config 3): one 12-step block
        mma12_ts_ss(tbase + a.acc1, tbase, tbase + a.acc2, sdesc_kmajor(smem_u32(A2), 64 * 16, 128),
                    (2 * 64 * 16) >> 4, bd, (2 * LBO) >> 4, idesc1, idesc2, 0);
      } else if (a.R2) {
        mma_run_ts_ss(tbase + a.acc1, tbase, tbase + a.acc2, sdesc_kmajor(smem_u32(A2), 64 * 16, 128),
                      (2 * 64 * 16) >> 4, bd, (2 * LBO) >> 4, idesc1, idesc2, K / 16);
      } else {
        mma_run_ts(tbase + a.acc1, tbase, 8, bd, (2 * LBO) >> 4, idesc1, K / 16);
      }
      if (elect_one()) mma_commit(&bars[0]);
      __syncwarp();
    }
    // Off the critical path, while MMA(t) runs: the trace of step t-1 and the
    // x_{t+1} prefetch (predicated loads: issuing never waits for them).
    if (valid) {
      if (t > 0) {
        bf16* gdst = gates + (size_t)(t - 1) * gstep + so;
        bf16* sdst = states + (size_t)t * sstep + so;
#pragma unroll
        for (int j = 0; j < NG; ++j) st2(gdst, (size_t)j * B * D, gsave[j][0], gsave[j][1]);
#pragma unroll
        for (int s = 0; s < NS; ++s) st2(sdst, (size_t)s * B * D, nsave[s][0], nsave[s][1]);
      }
      if (t + 1 < T) {
        const bf16* xp = x + (size_t)(t + 1) * gstep + xo;
#pragma unroll
        for (int j = 0; j < NG; ++j)
          if (p.inp[j]) xn[j] = ld2(xp, (size_t)j * D);
      }
      // x two steps ahead into L2 (no registers): next step's register loads then
      // wait for L2, not HBM (one prefetch per 32-byte sector of a row)
      if (a.xpf && t + 2 < T && (u & 15) == 0) {
        const bf16* xq = x + (size_t)(t + 2) * gstep + xo;
#pragma unroll
        for (int j = 0; j < NG; ++j)
          if (p.inp[j]) prefetch_l2(xq + (size_t)j * D);
      }
    }
    if (w == 0) mbar_wait(&bars[0], t & 1);  // (the issuing warp spins)
    else mbar_wait_idle(&bars[0], t & 1, a.waitmode);
    tc_fence_after();
    FRNN_PROF(2, t);
    // accumulators -> xs[b][row]: warps 0-3 drain the M=128 block, warps 4-7 (same
    // lane quadrants) the M=64 block in parallel
    if (w < 4) {
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(32 * w) << 16) + a.acc1, v);
      if (Ks && !m64) {  // (m64: accumulator 2 is an M=64 tile, added below)
        float v2[16];
        tmem_ld16(tbase + ((uint32_t)(32 * w) << 16) + a.acc2, v2);
#pragma unroll
        for (int n = 0; n < N; ++n) v[n] += v2[n];
      }
      if (32 * w + l < a.R1) {
#pragma unroll
        for (int n = 0; n < N; ++n) xs[n * XP + xs_row(32 * w + l)] = v[n];
      }
    } else if (w < 8 && a.R2) {  // M=64 layout: rows 16q..16q+15 in lanes 32q..32q+15
      const int q = w & 3;
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + a.acc2, v);
      if (l < 16 && 16 * q + l < a.R2) {
#pragma unroll
        for (int n = 0; n < N; ++n) xs[n * XP + xs_row(a.R1 + 16 * q + l)] = v[n];
      }
    }
    if (m64) {  // the split block's M=64 SMEM half, added to the drained M=128 half
      __syncthreads();
      if (w < 4) {
        float v2[16];
        tmem_ld16(tbase + ((uint32_t)(32 * w) << 16) + a.acc2, v2);
        if (l < 16 && 16 * w + l < a.R1) {
#pragma unroll
          for (int n = 0; n < N; ++n) xs[n * XP + xs_row(16 * w + l)] += v2[n];
        }
      }
    }
    tc_fence_before();
    __syncthreads();
    if (!MC) FRNN_PROF(5, t);
    float gout[NG][2], nout[NS][2];
    if (own) {
      float y[2][4];  // the pair's 2*NGP consecutive gate rows at column b
      if (NGP == 4) {
        const float4 y0 = *reinterpret_cast<const float4*>(xs + b * XP + xs_row(u * 4));
        const float4 y1 = *reinterpret_cast<const float4*>(xs + b * XP + xs_row(u * 4 + 4));
        y[0][0] = y0.x, y[0][1] = y0.y, y[0][2] = y0.z, y[0][3] = y0.w;
        y[1][0] = y1.x, y[1][1] = y1.y, y[1][2] = y1.z, y[1][3] = y1.w;
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int j = 0; j < NG; ++j) y[h][j] = xs[b * XP + xs_row((u + h) * NGP + j)];
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float g[4], prev[4], nx[4];
#pragma unroll
        for (int j = 0; j < NG; ++j) {  // x, then b, then y (engine.hpp:183-187)
          g[j] = (h ? hi16(xr[j]) : lo16(xr[j])) + bj[j][h] + y[h][j];
          gout[j][h] = g[j];
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) prev[s] = st[s][h];
        if (a.skeleton) {
#pragma unroll
          for (int s = 0; s < NS; ++s) nx[s] = g[s & 3];
        } else {
          C::template fwd<M>(prev, g, nx);
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) st[s][h] = nout[s][h] = nx[s];
      }
      if (!MC) FRNN_PROF(6, t);
      const uint32_t hword = b < nb ? pack_bf16(nout[0][0], nout[0][1]) : 0u;  // padding rows stay zero
      if (a.hdirect && t + 1 < T) {  // straight into the global staging slice (the multicast source)
        uint8_t* gst = reinterpret_cast<uint8_t*>(a.xstage) + (((size_t)grp * 2 + ((t + 1) & 1)) * NSL + gq) * a.slice;
        *reinterpret_cast<uint32_t*>(gst + kmaj(b, u, N)) = hword;
        fence_proxy_async_global();  // this writer's generic store -> the multicast's async-proxy read
      } else {
        *reinterpret_cast<uint32_t*>(hs + kmaj(b, u, N)) = hword;
      }
    }
    __syncthreads();
    FRNN_PROF(3, t);
    if (t + 1 < T) {  // publish h_{t+1}: slice -> global staging -> multicast to the cluster
      const int nbuf = (t + 1) & 1;
      uint8_t* gst = reinterpret_cast<uint8_t*>(a.xstage) + (((size_t)grp * 2 + nbuf) * NSL + gq) * a.slice;
      if (!a.hdirect) {
        for (int i = tid; i < (int)(a.slice / 16); i += NT)
          reinterpret_cast<uint4*>(gst)[i] = reinterpret_cast<const uint4*>(hs)[i];
        if (tid < (int)(a.slice / 16)) fence_proxy_async_global();  // the writers' generic -> async proxy order
        __syncthreads();
      }
      FRNN_PROF(7, t);
      if constexpr (!MC) {
        if (tid == 0) {
          mbar_arrive_expect_tx(&bars[1 + buf], (uint32_t)a.CL * a.slice);  // re-arm for step t+2
          fence_proxy_async_global();
          bulk_g2s_multicast((nbuf ? hB1 : hB0) + me * a.slice, gst, a.slice, &bars[1 + nbuf], mask);
        }
      } else {
      uint8_t* hBn = nbuf ? hB1 : hB0;
      if (tid == 0) {
        mbar_arrive_expect_tx(&bars[1 + buf], (uint32_t)a.CL * a.slice);  // re-arm for step t+2
        if (NCL > 1) mbar_arrive_expect_tx(&bars[3 + buf], (uint32_t)(NCL - 1) * a.CL * a.slice);
        fence_proxy_async_global();
        bulk_g2s_multicast(hBn + gq * a.slice, gst, a.slice, &bars[1 + nbuf], mask);
        if (NCL > 1 && !a.mcrelw) {  // release the slice to the group's other clusters
          if (a.mcfence) __threadfence();
          st_release_gpu(a.xflags + (size_t)grp * NSL + gq, (uint32_t)(t + 1));
        }
      }
      if (NCL > 1 && w == a.mcwarp) {
        // Import the other clusters' slices at this CTA's position: lane c of warp
        // 1 (not the MMA-issuing warp 0) pulls slice (c, me) of cluster c from L2
        // and multicasts it to this cluster, all clusters in parallel.  Double-
        // buffered staging is safe: the writer of step t+3 has consumed h_{t+2},
        // which needs every importer's step t+1.
        uint32_t* fl = a.xflags + (size_t)grp * NSL;
        if (a.mcrelw && l == 0) {  // the release (it waits for the slice stores) off the MMA-issuing warp
          if (a.mcfence) __threadfence();
          st_release_gpu(fl + gq, (uint32_t)(t + 1));
        }
        __syncwarp();
        for (int c = l; c < NCL; c += 32) {
          if (c == cl) continue;
          const int q = c * a.CL + (int)me;
          if (a.mcpoll) spin_until_geq_relaxed(fl + q, (uint32_t)(t + 1));
          else spin_until_geq(fl + q, (uint32_t)(t + 1));
          if (a.prof && c == (cl == 0 ? 1 : 0) && t + 1 < a.prof_steps)  // remote flag seen (step t+1's data)
            a.prof[((size_t)blockIdx.x * a.prof_steps + (t + 1)) * 8 + 6] = clock64();
          fence_proxy_async_global();
          const uint8_t* rsrc =
              reinterpret_cast<const uint8_t*>(a.xstage) + (((size_t)grp * 2 + nbuf) * NSL + q) * a.slice;
          bulk_g2s_multicast(hBn + q * a.slice, rsrc, a.slice, &bars[3 + nbuf], mask);
        }
        __syncwarp();
      }
      }
    }
    FRNN_PROF(4, t);
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      gsave[j][0] = gout[j][0];
      gsave[j][1] = gout[j][1];
      xr[j] = xn[j];
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      nsave[s][0] = nout[s][0];
      nsave[s][1] = nout[s][1];
    }
  }
  if (valid && T > 0) {  // the last step's trace
    bf16* gdst = gates + (size_t)(T - 1) * gstep + so;
    bf16* sdst = states + (size_t)T * sstep + so;
#pragma unroll
    for (int j = 0; j < NG; ++j) st2(gdst, (size_t)j * B * D, gsave[j][0], gsave[j][1]);
#pragma unroll
    for (int s = 0; s < NS; ++s) st2(sdst, (size_t)s * B * D, nsave[s][0], nsave[s][1]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while a peer's multicast may target it
  if (w == 0) tmem_dealloc(tbase, a.tmem_cols);
}

// Backward MMA issue for a tiling known at compile time: MBT TMEM-A blocks, MS
// SMEM-A blocks of 128 columns (paired with the first MS TMEM blocks), NK K-steps
// per block, N=16 -- every offset a constant, straight-line issue (the generic
// runtime loop is markedly slower at N=16, see DESIGN 8c).
template <int MBT_, int MS_, int NK>
__device__ __noinline__ void issue_bwd_fixed(uint32_t tbase, uint32_t acc1, uint64_t bd, uint64_t ad, uint32_t idesc,
                                                uint32_t idesc2, uint64_t* blkbar) {
  constexpr int NP = MBT_ > MS_ ? MBT_ : MS_, CB = NK * 8;
  constexpr uint64_t bk = (2 * 16 * 16) >> 4, a2k = (2 * 128 * 16) >> 4, blk16 = (uint64_t)128 * NK * 16 * 2 >> 4;
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const uint32_t accT = acc1 + i * 16, accS = acc1 + (MBT_ + i) * 16;
    if (i < MBT_ && i < MS_) mma_run_ts_ss(accT, tbase + i * CB, accS, ad + i * blk16, a2k, bd, bk, idesc, idesc2, NK);
    else if (i < MBT_) mma_run_ts(accT, tbase + i * CB, 8, bd, bk, idesc, NK);
    else mma_run_ss(accS, ad + i * blk16, a2k, bd, bk, idesc2, NK);
    if (elect_one()) mma_commit(&blkbar[i]);
    __syncwarp();
  }
}

// Every backward tiling (TMEM blocks MBT, SMEM blocks MS of 128 columns, K steps
// NK) the planner launches for 16 <= DH <= 1024 and any cell (enumerated with
// scripts/tilings.py / frnn_debug_cluster_shape), each a straight-line issue
// instance; (4,2,12), (6,0,3) and (2,0,12) are spelled out in the kernel.
#define FRNN_BWD_TILINGS(X)                                                                                       \
  X(1, 0, 1) X(1, 0, 2) X(1, 0, 3) X(1, 0, 4) X(1, 0, 8) X(1, 0, 10) X(1, 0, 12) X(2, 0, 1) X(2, 0, 2) X(2, 0, 3) \
  X(2, 0, 4) X(2, 0, 8) X(2, 0, 10) X(3, 0, 2) X(3, 0, 3) X(3, 0, 8) X(3, 0, 10) X(3, 0, 12) X(4, 0, 2)          \
  X(4, 0, 3) X(4, 0, 8) X(4, 0, 10) X(4, 0, 12) X(4, 1, 12) X(5, 0, 3) X(5, 0, 10) X(3, 4, 14)            \
  X(1, 0, 6) X(1, 0, 9) X(2, 0, 6) X(2, 0, 9) X(3, 0, 6) X(3, 0, 9) X(4, 0, 6) X(4, 0, 9) X(5, 0, 9) X(5, 1, 9)
__device__ __forceinline__ bool issue_bwd_table(int MBT, int MS, int nk, uint32_t tbase, uint32_t acc1, uint64_t bd,
                                                uint64_t ad, uint32_t idesc, uint32_t idesc2, uint64_t* blkbar) {
  switch (MBT * 1000 + MS * 100 + nk) {
#define FRNN_BWD_CASE(M_, S_, K_)                                   \
  case M_ * 1000 + S_ * 100 + K_:                                   \
    issue_bwd_fixed<M_, S_, K_>(tbase, acc1, bd, ad, idesc, idesc2, blkbar); \
    return true;
    FRNN_BWD_TILINGS(FRNN_BWD_CASE)
#undef FRNN_BWD_CASE
  }
  return false;
}

// The multi-cluster backward's tilings (H = 896 / 1024 / 1152 4-gate), a separate
// table so that the single-cluster instances keep their code (adding cases to
// the shared switch moved their register allocation: NH=12 backward +2 %).
__device__ __forceinline__ bool issue_bwd_table_mc(int MBT, int MS, int nk, uint32_t tbase, uint32_t acc1, uint64_t bd,
                                                   uint64_t ad, uint32_t idesc, uint32_t idesc2, uint64_t* blkbar) {
  switch (MBT * 1000 + MS * 100 + nk) {
#define FRNN_BWD_CASE(M_, S_, K_)                                             \
  case M_ * 1000 + S_ * 100 + K_:                                             \
    issue_bwd_fixed<M_, S_, K_>(tbase, acc1, bd, ad, idesc, idesc2, blkbar); \
    return true;
    FRNN_BWD_CASE(6, 1, 8) FRNN_BWD_CASE(6, 2, 8) FRNN_BWD_CASE(7, 2, 6)
#undef FRNN_BWD_CASE
  }
  return false;
}

constexpr bool mc_issue_instance(int MBT, int MS, int nk) {
  return (MBT == 6 && MS == 1 && nk == 8) || (MBT == 6 && MS == 2 && nk == 8) || (MBT == 7 && MS == 2 && nk == 6);
}

// ----------------------------------------------------------- backward ----
// L = 1: the H=768 4-gate layout (every tiling branch fixed at compile time);
// L = 4: multi-cluster (NCL > 1, 4-gate cells, bf16 column-pair exchange)
template <int V, int N, int L>
__global__ void __launch_bounds__(MAXT, 1) cl_bwd_kernel(CArgs a) {
  using C = Cell<V>;
  constexpr int NS = C::NS, NG = C::NG, NGP = C::NGP;
  // backward K rows per unit: the padded NGP, or (a.kcompact, GRU) only the gates with R
  const int NGK = a.kcompact ? C::NGK : NGP;
  auto kgate = [&](int q) { return a.kcompact ? C::kgate(q) : q; };
  using M = Math<true>;
  const Problem& p = a.p;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31, NT = blockDim.x;
  const uint32_t me = cluster_ctarank();
  // L == 4: the head's units over NCL clusters; partials for owners in other
  // clusters travel through L2 (pstage) behind per-source release counters
  constexpr bool MCB = L == 4;
  const int NCL = MCB ? a.NCL : 1, NSL = a.CL * NCL;
  const int grp = blockIdx.x / NSL;
  const int cl = MCB ? (blockIdx.x / a.CL) % NCL : 0;
  const int gq = MCB ? cl * a.CL + (int)me : (int)me;
  const int hd = grp / a.NBT, b0 = (grp % a.NBT) * N;
  const int nb = min(N, p.B - b0);
  const int unit0 = gq * a.UPC;
  const int DH = p.DH, D = p.D, B = p.B, T = p.T, KBP = a.KBP, MB = a.MB, MBT = a.MBT;
  const bool recur = p.clip_mode != 2;
  const float mag = p.clip_mag;
  const bf16* R = static_cast<const bf16*>(p.R);
  const bf16* states = static_cast<const bf16*>(p.cstates);
  const bf16* gates = static_cast<const bf16*>(p.cgates);
  const bf16* dsf = static_cast<const bf16*>(p.dsf);
  const bf16* dh = static_cast<const bf16*>(p.dh);
  bf16* dx = static_cast<bf16*>(p.dx);
  bf16* ds0 = static_cast<bf16*>(p.ds0);
  // L == 1 pins the headline tiling (MBT 4 x TMEM + MS 2 x SMEM 128-column blocks,
  // K = 192, UPC 48, 16 CTAs, 384 threads, DSMEM row exchange of bf16 column
  // pairs): every runtime tiling branch below folds away, so the step loop is a
  // fraction of the generic kernel's code (i-cache: the generic instantiation is
  // ~16 k SASS instructions).
  constexpr bool FX = L == 1;
  // L >= 1 (lean): only the default exchange (DSMEM row pushes; bf16 column pairs
  // for 4-gate cells; unrolled absorb) is compiled in -- the A/B variants of the
  // generic L = 0 instance cost the other tilings up to 25 % through code
  // generation alone (same runtime path, measured)
  constexpr bool LEAN = L >= 1;
  // L == 3: lean, and no coefficient split, A/B or debug switch compiled in
  constexpr bool RAW = L == 3;
  const bool k_noxchg = !RAW && a.noxchg, k_nodx = !RAW && a.nodx, k_noload = !RAW && a.noload;
  const bool dxearly = !RAW && a.dxearly;
  const bool pbf = FX || (a.pbf16 && a.dsm == 2);  // partials exchanged as bf16 pairs
  const int PW = pair_pitch(a.UPC);        // pvec 2 receive row pitch (words)
  const uint32_t recv_bytes = (uint32_t)a.CL * N * a.UPC * (pbf ? 2 : 4);  // exchanged bytes (expect_tx)
  const uint32_t recv_span = pbf && a.pvec == 2 ? (uint32_t)a.CL * N * PW * 4 : recv_bytes;  // buffer bytes
  const int MS = a.MS, SSM = a.SSM, NPAIR = max(MBT, MS);
  const size_t blk_bytes = (size_t)SSM * KBP * 2;  // one SMEM-A block

  extern __shared__ __align__(1024) uint8_t smem[];
  const bool dsm = LEAN || a.dsm != 0;
  const int TP = a.UPC + 2;                                              // term pitch (bank spread)
  uint8_t* AS = smem;                                                    // MS x [SSM x KBP] K-major
  float* recv = reinterpret_cast<float*>(AS + MS * blk_bytes);          // global mode: [CL src][N][UPC]
  float* recv1 = dsm ? recv + recv_span / 4 : recv;                     // DSMEM mode: 2 x [CL src][UPC][N]
  uint8_t* dgB = reinterpret_cast<uint8_t*>(recv1) + recv_span;         // [N x KBP] K-major
  // db scratch [NG][N][UPC] (after the loop only): aliases the receive buffers when
  // they are large enough -- keeping the CTA's shared memory small leaves the SM's
  // unified L1 room for the per-thread trace loads / dx stores (cluster_shape)
  const bool dbs_alias = (uint32_t)NG * N * a.UPC * 4 <= (dsm ? 2u : 1u) * recv_span;
  float* after_dg = reinterpret_cast<float*>(dgB + N * KBP * 2);
  float* dbs = dbs_alias ? recv : after_dg;
  float* term = dbs_alias ? after_dg : after_dg + NG * N * a.UPC;     // dsm 1 only: [N][TP] summed R^T dg
  uint64_t* bars = reinterpret_cast<uint64_t*>(term + (!FX && a.dsm == 1 ? N * TP : 0));  // -, rcv, rdy0|rcv0, rdy1|rcv1
  uint64_t* blkbar = bars + 4;  // [NPAIR]: MMAs of block pair i (and all before it) complete
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(blkbar + 16);
  // MCB: barrier + receive buffer [remote src][N][PW] words for the other clusters' partials
  uint64_t* rbar = blkbar + 17;
  uint32_t* rrecv = reinterpret_cast<uint32_t*>(blkbar + 18);

  // Column rotation: CTA `me` lays out its R^T column blocks starting at column
  // me*UPC, so the block it computes LAST (whose partials arrive after the MMAs)
  // belongs to different owners in every CTA.  Unrotated, all 16 CTAs' last
  // blocks hit the same 3 owners, whose DSMEM ingress then serialises the tail.
  const int crot = (!RAW && a.rot) ? (int)(((long long)me * a.UPC) % DH) : 0;
  auto rotc = [&](int c) { return c < DH ? (c + crot) % DH : c; };  // padding columns stay padding
  if (w == 0) tmem_alloc(tbase_s, a.tmem_cols);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], dsm ? 1 : a.CL);
    mbar_init(&bars[3], dsm ? 1 : a.CL);
    for (int i = 0; i < NPAIR; ++i) mbar_init(&blkbar[i], 1);
    if (MCB) mbar_init(rbar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < N * KBP * 2 / 16; i += NT) reinterpret_cast<uint4*>(dgB)[i] = make_uint4(0, 0, 0, 0);
  if (recur) {  // R_slice^T blocks in SMEM: element (column m, row k) of block ib
    for (int ib = 0; ib < MS; ++ib) {
      uint8_t* blk = AS + ib * blk_bytes;
      for (int i = tid; i < SSM * KBP; i += NT) {
        const int m = i % SSM, k = i / SSM, c = rotc(MBT * 128 + ib * SSM + m), uu = k / NGK, g = kgate(k % NGK);
        const float v = (c < DH && uu < a.UPC && g < NG && p.rec[g])
                            ? bf(R, ((size_t)(hd * NG + g) * DH + unit0 + uu) * DH + c) : 0.f;
        *reinterpret_cast<bf16*>(blk + kmaj(m, k, SSM)) = __float2bfloat16_rn(v);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, *tbase_s, 0);
  if (recur && w < 4) {  // R_slice^T blocks in TMEM: lane = state column, columns = row pairs
    for (int mb = 0; mb < MBT; ++mb) {
      const int c = rotc(mb * 128 + 32 * w + l);
      for (int c0 = 0; c0 < KBP / 2; c0 += 16) {
        uint32_t v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float f[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = 2 * (c0 + q) + h, uu = row / NGK, g = kgate(row % NGK);
            f[h] = (c < DH && uu < a.UPC && g < NG && p.rec[g])
                       ? bf(R, ((size_t)(hd * NG + g) * DH + unit0 + uu) * DH + c) : 0.f;
          }
          v[q] = pack_bf16(f[0], f[1]);
        }
        tmem_st16(tbase + ((uint32_t)(32 * w) << 16) + mb * (KBP / 2) + c0, v);
      }
    }
    tmem_st_wait();
  }
  fence_proxy_async_smem();
  // ---- element ownership: one pair (u, u+1) of one batch row b per thread
  const int NP = a.UPC / 2;
  const bool own = tid < NP * N;
  int u, b;
  own_pair(tid, NP, u, b, a.map);
  const bool valid = own && b < nb;
  const int e = hd * DH + unit0 + u;
  const size_t so = (size_t)(b0 + b) * D + e;       // [.][B][D]
  const size_t xo = (size_t)(b0 + b) * p.NG * D + e;  // [.][B][NG][D]
  const size_t sstep = (size_t)NS * B * D, gstep = (size_t)NG * B * D;
  float ds[NS][2], dbv[NG][2];
  float kc[2][C::NK];  // Jacobian coefficients of the step about to be applied
  uint32_t pv[NS], gv[NG], hv = 0;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const uint32_t v = valid ? ld2(dsf, (size_t)s * B * D + so) : 0u;
    ds[s][0] = lo16(v);
    ds[s][1] = hi16(v);
    pv[s] = 0;
  }
#pragma unroll
  for (int j = 0; j < NG; ++j) {
    dbv[j][0] = dbv[j][1] = 0.f;
    gv[j] = 0;
  }
  // Predicated loads (no select on the loaded value): issuing the prefetch
  // never waits for it.  The trace of step t is loaded two steps ahead: its
  // Jacobian coefficients are formed during step t+1's MMA window.
  auto load_trace = [&](int t) {
    if (valid && t >= 0 && !k_noload) {
#pragma unroll
      for (int s = 0; s < NS; ++s) pv[s] = ld2(states, (size_t)t * sstep + (size_t)s * B * D + so);
#pragma unroll
      for (int j = 0; j < NG; ++j) gv[j] = ld2(gates, (size_t)t * gstep + (size_t)j * B * D + so);
    }
  };
  auto load_dh = [&](int t) {
    if (valid && t >= 0 && dh) hv = ld2(dh, (size_t)t * B * D + so);
  };
  auto coefs = [&]() {  // kc <- Jacobian coefficients of the trace in pv/gv (cell.hpp:108-201)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float prev[4], g[4];
#pragma unroll
      for (int s = 0; s < NS; ++s) prev[s] = h ? hi16(pv[s]) : lo16(pv[s]);
#pragma unroll
      for (int j = 0; j < NG; ++j) g[j] = h ? hi16(gv[j]) : lo16(gv[j]);
      C::template coef<M>(prev, g, kc[h]);
    }
  };
  load_trace(T - 1);
  load_dh(T - 1);
  // csplit: the coefficients of step t-1 are formed under step t's MMAs (trace
  // loaded two steps ahead); otherwise (short MMA windows, where the extra MUFU
  // work competes with the MMA-issuing warp) right before they are applied.
  const bool csplit = !RAW && a.csplit != 0;
  if (csplit) {
    if (T > 0) coefs();
    load_trace(T - 2);
  }
  __syncthreads();
  cluster_sync_all();  // barrier inits visible before any remote arrive

  // Partials of step s are in pstage[grp][s&1][me][*]: wait for the CL
  // producers, pull them with one bulk load, sum, clip, add to ds_h.
  uint32_t rcv_phase = 0, par_phase = 0, rphase = 0;
  auto absorb_dsm = [&](int s) {  // partials pushed into my recv[s&1] by every peer (st.async)
    const int pb = s & 1;
    if (tid == 0) mbar_arrive_expect_tx(&bars[2 + pb], recv_bytes);
    mbar_wait_cluster(&bars[2 + pb], (par_phase >> pb) & 1u);
    par_phase ^= 1u << pb;
    const float* rb = pb ? recv1 : recv;  // [src][cu][N]
    if (tid < a.UPC * (N / 4)) {          // sum over sources: one float4 of 4 batch rows per thread
      const int cu = tid / (N / 4), g = tid % (N / 4);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q = 0; q < a.CL; ++q) {  // fixed source order: deterministic
        const float4 v = *reinterpret_cast<const float4*>(rb + ((size_t)q * a.UPC + cu) * N + 4 * g);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      term[(4 * g + 0) * TP + cu] = acc.x;
      term[(4 * g + 1) * TP + cu] = acc.y;
      term[(4 * g + 2) * TP + cu] = acc.z;
      term[(4 * g + 3) * TP + cu] = acc.w;
    }
    __syncthreads();
    if (own) {
      const float2 v = *reinterpret_cast<const float2*>(term + b * TP + u);
      float t0 = v.x, t1 = v.y;
      if (p.clip_mode == 1) {
        t0 = fminf(fmaxf(t0, -mag), mag);
        t1 = fminf(fmaxf(t1, -mag), mag);
      }
      ds[0][0] += t0;
      ds[0][1] += t1;
    }
  };
  auto absorb_rows = [&](int s) {  // DSMEM mode 2: recv[s&1] is [src][n][cu], like the global staging
    const int pb = s & 1;
    if (!k_noxchg) {
      if (tid == 0) mbar_arrive_expect_tx(&bars[2 + pb], recv_bytes);
      if (MCB && NCL > 1) {
        // The other clusters' sources: lane `src` of warp 0 waits for that source's
        // release counter, then pulls its [N][PW] block from L2 into rrecv (TMA).
        if (w == 0) {
          const uint32_t blk = (uint32_t)N * PW * 4;
          if (l == 0) mbar_arrive_expect_tx(rbar, (uint32_t)(NSL - a.CL) * blk);
          __syncwarp();
          const uint32_t* fl = a.bflags + (size_t)grp * NSL;
          const uint8_t* gsrc = reinterpret_cast<const uint8_t*>(a.pstage) + (((size_t)grp * 2 + pb) * NSL + gq) * NSL * blk;
          for (int src = l; src < NSL; src += 32)
            if (src / a.CL != cl) {
              if (!(a.mcdbg & 4)) spin_until_geq(fl + src, (uint32_t)(T - s));
              fence_proxy_async_global();
              const int ri = src < cl * a.CL ? src : src - a.CL;
              bulk_g2s(reinterpret_cast<uint8_t*>(rrecv) + ri * blk, gsrc + (size_t)src * blk, blk, rbar);
            }
        }
        mbar_wait(rbar, rphase);
        rphase ^= 1u;
      }
      mbar_wait_cluster(&bars[2 + pb], (par_phase >> pb) & 1u);
      par_phase ^= 1u << pb;
    }
    FRNN_PROF(5, T - 1 - (s - 1));
    if (own && pbf && a.pvec == 2) {  // words [src][n][PW]: one word per source = units (u, u+1) of row b
      const uint32_t* rp = reinterpret_cast<const uint32_t*>(pb ? recv1 : recv) + (size_t)b * PW + (u >> 1);
      const size_t qs = (size_t)N * PW;
      float t0 = 0.f, t1 = 0.f;
      if (a.CL == 16) {  // all loads in flight first, then the fixed-order sums (deterministic)
        uint32_t v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = rp[q * qs];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          t0 += lo16(v[q]);
          t1 += hi16(v[q]);
        }
      } else {
        for (int q = 0; q < a.CL; ++q) {
          const uint32_t v = rp[q * qs];
          t0 += lo16(v);
          t1 += hi16(v);
        }
      }
      if (MCB && NCL > 1 && !(a.mcdbg & 1)) {  // then the other clusters' sources, fixed order (deterministic)
        const uint32_t* r2 = rrecv + (size_t)b * PW + (u >> 1);
        const int nrs = NSL - a.CL;
        for (int q0 = 0; q0 < nrs; q0 += 16) {
          uint32_t v[16];
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (q0 + q < nrs) v[q] = r2[(q0 + q) * qs];
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (q0 + q < nrs) {
              t0 += lo16(v[q]);
              t1 += hi16(v[q]);
            }
        }
      }
      if (p.clip_mode == 1) {
        t0 = fminf(fmaxf(t0, -mag), mag);
        t1 = fminf(fmaxf(t1, -mag), mag);
      }
      ds[0][0] += t0;
      ds[0][1] += t1;
    } else if ((!LEAN || a.pvec == 0) && own && pbf) {  // [src][u/2][b/2][2] (push_pair_cols) or [src][b/2][cu]: half b&1
      const uint32_t* rp = reinterpret_cast<const uint32_t*>(pb ? recv1 : recv) +
                           (a.pvec ? (size_t)(u >> 1) * N + (b >> 1) * 2 : (size_t)(b >> 1) * a.UPC + u);
      const size_t qs = (size_t)(N / 2) * a.UPC;
      float t0 = 0.f, t1 = 0.f;
      const int sh = (b & 1) ? 0 : 16;  // lo16 = bits << 16, hi16 = bits & 0xffff0000
      if (FX || (a.CL == 16 && (LEAN || a.absu))) {  // all loads in flight first, then the fixed-order sums (deterministic)
        uint2 v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = *reinterpret_cast<const uint2*>(rp + q * qs);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          t0 += __uint_as_float((v[q].x << sh) & 0xFFFF0000u);
          t1 += __uint_as_float((v[q].y << sh) & 0xFFFF0000u);
        }
      } else {
        for (int q = 0; q < a.CL; ++q) {  // fixed source order: deterministic
          const uint2 v = *reinterpret_cast<const uint2*>(rp + q * qs);
          t0 += (b & 1) ? hi16(v.x) : lo16(v.x);
          t1 += (b & 1) ? hi16(v.y) : lo16(v.y);
        }
      }
      if (p.clip_mode == 1) {
        t0 = fminf(fmaxf(t0, -mag), mag);
        t1 = fminf(fmaxf(t1, -mag), mag);
      }
      ds[0][0] += t0;
      ds[0][1] += t1;
    } else if (own) {
      const float* rp = (pb ? recv1 : recv) + (size_t)b * a.UPC + u;
      const size_t qs = (size_t)N * a.UPC;
      float t0 = 0.f, t1 = 0.f;
      if (FX || (a.CL == 16 && (LEAN || a.absu))) {  // all loads in flight first, then the fixed-order sums
        float2 v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = *reinterpret_cast<const float2*>(rp + q * qs);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          t0 += v[q].x;
          t1 += v[q].y;
        }
      } else {
        for (int q = 0; q < a.CL; ++q) {  // fixed source order: deterministic
          const float2 v = *reinterpret_cast<const float2*>(rp + q * qs);
          t0 += v.x;
          t1 += v.y;
        }
      }
      if (p.clip_mode == 1) {
        t0 = fminf(fmaxf(t0, -mag), mag);
        t1 = fminf(fmaxf(t1, -mag), mag);
      }
      ds[0][0] += t0;
      ds[0][1] += t1;
    }
  };
  auto absorb = [&](int s) {
    if (LEAN || a.dsm == 2) {
      absorb_rows(s);
      return;
    }
    if (dsm) {
      absorb_dsm(s);
      return;
    }
    const int pb = s & 1;
    const int kpub = T - 1 - s;  // publish order of step s
    if (w == 0) {
      mbar_wait_cluster(&bars[2 + pb], (uint32_t)(kpub >> 1) & 1u);
      if (elect_one()) {
        mbar_arrive_expect_tx(&bars[1], recv_bytes);
        bulk_g2s(recv, a.pstage + (((size_t)grp * 2 + pb) * a.CL + me) * a.CL * N * a.UPC, recv_bytes, &bars[1]);
      }
      __syncwarp();
    }
    mbar_wait(&bars[1], rcv_phase);
    rcv_phase ^= 1;
    if (own) {
      float t0 = 0.f, t1 = 0.f;
      const float* rp = recv + (size_t)b * a.UPC + u;
      const size_t qs = (size_t)N * a.UPC;
      for (int q = 0; q < a.CL; ++q) {
        const float2 v = *reinterpret_cast<const float2*>(rp + q * qs);
        t0 += v.x;
        t1 += v.y;
      }
      if (p.clip_mode == 1) {
        t0 = fminf(fmaxf(t0, -mag), mag);
        t1 = fminf(fmaxf(t1, -mag), mag);
      }
      ds[0][0] += t0;
      ds[0][1] += t1;
    }
    __syncthreads();  // recv is reloaded next step
  };

  const uint32_t idesc = idesc_bf16(128, N);
  constexpr uint32_t LBO = N * 16, SBO = 128;
  uint32_t mma_phase = 0;
  for (int t = T - 1; t >= 0; --t) {
    const int k = T - 1 - t;
    FRNN_PROF(0, k);
    if (recur && t + 1 < T) absorb(t + 1);
    FRNN_PROF(1, k);
    float dgv[NG][2];
    // dx = dg for input-wired gates, engine.hpp:311-316 (off the critical path)
    auto store_dx = [&]() {
      if (valid && !k_nodx) {
        bf16* dxg = dx + (size_t)t * gstep + xo;
#pragma unroll
        for (int j = 0; j < NG; ++j) {
          if (p.inp[j]) st2(dxg, (size_t)j * D, dgv[j][0], dgv[j][1]);
          else *reinterpret_cast<uint32_t*>(dxg + (size_t)j * D) = 0u;
          if (a.dgw) st2(a.dgw + (size_t)t * gstep + xo, (size_t)j * D, dgv[j][0], dgv[j][1]);
        }
      }
    };
    if (own) {
      uint32_t pk[2][2] = {{0u, 0u}, {0u, 0u}};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float dsl[4], dg[4], dsp[4];
#pragma unroll
        for (int s = 0; s < NS; ++s) dsl[s] = ds[s][h];
        dsl[0] += h ? hi16(hv) : lo16(hv);  // engine.hpp:258-263
        if (a.skeleton) {
#pragma unroll
          for (int j = 0; j < NG; ++j) dg[j] = dsl[0];
#pragma unroll
          for (int s = 0; s < NS; ++s) dsp[s] = dsl[s];
        } else if (!csplit) {  // Jacobian formed and contracted here (cell.hpp:108-201, engine.hpp:275-284)
          float prev[4], g[4];
#pragma unroll
          for (int s = 0; s < NS; ++s) prev[s] = h ? hi16(pv[s]) : lo16(pv[s]);
#pragma unroll
          for (int j = 0; j < NG; ++j) g[j] = h ? hi16(gv[j]) : lo16(gv[j]);
          C::template bwd<M>(prev, g, dsl, dg, dsp);
        } else {
          C::apply(kc[h], dsl, dg, dsp);  // engine.hpp:275-284 with the coefficients formed last step
        }
#pragma unroll
        for (int j = 0; j < NG; ++j) {
          const float d = b < nb ? dg[j] : 0.f;
          dgv[j][h] = d;
          dbv[j][h] += d;
          pk[h][j >> 1] |= (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(d)) << (16 * (j & 1));
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) ds[s][h] = dsp[s];
      }
      // The pair's NGK*2 gate rows are contiguous along K of the dg tile.
      if (C::NGK == 3 && a.kcompact) {  // GRU: rows (u:z, u:r, u:g, u+1:z, u+1:r, u+1:g) from k = 3u, as 3 bf16 pairs
        const uint32_t lo = pk[0][0], hi = pk[1][0];
        const uint32_t g0 = pk[0][1] >> 16, g1 = pk[1][1] >> 16;  // dg of gate 3 (j = 3: high half)
        *reinterpret_cast<uint32_t*>(dgB + kmaj(b, 3 * u, N)) = lo;
        *reinterpret_cast<uint32_t*>(dgB + kmaj(b, 3 * u + 2, N)) = g0 | (hi << 16);
        *reinterpret_cast<uint32_t*>(dgB + kmaj(b, 3 * u + 4, N)) = (hi >> 16) | (g1 << 16);
      } else if (NGP == 4)
        *reinterpret_cast<uint4*>(dgB + kmaj(b, u * 4, N)) = make_uint4(pk[0][0], pk[0][1], pk[1][0], pk[1][1]);
      else if (NGP == 2)
        *reinterpret_cast<uint2*>(dgB + kmaj(b, u * 2, N)) = make_uint2(pk[0][0], pk[1][0]);
      else
        *reinterpret_cast<uint32_t*>(dgB + kmaj(b, u, N)) = (pk[0][0] & 0xFFFFu) | (pk[1][0] << 16);
    }
    load_dh(t - 1);
    if (!csplit) load_trace(t - 1);  // (the fused Jacobian path: next step's trace, one step ahead)
    if (recur) {
      fence_proxy_async_smem();
      __syncthreads();
      FRNN_PROF(2, k);
      if (w == 0) {  // block pairs in order: TMEM-A block i interleaved step by step with SMEM-A
                     // block i (the two operand paths overlap), one commit per pair so the drain +
                     // exchange of pair i overlaps the MMAs of the later pairs
        tc_fence_after();
        const uint64_t bd = sdesc_kmajor(smem_u32(dgB), LBO, SBO);
        const uint64_t ad = sdesc_kmajor(smem_u32(AS), SSM * 16, 128);
        const uint32_t idesc2 = idesc_bf16(SSM, N);
        const int nk = KBP / 16, cb = KBP / 2;
        if (FX ? !a.skeleton : (MBT == 4 && MS == 2 && nk == 12 && !a.skeleton)) {  // the H=768, 4-gate layout
          const uint64_t a2k = (2 * SSM * 16) >> 4, bk = (2 * LBO) >> 4, bs = blk_bytes >> 4;
          const uint32_t acc = tbase + a.acc1;
          mma12_ts_ss(acc, tbase, acc + 4 * N, ad, a2k, bd, bk, idesc, idesc2, 0);
          if (elect_one()) mma_commit(&blkbar[0]);
          __syncwarp();
          mma12_ts_ss(acc + N, tbase + cb, acc + 5 * N, ad + bs, a2k, bd, bk, idesc, idesc2, 0);
          if (elect_one()) mma_commit(&blkbar[1]);
          __syncwarp();
          mma12_ts(acc + 2 * N, tbase + 2 * cb, bd, bk, idesc, 0);
          if (elect_one()) mma_commit(&blkbar[2]);
          __syncwarp();
          mma12_ts(acc + 3 * N, tbase + 3 * cb, bd, bk, idesc, 0);
          if (elect_one()) mma_commit(&blkbar[3]);
          __syncwarp();
        } else if (MBT == 6 && MS == 0 && nk == 3 && !a.skeleton) {  // single-gate cells at H=768 (Elman)
          const uint64_t bk = (2 * LBO) >> 4;
          const uint32_t acc = tbase + a.acc1;
          mma3_ts(acc, tbase, bd, bk, idesc, 0);
          if (elect_one()) mma_commit(&blkbar[0]);
          __syncwarp();
          mma3_ts(acc + N, tbase + cb, bd, bk, idesc, 0);
          if (elect_one()) mma_commit(&blkbar[1]);
          __syncwarp();
          mma3_ts(acc + 2 * N, tbase + 2 * cb, bd, bk, idesc, 0);
          if (elect_one()) mma_commit(&blkbar[2]);
          __syncwarp();
          mma3_ts(acc + 3 * N, tbase + 3 * cb, bd, bk, idesc, 0);
          if (elect_one()) mma_commit(&blkbar[3]);
          __syncwarp();
          mma3_ts(acc + 4 * N, tbase + 4 * cb, bd, bk, idesc, 0);
          if (elect_one()) mma_commit(&blkbar[4]);
          __syncwarp();
          mma3_ts(acc + 5 * N, tbase + 5 * cb, bd, bk, idesc, 0);
          if (elect_one()) mma_commit(&blkbar[5]);
          __syncwarp();
        } else if (MCB && N == 16 && SSM == 128 && !a.skeleton && a.itab &&
                   issue_bwd_table_mc(MBT, MS, nk, tbase, tbase + a.acc1, bd, ad, idesc, idesc2, blkbar)) {
          // the multi-cluster tilings: compile-time issue (H=1024 backward 8.8 -> 7.6 us/step)
        } else if (!MCB && !FX && N == 16 && SSM == 128 && !a.skeleton && a.itab &&
                   issue_bwd_table(MBT, MS, nk, tbase, tbase + a.acc1, bd, ad, idesc, idesc2, blkbar)) {
          // every other tiling the planner reaches: compile-time issue instance (scripts/tilings.py)
        } else if (MBT == 2 && MS == 0 && nk == 12 && !a.skeleton) {  // DH=192 per head (config 3)
          const uint64_t bk = (2 * LBO) >> 4;
          mma12_ts(tbase + a.acc1, tbase, bd, bk, idesc, 0);
          if (elect_one()) mma_commit(&blkbar[0]);
          __syncwarp();
          mma12_ts(tbase + a.acc1 + N, tbase + cb, bd, bk, idesc, 0);
          if (elect_one()) mma_commit(&blkbar[1]);
          __syncwarp();
        } else
        for (int i = 0; i < NPAIR; ++i) {
          const uint32_t accT = tbase + a.acc1 + i * N, accS = tbase + a.acc1 + (MBT + i) * N;
          const uint64_t adS = ad + (uint64_t)(i * (blk_bytes >> 4));
          if (a.skeleton) {
          } else if (i < MBT && i < MS) {
            if (nk == 12) mma12_ts_ss(accT, tbase + i * cb, accS, adS, (2 * SSM * 16) >> 4, bd, (2 * LBO) >> 4,
                                      idesc, idesc2, 0);
            else mma_run_ts_ss(accT, tbase + i * cb, accS, adS, (2 * SSM * 16) >> 4, bd, (2 * LBO) >> 4, idesc,
                               idesc2, nk);
          } else if (i < MBT) {
            if (nk == 12) mma12_ts(accT, tbase + i * cb, bd, (2 * LBO) >> 4, idesc, 0);
            else mma_run_ts(accT, tbase + i * cb, 8, bd, (2 * LBO) >> 4, idesc, nk);
          } else {
            mma_run_ss(accS, adS, (2 * SSM * 16) >> 4, bd, (2 * LBO) >> 4, idesc2, nk);
          }
          if (elect_one()) mma_commit(&blkbar[i]);
          __syncwarp();
        }
      }
    }
    // Under step t's MMAs: the Jacobian of step t-1 (its trace landed during step
    // t+1), then the trace loads for step t-2.
    if (csplit) {
      if (t > 0 && !a.skeleton) coefs();
      load_trace(t - 2);
    }
    if (dxearly) store_dx();
    if (recur) {
      FRNN_PROF(3, k);
      // partial R_p^T dg_p, column c -> owner CTA c / UPC, layout [dest][src][b][u];
      // every warp drains the TMEM lane quadrant w%4 of blocks w/4, w/4+NT/128, ...
      float* base = a.pstage + (((size_t)grp * 2 + (t & 1)) * a.CL) * a.CL * N * a.UPC;
      const int qd = w & 3;
      const uint32_t rb = smem_u32((t & 1) ? recv1 : recv), rbar = smem_u32(&bars[2 + (t & 1)]);
      // the MBT + MS accumulator blocks (pair order: TMEM-A block i, then SMEM-A block i)
      // are dealt round-robin to the NT/128 warp groups
      const int both = min(MBT, MS), nent = MBT + MS, ngrp = NT >> 7;
      const bool fixed = FX || (MBT == 4 && MS == 2 && SSM == 128 && NT == 384 && a.UPC == 48 && a.dsm == 2 && DH == 768);
      if (fixed) {  // the H=768 layout spelled out: warp group -> (pair, column base, accumulator block)
        const int wg = w >> 2;
        const int i0 = wg == 2 ? 1 : 0, c0 = wg == 0 ? 0 : wg == 1 ? 512 : 128, a0 = wg == 0 ? 0 : wg == 1 ? 4 : 1;
        const int i1 = wg == 0 ? 1 : wg == 1 ? 2 : 3, c1 = wg == 0 ? 640 : wg == 1 ? 256 : 384,
                  a1 = wg == 0 ? 5 : wg == 1 ? 2 : 3;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          mbar_wait_idle(&blkbar[e ? i1 : i0], mma_phase, a.waitmode);
          FRNN_PROF_AT(6, k, NT - 32);  // the last warp's last block complete
          tc_fence_after();
          const int c = rotc((e ? c1 : c0) + 32 * qd + l), q = c / 48, cu = c % 48;
          float v[16];
          tmem_ld16(tbase + ((uint32_t)(32 * qd) << 16) + a.acc1 + (e ? a1 : a0) * N, v);
          const uint32_t mbr = mapa_shared(rbar, q);
          if (FX || (pbf && a.pvec == 2)) {
            push_col_pairs<N>(v, l, !k_noxchg, cu, pair_pitch(48), rb + (uint32_t)(me * N * pair_pitch(48) * 4), q, mbr);
          } else if (pbf && a.pvec) {
            push_pair_cols<N>(v, l, true, cu, rb + (uint32_t)(me * (N / 2) * 48 * 4), q, mbr);
          } else if (pbf) {  // words [src][n/2][cu] = bf16 (n even, n odd)
            const uint32_t dst = mapa_shared(rb + (uint32_t)((me * (N / 2) * 48 + cu) * 4), q);
#pragma unroll
            for (int n2 = 0; n2 < N / 2; ++n2)
              st_async_b32(dst + (uint32_t)(n2 * 48 * 4), __uint_as_float(pack_bf16(v[2 * n2], v[2 * n2 + 1])), mbr);
          } else {
            const uint32_t dst = mapa_shared(rb + (uint32_t)((me * N * 48 + cu) * 4), q);
#pragma unroll
            for (int n = 0; n < N; ++n) st_async_b32(dst + (uint32_t)(n * 48 * 4), v[n], mbr);
          }
        }
      }
      for (int ent = fixed ? nent : w >> 2; ent < nent; ent += ngrp) {
        int i, sblk;
        if (ent < 2 * both) {
          i = ent >> 1;
          sblk = ent & 1;
        } else {
          i = both + (ent - 2 * both);
          sblk = MS > MBT;
        }
        mbar_wait_idle(&blkbar[i], mma_phase, a.waitmode);
        FRNN_PROF_AT(6, k, NT - 32);  // the last warp's last block complete
        tc_fence_after();
        int c;
        bool lane_ok = true;
        if (!sblk) {
          c = i * 128 + 32 * qd + l;
        } else if (SSM == 64) {  // M=64 layout: rows 16q..16q+15 in lanes 32q..32q+15
          c = MBT * 128 + i * 64 + 16 * qd + l;
          lane_ok = l < 16;
        } else {
          c = MBT * 128 + i * 128 + 32 * qd + l;
        }
        c = rotc(c);
        float v[16];
        tmem_ld16(tbase + ((uint32_t)(32 * qd) << 16) + a.acc1 + (sblk ? MBT + i : i) * N, v);
        if (MCB) {  // whole warp (shuffles inside); owners in other clusters through pstage
          const int qg = min(c / a.UPC, NSL - 1), cu = c % a.UPC, q = qg % a.CL;
          uint32_t* gd = reinterpret_cast<uint32_t*>(a.pstage) +
                         ((((size_t)grp * 2 + (t & 1)) * NSL + qg) * NSL + gq) * N * PW;
          push_col_pairs_mc<N>(v, l, lane_ok && c < DH && !k_noxchg && (qg / a.CL == cl || !(a.mcdbg & 2)), qg / a.CL == cl, cu, PW,
                               rb + (uint32_t)(me * N * PW * 4), q, mapa_shared(rbar, q), gd);
        } else if (FX || (pbf && a.pvec == 2)) {  // whole warp (shuffles inside)
          const int q = min(c / a.UPC, a.CL - 1), cu = c % a.UPC;  // (clamped for lanes past DH)
          push_col_pairs<N>(v, l, lane_ok && c < DH && !k_noxchg, cu, PW, rb + (uint32_t)(me * N * PW * 4), q,
                            mapa_shared(rbar, q));
        } else if (!LEAN && pbf && a.pvec) {  // whole warp (shuffles inside)
          const int q = min(c / a.UPC, a.CL - 1), cu = c % a.UPC;  // (clamped for lanes past DH)
          push_pair_cols<N>(v, l, lane_ok && c < DH, cu, rb + (uint32_t)(me * (N / 2) * a.UPC * 4), q,
                            mapa_shared(rbar, q));
        } else if (lane_ok && c < DH) {
          const bool u48 = a.UPC == 48;  // the H=768 tiling: constant divisor and stride
          const int q = u48 ? c / 48 : c / a.UPC, cu = u48 ? c % 48 : c % a.UPC;
          if (LEAN || a.dsm == 2) {  // 4-byte pushes into the owner's recv[t&1][me][n][cu]: a warp writes
                             // 32 consecutive columns = one contiguous 128-byte row segment per n
            const uint32_t mbr = mapa_shared(rbar, q);
            if (pbf) {
              const uint32_t dst = mapa_shared(rb + (uint32_t)((me * (N / 2) * a.UPC + cu) * 4), q);
#pragma unroll
              for (int n2 = 0; n2 < N / 2; ++n2)
                st_async_b32(dst + (uint32_t)(n2 * a.UPC * 4), __uint_as_float(pack_bf16(v[2 * n2], v[2 * n2 + 1])),
                             mbr);
            } else if (u48) {
              const uint32_t dst = mapa_shared(rb + (uint32_t)((me * N * 48 + cu) * 4), q);
#pragma unroll
              for (int n = 0; n < N; ++n) st_async_b32(dst + (uint32_t)(n * 48 * 4), v[n], mbr);
            } else {
              const uint32_t dst = mapa_shared(rb + (uint32_t)((me * N * a.UPC + cu) * 4), q);
#pragma unroll
              for (int n = 0; n < N; ++n) st_async_b32(dst + (uint32_t)(n * a.UPC * 4), v[n], mbr);
            }
          } else if (!LEAN && dsm) {  // push straight into the owner's recv[t&1][me][cu][:], on its mbarrier
            const uint32_t dst = mapa_shared(rb + (uint32_t)(((me * a.UPC + cu) * N) * 4), q);
            const uint32_t mbr = mapa_shared(rbar, q);
#pragma unroll
            for (int i = 0; i < N / 4; ++i) st_async_v4(dst + 16 * i, v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3], mbr);
          } else if (!LEAN) {
            float* dst = base + (((size_t)q * a.CL + me) * N) * a.UPC + cu;
#pragma unroll
            for (int n = 0; n < N; ++n) dst[(size_t)n * a.UPC] = v[n];
          }
        }
      }
      FRNN_PROF_AT(7, k, NT - 32);  // the last warp's pushes issued
      mma_phase ^= 1;
      if (!dsm) fence_proxy_async_global();
      tc_fence_before();
      __syncthreads();
      if (!dsm && tid < a.CL) mbar_arrive_remote(mapa_shared(smem_u32(&bars[2 + (t & 1)]), tid));
      if (MCB && NCL > 1 && tid == 0)  // this CTA's partials of step t for the other clusters are stored
        st_release_gpu(a.bflags + (size_t)grp * NSL + gq, (uint32_t)(k + 1));
      FRNN_PROF(4, k);
    }
    if (!dxearly) store_dx();
  }
  if (recur && T > 0) absorb(0);
  if (valid) {
#pragma unroll
    for (int s = 0; s < NS; ++s) st2(ds0, (size_t)s * B * D + so, ds[s][0], ds[s][1]);
  }
  if (a.dbacc) {  // db: fixed-order sum over the tile's batch rows (deterministic)
    __syncthreads();  // (dbs may alias the receive buffers the last absorb just read)
    if (own) {
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        dbs[((size_t)j * N + b) * a.UPC + u] = dbv[j][0];
        dbs[((size_t)j * N + b) * a.UPC + u + 1] = dbv[j][1];
      }
    }
    __syncthreads();
    const int tile = grp % a.NBT;
    for (int q = tid; q < NG * a.UPC; q += NT) {
      const int j = q / a.UPC, uu = q % a.UPC;
      float sum = 0.f;
      for (int bb = 0; bb < nb; ++bb) sum += dbs[((size_t)j * N + bb) * a.UPC + uu];
      a.dbacc[((size_t)tile * NG + j) * D + hd * DH + unit0 + uu] = sum;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (w == 0) tmem_dealloc(tbase, a.tmem_cols);
}

uint32_t pow2_cols(uint32_t c) {
  uint32_t r = 32;
  while (r < c) r <<= 1;
  return r;
}

int ngp_of(int NG) { return NG <= 1 ? 1 : NG <= 2 ? 2 : 4; }
int NSof(const Problem& p) { return p.NS; }
// GRU backward without the n gate's zero R rows in K (FRNN_GRU_COMPACT=1): correct
// and 25 % fewer MMAs, but measured slower at H=768 (the padded layout keeps the
// compile-time headline instance) -- off by default
bool gru_compact(const Problem& p) {
  const char* e = getenv("FRNN_GRU_COMPACT");
  return p.variant == kGru && e && atoi(e) != 0;
}

}  // namespace

// ---------------------------------------------------------------- host ----
ClusterShape cluster_shape(const Problem& p, int UPC, int N, bool backward, int ncl) {
  ClusterShape s{};
  const int NGP = ngp_of(p.NG);
  s.UPC = UPC;
  s.NCL = std::max(1, ncl);
  s.CL = p.DH / (UPC * s.NCL);
  const int rows = UPC * NGP;
  s.R1 = rows < 128 ? rows : 128;
  s.R2 = rows - s.R1;
  s.K = p.DH;
  // backward K rows per unit: only gates with R (GRU's n gate has none, cell.hpp:43)
  const int ngk = gru_compact(p) ? 3 : NGP;
  s.KBP = (UPC * (backward ? ngk : NGP) + 15) / 16 * 16;
  s.MB = (p.DH + 127) / 128;
  s.slice = (uint32_t)UPC * N * 2;
  const int NBT = (p.B + N - 1) / N;
  s.groups = p.NH * NBT;
  const int pairs = UPC / 2 * N;
  s.threads = (int)align_up(pairs, 128);
  s.EPT = pairs <= MAXT ? 1 : 0;  // one unit pair per thread (0 = unsupported)
  if (!backward) {
    // One M=128 block whose K/2 TMEM columns + two accumulators exceed TMEM
    // (DH > 960): the tail of K moves to an SMEM M=128 tile with its own
    // accumulator, sized so the two operand paths take about equally long
    // (TMEM-A ~50, SMEM-A M=128 ~90 cycles per K=16 step at N=16, DESIGN 4).
    s.Ks = 0;
    // (multi-cluster: split even when K fits TMEM -- the two operand paths overlap)
    if (s.R2 == 0 && ((int)align_up(s.K / 2, 32) + 2 * N > 512 || (s.NCL > 1 && !getenv("FRNN_FWD_NOSPLIT")))) {
      const int nk = s.K / 16;
      int nts = (nk * 90 + 139) / 140;
      const char* kt = getenv("FRNN_FWD_KT");  // A/B hook: TMEM K columns of the split
      if (kt) nts = atoi(kt) / 16;
      nts = std::min(std::max(nk / 2, nts), (512 - 2 * N) / 8);  // (the TMEM cap wins)
      s.Ks = s.K - 16 * nts;
    }
    s.acc1 = (uint32_t)align_up((s.K - s.Ks) / 2, 32);
    s.acc2 = s.acc1 + N;
    s.tmem_cols = pow2_cols(s.acc2 + N);
    s.m64 = s.NCL > 1 && rows <= 64 && !getenv("FRNN_FWD_NOM64");
    s.smem = (size_t)2 * N * s.K * 2 + (s.R2 ? (size_t)64 * s.K * 2 : (size_t)(s.m64 ? 64 : 128) * s.Ks * 2) +
             (size_t)N * xs_pitch(rows) * 4 + align_up(s.slice, 16) + 64;
    // (x and the trace move by per-thread loads/stores: TMA tiles measured slower)
    s.ws = align_up((size_t)s.groups * 2 * s.NCL * s.CL * s.slice, 256);
    if (s.NCL > 1) s.ws += align_up(sizeof(uint32_t) * s.groups * s.NCL * s.CL, 256);  // release flags
  } else {
    // R_p^T column blocks: MBT of 128 columns with A in TMEM, then MS of SSM
    // columns with A in SMEM, issued as pairs (TMEM block i interleaved with
    // SMEM block i, the two operand paths overlap); accumulators (MBT + MS) x N.
    // SSM = 128 measured best (sLSTM H=768 backward 4.42 us/step vs 4.84 with
    // 64-column SMEM blocks and 4.75 with no interleaving).
    const int colblk = s.KBP / 2;
    const char* se = getenv("FRNN_BWD_SSM");  // A/B hook: 64 = SMEM blocks of 64 columns
    s.SSM = se && atoi(se) == 64 ? 64 : 128;
    auto ms_of = [&](int mbt) { return p.DH > 128 * mbt ? (p.DH - 128 * mbt + s.SSM - 1) / s.SSM : 0; };
    int mbt = s.MB;
    while (mbt > 0 && mbt * colblk + (mbt + ms_of(mbt)) * N > 512) --mbt;
    s.MBT = mbt;
    s.MS = ms_of(mbt);
    if (std::max(s.MBT, s.MS) > 16) s.EPT = 0;  // 16 block-pair mbarriers
    s.acc1 = (uint32_t)(s.MBT * colblk);
    s.tmem_cols = pow2_cols(s.acc1 + (s.MBT + s.MS) * N);
    s.smem = (size_t)s.MS * s.SSM * s.KBP * 2 + (size_t)s.CL * N * UPC * 4 + (size_t)N * s.KBP * 2 +
             (size_t)p.NG * N * UPC * 4 + 192;  // + 4 exchange and 16 block-pair mbarriers, TMEM base
    // DSMEM exchange: a second (parity) receive buffer + the summed-term tile
    const size_t dsm_smem = s.smem + (size_t)s.CL * N * UPC * 4 + (size_t)N * (UPC + 2) * 4;
    const char* xe = getenv("FRNN_XCHG");  // A/B hook: 0 = global + TMA bulk load, 1 = DSMEM v4 [cu][n], 2 = rows
    s.dsm = (!xe || atoi(xe) != 0) && dsm_smem <= (size_t)kSmemOptin && (UPC % 4) == 0;
    if (s.dsm) s.dsm = xe ? atoi(xe) : 2;
    if (s.dsm) s.smem = dsm_smem;
    // 4-gate cells exchange the R^T.dg partials as bf16 pairs by default (half the DSMEM
    // bytes and pushes; gradient errors vs the f64 oracle 1.75e-3 -> 1.82e-3 normwise),
    // in the column-pair receive layout; FRNN_PBF16 / FRNN_PVEC override.
    s.pbf16 = s.dsm == 2 && (getenv("FRNN_PBF16") ? atoi(getenv("FRNN_PBF16")) : (p.NG == 4 ? 1 : 0));
    s.pvec = getenv("FRNN_PVEC") ? atoi(getenv("FRNN_PVEC")) : 2;
    {  // final footprint: receive buffers at their exchanged size; db scratch aliased onto
       // them when it fits, the summed-term tile only for dsm 1.  A footprint at or under
       // 164 KB lets the driver pick the 164 KB carveout, leaving ~92 KB of L1 for the
       // per-thread trace loads and dx stores (sLSTM H=768 backward 3.93 -> 3.33 us/step)
      const size_t span = (s.dsm == 2 && s.pbf16) ? (s.pvec == 2 ? (size_t)s.CL * N * pair_pitch(UPC) * 4
                                                                  : (size_t)s.CL * N * UPC * 2)
                                                  : (size_t)s.CL * N * UPC * 4;
      const size_t nrecv = s.dsm ? 2 : 1, dbs = (size_t)p.NG * N * UPC * 4;
      s.smem = (size_t)s.MS * s.SSM * s.KBP * 2 + nrecv * span + (size_t)N * s.KBP * 2 +
               (dbs > nrecv * span ? dbs : 0) + (s.dsm == 1 ? (size_t)N * (UPC + 2) * 4 : 0) + 192;
    }
    // (per-thread trace loads / dx stores: TMA tiles measured slower)
    s.ws = align_up((size_t)s.groups * 2 * s.CL * s.CL * N * UPC * 4, 256);
    if (s.NCL > 1) {
      // the other clusters' partials land in SMEM too ([remote src][N][PW] words, after the
      // barriers), and 384 threads drain the MB accumulator blocks (3 warp groups)
      s.smem += (size_t)(s.NCL - 1) * s.CL * N * pair_pitch(UPC) * 4 + 64;
      s.threads = getenv("FRNN_MCB_THREADS") ? std::max(s.threads, atoi(getenv("FRNN_MCB_THREADS"))) : MAXT;  // partials for other clusters' owners [grp][2][dest][src][N][PW] words + release counters
      const size_t nsl = (size_t)s.NCL * s.CL;
      s.ws = align_up((size_t)s.groups * 2 * nsl * nsl * N * pair_pitch(UPC) * 4, 256) +
             align_up(sizeof(uint32_t) * s.groups * nsl, 256);
    }
  }
  // Multi-cluster kernels spin on other clusters' counters, and every CTA holds all
  // 512 TMEM columns: two CTAs on one SM would wait on each other's allocation.
  // More than half the SM's shared memory keeps them one per SM.
  if (s.NCL > 1) s.smem = std::max(s.smem, (size_t)118 * 1024);
  return s;
}

bool cluster_ept_supported(int ept) { return ept == 1; }
bool cluster_mc_bwd_instance(const ClusterShape& cs) { return mc_issue_instance(cs.MBT, cs.MS, cs.KBP / 16); }

namespace {

// Clusters per group of a forward plan (ctas_per_group = NCL x cluster).
int plan_ncl(const Plan& pl) { return pl.cluster > 0 ? std::max(1, pl.ctas_per_group / pl.cluster) : 1; }

CArgs make_cargs(const Problem& p, const Plan& pl, void* ws, bool backward, ClusterShape& cs) {
  const int N = pl.batch_tile;
  cs = cluster_shape(p, pl.units_per_cta, N, backward, plan_ncl(pl));
  CArgs a{};
  a.NCL = cs.NCL;
  a.Ks = cs.Ks;
  a.m64 = backward ? 0 : cs.m64;
  // (the slice writers' stores reach the flag's release through bar.sync; a full
  // fence before it measured 0.47 us/step slower at H=1024 and is not needed)
  a.mcfence = getenv("FRNN_MC_FENCE") ? atoi(getenv("FRNN_MC_FENCE")) : 0;
  a.mcpoll = getenv("FRNN_MC_POLL") ? atoi(getenv("FRNN_MC_POLL")) : 0;
  a.mcwarp = getenv("FRNN_MC_WARP") ? atoi(getenv("FRNN_MC_WARP")) : 1;
  // own-cluster K steps first, each group split TMEM|SMEM in the block's ratio (H=896 3.59 -> 3.39,
  // H=1024 3.80 -> 3.68 us/step forward; two clusters only by default)
  a.mclocal = getenv("FRNN_MC_LOCAL") ? atoi(getenv("FRNN_MC_LOCAL")) : 1;
  a.mcrelw = getenv("FRNN_MC_RELW") ? atoi(getenv("FRNN_MC_RELW")) : 1;
  a.mcdbg = getenv("FRNN_MC_DBG") ? atoi(getenv("FRNN_MC_DBG")) : 0;
  a.p = p;
  a.UPC = cs.UPC;
  a.CL = cs.CL;
  a.NBT = (p.B + N - 1) / N;
  a.R1 = cs.R1;
  a.R2 = cs.R2;
  a.K = cs.K;
  a.KBP = cs.KBP;
  a.MB = cs.MB;
  a.MBT = cs.MBT;
  a.MS = cs.MS;
  a.SSM = cs.SSM;
  a.tmem_cols = cs.tmem_cols;
  a.acc1 = cs.acc1;
  a.acc2 = cs.acc2;
  a.slice = cs.slice;
  a.prof = g_prof_buf;
  a.prof_steps = g_prof_steps;
  a.dsm = backward ? cs.dsm : 0;
  // 4-gate cells exchange the R^T.dg partials as bf16 pairs by default (half the DSMEM
  // bytes and pushes; backward 4.10 -> 3.58 us/step at H=768, gradient errors vs the
  // f64 oracle 1.75e-3 -> 1.82e-3 normwise); FRNN_PBF16=0/1 overrides.
  a.pbf16 = backward ? cs.pbf16 : 0;
  a.dxearly = getenv("FRNN_DXEARLY") ? atoi(getenv("FRNN_DXEARLY")) : 0;
  a.absu = getenv("FRNN_ABSU") ? atoi(getenv("FRNN_ABSU")) : 1;
  a.pvec = backward ? cs.pvec : 0;

  a.skeleton = g_skeleton || (getenv("FRNN_DBG_SKELETON") && atoi(getenv("FRNN_DBG_SKELETON")));
  {
    const char* cs_ = getenv("FRNN_COEFSPLIT");  // default: long MMA windows only
    a.csplit = cs_ ? atoi(cs_) : ((cs.KBP / 16) * (cs.MBT + cs.MS) >= 48);
  }
  // backward single-gate cells keep the unit-fastest ownership (Elman 3.92 -> 3.30 us/step)
  a.kcompact = backward && gru_compact(p);
  a.waitmode = getenv("FRNN_WAITMODE") ? atoi(getenv("FRNN_WAITMODE")) : 0;
  a.itab = getenv("FRNN_ISSUE_TABLE") ? atoi(getenv("FRNN_ISSUE_TABLE")) : 1;
  a.map = getenv(backward ? "FRNN_BMAP" : "FRNN_FMAP") ? atoi(getenv(backward ? "FRNN_BMAP" : "FRNN_FMAP"))
                                                       : (backward && p.NG == 1 ? 0 : 1);
  a.hdirect = getenv("FRNN_HDIRECT") ? atoi(getenv("FRNN_HDIRECT")) : 1;  // fwd 2.52 -> 2.44 us/step
  a.xpf = getenv("FRNN_XPF") ? atoi(getenv("FRNN_XPF")) : 0;
  a.rot = getenv("FRNN_ROT") ? atoi(getenv("FRNN_ROT")) : 0;  // measured neutral-to-slower (DESIGN 8c)
  a.noxchg = backward && getenv("FRNN_DBG_NOXCHG") && atoi(getenv("FRNN_DBG_NOXCHG"));
  a.nodx = getenv("FRNN_DBG_NODX") && atoi(getenv("FRNN_DBG_NODX"));        // fwd: trace stores
  a.noload = getenv("FRNN_DBG_NOLOAD") && atoi(getenv("FRNN_DBG_NOLOAD"));  // fwd: x loads
  char* w = static_cast<char*>(ws);
  if (!backward) {
    a.xstage = reinterpret_cast<bf16*>(w);
    if (cs.NCL > 1)
      a.xflags = reinterpret_cast<uint32_t*>(w + align_up((size_t)cs.groups * 2 * cs.NCL * cs.CL * cs.slice, 256));
  } else {
    a.pstage = reinterpret_cast<float*>(w);
    if (cs.NCL > 1) {
      const size_t nsl = (size_t)cs.NCL * cs.CL;
      a.bflags = reinterpret_cast<uint32_t*>(w + align_up((size_t)cs.groups * 2 * nsl * nsl * N * pair_pitch(cs.UPC) * 4, 256));
    }
    size_t off = cs.ws;
    bool all_in = true;
    for (int j = 0; j < p.NG; ++j) all_in = all_in && p.inp[j];
    if (!all_in) {
      a.dgw = reinterpret_cast<bf16*>(w + off);
      off += align_up((size_t)2 * p.T * p.B * p.NG * p.D, 256);
    }
    a.dbacc = dr_gemm_supported(p) ? reinterpret_cast<float*>(w + off) : nullptr;
  }
  return a;
}

template <class KernelT>
cudaError_t cluster_launch(KernelT kern, const CArgs& a, int grid, int threads, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (a.CL > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
    return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = a.CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  // Multi-cluster kernels spin on each other's counters: a cooperative launch
  // guarantees every cluster is resident (or fails) instead of trapping later
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = a.NCL > 1 ? 2 : 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// The compile-time backward layout (cl_bwd_kernel<V, N, 1>) applies when the
// solved tiling is exactly the headline one; anything else runs L = 0.
bool bwd_fixed_layout(const CArgs& a, const ClusterShape& cs) {
  return a.MBT == 4 && a.MS == 2 && a.SSM == 128 && a.KBP == 192 && a.UPC == 48 && a.CL == 16 && cs.threads == 384 &&
         a.dsm == 2 && a.pbf16 && a.pvec == 2 && a.absu && a.p.DH == 768 && !getenv("FRNN_BWD_GENERIC");
}

using KernelFn = void (*)(CArgs);
// The lean instance (L = 2) whenever the exchange is the default one.
bool bwd_lean_layout(const CArgs& a) {
  return a.dsm == 2 && (!a.pbf16 || a.pvec == 2 || a.pvec == 0) && a.absu && !getenv("FRNN_BWD_GENERIC");
}

// L = 3 (lean and plain) when no split coefficients and no experiment/debug switch is asked for.
bool bwd_plain(const CArgs& a) { return !a.csplit && !a.rot && !a.dxearly && !a.noxchg && !a.nodx && !a.noload; }

template <int V>
KernelFn bwd_kernel(int L) {
  if constexpr (V == kElman) {
    return L == 3 ? cl_bwd_kernel<V, 16, 3> : L ? cl_bwd_kernel<V, 16, 2> : cl_bwd_kernel<V, 16, 0>;
  } else {
    return L == 1 ? cl_bwd_kernel<V, 16, 1> : L == 2 ? cl_bwd_kernel<V, 16, 2>
         : L == 3 ? cl_bwd_kernel<V, 16, 3> : L == 4 ? cl_bwd_kernel<V, 16, 4> : cl_bwd_kernel<V, 16, 0>;
  }
}

template <int V>
KernelFn fwd_kernel(bool mc) {
  return mc ? cl_fwd_kernel<V, 16, 1> : cl_fwd_kernel<V, 16, 0>;
}

template <bool BWD>
cudaError_t launch_variant(int variant, const CArgs& a, const ClusterShape& cs, cudaStream_t s) {
  const int grid = cs.groups * cs.NCL * cs.CL;
  const int fx = !BWD ? 0 : a.NCL > 1 ? 4 : bwd_fixed_layout(a, cs) ? 1 : bwd_lean_layout(a) ? (bwd_plain(a) ? 3 : 2) : 0;
  const bool mc = a.NCL > 1 || a.Ks > 0;
  KernelFn k;
  switch (variant) {
    case kElman: k = BWD ? bwd_kernel<kElman>(fx) : fwd_kernel<kElman>(mc); break;
    case kLstm: k = BWD ? bwd_kernel<kLstm>(fx) : fwd_kernel<kLstm>(mc); break;
    case kGru: k = BWD ? bwd_kernel<kGru>(fx) : fwd_kernel<kGru>(mc); break;
    default: k = BWD ? bwd_kernel<kSlstm>(fx) : fwd_kernel<kSlstm>(mc); break;
  }
  return cluster_launch(k, a, grid, cs.threads, cs.smem, s);
}

}  // namespace

bool cluster_kernel_attrs(int variant, bool backward, int* regs, int* local_bytes, int* max_threads) {
  const void* f;
  switch (variant) {
    case kElman: f = backward ? (const void*)cl_bwd_kernel<kElman, 16, 0> : (const void*)cl_fwd_kernel<kElman, 16, 0>; break;
    case kLstm: f = backward ? (const void*)cl_bwd_kernel<kLstm, 16, 0> : (const void*)cl_fwd_kernel<kLstm, 16, 0>; break;
    case kGru: f = backward ? (const void*)cl_bwd_kernel<kGru, 16, 0> : (const void*)cl_fwd_kernel<kGru, 16, 0>; break;
    default: f = backward ? (const void*)cl_bwd_kernel<kSlstm, 16, 0> : (const void*)cl_fwd_kernel<kSlstm, 16, 0>; break;
  }
  cudaFuncAttributes at{};
  if (cudaFuncGetAttributes(&at, f) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  *regs = at.numRegs;
  *local_bytes = (int)at.localSizeBytes;
  *max_threads = at.maxThreadsPerBlock;
  return true;
}

size_t cluster_forward_ws(const Problem& p, const Plan& pl) {
  return cluster_shape(p, pl.units_per_cta, pl.batch_tile, false, plan_ncl(pl)).ws;
}

int cluster_max_active(const Problem& p, const ClusterShape& cs, bool backward) {
  const void* f;
  switch (p.variant) {
    case kElman: f = backward ? nullptr : (const void*)cl_fwd_kernel<kElman, 16, 1>; break;
    case kLstm: f = backward ? (const void*)cl_bwd_kernel<kLstm, 16, 4> : (const void*)cl_fwd_kernel<kLstm, 16, 1>; break;
    case kGru: f = backward ? (const void*)cl_bwd_kernel<kGru, 16, 4> : (const void*)cl_fwd_kernel<kGru, 16, 1>; break;
    default: f = backward ? (const void*)cl_bwd_kernel<kSlstm, 16, 4> : (const void*)cl_fwd_kernel<kSlstm, 16, 1>; break;
  }
  if (!f) return 0;
  if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs.smem) != cudaSuccess ||
      (cs.CL > 8 && cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cs.CL * cs.NCL * cs.groups);
  cfg.blockDim = dim3(cs.threads);
  cfg.dynamicSmemBytes = cs.smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs.CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, f, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

size_t cluster_backward_ws(const Problem& p, const Plan& pl) {
  size_t off = cluster_shape(p, pl.units_per_cta, pl.batch_tile, true, plan_ncl(pl)).ws;
  bool all_in = true;
  for (int j = 0; j < p.NG; ++j) all_in = all_in && p.inp[j];
  if (!all_in) off += align_up((size_t)2 * p.T * p.B * p.NG * p.D, 256);
  off += align_up(sizeof(float) * ((p.B + pl.batch_tile - 1) / pl.batch_tile) * p.NG * p.D, 256);  // db per tile
  return off;
}

cudaError_t cluster_forward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s) {
  ClusterShape cs;
  CArgs a = make_cargs(p, pl, ws, false, cs);
  if (a.xflags) {
    cudaError_t e = cudaMemsetAsync(a.xflags, 0, sizeof(uint32_t) * cs.groups * cs.NCL * cs.CL, s);
    if (e != cudaSuccess) return e;
  }
  kt_begin(KT_FWD, s);
  cudaError_t e = launch_variant<false>(p.variant, a, cs, s);
  kt_end(KT_FWD, s);
  return e;
}

cudaError_t cluster_backward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s) {
  ClusterShape cs;
  CArgs a = make_cargs(p, pl, ws, true, cs);
  if (a.bflags) {
    cudaError_t e = cudaMemsetAsync(a.bflags, 0, sizeof(uint32_t) * cs.groups * cs.NCL * cs.CL, s);
    if (e != cudaSuccess) return e;
  }
  kt_begin(KT_BWD, s);
  cudaError_t e = launch_variant<true>(p.variant, a, cs, s);
  kt_end(KT_BWD, s);
  if (e != cudaSuccess) return e;
  const void* dgp = a.dgw ? static_cast<const void*>(a.dgw) : p.dx;
  kt_begin(KT_PARAM, s);
  if (a.dbacc) {
    e = dr_gemm(p, dgp, s);
    if (e == cudaSuccess) e = db_convert(a.dbacc, p.dbias, p.NG * p.D, a.NBT, s);
  } else {
    DgView dg{dgp, (long long)p.B * p.NG * p.D, (long long)p.NG * p.D, (long long)p.D};
    e = param_grads(p, dg, nullptr, s);
  }
  kt_end(KT_PARAM, s);
  return e;
}

}  // namespace frnn
