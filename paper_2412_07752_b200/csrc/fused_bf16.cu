// fused_bf16.cu -- persistent fused recurrence kernels for bf16 (K1 forward,
// K2 backward), sm_100a / tcgen05.
//
// Decomposition.  A head's NG*DH gate rows are split into
// CPG = DH/UPC CTAs of UPC hidden units each; a CTA owns all NG gates of its
// units, so the cell pointwise update is CTA-local.  Row order inside a CTA is
// unit-major (row = u*NGP + g) so the gates of a unit sit in adjacent TMEM
// lanes of one warp.  One group of CPG CTAs per (head, batch tile of N rows);
// groups never talk (heads are independent: engine.hpp:139-142).
//
// K1 (forward, engine.hpp:170-201), per step t:
//   wait for the group's step-(t-1) release flags -> pull h_t (= states[t][0],
//   bf16, written by the peer CTAs through L2) into a K-major SMEM tile -> one
//   thread issues K/16 tcgen05.mma round-robin over NACC independent TMEM
//   accumulators (A = the CTA's R slice, RESIDENT IN TMEM for all T steps;
//   B = the h tile) -> tcgen05.ld + sum -> add x_t and b (x prefetched a step
//   ahead, kept raw) -> cell pointwise in registers (c/n/m stay fp32 in
//   registers) -> store h_{t+1}, release the step flag -> store the rest of the
//   trace (gates, other states) off the critical path.
// K2 (backward, engine.hpp:257-336), per reverse step t:
//   wait for the group's flags -> sum the CPG partial R^T.dg vectors for the
//   owned units, clip (engine.hpp:300-303) -> pointwise Jacobian -> dg (bf16)
//   into a SMEM B tile -> tcgen05.mma with A = R_slice^T (resident in TMEM, one
//   128-lane block per 128 state columns, one accumulator per block) gives
//   this CTA's partial R^T.dg for all DH columns -> store partials, release ->
//   store dx off the critical path.  dR/db come from param_grads (K = T*B).
#include <cuda_bf16.h>

#include <cstdlib>

#include "cells.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace frnn {
namespace {

using bf16 = __nv_bfloat16;
using namespace sm100;

struct FArgs {
  Problem p;
  int UPC, CPG, NBT, groups;
  int K;        // forward contraction length (DH padded to 32)
  int MB;       // backward: 128-column blocks of DH
  int nacc;     // forward: independent accumulator chains
  uint32_t tmem_cols, acc_col;
  uint32_t* flags;  // [groups][CPG] step counters (one writer each)
  float* part;      // backward partials [2][groups][CPG][MB*128][N]
  bf16* dgw;        // backward dg trace (only when a gate is not input-wired)
  float* dbacc;     // backward db accumulator [NG][D] fp32 (tcgen05 dR path)
  long long* prof;  // optional per-step phase timestamps (clock64), thread 0 of each CTA
  int prof_steps;
};

// Phase timestamp for step index `step` (debug instrumentation, off by default).
#define FRNN_PROF(slot, step)                                              \
  if (a.prof && threadIdx.x == 0 && (step) < a.prof_steps)                 \
    a.prof[((size_t)blockIdx.x * a.prof_steps + (step)) * 8 + (slot)] = clock64();

__device__ __forceinline__ float bf(const bf16* p, size_t i) { return __bfloat162float(p[i]); }
// Raw bf16 bits: a load whose conversion is deferred to the use, so a
// prefetch does not stall the issuing thread.
__device__ __forceinline__ unsigned short raw(const bf16* p, size_t i) {
  return reinterpret_cast<const unsigned short*>(p)[i];
}
__device__ __forceinline__ float cvt(unsigned short r) { return __uint_as_float((uint32_t)r << 16); }

// Offset (bytes) of element (row n, k) in a K-major no-swizzle operand tile with
// N rows: core matrix (k/8, n/8) at ((k/8)*(N/8) + n/8)*128.
template <int N>
__device__ __forceinline__ uint32_t kmaj_off(int n, int k) {
  return (uint32_t)(((k >> 3) * (N / 8) + (n >> 3)) * 128 + (n & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Warp 0 waits until every flag of the group reached `target`; then the CTA.
// The warp polls converged: one coalesced acquire load of all flags per
// iteration (lanes spinning separately would serialise the L2 round trips).
__device__ __forceinline__ void group_wait(const uint32_t* flags, int n, uint32_t target) {
  if (threadIdx.x < 32) {
    uint64_t t0 = 0;
    for (uint32_t it = 1;; ++it) {
      bool ok = true;
      for (int q = threadIdx.x; q < n; q += 32) ok = ok && ld_acquire(flags + q) >= target;
      if (__all_sync(0xffffffffu, ok)) break;
      if ((it & 1023u) == 0) {  // a peer that never arrives traps instead of hanging
        const uint64_t now = globaltimer_ns();
        if (t0 == 0) t0 = now;
        else if (now - t0 > 4000000000ull) __trap();
      }
    }
  }
  __syncthreads();
}

template <int V, int N>
__global__ void __launch_bounds__(128, 1) fused_fwd_kernel(FArgs a) {
  using C = Cell<V>;
  constexpr int NS = C::NS, NG = C::NG, NGP = C::NGP, UPW = 32 / NGP, EPT = N / NGP;
  constexpr int LB = 12;  // h-tile loads in flight per thread
  using M = Math<true>;
  const Problem& p = a.p;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int grp = blockIdx.x / a.CPG, cta = blockIdx.x % a.CPG;
  const int hd = grp / a.NBT, b0 = (grp % a.NBT) * N;
  const int nb = min(N, p.B - b0);
  const int unit0 = cta * a.UPC;
  const int DH = p.DH, D = p.D, B = p.B, K = a.K;
  const bf16* R = static_cast<const bf16*>(p.R);
  const bf16* bias = static_cast<const bf16*>(p.bias);
  const bf16* x = static_cast<const bf16*>(p.x);
  const bf16* s0 = static_cast<const bf16*>(p.s0);
  bf16* states = static_cast<bf16*>(p.states);
  bf16* gates = static_cast<bf16*>(p.gates);
  uint32_t* gflags = a.flags + grp * a.CPG;

  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* hB = smem;                                          // [N x K] bf16, K-major
  float* xs = reinterpret_cast<float*>(smem + N * K * 2);      // [128][N+1]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + N * K * 2 + 128 * (N + 1) * 4);
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(mbar + 1);

  if (w == 0) tmem_alloc(tbase_s, a.tmem_cols);
  if (tid == 0) {
    mbar_init(mbar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < N * K * 2 / 16; i += 128) reinterpret_cast<uint4*>(hB)[i] = make_uint4(0, 0, 0, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tbase_s;

  // ---- R slice -> TMEM: lane = row (u*NGP+g), columns = bf16 pairs along K.
  {
    const int row = 32 * w + l, u = row / NGP, g = row % NGP;
    const bool valid = u < a.UPC && g < NG && p.rec[g];
    const bf16* src = R + ((size_t)(hd * NG + (valid ? g : 0)) * DH + unit0 + (valid ? u : 0)) * DH;
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t v[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = 2 * c0 + 8 * q;
        uint4 r4 = make_uint4(0, 0, 0, 0);
        if (valid && k < DH) r4 = *reinterpret_cast<const uint4*>(src + k);
        v[4 * q + 0] = r4.x;
        v[4 * q + 1] = r4.y;
        v[4 * q + 2] = r4.z;
        v[4 * q + 3] = r4.w;
      }
      tmem_st16(tbase + ((uint32_t)(32 * w) << 16) + c0, v);
    }
    tmem_st_wait();
  }

  // ---- ownership for the pointwise phase: unit u, batch rows bo*EPT + i.
  const int uw = l % UPW, bo = l / UPW;
  const int u = w * UPW + uw;
  const bool own = u < a.UPC;
  const int e = hd * DH + unit0 + (own ? u : 0);
  float st[NS][EPT], bj[NG];
  unsigned short xr[NG][EPT];
#pragma unroll
  for (int j = 0; j < NG; ++j) bj[j] = own ? bf(bias, (size_t)j * D + e) : 0.f;
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int b = bo * EPT + i;
    const bool ok = own && b < nb;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const size_t gi = ((size_t)s * B + b0 + b) * D + e;
      st[s][i] = ok ? bf(s0, gi) : 0.f;
      if (ok) states[gi] = s0[gi];  // states[0] = s0
    }
#pragma unroll
    for (int j = 0; j < NG; ++j) xr[j][i] = (ok && p.inp[j] && p.T > 0) ? raw(x, ((size_t)(b0 + b) * NG + j) * D + e) : 0;
  }

  const uint32_t idesc = idesc_bf16(128, N);
  const uint32_t hB_s = smem_u32(hB);
  constexpr uint32_t LBO = N * 16, SBO = 128;
  // h tile loader: a warp instruction covers 8 rows x 4 consecutive 16-byte
  // chunks (conflict-free core-matrix stores, 64 B contiguous per row).
  const int nkc = DH / 8;
  const int nkb = (nkc + 3) / 4;
  const int ntile = (N / 8) * nkb;
  const int r8 = l & 7, kq = l >> 3;

  for (int t = 0; t < p.T; ++t) {
    const bf16* hsrc = (t == 0 ? s0 : states + (size_t)t * NS * B * D) + (size_t)b0 * D + hd * DH;
    FRNN_PROF(0, t);
    if (t > 0) group_wait(gflags, a.CPG, (uint32_t)t);
    FRNN_PROF(1, t);
    for (int it0 = w; it0 < ntile; it0 += 4 * LB) {
      uint4 v[LB];
#pragma unroll
      for (int q = 0; q < LB; ++q) {
        const int tile = it0 + 4 * q;
        const int b = (tile % (N / 8)) * 8 + r8, kc = (tile / (N / 8)) * 4 + kq;
        // Weak loads are safe here: group_wait's ld.acquire.gpu invalidated L1
        // (CCTL.IVALL) and bar.sync orders these after it.
        if (tile < ntile && b < nb && kc < nkc) v[q] = *reinterpret_cast<const uint4*>(hsrc + (size_t)b * D + kc * 8);
      }
#pragma unroll
      for (int q = 0; q < LB; ++q) {
        const int tile = it0 + 4 * q;
        const int b = (tile % (N / 8)) * 8 + r8, kc = (tile / (N / 8)) * 4 + kq;
        if (tile < ntile && b < nb && kc < nkc) *reinterpret_cast<uint4*>(hB + kmaj_off<N>(b, kc * 8)) = v[q];
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    FRNN_PROF(2, t);
    if (w == 0) {
      // Warp 0 issues (one elected lane), operands warp-uniform; every operand
      // advances by a constant (B descriptor start address by 2*LBO bytes, A by
      // 8 TMEM columns).
      tc_fence_after();
      const uint32_t tb = __shfl_sync(0xffffffffu, tbase, 0);
      const uint32_t dacc = tb + a.acc_col;
      uint64_t bd = sdesc_kmajor(hB_s, LBO, SBO);
      uint32_t at = tb;
      for (int ks = 0; ks < K / 16; ++ks) {
        if (elect_one()) mma_ts(dacc, at, bd, idesc, ks > 0 ? 1u : 0u);
        __syncwarp();
        bd += (2 * LBO) >> 4;
        at += 8;
      }
      if (elect_one()) mma_commit(mbar);
      __syncwarp();
    }
    mbar_wait(mbar, t & 1);
    tc_fence_after();
    FRNN_PROF(3, t);
#pragma unroll
    for (int n0 = 0; n0 < N; n0 += 16) {
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(32 * w) << 16) + a.acc_col + n0, v);
#pragma unroll
      for (int q = 0; q < 16; ++q) xs[(32 * w + l) * (N + 1) + n0 + q] = v[q];
    }
    __syncwarp();
    float gout[NG][EPT], nout[NS][EPT];
    bf16* sdst = states + (size_t)(t + 1) * NS * B * D;
    if (own) {
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int b = bo * EPT + i;
        float g[4], prev[4], nx[4];
#pragma unroll
        for (int j = 0; j < NG; ++j) {  // x, then b, then y (engine.hpp:183-187)
          g[j] = cvt(xr[j][i]) + bj[j] + xs[(32 * w + uw * NGP + j) * (N + 1) + b];
          gout[j][i] = g[j];
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) prev[s] = st[s][i];
        C::template fwd<M>(prev, g, nx);
#pragma unroll
        for (int s = 0; s < NS; ++s) st[s][i] = nout[s][i] = nx[s];
        if (b < nb) sdst[((size_t)b0 + b) * D + e] = __float2bfloat16_rn(nx[0]);  // h_{t+1}
      }
    }
    FRNN_PROF(4, t);
    tc_fence_before();
    __syncthreads();
    if (tid == 0) st_release(gflags + cta, (uint32_t)(t + 1));
    FRNN_PROF(5, t);
    // Off the critical path: the rest of the trace, and x_{t+1}.
    if (own) {
      bf16* gdst = gates + (size_t)t * NG * B * D;
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int b = bo * EPT + i;
        if (b < nb) {
#pragma unroll
          for (int j = 0; j < NG; ++j) gdst[((size_t)j * B + b0 + b) * D + e] = __float2bfloat16_rn(gout[j][i]);
#pragma unroll
          for (int s = 1; s < NS; ++s) sdst[((size_t)s * B + b0 + b) * D + e] = __float2bfloat16_rn(nout[s][i]);
        }
        if (t + 1 < p.T) {
#pragma unroll
          for (int j = 0; j < NG; ++j)
            xr[j][i] = (b < nb && p.inp[j]) ? raw(x, (((size_t)(t + 1) * B + b0 + b) * NG + j) * D + e) : 0;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tbase, a.tmem_cols);
}

template <int V, int N>
__global__ void __launch_bounds__(128, 1) fused_bwd_kernel(FArgs a) {
  using C = Cell<V>;
  constexpr int NS = C::NS, NG = C::NG, NGP = C::NGP, UPW = 32 / NGP, EPT = N / NGP;
  constexpr int KB = 128;  // contraction = the CTA's 128 gate rows
  constexpr int QB = EPT >= 16 ? 2 : 8;  // partial vectors in flight per thread
  using M = Math<true>;
  const Problem& p = a.p;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int grp = blockIdx.x / a.CPG, cta = blockIdx.x % a.CPG;
  const int hd = grp / a.NBT, b0 = (grp % a.NBT) * N;
  const int nb = min(N, p.B - b0);
  const int unit0 = cta * a.UPC;
  const int DH = p.DH, D = p.D, B = p.B, T = p.T, MB = a.MB, DHP = MB * 128;
  const bool recur = p.clip_mode != 2;
  const float mag = p.clip_mag;
  const bf16* R = static_cast<const bf16*>(p.R);
  const bf16* states = static_cast<const bf16*>(p.cstates);
  const bf16* gates = static_cast<const bf16*>(p.cgates);
  const bf16* dsf = static_cast<const bf16*>(p.dsf);
  const bf16* dh = static_cast<const bf16*>(p.dh);
  bf16* dx = static_cast<bf16*>(p.dx);
  bf16* ds0 = static_cast<bf16*>(p.ds0);
  uint32_t* gflags = a.flags + grp * a.CPG;

  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* dgB = smem;  // [N x KB] bf16, K-major
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + N * KB * 2);
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(mbar + 1);

  if (w == 0) tmem_alloc(tbase_s, a.tmem_cols);
  if (tid == 0) {
    mbar_init(mbar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < N * KB * 2 / 16; i += 128) reinterpret_cast<uint4*>(dgB)[i] = make_uint4(0, 0, 0, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tbase_s;

  // ---- R_slice^T -> TMEM: block mb, lane = state column c, columns = row pairs.
  if (recur) {
    for (int mb = 0; mb < MB; ++mb) {
      const int c = mb * 128 + 32 * w + l;
      for (int c0 = 0; c0 < KB / 2; c0 += 16) {
        uint32_t v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float f[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = 2 * (c0 + q) + h, uu = row / NGP, g = row % NGP;
            f[h] = (c < DH && uu < a.UPC && g < NG && p.rec[g])
                       ? bf(R, ((size_t)(hd * NG + g) * DH + unit0 + uu) * DH + c)
                       : 0.f;
          }
          v[q] = pack_bf16(f[0], f[1]);
        }
        tmem_st16(tbase + ((uint32_t)(32 * w) << 16) + mb * (KB / 2) + c0, v);
      }
    }
    tmem_st_wait();
  }

  const int uw = l % UPW, bo = l / UPW;
  const int u = w * UPW + uw;
  const bool own = u < a.UPC;
  const int e = hd * DH + unit0 + (own ? u : 0);
  float ds[NS][EPT], dbv[NG];  // dbv: this thread's share of db (engine.hpp:317)
  unsigned short pv[NS][EPT], gv[NG][EPT], hv[EPT];
#pragma unroll
  for (int j = 0; j < NG; ++j) dbv[j] = 0.f;
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int b = bo * EPT + i;
    const bool ok = own && b < nb;
#pragma unroll
    for (int s = 0; s < NS; ++s) ds[s][i] = ok ? bf(dsf, ((size_t)s * B + b0 + b) * D + e) : 0.f;
  }
  auto prefetch = [&](int t) {
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int b = bo * EPT + i;
      const bool ok = own && b < nb && t >= 0;
#pragma unroll
      for (int s = 0; s < NS; ++s) pv[s][i] = ok ? raw(states, (((size_t)t * NS + s) * B + b0 + b) * D + e) : 0;
#pragma unroll
      for (int j = 0; j < NG; ++j) gv[j][i] = ok ? raw(gates, (((size_t)t * NG + j) * B + b0 + b) * D + e) : 0;
      hv[i] = (ok && dh) ? raw(dh, ((size_t)t * B + b0 + b) * D + e) : 0;
    }
  };
  prefetch(T - 1);

  // Sum the CPG partials of R^T.dg for the owned (unit, batch) elements,
  // clip (engine.hpp:300-303) and add to ds_h.
  auto absorb = [&](int buf) {
    float term[EPT];
#pragma unroll
    for (int i = 0; i < EPT; ++i) term[i] = 0.f;
    if (own) {
      const float* src = a.part + ((size_t)(buf * a.groups + grp) * a.CPG * DHP + (unit0 + u)) * N + bo * EPT;
      const size_t stride = (size_t)DHP * N;
      for (int q0 = 0; q0 < a.CPG; q0 += QB) {
        float4 v[QB][EPT / 4];
#pragma unroll
        for (int q = 0; q < QB; ++q)
#pragma unroll
          for (int i4 = 0; i4 < EPT / 4; ++i4)
            if (q0 + q < a.CPG) v[q][i4] = reinterpret_cast<const float4*>(src + (q0 + q) * stride)[i4];
#pragma unroll
        for (int q = 0; q < QB; ++q)
#pragma unroll
          for (int i4 = 0; i4 < EPT / 4; ++i4)
            if (q0 + q < a.CPG) {
              term[4 * i4] += v[q][i4].x;
              term[4 * i4 + 1] += v[q][i4].y;
              term[4 * i4 + 2] += v[q][i4].z;
              term[4 * i4 + 3] += v[q][i4].w;
            }
      }
    }
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      float tv = term[i];
      if (p.clip_mode == 1) tv = fminf(fmaxf(tv, -mag), mag);
      ds[0][i] += tv;
    }
  };

  const uint32_t idesc = idesc_bf16(128, N);
  const uint32_t dgB_s = smem_u32(dgB);
  constexpr uint32_t LBO = N * 16, SBO = 128;
  uint32_t phase = 0;

  for (int t = T - 1; t >= 0; --t) {
    const int k = T - 1 - t;  // steps already published
    FRNN_PROF(0, k);
    if (recur && k > 0) {
      group_wait(gflags, a.CPG, (uint32_t)k);
      absorb((t + 1) & 1);
    }
    float dgv[NG][EPT];
    if (own) {
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int b = bo * EPT + i;
        float prev[4], g[4], dsl[4], dg[4], dsp[4];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          prev[s] = cvt(pv[s][i]);
          dsl[s] = ds[s][i];
        }
        dsl[0] += cvt(hv[i]);  // engine.hpp:258-263
#pragma unroll
        for (int j = 0; j < NG; ++j) g[j] = cvt(gv[j][i]);
        C::template bwd<M>(prev, g, dsl, dg, dsp);
#pragma unroll
        for (int j = 0; j < NG; ++j) {
          dgv[j][i] = dg[j];
          if (b < nb) dbv[j] += dg[j];
          if (b < nb)
            *reinterpret_cast<bf16*>(dgB + kmaj_off<N>(b, 32 * w + uw * NGP + j)) = __float2bfloat16_rn(dg[j]);
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) ds[s][i] = dsp[s];
      }
    }
    FRNN_PROF(1, k);
    prefetch(t - 1);
    if (recur) {
      fence_proxy_async_smem();
      __syncthreads();
      FRNN_PROF(2, k);
      if (w == 0) {
        tc_fence_after();
        const uint32_t tb = __shfl_sync(0xffffffffu, tbase, 0);
        const uint64_t bd0 = sdesc_kmajor(dgB_s, LBO, SBO);
        uint32_t dacc = tb + a.acc_col, at = tb;
        for (int mb = 0; mb < MB; ++mb) {
          uint64_t bd = bd0;
#pragma unroll
          for (int ks = 0; ks < KB / 16; ++ks) {
            if (elect_one()) mma_ts(dacc, at + ks * 8, bd, idesc, ks > 0 ? 1u : 0u);
            __syncwarp();
            bd += (2 * LBO) >> 4;
          }
          dacc += N;
          at += KB / 2;
        }
        if (elect_one()) mma_commit(mbar);
        __syncwarp();
      }
      mbar_wait(mbar, phase);
      phase ^= 1;
      tc_fence_after();
      FRNN_PROF(3, k);
      float* dst0 = a.part + ((size_t)((t & 1) * a.groups + grp) * a.CPG + cta) * DHP * N;
      for (int mb = 0; mb < MB; ++mb) {
        const int c = mb * 128 + 32 * w + l;
#pragma unroll
        for (int n0 = 0; n0 < N; n0 += 16) {
          float v[16];
          tmem_ld16(tbase + ((uint32_t)(32 * w) << 16) + a.acc_col + mb * N + n0, v);
          if (c < DH) {
            float* dst = dst0 + (size_t)c * N + n0;
#pragma unroll
            for (int q = 0; q < 16; q += 4)
              *reinterpret_cast<float4*>(dst + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
          }
        }
      }
      FRNN_PROF(4, k);
      tc_fence_before();
      __syncthreads();
      if (tid == 0) st_release(gflags + cta, (uint32_t)(k + 1));
      FRNN_PROF(5, k);
    }
    // Off the critical path: dx (= dg for input-wired gates, engine.hpp:311-316).
    if (own) {
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int b = bo * EPT + i;
        if (b >= nb) continue;
#pragma unroll
        for (int j = 0; j < NG; ++j) {
          const size_t xi = (((size_t)t * B + b0 + b) * NG + j) * D + e;
          const bf16 v = __float2bfloat16_rn(dgv[j][i]);
          dx[xi] = p.inp[j] ? v : __float2bfloat16_rn(0.f);
          if (a.dgw) a.dgw[xi] = v;
        }
      }
    }
  }
  if (recur && T > 0) {
    group_wait(gflags, a.CPG, (uint32_t)T);
    absorb(0);
  }
  if (own) {
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int b = bo * EPT + i;
      if (b >= nb) continue;
#pragma unroll
      for (int s = 0; s < NS; ++s) ds0[((size_t)s * B + b0 + b) * D + e] = __float2bfloat16_rn(ds[s][i]);
    }
  }
  if (a.dbacc) {  // db: sum this unit's batch shares across lanes, one fp32 atomic per (gate, unit, tile)
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      float v = dbv[j];
#pragma unroll
      for (int off = UPW; off < 32; off <<= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (own && bo == 0) a.dbacc[((size_t)(grp % a.NBT) * NG + j) * D + e] = v;  // one writer per (tile, gate, unit)
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tbase, a.tmem_cols);
}

uint32_t pow2_cols(uint32_t c) {
  uint32_t r = 32;
  while (r < c) r <<= 1;
  return r;
}

}  // namespace

long long* g_prof_buf = nullptr;
int g_prof_steps = 0;

namespace {

struct Layout {
  int K, MB, nacc;
  uint32_t acc_col, tmem_cols;
};

Layout tmem_layout(const Problem& p, int N, bool backward) {
  Layout L{};
  L.K = (int)align_up(p.DH, 32);
  L.MB = (p.DH + 127) / 128;
  if (!backward) {
    L.acc_col = (uint32_t)align_up(L.K / 2, 32);
    L.nacc = 1;
    L.tmem_cols = pow2_cols(L.acc_col + N);
  } else {
    L.acc_col = (uint32_t)(L.MB * 64);
    L.nacc = L.MB;
    L.tmem_cols = pow2_cols(L.acc_col + L.MB * N);
  }
  return L;
}

size_t flags_bytes(int groups, int CPG) { return align_up(sizeof(uint32_t) * groups * CPG, 256); }

FArgs make_args(const Problem& p, const Plan& pl, void* ws, bool backward) {
  FArgs a{};
  a.prof = g_prof_buf;
  a.prof_steps = g_prof_steps;
  a.p = p;
  a.UPC = pl.units_per_cta;
  a.CPG = pl.ctas_per_group;
  a.NBT = (p.B + pl.batch_tile - 1) / pl.batch_tile;
  a.groups = p.NH * a.NBT;
  const int N = pl.batch_tile;
  Layout L = tmem_layout(p, N, backward);
  a.K = L.K;
  a.MB = L.MB;
  a.nacc = L.nacc;
  a.acc_col = L.acc_col;
  a.tmem_cols = L.tmem_cols;
  char* w = static_cast<char*>(ws);
  a.flags = reinterpret_cast<uint32_t*>(w);
  size_t off = flags_bytes(a.groups, a.CPG);
  if (backward) {
    a.part = reinterpret_cast<float*>(w + off);
    off += align_up(sizeof(float) * 2 * a.groups * a.CPG * (size_t)a.MB * 128 * N, 256);
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

size_t fwd_smem(int N, int K) { return (size_t)N * K * 2 + 128 * (N + 1) * 4 + 16; }
size_t bwd_smem(int N) { return (size_t)N * 128 * 2 + 16; }

template <class KernelT>
cudaError_t coop_launch(KernelT kern, const FArgs& a, int grid, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  FArgs copy = a;
  void* args[] = {&copy};
  note_launch();
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(128), args, smem,
                                     s);
}

}  // namespace

uint32_t fused_tmem_cols(const Problem& p, int N, bool backward) { return tmem_layout(p, N, backward).tmem_cols; }

size_t fused_forward_ws(const Problem& p, const Plan& pl) {
  const int groups = p.NH * ((p.B + pl.batch_tile - 1) / pl.batch_tile);
  return flags_bytes(groups, pl.ctas_per_group);
}

size_t fused_backward_ws(const Problem& p, const Plan& pl) {
  const int N = pl.batch_tile;
  const int groups = p.NH * ((p.B + N - 1) / N);
  const int MB = (p.DH + 127) / 128;
  size_t off = flags_bytes(groups, pl.ctas_per_group);
  off += align_up(sizeof(float) * 2 * groups * pl.ctas_per_group * (size_t)MB * 128 * N, 256);
  bool all_in = true;
  for (int j = 0; j < p.NG; ++j) all_in = all_in && p.inp[j];
  if (!all_in) off += align_up((size_t)2 * p.T * p.B * p.NG * p.D, 256);
  off += align_up(sizeof(float) * ((p.B + N - 1) / N) * p.NG * p.D, 256);  // db per batch tile
  return off;
}

#define FRNN_FUSED_DISPATCH(KERNEL, N_)                                             \
  switch (p.variant) {                                                               \
    case kElman: e = coop_launch(KERNEL<kElman, N_>, a, pl.grid, smem, s); break;    \
    case kLstm: e = coop_launch(KERNEL<kLstm, N_>, a, pl.grid, smem, s); break;      \
    case kGru: e = coop_launch(KERNEL<kGru, N_>, a, pl.grid, smem, s); break;        \
    default: e = coop_launch(KERNEL<kSlstm, N_>, a, pl.grid, smem, s); break;        \
  }

cudaError_t fused_forward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s) {
  FArgs a = make_args(p, pl, ws, false);
  cudaError_t e = cudaMemsetAsync(a.flags, 0, sizeof(uint32_t) * a.groups * a.CPG, s);
  if (e != cudaSuccess) return e;
  const size_t smem = fwd_smem(pl.batch_tile, a.K);
  if (pl.batch_tile != 16) return cudaErrorInvalidValue;
  kt_begin(KT_FWD, s);
  FRNN_FUSED_DISPATCH(fused_fwd_kernel, 16)
  kt_end(KT_FWD, s);
  return e;
}

cudaError_t fused_backward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s) {
  FArgs a = make_args(p, pl, ws, true);
  cudaError_t e = cudaMemsetAsync(a.flags, 0, sizeof(uint32_t) * a.groups * a.CPG, s);
  if (e != cudaSuccess) return e;
  const size_t smem = bwd_smem(pl.batch_tile);
  if (pl.batch_tile != 16) return cudaErrorInvalidValue;
  kt_begin(KT_BWD, s);
  FRNN_FUSED_DISPATCH(fused_bwd_kernel, 16)
  kt_end(KT_BWD, s);
  if (e != cudaSuccess) return e;
  // dR / db from the dg trace (dx when every gate is input-wired).
  const void* dgp = a.dgw ? static_cast<const void*>(a.dgw) : p.dx;
  kt_begin(KT_PARAM, s);
  if (a.dbacc) {  // tcgen05 GEMM for dR; db was accumulated by the recurrence
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
