// alternating.cu -- K4/K5: the alternating path for hidden sizes whose R does
// not fit on-chip: the time loop runs on the
// host, and every step is ONE kernel that streams R from L2/HBM through a TMA
// ring into tcgen05.mma and applies the cell's pointwise map in the epilogue
// (the paper's separate matmul + pointwise kernels, fused).  Consecutive step
// kernels are chained with programmatic dependent launch: kernel t+1 starts
// while kernel t drains, allocates TMEM and prefetches its first R stages
// (R does not depend on the previous step) and only then waits for h_t.
//
// Forward step t (engine.hpp:170-201), one CTA per (unit tile, head, batch tile):
//   A = R rows of UPT units x NG gates (128 rows, gate-major, K-major in rnnkit's
//       R[NH][NG][DH][DH] layout: a 4-D tensor-map box (64 k, UPT units, NG, 1))
//   B = h_t = states[t][0] rows of the batch tile (K-major: states[t][0][b][:])
//   D = A.B^T in TMEM (M=128, N = batch tile), then per element
//   g = (x) + b + y (engine.hpp:183-187), pointwise_forward (cell.hpp:65-99),
//   gates[t], states[t+1] (bf16 trace) and the fp32 state carry are written.
//
// Backward kernel for step t (engine.hpp:257-336), reverse order; it first
// finishes step t+1's recurrent term and then runs step t's Jacobian:
//   A = R^T: 128 state columns c x K = (gate j, row r) over the gates that use
//       R, MN-major (c is contiguous in R[hd][j][r][:]), 2 x (64c x 64r) boxes
//   B = dg_{t+1}[b][j][hd*DH + r] (K-major, from dx -- or the dg workspace
//       when a gate has no input, GRU) -- 5-D box (64 r, 1, 1, N b, 1 t)
//   K is split over a thread-block cluster of KS CTAs; each CTA drains its
//   partial to shared memory and the owner of a column range sums the KS
//   partials in rank order through DSMEM (deterministic), clips
//   (engine.hpp:300-303), adds it to ds_h, then (unless t == -1, the final
//   ds0 kernel) applies the Jacobian (cell.hpp:108-201 contracted as
//   engine.hpp:275-284): dx[t] = dg (0 for un-wired gates), db += dg (fixed
//   order, per batch tile), and carries ds_prev in fp32.
// dR is one tcgen05 GEMM over K = T*B after the loop (dr_gemm.cu).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "cells.cuh"
#include "kernels.h"
#include "sm100.cuh"
#include "tmap.h"

namespace frnn {
extern long long* g_prof_buf;
extern int g_prof_steps;
namespace {

using bf16 = __nv_bfloat16;
using namespace sm100;

constexpr int ATHREADS = 256;
constexpr int MAXKS = 8;
constexpr uint32_t A_BYTES = 128 * 64 * 2;  // one A stage: 128 rows x 64 K (bf16)
constexpr int PC = 132;                     // backward partial pitch (floats): 128 columns + 4

struct AltArgs {
  Problem p;
  int t;          // forward: step; backward: Jacobian step (-1 = final ds0 kernel)
  int N;          // batch tile (MMA N)
  int UPT;        // forward: units per tile
  int numk;       // forward: K blocks (DH / 64)
  int stages;
  int KS, KT, kpg, nrec, has_gemm, first;
  int ka;         // 64-wide K atoms per pipeline stage (TMA boxes per operand)
  int dbg;        // experiment hook (FRNN_ALT_DBG): 1 skip R loads, 2 skip h loads, 4 skip MMA (timing only)
  int recg[4];
  uint32_t stage_bytes, a_bytes, region, tmem_cols;  // a_bytes: A part of a stage (ka atoms)
  float* carry;   // fp32 [NS][B][D]: forward state / backward ds carry
  bf16* dgw;      // backward: dg trace when some gate is not input-wired
  float* dbacc;   // backward: [NBT][NG][D]
  long long* prof;  // frnn_debug_profile: globaltimer stamps [launch][cta][4]
  int prof_slot;    // launch index (-1: off)
};

// Stamp k of this CTA by thread `who`: 0 start, 1 dependency released (an idle
// warp), 2 GEMM done, 3 end, 4 producer finished issuing.
#define ALT_PROF_BY(k, who)                                                                           \
  if (a.prof && a.prof_slot >= 0 && threadIdx.x == (who))                                             \
    a.prof[(((size_t)a.prof_slot * gridDim.x * gridDim.y * gridDim.z) +                               \
            (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 8 + (k)] = (long long)globaltimer_ns();
#define ALT_PROF(k) ALT_PROF_BY(k, 0)

__device__ __forceinline__ float bf(const bf16* p, size_t i) { return __bfloat162float(p[i]); }

__device__ __forceinline__ float4 ld_dsmem_f4(const void* local, uint32_t rank) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(mapa_shared(smem_u32(local), rank))
               : "memory");
  return v;
}

struct Smem {
  uint8_t* stage0;
  uint64_t *full, *empty, *done;
  uint32_t* tbase_s;
};

__device__ __forceinline__ Smem carve(uint8_t* raw, const AltArgs& a) {
  Smem s;
  s.stage0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  s.full = reinterpret_cast<uint64_t*>(s.stage0 + a.region);
  s.empty = s.full + a.stages;
  s.done = s.empty + a.stages;
  s.tbase_s = reinterpret_cast<uint32_t*>(s.done + 1);
  return s;
}

__device__ __forceinline__ uint32_t prologue(const Smem& s, const AltArgs& a, const void* m0, const void* m1) {
  const int tid = threadIdx.x, w = tid >> 5;
  if (w == 2) tmem_alloc(s.tbase_s, a.tmem_cols);
  if (tid == 32) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    mbar_init(s.done, 1);
    fence_mbar_init();
  }
  if (tid == 0) {
    prefetch_tensormap(m0);
    prefetch_tensormap(m1);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  return *s.tbase_s;
}

// Drain the fp32 accumulator (lane = row m, column = batch b) of M=128 x N.
// to_rows: dst[m * pitch + b] (forward); else dst[b * pitch + m] (backward).
__device__ __forceinline__ void drain(uint32_t tbase, int N, float* dst, int pitch, bool to_rows) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int q = w & 3, half = w >> 2;
  for (int ch = half; ch < N / 16; ch += 2) {
    float v[16];
    tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + ch * 16, v);
    const int m = 32 * q + l;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (to_rows) dst[m * pitch + ch * 16 + i] = v[i];
      else dst[(ch * 16 + i) * pitch + m] = v[i];
    }
  }
}

// ------------------------------------------------------------ forward ----
template <int V>
__global__ void __launch_bounds__(ATHREADS, 1)
    alt_fwd_kernel(const __grid_constant__ CUtensorMap mapR, const __grid_constant__ CUtensorMap mapH, AltArgs a) {
  using C = Cell<V>;
  constexpr int NS = C::NS, NG = C::NG;
  using M = Math<true>;
  const Problem& p = a.p;
  const int tid = threadIdx.x, w = tid >> 5;
  const int hd = blockIdx.y, b0 = blockIdx.z * a.N, nb = min(a.N, p.B - b0);
  const int UPT = a.UPT, unit0 = blockIdx.x * UPT;
  const int t = a.t, N = a.N, DH = p.DH, D = p.D, B = p.B;

  ALT_PROF(0);
  extern __shared__ uint8_t smem_raw[];
  const Smem s = carve(smem_raw, a);
  const uint32_t tbase = prologue(s, a, &mapR, &mapH);
  griddep_launch_dependents();

  if (w == 0) {  // TMA producer: R prefetch before the dependency, then h_t
    if (elect_one()) {
      const uint64_t pol = l2_evict_last_policy();
      const int npre = min(a.stages, a.numk);
      const bool lr = !(a.dbg & 1), lh = !(a.dbg & 2);
      const uint32_t sb = (lr ? a.a_bytes : 0u) + (lh ? a.stage_bytes - a.a_bytes : 0u);
      const uint32_t bat = (uint32_t)N * 128;  // one B atom
      auto load_r = [&](int kb, uint8_t* sp, uint64_t* bar) {
        for (int q = 0; q < a.ka; ++q)
          tma_load_4d_hint(sp + q * A_BYTES, &mapR, (kb * a.ka + q) * 64, unit0, 0, hd, bar, pol);
      };
      auto load_h = [&](int kb, uint8_t* sp, uint64_t* bar) {
        for (int q = 0; q < a.ka; ++q)
          tma_load_4d(sp + a.a_bytes + q * bat, &mapH, (kb * a.ka + q) * 64, hd, b0, t * NS, bar);
      };
      for (int kb = 0; kb < npre; ++kb) {
        mbar_arrive_expect_tx(&s.full[kb], sb);
        if (lr) load_r(kb, s.stage0 + kb * a.stage_bytes, &s.full[kb]);
      }
      griddep_wait();
      ALT_PROF(5);
      for (int kb = 0; kb < npre; ++kb)
        if (lh) load_h(kb, s.stage0 + kb * a.stage_bytes, &s.full[kb]);
      for (int kb = npre; kb < a.numk; ++kb) {
        const int st = kb % a.stages;
        mbar_wait(&s.empty[st], ((kb / a.stages) - 1) & 1);
        if (kb == npre) ALT_PROF(6);
        uint8_t* sp = s.stage0 + st * a.stage_bytes;
        mbar_arrive_expect_tx(&s.full[st], sb);
        if (lr) load_r(kb, sp, &s.full[st]);
        if (lh) load_h(kb, sp, &s.full[st]);
      }
      ALT_PROF(4);
    }
    __syncwarp();
  } else if (w == 1) {  // MMA issuer
    const uint32_t idesc = idesc_bf16(128, N);
    for (int kb = 0; kb < a.numk; ++kb) {
      const int st = kb % a.stages;
      mbar_wait(&s.full[st], (kb / a.stages) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(s.stage0 + st * a.stage_bytes);
      if (!(a.dbg & 4)) {
        for (int q = 0; q < a.ka; ++q) {
          const uint64_t ad = sdesc_k_sw128(sa + q * A_BYTES), bd = sdesc_k_sw128(sa + a.a_bytes + q * N * 128);
          mma4_ss(tbase, ad, 2, bd, 2, idesc, (kb | q) ? 1u : 0u);  // the atom's 4 K=16 steps
        }
      }
      if (elect_one()) {
        if (a.dbg & 8) mbar_arrive(&s.empty[st]);  // experiment: plain arrive (valid only without MMAs)
        else mma_commit(&s.empty[st]);
      }
      __syncwarp();
      if (kb == 0) ALT_PROF_BY(7, 32);
    }
    if (elect_one()) mma_commit(s.done);
    __syncwarp();
  }
  griddep_wait();
  ALT_PROF_BY(1, 64);
  // ---- epilogue operands, prefetched while the GEMM streams: each thread owns
  // a pair of adjacent units of FP rows (bf16x2 / float2 accesses).
  const bf16* x = static_cast<const bf16*>(p.x);
  const bf16* bias = static_cast<const bf16*>(p.bias);
  bf16* gates = static_cast<bf16*>(p.gates);
  bf16* states = static_cast<bf16*>(p.states);
  const size_t sBD = (size_t)B * D;
  const int NPAIR = UPT / 2, RPP = ATHREADS / NPAIR;
  const int pu = tid % NPAIR, r0 = tid / NPAIR, u = 2 * pu;
  const bool uvalid = unit0 + u < DH;
  const int e = hd * DH + unit0 + u;
  uint32_t bj[NG];
#pragma unroll
  for (int j = 0; j < NG; ++j) bj[j] = uvalid ? *reinterpret_cast<const uint32_t*>(bias + (size_t)j * D + e) : 0u;
  constexpr int FP = 4;  // rows prefetched per chunk
  uint32_t xv[FP][NG];
  float2 cv[FP][NS];
  auto load_chunk = [&](int pass0) {
#pragma unroll
    for (int k = 0; k < FP; ++k) {
      const int b = r0 + RPP * (pass0 + k);
      if (uvalid && b < nb) {
        const size_t so = (size_t)(b0 + b) * D + e;
        const size_t xo = ((size_t)t * B + b0 + b) * NG * D + e;
#pragma unroll
        for (int j = 0; j < NG; ++j)
          if (p.inp[j]) xv[k][j] = *reinterpret_cast<const uint32_t*>(x + xo + (size_t)j * D);
#pragma unroll
        for (int q = 0; q < NS; ++q) cv[k][q] = *reinterpret_cast<const float2*>(a.carry + q * sBD + so);
      }
    }
  };
  load_chunk(0);
  mbar_wait(s.done, 0);
  ALT_PROF(2);
  tc_fence_after();
  float* xs = reinterpret_cast<float*>(s.stage0);  // the ring is drained: reuse it
  const int XP = N + 1;
  drain(tbase, N, xs, XP, true);
  tc_fence_before();
  __syncthreads();

  const int passes = (nb + RPP - 1) / RPP;
  for (int pass0 = 0; pass0 < passes; pass0 += FP) {
    if (pass0 > 0) load_chunk(pass0);
#pragma unroll
    for (int k = 0; k < FP; ++k) {
      const int b = r0 + RPP * (pass0 + k);
      if (!uvalid || b >= nb) continue;
      const size_t so = (size_t)(b0 + b) * D + e;
      float gout[2][4], nout[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float g[4], prev[4], nx[4];
#pragma unroll
        for (int j = 0; j < NG; ++j) {  // x, then b, then y (engine.hpp:183-187)
          float acc = p.inp[j] ? __uint_as_float(h ? (xv[k][j] & 0xFFFF0000u) : (xv[k][j] << 16)) : 0.f;
          acc += __uint_as_float(h ? (bj[j] & 0xFFFF0000u) : (bj[j] << 16));
          acc += p.rec[j] ? xs[(j * UPT + u + h) * XP + b] : 0.f;
          g[j] = gout[h][j] = acc;
        }
#pragma unroll
        for (int q = 0; q < NS; ++q) prev[q] = h ? cv[k][q].y : cv[k][q].x;
        C::template fwd<M>(prev, g, nx);
#pragma unroll
        for (int q = 0; q < NS; ++q) nout[h][q] = nx[q];
      }
#pragma unroll
      for (int j = 0; j < NG; ++j)
        *reinterpret_cast<uint32_t*>(gates + ((size_t)t * NG + j) * sBD + so) = pack_bf16(gout[0][j], gout[1][j]);
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        *reinterpret_cast<uint32_t*>(states + ((size_t)(t + 1) * NS + q) * sBD + so) =
            pack_bf16(nout[0][q], nout[1][q]);
        *reinterpret_cast<float2*>(a.carry + q * sBD + so) = make_float2(nout[0][q], nout[1][q]);
      }
    }
  }
  ALT_PROF(3);
  fence_proxy_async_global();  // states[t+1][0] is the next step's TMA operand
  tc_fence_before();
  __syncthreads();
  if (w == 2) tmem_dealloc(tbase, a.tmem_cols);
}

// states[0] = s0 and the fp32 carry
__global__ void alt_fwd_init(const bf16* s0, bf16* states, float* carry, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const bf16 v = s0[i];
    states[i] = v;
    carry[i] = __bfloat162float(v);
  }
}

// ----------------------------------------------------------- backward ----
template <int V>
__global__ void __launch_bounds__(ATHREADS, 1)
    alt_bwd_kernel(const __grid_constant__ CUtensorMap mapRT, const __grid_constant__ CUtensorMap mapDG, AltArgs a) {
  using C = Cell<V>;
  constexpr int NS = C::NS, NG = C::NG;
  using M = Math<true>;
  const Problem& p = a.p;
  const int tid = threadIdx.x, w = tid >> 5;
  const int KS = a.KS;
  const int rank = KS > 1 ? (int)cluster_ctarank() : 0;
  const int c0 = (blockIdx.x / KS) * 128;
  const int hd = blockIdx.y, bt = blockIdx.z, b0 = bt * a.N, nb = min(a.N, p.B - b0);
  const int t = a.t, N = a.N, DH = p.DH, D = p.D, B = p.B;
  const int kb0 = rank * a.KT / KS, kb1 = (rank + 1) * a.KT / KS, numk = a.has_gemm ? kb1 - kb0 : 0;

  ALT_PROF(0);
  extern __shared__ uint8_t smem_raw[];
  const Smem s = carve(smem_raw, a);
  const uint32_t tbase = prologue(s, a, &mapRT, &mapDG);
  griddep_launch_dependents();

  if (numk > 0) {
    if (w == 0) {
      if (elect_one()) {
        const uint64_t pol = l2_evict_last_policy();
        const int npre = min(a.stages, numk);
        auto load_a = [&](int i, uint8_t* sp, uint64_t* bar) {
          const int kb = kb0 + i, g = a.recg[kb / a.kpg], rb = kb % a.kpg;
          for (int q = 0; q < a.ka; ++q) {
            const int r = (rb * a.ka + q) * 64;
            tma_load_4d_hint(sp + q * A_BYTES, &mapRT, c0, r, g, hd, bar, pol);
            tma_load_4d_hint(sp + q * A_BYTES + A_BYTES / 2, &mapRT, c0 + 64, r, g, hd, bar, pol);
          }
        };
        auto load_b = [&](int i, uint8_t* sp, uint64_t* bar) {
          const int kb = kb0 + i, g = a.recg[kb / a.kpg], rb = kb % a.kpg;
          for (int q = 0; q < a.ka; ++q)
            tma_load_5d(sp + a.a_bytes + q * N * 128, &mapDG, (rb * a.ka + q) * 64, hd, g, b0, t + 1, bar);
        };
        for (int i = 0; i < npre; ++i) {
          mbar_arrive_expect_tx(&s.full[i], a.stage_bytes);
          load_a(i, s.stage0 + i * a.stage_bytes, &s.full[i]);
        }
        griddep_wait();
        for (int i = 0; i < npre; ++i) load_b(i, s.stage0 + i * a.stage_bytes, &s.full[i]);
        for (int i = npre; i < numk; ++i) {
          const int st = i % a.stages;
          mbar_wait(&s.empty[st], ((i / a.stages) - 1) & 1);
          uint8_t* sp = s.stage0 + st * a.stage_bytes;
          mbar_arrive_expect_tx(&s.full[st], a.stage_bytes);
          load_a(i, sp, &s.full[st]);
          load_b(i, sp, &s.full[st]);
        }
        ALT_PROF(4);
      }
      __syncwarp();
    } else if (w == 1) {
      const uint32_t idesc = idesc_bf16(128, N) | (1u << 15);  // A (R^T) MN-major, B K-major
      for (int i = 0; i < numk; ++i) {
        const int st = i % a.stages;
        mbar_wait(&s.full[st], (i / a.stages) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(s.stage0 + st * a.stage_bytes);
        for (int q = 0; q < a.ka; ++q) {
          const uint64_t ad = sdesc_mn_sw128_chunk(sa + q * A_BYTES, A_BYTES / 2),
                         bd = sdesc_k_sw128(sa + a.a_bytes + q * N * 128);
          mma4_ss(tbase, ad, 128, bd, 2, idesc, (i | q) ? 1u : 0u);
        }
        if (elect_one()) mma_commit(&s.empty[st]);
        __syncwarp();
      }
      if (elect_one()) mma_commit(s.done);
      __syncwarp();
    }
  }
  griddep_wait();
  ALT_PROF_BY(1, 64);
  // This rank finishes columns [cb, ce) of the tile; an item is 4 adjacent
  // columns x 1 batch row (8-byte bf16 / 16-byte fp32 accesses).
  const int CW = (((128 + KS - 1) / KS) + 3) & ~3;
  const int cb = min(128, rank * CW), ce = min(128, cb + CW);
  const int G = (ce - cb) / 4;  // column groups
  const int NBL = G > 0 ? ATHREADS / G : 1;
  const int cg = G > 0 ? tid % G : 0, bl = G > 0 ? tid / G : NBL;
  const int cl = cb + 4 * cg;
  const bool cvalid = G > 0 && bl < NBL && c0 + cl < DH;
  const int e = hd * DH + c0 + cl;
  const bool recur = a.has_gemm != 0;
  const float mag = p.clip_mag;
  const bf16* states = static_cast<const bf16*>(p.cstates);
  const bf16* gates = static_cast<const bf16*>(p.cgates);
  const bf16* dsf = static_cast<const bf16*>(p.dsf);
  const bf16* dh = static_cast<const bf16*>(p.dh);
  bf16* dx = static_cast<bf16*>(p.dx);
  bf16* ds0 = static_cast<bf16*>(p.ds0);
  const size_t sBD = (size_t)B * D;
  constexpr int FB = 2;  // items prefetched per chunk
  uint2 pv[FB][NS], gv[FB][NG], hv[FB];
  float4 dv[FB][NS];
  auto unpack4 = [](uint2 v, float* f) {
    f[0] = __uint_as_float(v.x << 16);
    f[1] = __uint_as_float(v.x & 0xFFFF0000u);
    f[2] = __uint_as_float(v.y << 16);
    f[3] = __uint_as_float(v.y & 0xFFFF0000u);
  };
  auto load_chunk = [&](int k0) {
#pragma unroll
    for (int k = 0; k < FB; ++k) {
      const int b = bl + NBL * (k0 + k);
      if (cvalid && b < nb) {
        const size_t so = (size_t)(b0 + b) * D + e;
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          if (a.first) {
            float f[4];
            unpack4(*reinterpret_cast<const uint2*>(dsf + q * sBD + so), f);
            dv[k][q] = make_float4(f[0], f[1], f[2], f[3]);
          } else {
            dv[k][q] = *reinterpret_cast<const float4*>(a.carry + q * sBD + so);
          }
        }
        if (t >= 0) {
#pragma unroll
          for (int q = 0; q < NS; ++q)
            pv[k][q] = *reinterpret_cast<const uint2*>(states + ((size_t)t * NS + q) * sBD + so);
#pragma unroll
          for (int j = 0; j < NG; ++j)
            gv[k][j] = *reinterpret_cast<const uint2*>(gates + ((size_t)t * NG + j) * sBD + so);
          hv[k] = dh ? *reinterpret_cast<const uint2*>(dh + (size_t)t * sBD + so) : make_uint2(0u, 0u);
        }
      }
    }
  };
  load_chunk(0);

  float* part = reinterpret_cast<float*>(s.stage0);  // [b][PC]: partial R^T dg of my K range
  if (numk > 0) {
    mbar_wait(s.done, 0);
    tc_fence_after();
    drain(tbase, N, part, PC, false);
  }
  tc_fence_before();
  __syncthreads();
  if (a.has_gemm && KS > 1) cluster_sync_all();  // every rank's partial is in its smem
  ALT_PROF(2);

  float dbp[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) dbp[j][i] = 0.f;
  const int items = (nb + NBL - 1) / NBL;
  for (int k0 = 0; k0 < items; k0 += FB) {
    if (k0 > 0) load_chunk(k0);
#pragma unroll
    for (int k = 0; k < FB; ++k) {
      const int b = bl + NBL * (k0 + k);
      if (!cvalid || b >= nb) continue;
      const size_t so = (size_t)(b0 + b) * D + e;
      float term[4] = {0.f, 0.f, 0.f, 0.f};
      if (recur) {
        float4 v[MAXKS];
        const float* src = part + b * PC + cl;
#pragma unroll
        for (int r = 0; r < MAXKS; ++r)
          if (r < KS) v[r] = KS > 1 ? ld_dsmem_f4(src, r) : *reinterpret_cast<const float4*>(src);
#pragma unroll
        for (int r = 0; r < MAXKS; ++r)
          if (r < KS) {  // fixed rank order: deterministic
            term[0] += v[r].x;
            term[1] += v[r].y;
            term[2] += v[r].z;
            term[3] += v[r].w;
          }
      }
      float dsv[4][4], prv[4][4], gtv[4][4], dhv[4];
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        dsv[q][0] = dv[k][q].x;
        dsv[q][1] = dv[k][q].y;
        dsv[q][2] = dv[k][q].z;
        dsv[q][3] = dv[k][q].w;
      }
      if (recur) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float tv = term[i];
          if (p.clip_mode == 1) tv = fminf(fmaxf(tv, -mag), mag);  // engine.hpp:300-303
          dsv[0][i] += tv;
        }
      }
      if (t < 0) {  // final: ds0 = d states[0]
#pragma unroll
        for (int q = 0; q < NS; ++q)
          *reinterpret_cast<uint2*>(ds0 + q * sBD + so) =
              make_uint2(pack_bf16(dsv[q][0], dsv[q][1]), pack_bf16(dsv[q][2], dsv[q][3]));
        continue;
      }
#pragma unroll
      for (int q = 0; q < NS; ++q) unpack4(pv[k][q], prv[q]);
#pragma unroll
      for (int j = 0; j < NG; ++j) unpack4(gv[k][j], gtv[j]);
      unpack4(hv[k], dhv);
      float dgo[4][4], dso[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float ds[4], prev[4], g[4], dg[4], dsp[4];
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          ds[q] = dsv[q][i];
          prev[q] = prv[q][i];
        }
        ds[0] += dhv[i];  // engine.hpp:258-263 (zero when no step gradients)
#pragma unroll
        for (int j = 0; j < NG; ++j) g[j] = gtv[j][i];
        C::template bwd<M>(prev, g, ds, dg, dsp);
#pragma unroll
        for (int j = 0; j < NG; ++j) {
          dgo[j][i] = dg[j];
          dbp[j][i] += dg[j];
        }
#pragma unroll
        for (int q = 0; q < NS; ++q) dso[q][i] = dsp[q];
      }
      const size_t xo = ((size_t)t * B + b0 + b) * NG * D + e;
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        const uint2 d = make_uint2(pack_bf16(dgo[j][0], dgo[j][1]), pack_bf16(dgo[j][2], dgo[j][3]));
        *reinterpret_cast<uint2*>(dx + xo + (size_t)j * D) = p.inp[j] ? d : make_uint2(0u, 0u);
        if (a.dgw) *reinterpret_cast<uint2*>(a.dgw + xo + (size_t)j * D) = d;
      }
#pragma unroll
      for (int q = 0; q < NS; ++q)
        *reinterpret_cast<float4*>(a.carry + q * sBD + so) = make_float4(dso[q][0], dso[q][1], dso[q][2], dso[q][3]);
    }
  }
  if (a.has_gemm && KS > 1) cluster_sync_all();  // peers are done reading my partials
  if (t >= 0 && G > 0) {  // db: fixed-order sum over this tile's batch rows (deterministic)
    float* dbs = part;    // [NG][NBL][G*4]
    const int W4 = G * 4;
    __syncthreads();
    if (bl < NBL) {
#pragma unroll
      for (int j = 0; j < NG; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) dbs[(j * NBL + bl) * W4 + 4 * cg + i] = dbp[j][i];
    }
    __syncthreads();
    for (int q = tid; q < NG * W4; q += ATHREADS) {
      const int j = q / W4, cc = q % W4, c = c0 + cb + cc;
      if (c >= DH) continue;
      const int nbl = min(NBL, nb);
      float sum = 0.f;
      for (int k = 0; k < nbl; ++k) sum += dbs[(j * NBL + k) * W4 + cc];
      a.dbacc[((size_t)bt * NG + j) * D + hd * DH + c] += sum;
    }
  }
  ALT_PROF(3);
  fence_proxy_async_global();  // dg_t is the next kernel's TMA operand
  tc_fence_before();
  __syncthreads();
  if (w == 2) tmem_dealloc(tbase, a.tmem_cols);
}

// ---------------------------------------------------------------- host ----
uint32_t pow2_at_least(uint32_t c, uint32_t lo) {
  uint32_t r = lo;
  while (r < c) r <<= 1;
  return r;
}

bool all_inputs(const Problem& p) {
  for (int j = 0; j < p.NG; ++j)
    if (!p.inp[j]) return false;
  return true;
}

template <class K, class... Args>
cudaError_t launch_step(K kern, dim3 grid, size_t smem, int cluster, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(ATHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  static const bool pdl = getenv("FRNN_ALT_NOPDL") == nullptr;
  if (pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  if (e == cudaSuccess) note_launch();
  return e;
}

using StepKernel = void (*)(CUtensorMap, CUtensorMap, AltArgs);

StepKernel pick(int variant, bool bwd) {
  switch (variant) {
    case kElman: return bwd ? alt_bwd_kernel<kElman> : alt_fwd_kernel<kElman>;
    case kLstm: return bwd ? alt_bwd_kernel<kLstm> : alt_fwd_kernel<kLstm>;
    case kGru: return bwd ? alt_bwd_kernel<kGru> : alt_fwd_kernel<kGru>;
    default: return bwd ? alt_bwd_kernel<kSlstm> : alt_fwd_kernel<kSlstm>;
  }
}

}  // namespace

// Derived geometry of one alternating pass for the solver's choices (planner.cpp):
// batch tile N, backward cluster K-split KS, K atoms per stage ka, ring stages.
AltShape alt_shape(const Problem& p, bool backward, int N, int KS, int ka, int stages) {
  AltShape s{};
  s.N = N;
  s.NBT = (p.B + N - 1) / N;
  s.ka = ka;
  s.a_bytes = A_BYTES * ka;
  s.stage_bytes = ka * (A_BYTES + (uint32_t)N * 128);
  s.kpg = p.DH / (64 * ka);
  size_t epi;
  if (!backward) {
    s.UPT = p.NG == 1 ? 128 : 32;
    s.tiles = (p.DH + s.UPT - 1) / s.UPT;
    s.numk = s.kpg;
    s.KS = 1;
    epi = (size_t)128 * (N + 1) * 4;
  } else {
    s.tiles = (p.DH + 127) / 128;
    s.nrec = 0;
    for (int j = 0; j < p.NG; ++j)
      if (p.rec[j]) s.recg[s.nrec++] = j;
    s.KT = s.nrec * s.kpg;
    s.KS = KS;
    s.numk = (s.KT + KS - 1) / KS;
    epi = (size_t)N * PC * 4;
  }
  s.stages = stages;
  s.region = (uint32_t)std::max<size_t>((size_t)stages * s.stage_bytes, epi);
  s.region = (s.region + 1023) & ~1023u;
  s.smem = 1024 + s.region + 256;
  s.tmem_cols = pow2_at_least((uint32_t)N, 32);
  s.grid = (backward ? s.tiles * s.KS : s.tiles) * p.NH * s.NBT;
  return s;
}

bool alt_supported(const Problem& p, std::string* why) {
  if (!p.bf16) {
    *why = "alternating path: bf16 only";
    return false;
  }
  if (p.DH % 64) {
    *why = "alternating path: head_dim must be a multiple of 64 (TMA K blocks)";
    return false;
  }
  if (p.NG != 1 && p.NG != 4) {
    *why = "alternating path: 1 or 4 gates";
    return false;
  }
  return true;
}

size_t alt_forward_ws(const Problem& p, const Plan& pl) {
  if (!p.bf16 || pl.ffma) return alt32_forward_ws(p);
  return align_up(sizeof(float) * (size_t)p.NS * p.B * p.D, 256);
}

size_t alt_backward_ws(const Problem& p, const Plan& pl) {
  if (!p.bf16 || pl.ffma) return alt32_backward_ws(p);
  size_t off = align_up(sizeof(float) * (size_t)p.NS * p.B * p.D, 256);
  if (!all_inputs(p)) off += align_up((size_t)2 * p.T * p.B * p.NG * p.D, 256);
  const int N = pl.batch_tile > 0 ? pl.batch_tile : 16;
  off += align_up(sizeof(float) * (size_t)((p.B + N - 1) / N) * p.NG * p.D, 256);
  return off;
}

cudaError_t alt_forward(const Problem& p, const Plan& pl, void* ws, cudaStream_t st) {
  if (!p.bf16 || pl.ffma) return alt32_forward(p, ws, st);
  std::string why;
  if (!alt_supported(p, &why) || !tmap_encoder()) return cudaErrorNotSupported;
  const AltShape sh = alt_shape(p, false, pl.batch_tile, 1, pl.ka, pl.stages);
  CUtensorMap mR, mH;
  {  // R[NH][NG][DH][DH]: (k, unit, gate, head), box = (64, UPT, NG, 1)
    cuuint64_t dims[4] = {(cuuint64_t)p.DH, (cuuint64_t)p.DH, (cuuint64_t)p.NG, (cuuint64_t)p.NH};
    cuuint64_t str[3] = {(cuuint64_t)p.DH * 2, (cuuint64_t)p.DH * p.DH * 2, (cuuint64_t)p.NG * p.DH * p.DH * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)sh.UPT, (cuuint32_t)p.NG, 1};
    if (!tmap_bf16(&mR, p.R, 4, dims, str, box)) return cudaErrorInvalidValue;
  }
  {  // states[T+1][NS][B][D] as (k, head, b, t*NS+s), box = (64, 1, N, 1)
    cuuint64_t dims[4] = {(cuuint64_t)p.DH, (cuuint64_t)p.NH, (cuuint64_t)p.B, (cuuint64_t)(p.T + 1) * p.NS};
    cuuint64_t str[3] = {(cuuint64_t)p.DH * 2, (cuuint64_t)p.D * 2, (cuuint64_t)p.B * p.D * 2};
    cuuint32_t box[4] = {64, 1, (cuuint32_t)sh.N, 1};
    if (!tmap_bf16(&mH, p.states, 4, dims, str, box)) return cudaErrorInvalidValue;
  }
  AltArgs a{};
  a.p = p;
  a.N = sh.N;
  a.UPT = sh.UPT;
  a.numk = sh.numk;
  a.stages = sh.stages;
  a.KS = 1;
  a.stage_bytes = sh.stage_bytes;
  a.a_bytes = sh.a_bytes;
  a.ka = sh.ka;
  a.region = sh.region;
  a.tmem_cols = sh.tmem_cols;
  a.carry = static_cast<float*>(ws);
  a.dbg = getenv("FRNN_ALT_DBG") ? atoi(getenv("FRNN_ALT_DBG")) : 0;
  const size_t n = (size_t)p.NS * p.B * p.D;
  kt_begin(KT_FWD, st);
  alt_fwd_init<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256, 0, st>>>(
      static_cast<const bf16*>(p.s0), static_cast<bf16*>(p.states), a.carry, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  note_launch();
  const StepKernel kern = pick(p.variant, false);
  if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.smem)) != cudaSuccess)
    return e;
  const dim3 grid(sh.tiles, p.NH, sh.NBT);
  a.prof = g_prof_buf;
  for (int t = 0; t < p.T && e == cudaSuccess; ++t) {
    a.t = t;
    a.prof_slot = t < g_prof_steps ? t : -1;
    e = launch_step(kern, grid, sh.smem, 1, st, mR, mH, a);
  }
  kt_end(KT_FWD, st);
  return e;
}

cudaError_t alt_backward(const Problem& p, const Plan& pl, void* ws, cudaStream_t st) {
  if (!p.bf16 || pl.ffma) return alt32_backward(p, ws, st);
  std::string why;
  if (!alt_supported(p, &why) || !tmap_encoder()) return cudaErrorNotSupported;
  const AltShape sh = alt_shape(p, true, pl.batch_tile, pl.k_split, pl.ka, pl.stages);
  char* w = static_cast<char*>(ws);
  size_t off = 0;
  float* carry = reinterpret_cast<float*>(w);
  off += align_up(sizeof(float) * (size_t)p.NS * p.B * p.D, 256);
  bf16* dgw = nullptr;
  if (!all_inputs(p)) {
    dgw = reinterpret_cast<bf16*>(w + off);
    off += align_up((size_t)2 * p.T * p.B * p.NG * p.D, 256);
  }
  float* dbacc = reinterpret_cast<float*>(w + off);
  const void* dg_trace = dgw ? static_cast<const void*>(dgw) : p.dx;
  CUtensorMap mRT, mDG;
  {  // R as (c, r, gate, head), box = (64 c, 64 r, 1, 1): MN-major A = R^T
    cuuint64_t dims[4] = {(cuuint64_t)p.DH, (cuuint64_t)p.DH, (cuuint64_t)p.NG, (cuuint64_t)p.NH};
    cuuint64_t str[3] = {(cuuint64_t)p.DH * 2, (cuuint64_t)p.DH * p.DH * 2, (cuuint64_t)p.NG * p.DH * p.DH * 2};
    cuuint32_t box[4] = {64, 64, 1, 1};
    if (!tmap_bf16(&mRT, p.R, 4, dims, str, box)) return cudaErrorInvalidValue;
  }
  {  // dg[T][B][NG][D] as (r, head, gate, b, t), box = (64, 1, 1, N, 1)
    cuuint64_t dims[5] = {(cuuint64_t)p.DH, (cuuint64_t)p.NH, (cuuint64_t)p.NG, (cuuint64_t)p.B, (cuuint64_t)p.T};
    cuuint64_t str[4] = {(cuuint64_t)p.DH * 2, (cuuint64_t)p.D * 2, (cuuint64_t)p.NG * p.D * 2,
                         (cuuint64_t)p.B * p.NG * p.D * 2};
    cuuint32_t box[5] = {64, 1, 1, (cuuint32_t)sh.N, 1};
    if (!tmap_bf16(&mDG, dg_trace, 5, dims, str, box)) return cudaErrorInvalidValue;
  }
  AltArgs a{};
  a.p = p;
  a.N = sh.N;
  a.stages = sh.stages;
  a.KS = sh.KS;
  a.KT = sh.KT;
  a.kpg = sh.kpg;
  a.nrec = sh.nrec;
  for (int j = 0; j < 4; ++j) a.recg[j] = sh.recg[j];
  a.stage_bytes = sh.stage_bytes;
  a.a_bytes = sh.a_bytes;
  a.ka = sh.ka;
  a.region = sh.region;
  a.tmem_cols = sh.tmem_cols;
  a.carry = carry;
  a.dgw = dgw;
  a.dbacc = dbacc;
  cudaError_t e = cudaMemsetAsync(dbacc, 0, sizeof(float) * (size_t)sh.NBT * p.NG * p.D, st);
  if (e != cudaSuccess) return e;
  const StepKernel kern = pick(p.variant, true);
  if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.smem)) != cudaSuccess)
    return e;
  if (sh.KS > 8 &&
      (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
    return e;
  const dim3 grid(sh.tiles * sh.KS, p.NH, sh.NBT);
  const bool recur = p.clip_mode != 2 && sh.nrec > 0;
  kt_begin(KT_BWD, st);
  a.prof = g_prof_buf;
  for (int t = p.T - 1; t >= -1 && e == cudaSuccess; --t) {
    a.t = t;
    a.prof_slot = p.T - 1 - t < g_prof_steps ? p.T - 1 - t : -1;
    a.first = t == p.T - 1;
    a.has_gemm = recur && t < p.T - 1;
    e = launch_step(kern, grid, sh.smem, sh.KS, st, mRT, mDG, a);
  }
  kt_end(KT_BWD, st);
  if (e != cudaSuccess) return e;
  kt_begin(KT_PARAM, st);
  if (dr_gemm_supported(p)) {
    e = dr_gemm(p, dg_trace, st);
    if (e == cudaSuccess) e = db_convert(dbacc, p.dbias, p.NG * p.D, sh.NBT, st);
  } else {
    DgView dg{dg_trace, (long long)p.B * p.NG * p.D, (long long)p.NG * p.D, (long long)p.D};
    e = param_grads(p, dg, nullptr, st);
  }
  kt_end(KT_PARAM, st);
  return e;
}

}  // namespace frnn
