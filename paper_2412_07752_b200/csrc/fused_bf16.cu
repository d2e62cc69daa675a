// fused_bf16.cu -- persistent fused recurrence kernels for bf16 (K1 forward,
// K2 backward), sm_100a / tcgen05.
//
// Decomposition.  A head's NG*DH gate rows are split into
// CPG = DH/UPC CTAs of UPC hidden units each; a CTA owns all NG gates of its
// units, so the cell pointwise update is CTA-local.  Row order inside a CTA is
// unit-major (row = u*NGP + g) so the 4 gates of a unit sit in 4 adjacent TMEM
// lanes of one warp.  One group of CPG CTAs per (head, batch tile of N rows);
// groups never talk (heads are independent: engine.hpp:139-142).
//
// K1 (forward, engine.hpp:170-201), per step t:
//   wait for the group's step-(t-1) flag -> pull h_t (= states[t][0], bf16,
//   written by the peer CTAs through L2) into a K-major SMEM tile -> one thread
//   issues K/16 tcgen05.mma (A = the CTA's R slice, RESIDENT IN TMEM for all T
//   steps; B = h tile; D = fp32 accumulator in TMEM) -> tcgen05.ld -> add x_t
//   and b (x prefetched a step ahead) -> cell pointwise in registers (c/n/m
//   states stay fp32 in registers) -> write gates/states trace -> release flag.
// K2 (backward, engine.hpp:257-336), per reverse step t:
//   wait for the group's partial R^T.dg sums of step t+1 -> reduce the CPG
//   partials for the owned units, clip (engine.hpp:300-303) -> pointwise
//   Jacobian -> dx, and dg (bf16) into a SMEM B tile -> tcgen05.mma with
//   A = R_slice^T (resident in TMEM, one 128-lane block per 128 state columns)
//   gives this CTA's partial R^T.dg for all DH columns -> write partials,
//   release flag.  dR/db come from param_grads (post-loop, K = T*B).
#include <cuda_bf16.h>

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
  uint32_t tmem_cols, acc_col;
  uint32_t* counters;
  float* part;  // backward partials [2][groups][CPG][MB*128][N]
  bf16* dgw;    // backward dg trace (only when a gate is not input-wired)
};

__device__ __forceinline__ float bf(const bf16* p, size_t i) { return __bfloat162float(p[i]); }

// Offset (bytes) of element (row n, k) in a K-major no-swizzle operand tile with
// N rows: core matrix (k/8, n/8) at ((k/8)*(N/8) + n/8)*128.
template <int N>
__device__ __forceinline__ uint32_t kmaj_off(int n, int k) {
  return (uint32_t)(((k >> 3) * (N / 8) + (n >> 3)) * 128 + (n & 7) * 16 + (k & 7) * 2);
}

template <int V, int N>
__global__ void __launch_bounds__(128, 1) fused_fwd_kernel(FArgs a) {
  using C = Cell<V>;
  constexpr int NS = C::NS, NG = C::NG, NGP = C::NGP, UPW = 32 / NGP, EPT = N / NGP;
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
  float st[NS][EPT], bj[NG], xr[NG][EPT];
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
    for (int j = 0; j < NG; ++j)
      xr[j][i] = (ok && p.inp[j] && p.T > 0) ? bf(x, (((size_t)0 * B + b0 + b) * NG + j) * D + e) : 0.f;
  }

  const uint32_t idesc = idesc_bf16(128, N);
  const uint32_t hB_s = smem_u32(hB);
  constexpr uint32_t LBO = N * 16, SBO = 128;
  const int nchunk = nb * (DH / 16);  // 32-byte chunks of the h tile

  for (int t = 0; t < p.T; ++t) {
    const bf16* hsrc = t == 0 ? s0 : states + (size_t)t * NS * B * D;
    if (t > 0) {
      if (tid == 0) spin_until_geq(a.counters + grp, (uint32_t)(a.CPG * t));
      __syncthreads();
    }
    // h_t tile -> SMEM (K-major core matrices), all loads in flight first.
    for (int base = tid; base < nchunk; base += 128 * 8) {
      uint4 v[8][2];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = base + q * 128;
        if (i < nchunk) {
          const int b = i % nb, kp = i / nb;
          const uint4* src = reinterpret_cast<const uint4*>(hsrc + (size_t)(b0 + b) * D + hd * DH + kp * 16);
          v[q][0] = __ldcg(src);
          v[q][1] = __ldcg(src + 1);
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = base + q * 128;
        if (i < nchunk) {
          const int b = i % nb, kp = i / nb;
          const uint32_t off = kmaj_off<N>(b, kp * 16);
          *reinterpret_cast<uint4*>(hB + off) = v[q][0];
          *reinterpret_cast<uint4*>(hB + off + LBO) = v[q][1];
        }
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      for (int ks = 0; ks < K / 16; ++ks)
        mma_ts(tbase + a.acc_col, tbase + ks * 8, sdesc_kmajor(hB_s + ks * 2 * LBO, LBO, SBO), idesc,
               ks > 0);
      mma_commit(mbar);
    }
    mbar_wait(mbar, t & 1);
    tc_fence_after();
#pragma unroll
    for (int n0 = 0; n0 < N; n0 += 16) {
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(32 * w) << 16) + a.acc_col + n0, v);
#pragma unroll
      for (int q = 0; q < 16; ++q) xs[(32 * w + l) * (N + 1) + n0 + q] = v[q];
    }
    __syncwarp();
    if (own) {
      bf16* gdst = gates + (size_t)t * NG * B * D;
      bf16* sdst = states + (size_t)(t + 1) * NS * B * D;
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int b = bo * EPT + i;
        if (b < nb) {
          float g[4], prev[4], nx[4];
#pragma unroll
          for (int j = 0; j < NG; ++j) {
            g[j] = xr[j][i] + bj[j] + xs[(32 * w + uw * NGP + j) * (N + 1) + b];
            gdst[((size_t)j * B + b0 + b) * D + e] = __float2bfloat16_rn(g[j]);
          }
#pragma unroll
          for (int s = 0; s < NS; ++s) prev[s] = st[s][i];
          C::template fwd<M>(prev, g, nx);
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            st[s][i] = nx[s];
            sdst[((size_t)s * B + b0 + b) * D + e] = __float2bfloat16_rn(nx[s]);
          }
        }
      }
      if (t + 1 < p.T) {  // prefetch x_{t+1}
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
          const int b = bo * EPT + i;
#pragma unroll
          for (int j = 0; j < NG; ++j)
            xr[j][i] = (b < nb && p.inp[j]) ? bf(x, (((size_t)(t + 1) * B + b0 + b) * NG + j) * D + e) : 0.f;
        }
      }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      red_release_add(a.counters + grp, 1u);
    }
  }
  __syncthreads();
  if (w == 0) tmem_dealloc(tbase, a.tmem_cols);
}

template <int V, int N>
__global__ void __launch_bounds__(128, 1) fused_bwd_kernel(FArgs a) {
  using C = Cell<V>;
  constexpr int NS = C::NS, NG = C::NG, NGP = C::NGP, UPW = 32 / NGP, EPT = N / NGP;
  constexpr int KB = 128;  // contraction = the CTA's 128 gate rows
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
  float ds[NS][EPT], pv[NS][EPT], gv[NG][EPT];
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
      for (int s = 0; s < NS; ++s) pv[s][i] = ok ? bf(states, (((size_t)t * NS + s) * B + b0 + b) * D + e) : 0.f;
#pragma unroll
      for (int j = 0; j < NG; ++j) gv[j][i] = ok ? bf(gates, (((size_t)t * NG + j) * B + b0 + b) * D + e) : 0.f;
    }
  };
  prefetch(T - 1);

  auto part_at = [&](int buf, int src_cta) -> float* {
    return a.part + ((size_t)((buf * a.groups + grp) * a.CPG + src_cta) * DHP) * N;
  };
  // Sum the CPG partials of R^T.dg for the owned (unit, batch) elements,
  // clip (engine.hpp:300-303) and add to ds_h.
  auto absorb = [&](int buf) {
    float term[EPT];
#pragma unroll
    for (int i = 0; i < EPT; ++i) term[i] = 0.f;
    if (own) {
      for (int q = 0; q < a.CPG; ++q) {
        const float* src = part_at(buf, q) + (size_t)(unit0 + u) * N + bo * EPT;
#pragma unroll
        for (int i = 0; i < EPT; i += 4) {
          float4 v = __ldcg(reinterpret_cast<const float4*>(src + i));
          term[i] += v.x;
          term[i + 1] += v.y;
          term[i + 2] += v.z;
          term[i + 3] += v.w;
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
    if (recur && k > 0) {
      if (tid == 0) spin_until_geq(a.counters + grp, (uint32_t)(a.CPG * k));
      __syncthreads();
      absorb((t + 1) & 1);
    }
    if (own) {
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const int b = bo * EPT + i;
        if (b >= nb) continue;
        float prev[4], g[4], dsl[4], dg[4], dsp[4];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          prev[s] = pv[s][i];
          dsl[s] = ds[s][i];
        }
        if (dh) dsl[0] += bf(dh, ((size_t)t * B + b0 + b) * D + e);  // engine.hpp:258-263
#pragma unroll
        for (int j = 0; j < NG; ++j) g[j] = gv[j][i];
        C::template bwd<M>(prev, g, dsl, dg, dsp);
#pragma unroll
        for (int j = 0; j < NG; ++j) {
          const size_t xi = (((size_t)t * B + b0 + b) * NG + j) * D + e;
          const bf16 v = __float2bfloat16_rn(dg[j]);
          dx[xi] = p.inp[j] ? v : __float2bfloat16_rn(0.f);
          if (a.dgw) a.dgw[xi] = v;
          *reinterpret_cast<bf16*>(dgB + kmaj_off<N>(b, 32 * w + uw * NGP + j)) = v;
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) ds[s][i] = dsp[s];
      }
    }
    prefetch(t - 1);
    if (recur) {
      fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        for (int mb = 0; mb < MB; ++mb)
          for (int ks = 0; ks < KB / 16; ++ks)
            mma_ts(tbase + a.acc_col + mb * N, tbase + mb * (KB / 2) + ks * 8,
                   sdesc_kmajor(dgB_s + ks * 2 * LBO, LBO, SBO), idesc, ks > 0);
        mma_commit(mbar);
      }
      mbar_wait(mbar, phase);
      phase ^= 1;
      tc_fence_after();
      for (int mb = 0; mb < MB; ++mb) {
        const int c = mb * 128 + 32 * w + l;
        float* dst = part_at(t & 1, cta) + (size_t)c * N;
#pragma unroll
        for (int n0 = 0; n0 < N; n0 += 16) {
          float v[16];
          tmem_ld16(tbase + ((uint32_t)(32 * w) << 16) + a.acc_col + mb * N + n0, v);
          if (c < DH) {
#pragma unroll
            for (int q = 0; q < 16; q += 4)
              __stcg(reinterpret_cast<float4*>(dst + n0 + q), make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]));
          }
        }
      }
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        red_release_add(a.counters + grp, 1u);
      }
    }
  }
  if (recur && T > 0) {
    if (tid == 0) spin_until_geq(a.counters + grp, (uint32_t)(a.CPG * T));
    __syncthreads();
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
  __syncthreads();
  if (w == 0) tmem_dealloc(tbase, a.tmem_cols);
}

uint32_t pow2_cols(uint32_t c) {
  uint32_t r = 32;
  while (r < c) r <<= 1;
  return r;
}

FArgs make_args(const Problem& p, const Plan& pl, void* ws, bool backward) {
  FArgs a{};
  a.p = p;
  a.UPC = pl.units_per_cta;
  a.CPG = pl.ctas_per_group;
  a.NBT = (p.B + pl.batch_tile - 1) / pl.batch_tile;
  a.groups = p.NH * a.NBT;
  a.K = (int)align_up(p.DH, 32);
  a.MB = (p.DH + 127) / 128;
  const int N = pl.batch_tile;
  if (!backward) {
    a.acc_col = (uint32_t)align_up(a.K / 2, 32);
    a.tmem_cols = pow2_cols(a.acc_col + N);
  } else {
    a.acc_col = (uint32_t)(a.MB * 64);
    a.tmem_cols = pow2_cols(a.acc_col + a.MB * N);
  }
  char* w = static_cast<char*>(ws);
  a.counters = reinterpret_cast<uint32_t*>(w);
  size_t off = align_up(sizeof(uint32_t) * a.groups, 256);
  if (backward) {
    a.part = reinterpret_cast<float*>(w + off);
    off += align_up(sizeof(float) * 2 * a.groups * a.CPG * (size_t)a.MB * 128 * N, 256);
    bool all_in = true;
    for (int j = 0; j < p.NG; ++j) all_in = all_in && p.inp[j];
    a.dgw = all_in ? nullptr : reinterpret_cast<bf16*>(w + off);
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
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(128), args, smem,
                                     s);
}

}  // namespace

size_t fused_forward_ws(const Problem& p, const Plan& pl) {
  const int groups = p.NH * ((p.B + pl.batch_tile - 1) / pl.batch_tile);
  return align_up(sizeof(uint32_t) * groups, 256);
}

size_t fused_backward_ws(const Problem& p, const Plan& pl) {
  const int N = pl.batch_tile;
  const int groups = p.NH * ((p.B + N - 1) / N);
  const int MB = (p.DH + 127) / 128;
  size_t off = align_up(sizeof(uint32_t) * groups, 256);
  off += align_up(sizeof(float) * 2 * groups * pl.ctas_per_group * (size_t)MB * 128 * N, 256);
  bool all_in = true;
  for (int j = 0; j < p.NG; ++j) all_in = all_in && p.inp[j];
  if (!all_in) off += align_up((size_t)2 * p.T * p.B * p.NG * p.D, 256);
  return off;
}

#define FRNN_FUSED_DISPATCH(KERNEL, N_)                                   \
  switch (p.variant) {                                                     \
    case kElman: e = coop_launch(KERNEL<kElman, N_>, a, pl.grid, smem, s); break; \
    case kLstm: e = coop_launch(KERNEL<kLstm, N_>, a, pl.grid, smem, s); break;   \
    case kGru: e = coop_launch(KERNEL<kGru, N_>, a, pl.grid, smem, s); break;     \
    default: e = coop_launch(KERNEL<kSlstm, N_>, a, pl.grid, smem, s); break;     \
  }

cudaError_t fused_forward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s) {
  FArgs a = make_args(p, pl, ws, false);
  cudaError_t e = cudaMemsetAsync(a.counters, 0, sizeof(uint32_t) * a.groups, s);
  if (e != cudaSuccess) return e;
  const size_t smem = fwd_smem(pl.batch_tile, a.K);
  if (pl.batch_tile == 16) {
    FRNN_FUSED_DISPATCH(fused_fwd_kernel, 16)
  } else {
    return cudaErrorInvalidValue;
  }
  return e;
}

cudaError_t fused_backward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s) {
  FArgs a = make_args(p, pl, ws, true);
  cudaError_t e = cudaMemsetAsync(a.counters, 0, sizeof(uint32_t) * a.groups, s);
  if (e != cudaSuccess) return e;
  const size_t smem = bwd_smem(pl.batch_tile);
  if (pl.batch_tile == 16) {
    FRNN_FUSED_DISPATCH(fused_bwd_kernel, 16)
  } else {
    return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  // dR / db from the dg trace (dx when every gate is input-wired).
  DgView dg{a.dgw ? static_cast<const void*>(a.dgw) : p.dx, (long long)p.B * p.NG * p.D,
            (long long)p.NG * p.D, (long long)p.D};
  return param_grads(p, dg, nullptr, s);
}

}  // namespace frnn
