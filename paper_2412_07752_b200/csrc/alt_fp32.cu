// alt_fp32.cu -- FFMA step kernels of the alternating path.  Two users:
//  * fp32 mode for head dims whose R block does not fit in shared memory (the
//    SIMT kernels of simt_fp32.cu hold a head's whole R on-chip, so they stop
//    near DH ~ 110 for 4-gate cells) -- the rel 1e-5 parity mode of BASELINE
//    config 1 extended to any head dim;
//  * bf16 shapes no tensor-core kernel can tile (head dims not a multiple of
//    8, or beyond the fused limits and not a multiple of 64): bf16 storage,
//    fp32 arithmetic (Plan::ffma).
// The time loop runs on the host, every step is one FFMA kernel that streams R
// tiles from L2 through shared memory (R is re-read every step, L2-resident:
// 9.4 MB fp32 at H=768) and applies the cell in the epilogue with the accurate
// (libdevice) transcendentals.
//
//   forward step t  (engine.hpp:170-201): CTA = 32 gate rows (32/NG units x
//     NG gates) x 16 batch rows; y = R.h_t accumulated over ascending K
//     chunks; g = (x) + b + y; pointwise_forward; gates[t], states[t+1].
//   backward step t (engine.hpp:257-336): CTA = 32 state columns x 16 batch
//     rows; term = R^T dg_{t+1} over the R-gates; clip; ds_h += term; then
//     the Jacobian of step t (dx, the dg trace for dR/db, the fp32 ds carry);
//     a final launch (t = -1) adds R^T dg_0 for ds0.
// dR / db come from param_grads.cu over the dg trace, as in the SIMT path.
#include <cuda_bf16.h>

#include "cells.cuh"
#include "kernels.h"

namespace frnn {
namespace {

constexpr int TH = 256, ROWS = 32, BB = 16, KC = 64;

// Storage type E (float, or bf16 for head dims the tensor-core kernels cannot
// tile); arithmetic is always fp32 with the accurate cell math.
__device__ __forceinline__ float ldf(float v) { return v; }
__device__ __forceinline__ float ldf(__nv_bfloat16 v) { return __bfloat162float(v); }
template <class E>
__device__ __forceinline__ E stf(float v);
template <>
__device__ __forceinline__ float stf<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 stf<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

struct A32 {
  Problem p;
  int t, first, has_gemm;
  float* dsw;  // [NS][B][D] fp32 ds carry
  void* dgw;   // [T][NG][B][D] dg trace (storage type)
};

template <int V, class E>
__global__ void __launch_bounds__(TH) alt32_fwd_kernel(A32 a) {
  using C = Cell<V>;
  constexpr int NS = C::NS, NG = C::NG, UPT = ROWS / NG;
  using M = Math<false>;
  const Problem& p = a.p;
  const int t = a.t, DH = p.DH, D = p.D, B = p.B;
  const int unit0 = blockIdx.x * UPT, hd = blockIdx.y, b0 = blockIdx.z * BB, nb = min(BB, B - b0);
  const E* R = static_cast<const E*>(p.R);
  const E* bias = static_cast<const E*>(p.bias);
  const E* x = static_cast<const E*>(p.x);
  E* states = static_cast<E*>(p.states);
  E* gates = static_cast<E*>(p.gates);
  __shared__ float Rt[ROWS][KC + 1];
  __shared__ float Ht[BB][KC + 1];
  __shared__ float ys[ROWS][BB + 1];
  const int tid = threadIdx.x, row = tid % ROWS, bq = tid / ROWS;  // 2 outputs: batch bq, bq + 8
  const int rj = row / UPT, ru = row % UPT;                      // gate-major rows
  const bool rvalid = unit0 + ru < DH && p.rec[rj];
  float acc0 = 0.f, acc1 = 0.f;
  const size_t sBD = (size_t)B * D;
  const E* h = states + (size_t)t * NS * sBD;  // h_t = states[t][0]
  for (int k0 = 0; k0 < DH; k0 += KC) {
    for (int i = tid; i < ROWS * KC; i += TH) {
      const int rr = i / KC, kk = i % KC, j = rr / UPT, u = unit0 + rr % UPT, k = k0 + kk;
      Rt[rr][kk] = (u < DH && k < DH && p.rec[j]) ? ldf(R[((size_t)(hd * NG + j) * DH + u) * DH + k]) : 0.f;
    }
    for (int i = tid; i < BB * KC; i += TH) {
      const int b = i / KC, kk = i % KC, k = k0 + kk;
      Ht[b][kk] = (b < nb && k < DH) ? ldf(h[(size_t)(b0 + b) * D + hd * DH + k]) : 0.f;
    }
    __syncthreads();
#pragma unroll 16
    for (int kk = 0; kk < KC; ++kk) {  // ascending K (engine.hpp:181)
      const float r = Rt[row][kk];
      acc0 = fmaf(r, Ht[bq][kk], acc0);
      acc1 = fmaf(r, Ht[bq + 8][kk], acc1);
    }
    __syncthreads();
  }
  ys[row][bq] = rvalid ? acc0 : 0.f;
  ys[row][bq + 8] = rvalid ? acc1 : 0.f;
  __syncthreads();
  for (int i = tid; i < UPT * nb; i += TH) {
    const int u = i % UPT, b = i / UPT, unit = unit0 + u;
    if (unit >= DH) continue;
    const int e = hd * DH + unit;
    const size_t so = (size_t)(b0 + b) * D + e;
    float g[4], prev[4], nx[4];
#pragma unroll
    for (int j = 0; j < NG; ++j) {  // x, then b, then y (engine.hpp:183-187)
      float v = p.inp[j] ? ldf(x[(((size_t)t * B + b0 + b) * NG + j) * D + e]) : 0.f;
      v += ldf(bias[(size_t)j * D + e]);
      v += ys[j * UPT + u][b];
      g[j] = v;
      gates[((size_t)t * NG + j) * sBD + so] = stf<E>(v);
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) prev[s] = ldf(states[((size_t)t * NS + s) * sBD + so]);
    C::template fwd<M>(prev, g, nx);
#pragma unroll
    for (int s = 0; s < NS; ++s) states[((size_t)(t + 1) * NS + s) * sBD + so] = stf<E>(nx[s]);
  }
}

template <int V, class E>
__global__ void __launch_bounds__(TH) alt32_bwd_kernel(A32 a) {
  using C = Cell<V>;
  constexpr int NS = C::NS, NG = C::NG;
  using M = Math<false>;
  const Problem& p = a.p;
  const int t = a.t, DH = p.DH, D = p.D, B = p.B;
  const int c0 = blockIdx.x * ROWS, hd = blockIdx.y, b0 = blockIdx.z * BB, nb = min(BB, B - b0);
  const E* R = static_cast<const E*>(p.R);
  const E* states = static_cast<const E*>(p.cstates);
  const E* gates = static_cast<const E*>(p.cgates);
  const E* dsf = static_cast<const E*>(p.dsf);
  const E* dh = static_cast<const E*>(p.dh);
  E* dx = static_cast<E*>(p.dx);
  E* ds0 = static_cast<E*>(p.ds0);
  E* dgw = static_cast<E*>(a.dgw);
  __shared__ float Rt[KC][ROWS + 1];  // [r][c]
  __shared__ float Gt[BB][KC + 1];    // [b][r]
  __shared__ float ts[ROWS][BB + 1];
  const int tid = threadIdx.x, col = tid % ROWS, bq = tid / ROWS;
  const size_t sBD = (size_t)B * D;
  if (a.has_gemm) {
    float acc0 = 0.f, acc1 = 0.f;
    for (int j = 0; j < NG; ++j) {
      if (!p.rec[j]) continue;
      const E* dgj = dgw + ((size_t)(t + 1) * NG + j) * sBD;  // dg_{t+1}, gate j
      for (int r0 = 0; r0 < DH; r0 += KC) {
        for (int i = tid; i < KC * ROWS; i += TH) {
          const int rr = i / ROWS, cc = i % ROWS, r = r0 + rr, c = c0 + cc;
          Rt[rr][cc] = (r < DH && c < DH) ? ldf(R[((size_t)(hd * NG + j) * DH + r) * DH + c]) : 0.f;
        }
        for (int i = tid; i < BB * KC; i += TH) {
          const int b = i / KC, rr = i % KC, r = r0 + rr;
          Gt[b][rr] = (b < nb && r < DH) ? ldf(dgj[(size_t)(b0 + b) * D + hd * DH + r]) : 0.f;
        }
        __syncthreads();
#pragma unroll 16
        for (int rr = 0; rr < KC; ++rr) {
          const float rv = Rt[rr][col];
          acc0 = fmaf(rv, Gt[bq][rr], acc0);
          acc1 = fmaf(rv, Gt[bq + 8][rr], acc1);
        }
        __syncthreads();
      }
    }
    ts[col][bq] = acc0;
    ts[col][bq + 8] = acc1;
  }
  __syncthreads();
  const float mag = p.clip_mag;
  for (int i = tid; i < ROWS * nb; i += TH) {
    const int cc = i % ROWS, b = i / ROWS, c = c0 + cc;
    if (c >= DH) continue;
    const int e = hd * DH + c;
    const size_t so = (size_t)(b0 + b) * D + e;
    float ds[4], prev[4], g[4], dg[4], dsp[4];
#pragma unroll
    for (int s = 0; s < NS; ++s) ds[s] = a.first ? ldf(dsf[s * sBD + so]) : a.dsw[s * sBD + so];
    if (a.has_gemm) {
      float term = ts[cc][b];
      if (p.clip_mode == 1) term = fminf(fmaxf(term, -mag), mag);  // engine.hpp:300-303
      ds[0] += term;
    }
    if (t < 0) {
#pragma unroll
      for (int s = 0; s < NS; ++s) ds0[s * sBD + so] = stf<E>(ds[s]);
      continue;
    }
    if (dh) ds[0] += ldf(dh[(size_t)t * sBD + so]);  // engine.hpp:258-263
#pragma unroll
    for (int s = 0; s < NS; ++s) prev[s] = ldf(states[((size_t)t * NS + s) * sBD + so]);
#pragma unroll
    for (int j = 0; j < NG; ++j) g[j] = ldf(gates[((size_t)t * NG + j) * sBD + so]);
    C::template bwd<M>(prev, g, ds, dg, dsp);
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      dx[(((size_t)t * B + b0 + b) * NG + j) * D + e] = stf<E>(p.inp[j] ? dg[j] : 0.f);
      dgw[((size_t)t * NG + j) * sBD + so] = stf<E>(dg[j]);
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) a.dsw[s * sBD + so] = dsp[s];
  }
}

template <bool BWD, class E>
cudaError_t launch_e(const A32& a, dim3 grid, cudaStream_t s) {
  switch (a.p.variant) {
    case kElman: BWD ? alt32_bwd_kernel<kElman, E><<<grid, TH, 0, s>>>(a) : alt32_fwd_kernel<kElman, E><<<grid, TH, 0, s>>>(a); break;
    case kLstm: BWD ? alt32_bwd_kernel<kLstm, E><<<grid, TH, 0, s>>>(a) : alt32_fwd_kernel<kLstm, E><<<grid, TH, 0, s>>>(a); break;
    case kGru: BWD ? alt32_bwd_kernel<kGru, E><<<grid, TH, 0, s>>>(a) : alt32_fwd_kernel<kGru, E><<<grid, TH, 0, s>>>(a); break;
    default: BWD ? alt32_bwd_kernel<kSlstm, E><<<grid, TH, 0, s>>>(a) : alt32_fwd_kernel<kSlstm, E><<<grid, TH, 0, s>>>(a); break;
  }
  note_launch();
  return cudaGetLastError();
}

template <bool BWD>
cudaError_t launch(const A32& a, dim3 grid, cudaStream_t s) {
  return a.p.bf16 ? launch_e<BWD, __nv_bfloat16>(a, grid, s) : launch_e<BWD, float>(a, grid, s);
}

}  // namespace

size_t alt32_forward_ws(const Problem&) { return 0; }

size_t alt32_backward_ws(const Problem& p) {
  return align_up(sizeof(float) * (size_t)p.NS * p.B * p.D, 256) +
         align_up((p.bf16 ? 2 : 4) * (size_t)p.T * p.NG * p.B * p.D, 256) + param_grads_ws(p);
}

cudaError_t alt32_forward(const Problem& p, void*, cudaStream_t s) {
  cudaError_t e =
      cudaMemcpyAsync(p.states, p.s0, (p.bf16 ? 2 : 4) * (size_t)p.NS * p.B * p.D, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return e;
  A32 a{};
  a.p = p;
  const int NGu = p.NG == 1 ? 1 : 4;
  const dim3 grid((p.DH + ROWS / NGu - 1) / (ROWS / NGu), p.NH, (p.B + BB - 1) / BB);
  kt_begin(KT_FWD, s);
  for (int t = 0; t < p.T && e == cudaSuccess; ++t) {
    a.t = t;
    e = launch<false>(a, grid, s);
  }
  kt_end(KT_FWD, s);
  return e;
}

cudaError_t alt32_backward(const Problem& p, void* ws, cudaStream_t s) {
  char* w = static_cast<char*>(ws);
  A32 a{};
  a.p = p;
  a.dsw = reinterpret_cast<float*>(w);
  a.dgw = w + align_up(sizeof(float) * (size_t)p.NS * p.B * p.D, 256);
  bool recur = p.clip_mode != 2;
  bool any_rec = false;
  for (int j = 0; j < p.NG; ++j) any_rec = any_rec || p.rec[j];
  recur = recur && any_rec;
  const dim3 grid((p.DH + ROWS - 1) / ROWS, p.NH, (p.B + BB - 1) / BB);
  cudaError_t e = cudaSuccess;
  kt_begin(KT_BWD, s);
  for (int t = p.T - 1; t >= -1 && e == cudaSuccess; --t) {
    a.t = t;
    a.first = t == p.T - 1;
    a.has_gemm = recur && t < p.T - 1;
    e = launch<true>(a, grid, s);
  }
  kt_end(KT_BWD, s);
  if (e != cudaSuccess) return e;
  kt_begin(KT_PARAM, s);
  DgView dg{a.dgw, (long long)p.NG * p.B * p.D, (long long)p.D, (long long)p.B * p.D};
  e = param_grads(p, dg, nullptr, s);
  kt_end(KT_PARAM, s);
  return e;
}

}  // namespace frnn
