// simt_fp32.cu -- persistent fp32 FFMA kernels for the fp32 parity mode
// (BASELINE config 1: LSTM fp32, NH=1, D=64, B=8, T=64; rel 1e-5 vs fp64).
//
// Blackwell has no fp32 tensor-core path that meets 1e-5 (only TF32), so this
// mode runs on the FFMA pipes.  One CTA per (head, batch tile of BT rows) runs
// all T steps; the head's R block lives in shared memory for the whole run
// (padded row stride so both R.h (row-parallel) and R^T.dg (column-parallel)
// are bank-conflict free), the tile's states live in shared memory, and every
// step is: gate pre-activations (x + b + R.h, the order of engine.hpp:183-187)
// -> pointwise (cell.hpp:65) -> trace writes.  Backward mirrors
// engine.hpp:257-336.  dR/db are produced by param_grads.cu from the dg trace.
#include "cells.cuh"
#include "kernels.h"

namespace frnn {
namespace {

constexpr int BT = 8;        // batch rows per CTA
constexpr int THREADS = 256;

__host__ __device__ inline int rpad(int DH) { return DH | 1; }  // odd row stride

template <int V>
__global__ void __launch_bounds__(THREADS) simt_fwd_kernel(Problem p) {
  using C = Cell<V>;
  constexpr int NS = C::NS, NG = C::NG;
  using M = Math<false>;
  const int DH = p.DH, D = p.D, B = p.B, P = rpad(DH);
  const int hd = blockIdx.x % p.NH;
  const int b0 = (blockIdx.x / p.NH) * BT;
  const int nb = min(BT, B - b0);
  const float* R = static_cast<const float*>(p.R);
  const float* bias = static_cast<const float*>(p.bias);
  const float* x = static_cast<const float*>(p.x);
  const float* s0 = static_cast<const float*>(p.s0);
  float* states = static_cast<float*>(p.states);
  float* gates = static_cast<float*>(p.gates);

  extern __shared__ float sm[];
  float* Rs = sm;                         // [NG*DH][P]
  float* st = Rs + (size_t)NG * DH * P;   // [NS][BT][DH]
  float* gs = st + NS * BT * DH;          // [NG][BT][DH]

  for (int i = threadIdx.x; i < NG * DH * DH; i += THREADS) {
    int j = i / (DH * DH), r = (i / DH) % DH, c = i % DH;
    Rs[(j * DH + r) * P + c] = p.rec[j] ? R[((size_t)(hd * NG + j) * DH + r) * DH + c] : 0.f;
  }
  for (int i = threadIdx.x; i < NS * BT * DH; i += THREADS) {
    int s = i / (BT * DH), b = (i / DH) % BT, r = i % DH;
    float v = 0.f;
    if (b < nb) {
      size_t gi = ((size_t)s * B + b0 + b) * D + hd * DH + r;
      v = s0[gi];
      states[gi] = v;  // states[0] = s0 (engine.hpp:161-164)
    }
    st[i] = v;
  }
  __syncthreads();

  for (int t = 0; t < p.T; ++t) {
    for (int row = threadIdx.x; row < NG * DH; row += THREADS) {
      const int j = row / DH, r = row % DH, e = hd * DH + r;
      float acc[BT];
#pragma unroll
      for (int b = 0; b < BT; ++b) acc[b] = 0.f;
      if (p.rec[j]) {
        const float* rr = Rs + row * P;
        for (int c = 0; c < DH; ++c) {  // ascending c (engine.hpp:181)
          float rv = rr[c];
#pragma unroll
          for (int b = 0; b < BT; ++b) acc[b] = fmaf(rv, st[b * DH + c], acc[b]);
        }
      }
      const float bj = bias[(size_t)j * D + e];
#pragma unroll
      for (int b = 0; b < BT; ++b) {
        if (b < nb) {
          float xv = p.inp[j] ? x[(((size_t)t * B + b0 + b) * NG + j) * D + e] : 0.f;
          float g = xv + bj + acc[b];  // x, then b, then y (engine.hpp:183-187)
          gs[(j * BT + b) * DH + r] = g;
          gates[(((size_t)t * NG + j) * B + b0 + b) * D + e] = g;
        }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb * DH; i += THREADS) {
      const int b = i / DH, r = i % DH, e = hd * DH + r;
      float prev[4], g[4], nx[4];
#pragma unroll
      for (int s = 0; s < NS; ++s) prev[s] = st[(s * BT + b) * DH + r];
#pragma unroll
      for (int j = 0; j < NG; ++j) g[j] = gs[(j * BT + b) * DH + r];
      C::template fwd<M>(prev, g, nx);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        st[(s * BT + b) * DH + r] = nx[s];
        states[(((size_t)(t + 1) * NS + s) * B + b0 + b) * D + e] = nx[s];
      }
    }
    __syncthreads();
  }
}

template <int V>
__global__ void __launch_bounds__(THREADS) simt_bwd_kernel(Problem p, float* dgw) {
  using C = Cell<V>;
  constexpr int NS = C::NS, NG = C::NG;
  using M = Math<false>;
  const int DH = p.DH, D = p.D, B = p.B, P = rpad(DH);
  const int hd = blockIdx.x % p.NH;
  const int b0 = (blockIdx.x / p.NH) * BT;
  const int nb = min(BT, B - b0);
  const float* R = static_cast<const float*>(p.R);
  const float* states = static_cast<const float*>(p.cstates);
  const float* gates = static_cast<const float*>(p.cgates);
  const float* dsf = static_cast<const float*>(p.dsf);
  const float* dh = static_cast<const float*>(p.dh);
  float* dx = static_cast<float*>(p.dx);
  float* ds0 = static_cast<float*>(p.ds0);

  extern __shared__ float sm[];
  float* Rs = sm;                          // [NG*DH][P]
  float* ds = Rs + (size_t)NG * DH * P;    // [NS][BT][DH]  grad wrt states[t+1]
  float* dsn = ds + NS * BT * DH;          // [NS][BT][DH]  grad wrt states[t]
  float* dgs = dsn + NS * BT * DH;         // [NG][BT][DH]

  for (int i = threadIdx.x; i < NG * DH * DH; i += THREADS) {
    int j = i / (DH * DH), r = (i / DH) % DH, c = i % DH;
    Rs[(j * DH + r) * P + c] = p.rec[j] ? R[((size_t)(hd * NG + j) * DH + r) * DH + c] : 0.f;
  }
  for (int i = threadIdx.x; i < NS * BT * DH; i += THREADS) {
    int s = i / (BT * DH), b = (i / DH) % BT, r = i % DH;
    ds[i] = b < nb ? dsf[((size_t)s * B + b0 + b) * D + hd * DH + r] : 0.f;
  }
  __syncthreads();

  const float mag = p.clip_mag;
  for (int t = p.T - 1; t >= 0; --t) {
    // Pointwise Jacobian phase (engine.hpp:258-286).
    for (int i = threadIdx.x; i < nb * DH; i += THREADS) {
      const int b = i / DH, r = i % DH, e = hd * DH + r;
      float prev[4], g[4], dsl[4], dg[4], dsp[4];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        prev[s] = states[(((size_t)t * NS + s) * B + b0 + b) * D + e];
        dsl[s] = ds[(s * BT + b) * DH + r];
      }
      if (dh) dsl[0] += dh[((size_t)t * B + b0 + b) * D + e];
#pragma unroll
      for (int j = 0; j < NG; ++j) g[j] = gates[(((size_t)t * NG + j) * B + b0 + b) * D + e];
      C::template bwd<M>(prev, g, dsl, dg, dsp);
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        dgs[(j * BT + b) * DH + r] = dg[j];
        dx[(((size_t)t * B + b0 + b) * NG + j) * D + e] = p.inp[j] ? dg[j] : 0.f;
        dgw[(((size_t)t * NG + j) * B + b0 + b) * D + e] = dg[j];
      }
#pragma unroll
      for (int s = 0; s < NS; ++s) dsn[(s * BT + b) * DH + r] = dsp[s];
    }
    __syncthreads();
    // Recurrent term ds_h += clip(sum_j R_j^T dg_j) (engine.hpp:289-308).
    if (p.clip_mode != 2) {
      for (int i = threadIdx.x; i < nb * DH; i += THREADS) {
        const int b = i / DH, c = i % DH;
        float term = 0.f;
#pragma unroll
        for (int j = 0; j < NG; ++j) {
          if (!p.rec[j]) continue;
          const float* dgj = dgs + (j * BT + b) * DH;
          const float* rc = Rs + (size_t)j * DH * P + c;
          for (int r = 0; r < DH; ++r) term = fmaf(rc[r * P], dgj[r], term);
        }
        if (p.clip_mode == 1) term = fminf(fmaxf(term, -mag), mag);
        dsn[b * DH + c] += term;
      }
    }
    __syncthreads();
    float* tmp = ds;
    ds = dsn;
    dsn = tmp;
  }
  for (int i = threadIdx.x; i < NS * nb * DH; i += THREADS) {
    int s = i / (nb * DH), b = (i / DH) % nb, r = i % DH;
    ds0[((size_t)s * B + b0 + b) * D + hd * DH + r] = ds[(s * BT + b) * DH + r];
  }
}

}  // namespace

size_t simt_smem_bytes(const Problem& p, bool backward) {
  size_t r = (size_t)p.NG * p.DH * rpad(p.DH);
  size_t st = (size_t)p.NS * BT * p.DH;
  size_t g = (size_t)p.NG * BT * p.DH;
  return sizeof(float) * (backward ? r + 2 * st + g : r + st + g);
}

cudaError_t simt_forward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s) {
  size_t smem = simt_smem_bytes(p, false);
  int grid = p.NH * ((p.B + BT - 1) / BT);
  cudaError_t e = cudaSuccess;
#define LAUNCH_F(V)                                                                       \
  {                                                                                       \
    e = cudaFuncSetAttribute(simt_fwd_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)smem);                                                  \
    if (e == cudaSuccess) simt_fwd_kernel<V><<<grid, THREADS, smem, s>>>(p), note_launch(); \
  }
  switch (p.variant) {
    case kElman: LAUNCH_F(kElman); break;
    case kLstm: LAUNCH_F(kLstm); break;
    case kGru: LAUNCH_F(kGru); break;
    default: LAUNCH_F(kSlstm); break;
  }
#undef LAUNCH_F
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t simt_backward(const Problem& p, const Plan& pl, void* ws, cudaStream_t s) {
  size_t smem = simt_smem_bytes(p, true);
  int grid = p.NH * ((p.B + BT - 1) / BT);
  float* dgw = static_cast<float*>(ws);  // [T][NG][B][D] fp32 gate gradients
  cudaError_t e = cudaSuccess;
#define LAUNCH_B(V)                                                                       \
  {                                                                                       \
    e = cudaFuncSetAttribute(simt_bwd_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)smem);                                                  \
    if (e == cudaSuccess) simt_bwd_kernel<V><<<grid, THREADS, smem, s>>>(p, dgw), note_launch(); \
  }
  switch (p.variant) {
    case kElman: LAUNCH_B(kElman); break;
    case kLstm: LAUNCH_B(kLstm); break;
    case kGru: LAUNCH_B(kGru); break;
    default: LAUNCH_B(kSlstm); break;
  }
#undef LAUNCH_B
  if (e != cudaSuccess) return e;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  DgView dg{dgw, (long long)p.NG * p.B * p.D, (long long)p.D, (long long)p.B * p.D};
  size_t off = align_up(sizeof(float) * (size_t)p.T * p.NG * p.B * p.D, 256);
  return param_grads(p, dg, static_cast<char*>(ws) + off, s);
}

}  // namespace frnn
