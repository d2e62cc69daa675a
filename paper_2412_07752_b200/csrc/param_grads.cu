// param_grads.cu -- dR and db from the gate-gradient trace (SIMT reference
// version; the tcgen05 GEMM in dr_gemm.cu replaces it for bf16 when shapes allow).
//
//   dR[hd][j][r][c] = sum_{t,b} dg[t][b][j][hd*DH+r] * h_t[b][hd*DH+c]   (engine.hpp:321-334)
//   db[j][e]        = sum_{t,b} dg[t][b][j][e]                          (engine.hpp:311-320)
// h_t = states[t][0] is the pre-step hidden state.  Gates without the
// recurrent term get dR = 0 (engine.hpp:323).  fp32 accumulation.
#include <cuda_bf16.h>

#include "kernels.h"

namespace frnn {
namespace {

template <class T>
__device__ __forceinline__ float ld(const T* p, size_t i);
template <>
__device__ __forceinline__ float ld<float>(const float* p, size_t i) { return p[i]; }
template <>
__device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p, size_t i) {
  return __bfloat162float(p[i]);
}
template <class T>
__device__ __forceinline__ T cvt(float v);
template <>
__device__ __forceinline__ float cvt<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

constexpr int TILE = 64, KT = 16;

template <class T>
__global__ void __launch_bounds__(256) dr_db_kernel(Problem p, DgView dg) {
  const int DH = p.DH, D = p.D, B = p.B, NG = p.NG;
  const int hd = blockIdx.z / NG, j = blockIdx.z % NG;
  const int c0 = blockIdx.x * TILE, r0 = blockIdx.y * TILE;
  const T* dgp = static_cast<const T*>(dg.ptr);
  const T* st = static_cast<const T*>(p.cstates);
  const bool rec = p.rec[j];
  const bool do_db = blockIdx.x == 0;
  __shared__ float As[KT][TILE];
  __shared__ float Bs[KT][TILE];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  float dbacc = 0.f;
  const long long K = (long long)p.T * B;
  if (rec || do_db) {
    for (long long k0 = 0; k0 < K; k0 += KT) {
      for (int i = threadIdx.x; i < KT * TILE; i += 256) {
        int kk = i / TILE, m = i % TILE;
        long long k = k0 + kk;
        float a = 0.f, b = 0.f;
        if (k < K) {
          int t = (int)(k / B), bb = (int)(k % B);
          if (r0 + m < DH)
            a = ld(dgp, (size_t)(t * dg.ts + bb * dg.bs + j * dg.js) + hd * DH + r0 + m);
          if (rec && c0 + m < DH)
            b = ld(st, ((size_t)t * p.NS * B + bb) * D + hd * DH + c0 + m);  // states[t][0][b]
        }
        As[kk][m] = a;
        Bs[kk][m] = b;
      }
      __syncthreads();
      if (rec) {
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) {
          float av[4], bv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
          for (int i = 0; i < 4; ++i) bv[i] = Bs[kk][tx * 4 + i];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(av[i], bv[q], acc[i][q]);
        }
      }
      if (do_db && threadIdx.x < TILE) {
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) dbacc += As[kk][threadIdx.x];
      }
      __syncthreads();
    }
  }
  T* dR = static_cast<T*>(p.dR);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int r = r0 + ty * 4 + i, c = c0 + tx * 4 + q;
      if (r < DH && c < DH)
        dR[(((size_t)hd * NG + j) * DH + r) * DH + c] = cvt<T>(rec ? acc[i][q] : 0.f);
    }
  if (do_db && threadIdx.x < TILE && r0 + threadIdx.x < DH)
    static_cast<T*>(p.dbias)[(size_t)j * D + hd * DH + r0 + threadIdx.x] = cvt<T>(dbacc);
}

}  // namespace

size_t param_grads_ws(const Problem&) { return 0; }

cudaError_t param_grads(const Problem& p, DgView dg, void*, cudaStream_t s) {
  dim3 grid((p.DH + TILE - 1) / TILE, (p.DH + TILE - 1) / TILE, p.NH * p.NG);
  if (p.bf16)
    dr_db_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(p, dg);
  else
    dr_db_kernel<float><<<grid, 256, 0, s>>>(p, dg);
  note_launch();
  return cudaGetLastError();
}

}  // namespace frnn
