// wx_gemm.cu -- the input projection before the recurrence:
// rnnkit's engine takes gate pre-inputs x = W u that are computed outside it
// (the "w/ Linear" comparison PAPER.md:622-627).
// This is that GEMM on tcgen05, writing rnnkit's x[T][B][NG][D] layout directly:
//
//   x[m][n] = sum_k u[m][k] * W[n][k],   m = t*B + b (tokens), n = j*D + e (gate rows)
//
// u [tokens][Din] and W [NG*D][Din] are both K-major, so TMA streams 128x64 /
// 256x64 bf16 tiles (128B swizzle) into a 2-stage mbarrier ring; one elected
// lane of warp 1 issues tcgen05.mma (M=128, N=256, K=16, fp32 accumulator in
// TMEM); warps 0-3 drain TMEM (one token row per thread) to bf16.  Out-of-range
// tiles are zero-filled by TMA and masked on store.  Measured 608 TFLOP/s at
// 16384 x 3072 x 768 (127 us): with K = 768 a 128x256 tile moves 590 KB from L2
// for 50 MFLOP, so the kernel is L2-bandwidth bound (~7 TB/s); larger tiles or
// cluster multicast of the W slab are the next step.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"
#include "tmap.h"

namespace frnn {
namespace {

using namespace sm100;
using bf16 = __nv_bfloat16;

constexpr int BM = 128, BN = 256, BK = 64, MAXST = 4;
constexpr uint32_t A_STAGE = BM * BK * 2, B_STAGE = BN * BK * 2, STAGE = A_STAGE + B_STAGE;

struct WArgs {
  long long M;
  int N, K, numk, stages;
  bf16* x;
};

__global__ void __launch_bounds__(128, 2)
    wx_gemm_kernel(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapW, WArgs g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int STAGES = g.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const long long m0 = (long long)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;

  if (w == 2) tmem_alloc(tbase_s, BN);
  if (tid == 32) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (tid == 0) {
    prefetch_tensormap(&mapU);
    prefetch_tensormap(&mapW);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tbase_s;

  if (w == 0) {  // TMA producer
    if (elect_one()) {
      for (int kb = 0; kb < g.numk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        uint8_t* st = smem + s * STAGE;
        mbar_arrive_expect_tx(&full[s], STAGE);
        tma_load_2d(st, &mapU, kb * BK, (int)m0, &full[s]);
        tma_load_2d(st + A_STAGE, &mapW, kb * BK, n0, &full[s]);
      }
    }
    __syncwarp();
  } else if (w == 1) {  // MMA issuer
    const uint32_t idesc = idesc_bf16(BM, BN);
    for (int kb = 0; kb < g.numk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE);
      const uint64_t ad = sdesc_k_sw128(sa), bd = sdesc_k_sw128(sa + A_STAGE);
#pragma unroll
      for (int k = 0; k < BK / 16; ++k) {
        if (elect_one()) mma_ss(tbase, ad + 2 * k, bd + 2 * k, idesc, (kb | k) ? 1u : 0u);
        __syncwarp();
      }
      if (elect_one()) mma_commit(&empty[s]);
      __syncwarp();
    }
    if (elect_one()) mma_commit(done);
    __syncwarp();
  }
  // ---- epilogue: TMEM lane = token row, columns = gate rows; bf16 out
  mbar_wait(done, 0);
  tc_fence_after();
  const long long m = m0 + 32 * w + l;
  bf16* dst = g.x + m * g.N + n0;
  const bool row_ok = m < g.M;
  for (int c = 0; c < BN; c += 16) {
    float v[16];
    tmem_ld16(tbase + ((uint32_t)(32 * w) << 16) + c, v);
    if (!row_ok || n0 + c >= g.N) continue;
    uint4 o[2];
    uint32_t* op = reinterpret_cast<uint32_t*>(o);
#pragma unroll
    for (int q = 0; q < 8; ++q) op[q] = pack_bf16(v[2 * q], v[2 * q + 1]);
    if (n0 + c + 16 <= g.N && (g.N % 8) == 0) {
      reinterpret_cast<uint4*>(dst + c)[0] = o[0];
      reinterpret_cast<uint4*>(dst + c)[1] = o[1];
    } else {
      for (int q = 0; q < 16 && n0 + c + q < g.N; ++q) dst[c + q] = __float2bfloat16_rn(v[q]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 2) tmem_dealloc(tbase, BN);
}

}  // namespace

cudaError_t wx_gemm(const void* W, const void* u, void* x, long long M, int N, int K, cudaStream_t s) {
  if (!tmap_encoder()) return cudaErrorNotSupported;
  if (M < 1 || N < 1 || K < 1 || (K % 8) != 0) return cudaErrorInvalidValue;
  CUtensorMap mu, mw;
  {  // u [M][K], K-major, box (64 k, 128 rows)
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
    cuuint64_t str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {BK, BM};
    if (!tmap_bf16(&mu, u, 2, dims, str, box)) return cudaErrorInvalidValue;
  }
  {  // W [N][K], K-major, box (64 k, 256 rows)
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
    cuuint64_t str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {BK, BN};
    if (!tmap_bf16(&mw, W, 2, dims, str, box)) return cudaErrorInvalidValue;
  }
  // 2 stages (97 KB) let two CTAs share an SM, so one CTA's TMEM drain overlaps
  // the other's mainloop; FRNN_WX_STAGES overrides (experiments)
  const int st = getenv("FRNN_WX_STAGES") ? atoi(getenv("FRNN_WX_STAGES")) : 2;
  WArgs g{M, N, K, (K + BK - 1) / BK, st < 1 ? 1 : st > MAXST ? MAXST : st, static_cast<bf16*>(x)};
  const size_t smem = 1024 + g.stages * STAGE + 256;
  cudaError_t e = cudaFuncSetAttribute(wx_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN));
  wx_gemm_kernel<<<grid, 128, smem, s>>>(mu, mw, g);
  note_launch();
  return cudaGetLastError();
}

}  // namespace frnn
