// dr_gemm.cu -- K3: the recurrent-weight gradient as one tcgen05 GEMM per head
// (engine.hpp:321-334, summed over all steps at once):
//
//   dR[hd][j][r][c] = sum_{t,b} dg[t][b][j][hd*DH+r] * h_t[b][hd*DH+c]
//
// C[M = NG*DH rows (j,r)][N = DH cols c], K = T*B.  Both operands are MN-major
// in rnnkit's layouts (the reduction index (t,b) is the outer stride), so they
// are staged by TMA with 4-D tensor maps straight from dx / states (no
// transposes), 128-byte swizzle, into a 4-stage mbarrier ring; one elected
// thread issues tcgen05.mma (M=128, N=BN, K=16, bf16 -> fp32 in TMEM); the
// epilogue drains TMEM to bf16 dR (zero rows for gates without R, engine.hpp:323).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <mutex>

#include "kernels.h"
#include "sm100.cuh"

namespace frnn {
namespace {

using namespace sm100;
using bf16 = __nv_bfloat16;

constexpr int BM = 128, BK = 64, STAGES = 4;
constexpr uint32_t CHUNK = 64 * 64 * 2;  // one [64 k][64 mn] swizzled box = 8 KB

struct GArgs {
  int NG, DH, NH, B, numk, BN;
  // K tiling over k = (t, b): B <= 64: ksteps whole steps per tile (kreal = ksteps*B
  // rows, the rest of the 64-row B tile stays zero); B > 64: one step, 64-row
  // batch chunks (bchunks per step; rows past B are zero-filled by TMA)
  int ksteps, bchunks, kreal;
  bool rec[4];
  bf16* dR;
};

__device__ __forceinline__ void tma_load4(void* smem, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// MN-major, 128B-swizzle smem descriptor: LBO = stride between 64-element MN
// chunks (one 8 KB box), SBO = stride between 8-row K groups (1 KB).
__device__ __forceinline__ uint64_t sdesc_mn_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((CHUNK >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

__global__ void __launch_bounds__(128, 1) dr_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                                                          const __grid_constant__ CUtensorMap map_b, GArgs g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int BN = g.BN;
  const uint32_t stage_bytes = 2 * CHUNK + (BN / 64) * CHUNK;  // (B tiles keep a full 64-row chunk)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * stage_bytes);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int hd = blockIdx.z, m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;

  if (w == 0) tmem_alloc(tbase_s, BN <= 64 ? 64 : BN <= 128 ? 128 : 256);
  if (tid == 32) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (g.kreal < BK) {  // B tile rows kreal..63 are never written by TMA: zero them once
    for (int s = 0; s < STAGES; ++s)
      for (int q = 0; q < BN / 64; ++q) {
        uint8_t* sb = smem + s * stage_bytes + 2 * CHUNK + q * CHUNK;
        for (int i = g.kreal * 128 / 16 + tid; i < (int)(CHUNK / 16); i += blockDim.x)
          reinterpret_cast<uint4*>(sb)[i] = make_uint4(0, 0, 0, 0);
      }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, *tbase_s, 0);
  const uint32_t b_box_bytes = (uint32_t)(g.B <= 64 ? g.B * g.ksteps : 64) * 128;  // one 64-column chunk

  if (w == 0) {  // TMA producer
    if (elect_one()) {
      for (int kt = 0; kt < g.numk; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
        uint8_t* sa = smem + s * stage_bytes;
        uint8_t* sb = sa + 2 * CHUNK;
        mbar_arrive_expect_tx(&full[s], 2 * CHUNK + (BN / 64) * b_box_bytes);
        // this tile's first (t, b): A rows past the tile's real k meet zero B rows
        const int t0 = g.B <= 64 ? kt * g.ksteps : kt / g.bchunks;
        const int bb0 = g.B <= 64 ? 0 : (kt % g.bchunks) * 64;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = m0 + 64 * h;  // 64 rows of one gate (DH % 64 == 0)
          tma_load4(sa + h * CHUNK, &map_a, m % g.DH, hd, m / g.DH, t0 * g.B + bb0, &full[s]);
        }
        for (int q = 0; q < BN / 64; ++q)
          tma_load4(sb + q * CHUNK, &map_b, n0 + 64 * q, hd, bb0, t0, &full[s]);
      }
    }
    __syncwarp();
  } else if (w == 1) {  // MMA issuer
    const uint32_t idesc = idesc_bf16(BM, BN) | (1u << 15) | (1u << 16);  // A, B MN-major
    for (int kt = 0; kt < g.numk; ++kt) {
      const int s = kt % STAGES;
      mbar_wait(&full[s], (kt / STAGES) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * stage_bytes);
      const uint32_t sb = sa + 2 * CHUNK;
#pragma unroll
      for (int k = 0; k < BK / 16; ++k) {
        if (elect_one())
          mma_ss(tbase, sdesc_mn_sw128(sa + k * 2048), sdesc_mn_sw128(sb + k * 2048), idesc,
                 (kt > 0 || k > 0) ? 1u : 0u);
        __syncwarp();
      }
      if (elect_one()) mma_commit(&empty[s]);
      __syncwarp();
    }
    if (elect_one()) mma_commit(done);
    __syncwarp();
  }
  // ---- epilogue: TMEM -> bf16 dR rows (row = m, 16 columns per load)
  mbar_wait(done, 0);
  tc_fence_after();
  const int m = m0 + 32 * w + l;
  const int j = m / g.DH, r = m % g.DH;
  const bool rec = g.rec[j];
  bf16* dst = g.dR + (((size_t)hd * g.NG + j) * g.DH + r) * g.DH + n0;
  for (int c = 0; c < BN; c += 16) {
    float v[16];
    tmem_ld16(tbase + ((uint32_t)(32 * w) << 16) + c, v);
    uint4 o[2];
    uint32_t* op = reinterpret_cast<uint32_t*>(o);
#pragma unroll
    for (int q = 0; q < 8; ++q) op[q] = rec ? pack_bf16(v[2 * q], v[2 * q + 1]) : 0u;
    reinterpret_cast<uint4*>(dst + c)[0] = o[0];
    reinterpret_cast<uint4*>(dst + c)[1] = o[1];
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tbase, BN <= 64 ? 64 : BN <= 128 ? 128 : 256);
}

__global__ void db_convert_kernel(const float* acc, bf16* db, int n, int tiles) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float s = 0.f;
    for (int t = 0; t < tiles; ++t) s += acc[(size_t)t * n + i];
    db[i] = __float2bfloat16_rn(s);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

int pick_bn(int DH) {
  if (DH % 256 == 0) return 256;
  if (DH <= 256 && DH % 64 == 0) return DH;
  if (DH % 128 == 0) return 128;
  return 64;
}

}  // namespace

bool dr_gemm_supported(const Problem& p) {
  return p.bf16 && p.DH % 64 == 0 && (p.NG * p.DH) % BM == 0 && encoder() != nullptr;
}

// dg: the dx-layout gate-gradient trace [T][B][NG][D] (dx, or the dgw
// workspace when a gate is not input-wired); h from states[t][0].
cudaError_t dr_gemm(const Problem& p, const void* dg, cudaStream_t s) {
  EncodeFn enc = encoder();
  if (!enc) return cudaErrorNotSupported;
  const int BN = pick_bn(p.DH);
  CUtensorMap ma, mb;
  {  // A = dg: dims (r, head, gate, k = t*B + b)
    cuuint64_t dims[4] = {(cuuint64_t)p.DH, (cuuint64_t)p.NH, (cuuint64_t)p.NG, (cuuint64_t)p.T * p.B};
    cuuint64_t strides[3] = {(cuuint64_t)p.DH * 2, (cuuint64_t)p.D * 2, (cuuint64_t)p.NG * p.D * 2};
    cuuint32_t box[4] = {64, 1, 1, (cuuint32_t)BK};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(dg), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {  // B = h_t = states[t][0]: dims (c, head, b, t); one box = BK/B steps x B rows
    cuuint64_t dims[4] = {(cuuint64_t)p.DH, (cuuint64_t)p.NH, (cuuint64_t)p.B, (cuuint64_t)p.T};
    cuuint64_t strides[3] = {(cuuint64_t)p.DH * 2, (cuuint64_t)p.D * 2, (cuuint64_t)p.NS * p.B * p.D * 2};
    cuuint32_t box[4] = {64, 1, (cuuint32_t)std::min(p.B, BK), (cuuint32_t)(p.B <= BK ? BK / p.B : 1)};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(p.cstates), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  GArgs g{};
  g.NG = p.NG;
  g.DH = p.DH;
  g.NH = p.NH;
  g.B = p.B;
  g.BN = BN;
  g.ksteps = p.B <= BK ? BK / p.B : 1;
  g.bchunks = p.B <= BK ? 1 : (p.B + BK - 1) / BK;
  g.kreal = p.B <= BK ? g.ksteps * p.B : BK;
  g.numk = p.B <= BK ? (p.T + g.ksteps - 1) / g.ksteps : p.T * g.bchunks;
  for (int j = 0; j < 4; ++j) g.rec[j] = p.rec[j];
  g.dR = static_cast<bf16*>(p.dR);
  const uint32_t stage_bytes = 2 * CHUNK + (BN / 64) * CHUNK;
  const size_t smem = STAGES * stage_bytes + 1024 + 256;
  cudaError_t e = cudaFuncSetAttribute(dr_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(p.NG * p.DH / BM, p.DH / BN, p.NH);
  dr_gemm_kernel<<<grid, 128, smem, s>>>(ma, mb, g);
  note_launch();
  return cudaGetLastError();
}

cudaError_t db_convert(const float* acc, void* db, int n, int tiles, cudaStream_t s) {
  db_convert_kernel<<<(n + 255) / 256, 256, 0, s>>>(acc, static_cast<bf16*>(db), n, tiles);
  note_launch();
  return cudaGetLastError();
}

}  // namespace frnn
