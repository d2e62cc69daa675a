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
// tiles are zero-filled by TMA and masked on store.  That single-CTA form ran at
// 608 TFLOP/s at 16384 x 3072 x 768 (127 us): with K = 768 a 128x256 tile moves
// 590 KB from L2 for 50 MFLOP.  It is kept for out_features % 8 != 0 (no TMA
// store) and as the FRNN_WX_ALGO=1 A/B arm; the default is the CTA-pair
// persistent kernel below (59 us, 1309 TFLOP/s on the same shape).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
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

// ---------------------------------------------------------------------------
// CTA-pair persistent form (default when out_features % 8 == 0).  A cluster of
// two CTAs on one TPC computes 256x256 output tiles with tcgen05.mma.cta_group::2
// (M=256, N=256, K=16): CTA r stages token rows m0+128r and gate rows n0+128r of
// each 64-wide K slab, so a pair moves (256+256)x64 bf16 per slab where two
// independent 128x256 CTAs moved 2x(128+256)x64 -- a third less L2->SM traffic
// and half the B operand per SM.  One elected lane of the leader (rank 0)
// issues the MMAs; TMA completions of both CTAs land on the leader's `full`
// barrier (.cta_group::2), MMA completion is multicast to both CTAs' `empty`
// and `tfull` barriers.  The accumulator is double-buffered in TMEM (2 x 256
// columns), so the epilogue of tile i (warps 4-7: TMEM -> bf16 -> 128B-swizzled
// smem -> TMA store) overlaps the mainloop of tile i+1.  Grid = one pair per
// TPC, tiles strided over pairs.
constexpr int P_BM = 128, P_BN = 256, P_MAXST = 6;
constexpr uint32_t P_A = P_BM * BK * 2, P_B = (P_BN / 2) * BK * 2, P_STAGE = P_A + P_B;  // 16 KB + 16 KB
constexpr uint32_t P_OUT = P_BM * 64 * 2;                                                 // 128 rows x 128 B
inline size_t pair_smem(int stages) { return 1024 + 2 * P_OUT + stages * P_STAGE + 256; }

struct PArgs {
  int tiles_n, tiles_m, tiles, numk, stages, mfast;
};
// Tile t -> (token block, gate block): gate blocks fastest by default, so the
// pairs in flight share token slabs of u.
__device__ __forceinline__ int tile_m(const PArgs& g, int t) { return g.mfast ? t % g.tiles_m : t / g.tiles_n; }
__device__ __forceinline__ int tile_n(const PArgs& g, int t) { return g.mfast ? t / g.tiles_m : t % g.tiles_n; }

__device__ __forceinline__ void tma_load_2d_pair(void* smem, const void* map, int c0, int c1, uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const void* map, int c0, int c1, const void* smem) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(smem_u32(smem))
               : "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// Arrive on the barrier at this offset in both CTAs once the pair's MMAs are done.
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    wx_gemm_pair_kernel(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapW,
                        const __grid_constant__ CUtensorMap mapX, PArgs g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* outbuf = smem;
  smem += 2 * P_OUT;
  const uint32_t P_ST = g.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P_ST * P_STAGE);
  uint64_t* empty = full + P_ST;
  uint64_t* tfull = empty + P_ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (w == 2) {  // both CTAs of the pair allocate together: 2 accumulators x 256 columns
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 32) {
    for (uint32_t s = 0; s < P_ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2);  // one arrival per CTA epilogue
    }
    fence_mbar_init();
  }
  if (tid == 0) {
    prefetch_tensormap(&mapU);
    prefetch_tensormap(&mapW);
    prefetch_tensormap(&mapX);
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tbase = *tbase_s;

  if (w == 0) {  // TMA producer (both CTAs): own 128 token rows + own 128 gate rows
    if (elect_one()) {
      const uint32_t leader_full = mapa_shared(smem_u32(full), 0);
      uint32_t it = 0;
      for (int t = pair; t < g.tiles; t += npairs) {
        const int m0 = tile_m(g, t) * 2 * P_BM + (int)rank * P_BM;
        const int n0 = tile_n(g, t) * P_BN + (int)rank * (P_BN / 2);
        for (int kb = 0; kb < g.numk; ++kb, ++it) {
          const uint32_t s = it % P_ST;
          if (it >= P_ST) mbar_wait(&empty[s], ((it / P_ST) - 1) & 1);
          uint8_t* st = smem + s * P_STAGE;
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * P_STAGE);
          const uint32_t fb = leader_full + s * 8;
          tma_load_2d_pair(st, &mapU, kb * BK, m0, fb);
          tma_load_2d_pair(st + P_A, &mapW, kb * BK, n0, fb);
        }
      }
    }
    __syncwarp();
  } else if (w == 1 && rank == 0) {  // MMA issuer (leader only)
    constexpr uint32_t idesc = idesc_bf16(2 * P_BM, P_BN);
    uint32_t it = 0, tl = 0;
    for (int t = pair; t < g.tiles; t += npairs, ++tl) {
      const uint32_t acc = tl & 1, d = tbase + acc * P_BN;
      if (tl >= 2) mbar_wait_cluster(&tempty[acc], ((tl >> 1) - 1) & 1);
      tc_fence_after();
      for (int kb = 0; kb < g.numk; ++kb, ++it) {
        const uint32_t s = it % P_ST;
        mbar_wait(&full[s], (it / P_ST) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * P_STAGE);
        const uint64_t ad = sdesc_k_sw128(sa), bd = sdesc_k_sw128(sa + P_A);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) mma_pair(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) ? 1u : 0u);
          commit_pair(&empty[s]);
        }
        __syncwarp();
      }
      if (elect_one()) commit_pair(&tfull[acc]);
      __syncwarp();
    }
  } else if (w >= 4) {  // epilogue: TMEM lane quadrant w-4 = token rows 32(w-4)..+32 of this CTA
    const int q = w - 4, row = 32 * q + l;
    const uint32_t tempty_leader = mapa_shared(smem_u32(tempty), 0);
    uint32_t tl = 0, chunk = 0;
    for (int t = pair; t < g.tiles; t += npairs, ++tl) {
      const uint32_t acc = tl & 1;
      const int m0 = tile_m(g, t) * 2 * P_BM + (int)rank * P_BM;
      const int n0 = tile_n(g, t) * P_BN;
      mbar_wait_cluster(&tfull[acc], (tl >> 1) & 1);
      tc_fence_after();
      for (int c = 0; c < P_BN; c += 64, ++chunk) {
        uint8_t* ob = outbuf + (chunk & 1) * P_OUT;
        if (tid == 128) bulk_wait_group_read<1>();  // the store that last used `ob` has read it
        epi_sync();
        uint32_t r[64];
        const uint32_t ta = tbase + ((uint32_t)(32 * q) << 16) + acc * P_BN + c;
        tmem_ld32_nowait(ta, r);
        tmem_ld32_nowait(ta + 32, r + 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint8_t* rowp = ob + row * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint4 o;
          o.x = pack_bf16(__uint_as_float(r[8 * j + 0]), __uint_as_float(r[8 * j + 1]));
          o.y = pack_bf16(__uint_as_float(r[8 * j + 2]), __uint_as_float(r[8 * j + 3]));
          o.z = pack_bf16(__uint_as_float(r[8 * j + 4]), __uint_as_float(r[8 * j + 5]));
          o.w = pack_bf16(__uint_as_float(r[8 * j + 6]), __uint_as_float(r[8 * j + 7]));
          *reinterpret_cast<uint4*>(rowp + ((j ^ (row & 7)) << 4)) = o;
        }
        fence_proxy_async_smem();
        if (c + 64 == P_BN) tc_fence_before();
        epi_sync();
        if (tid == 128) {
          tma_store_2d(&mapX, n0 + c, m0, ob);
          bulk_commit_group();
          if (c + 64 == P_BN) {  // this CTA's half of accumulator `acc` is drained
            if (rank == 0)
              mbar_arrive(&tempty[acc]);
            else
              mbar_arrive_remote(tempty_leader + acc * 8);
          }
        }
      }
    }
    if (tid == 128) bulk_wait_group<0>();
  }
  tc_fence_before();
  cluster_sync_all();
  if (w == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
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
  const char* algo_env = getenv("FRNN_WX_ALGO");  // 1 = single-CTA tiles (A/B)
  if ((N % 8) == 0 && !(algo_env && atoi(algo_env) == 1)) {
    CUtensorMap mu2, mw2, mx;
    {  // per-CTA boxes: 128 token rows / 128 gate rows of a 64-wide K slab
      cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
      cuuint64_t str[1] = {(cuuint64_t)K * 2};
      cuuint32_t box[2] = {BK, P_BM};
      if (!tmap_bf16(&mu2, u, 2, dims, str, box)) return cudaErrorInvalidValue;
      cuuint64_t dw[2] = {(cuuint64_t)K, (cuuint64_t)N};
      cuuint32_t bw[2] = {BK, P_BN / 2};
      if (!tmap_bf16(&mw2, W, 2, dw, str, bw)) return cudaErrorInvalidValue;
    }
    {  // x [M][N]: 64-column x 128-row store boxes, 128B swizzle (matches the epilogue's smem layout)
      cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
      cuuint64_t str[1] = {(cuuint64_t)N * 2};
      cuuint32_t box[2] = {64, P_BM};
      if (!tmap_bf16(&mx, x, 2, dims, str, box)) return cudaErrorInvalidValue;
    }
    PArgs pa;
    pa.tiles_n = (N + P_BN - 1) / P_BN;
    const long long tiles_m = (M + 2 * P_BM - 1) / (2 * P_BM);
    if (tiles_m * pa.tiles_n > (1ll << 30)) return cudaErrorInvalidValue;
    pa.tiles = (int)(tiles_m * pa.tiles_n);
    pa.tiles_m = (int)tiles_m;
    pa.mfast = getenv("FRNN_WX_RASTER") ? atoi(getenv("FRNN_WX_RASTER")) : 0;
    pa.numk = (K + BK - 1) / BK;
    const char* st_env = getenv("FRNN_WX_PST");
    pa.stages = st_env ? std::max(2, std::min(P_MAXST, atoi(st_env))) : 5;
    cudaError_t e = cudaFuncSetAttribute(wx_gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)pair_smem(P_MAXST));
    if (e != cudaSuccess) return e;
    const int pairs = std::min(sm_count() / 2, pa.tiles);
    wx_gemm_pair_kernel<<<2 * pairs, 256, pair_smem(pa.stages), s>>>(mu2, mw2, mx, pa);
    note_launch();
    return cudaGetLastError();
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
