// mma_bwd_bench.cu -- the exact per-step MMA mixes of the cluster-resident
// kernels, timed in isolation on one CTA (clock64 from the first issue to the
// completion of the last commit's mbarrier):
//   fwd : 48 x (TS M=128 + SS M=64), N=16, K=768, two accumulators (interleaved)
//   bwd : 4 TMEM-A chains + 2 SMEM-A chains (M=128, N=16, K=192), 6 accumulators,
//         one commit at the end / one commit per block
//   bwd-ts / bwd-ss : only the TMEM-A or the SMEM-A chains
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbb tests/cuda/mma_bwd_bench.cu
#include <cuda_bf16.h>

#include <cstdio>

#include "../../paper_2412_07752_b200/csrc/sm100.cuh"

using namespace frnn::sm100;

constexpr int N = 16, KF = 768, KB = 192;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}
// random bf16 pair in (-1, 1): sign + exponent 2^-1..2^-8, random mantissa
__device__ __forceinline__ uint32_t rnd_pair(uint32_t i) {
  const uint32_t h = hash32(i * 2654435761u + 12345u);
  auto one = [](uint32_t r) { return (uint32_t)(((r & 1u) << 15) | ((119u + ((r >> 1) & 7u)) << 7) | ((r >> 4) & 0x7Fu)); };
  return one(h & 0xFFFFu) | (one(h >> 16) << 16);
}

__global__ void bench(int mode, int spin, int rnd, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  // forward: B [16 x 768], A2 [64 x 768]; backward: 2 x A [128 x 192], B [16 x 192]
  uint8_t* bufB = sm;                       // 24 KB
  uint8_t* bufA = sm + 32768;               // 96 KB
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, w = tid >> 5;
  if (w == 0) tmem_alloc(&tb, 512);
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < (32768 + 98304) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = rnd ? rnd_pair(i) : 0x3c003c00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tb;
  if (w < 4) {  // TMEM A columns 0..383: random or constant bf16 pairs
    for (int c0 = 0; c0 < 384; c0 += 16) {
      uint32_t v[16];
      for (int q = 0; q < 16; ++q) v[q] = rnd ? rnd_pair(0x100000u + (c0 + q) * 128 + 32 * w + (tid & 31)) : 0x3c003c00u;
      tmem_st16(t + ((uint32_t)(32 * w) << 16) + c0, v);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  long long best = 1ll << 60;
  for (int rep = 0; rep < 8; ++rep) {
    __syncthreads();
    const long long t0 = clock64();
    int nb = 1;
    if (w == 0) {
      tc_fence_after();
      if (mode >= 8) {  // 4 x (TS M=128 + SS M=64 interleaved), the forward's mix, over K=192
        const uint32_t LBO = N * 16;
        const uint64_t bd = sdesc_kmajor(smem_u32(bufB), LBO, 128);
        const uint32_t blk64 = 64 * KB * 2, cb = KB / 2;
        const bool per = mode == 9;
        nb = per ? 4 : 1;
        for (int i = 0; i < 4; ++i) {
          mma_chain_ts_ss(t + 384 + i * N, t + i * cb, 8, t + 448 + i * N,
                          sdesc_kmajor(smem_u32(bufA) + i * blk64, 64 * 16, 128), (2 * 64 * 16) >> 4, bd,
                          (2 * LBO) >> 4, idesc_bf16(128, N), idesc_bf16(64, N), KB / 16);
          if (per || i == 3) {
            if (elect_one()) mma_commit(&bar[per ? i : 0]);
            __syncwarp();
          }
        }
      } else if (mode >= 5) {  // K-outer interleaving over the accumulators / a single long chain
        const uint32_t LBO = N * 16;
        const uint64_t bd = sdesc_kmajor(smem_u32(bufB), LBO, 128);
        const uint64_t ad = sdesc_kmajor(smem_u32(bufA), 128 * 16, 128);
        const uint32_t blk = 128 * KB * 2, cb = KB / 2, id = idesc_bf16(128, N);
        if (mode == 5)
          mma_kloop_multi(t + 384, N, t, cb, 4, ad, blk >> 4, (2 * 128 * 16) >> 4, 2, bd, (2 * LBO) >> 4, id, KB / 16);
        else if (mode == 6)
          mma_kloop_multi(t + 384, N, t, cb, 4, ad, blk >> 4, (2 * 128 * 16) >> 4, 0, bd, (2 * LBO) >> 4, id, KB / 16);
        else  // one TS chain of 48 (forward-like, same instruction count as mode 3)
          mma_chain_ts(t + 384, t, 8, sdesc_kmajor(smem_u32(bufB), LBO, 128), (2 * LBO) >> 4, id, 48);
        if (elect_one()) mma_commit(&bar[0]);
      } else if (mode == 0) {  // forward mix
        const uint32_t LBO = N * 16;
        const uint64_t bd = sdesc_kmajor(smem_u32(bufB), LBO, 128);
        mma_chain_ts_ss(t + 384, t, 8, t + 400, sdesc_kmajor(smem_u32(bufA), 64 * 16, 128), (2 * 64 * 16) >> 4, bd,
                        (2 * LBO) >> 4, idesc_bf16(128, N), idesc_bf16(64, N), KF / 16);
        if (elect_one()) mma_commit(&bar[0]);
      } else {
        const uint32_t LBO = N * 16;
        const uint64_t bd = sdesc_kmajor(smem_u32(bufB), LBO, 128);
        const uint64_t ad = sdesc_kmajor(smem_u32(bufA), 128 * 16, 128);
        const uint32_t blk = 128 * KB * 2, cb = KB / 2, id = idesc_bf16(128, N);
        const bool ts = mode != 4, ss = mode != 3, per = mode == 2;
        nb = per ? 6 : 1;
        for (int mb = 0; mb < 6; ++mb) {
          if (mb < 4) {
            if (ts) mma_chain_ts(t + 384 + mb * N, t + mb * cb, 8, bd, (2 * LBO) >> 4, id, KB / 16);
          } else if (ss) {
            mma_chain_ss(t + 384 + mb * N, ad + (uint64_t)((mb - 4) * (blk >> 4)), (2 * 128 * 16) >> 4, bd,
                         (2 * LBO) >> 4, id, KB / 16);
          }
          if (per || mb == 5) {
            if (elect_one()) mma_commit(&bar[per ? mb : 0]);
            __syncwarp();
          }
        }
      }
      __syncwarp();
    }
    if (spin && w > 0) {  // the other warps poll the last barrier (test_wait spin), as drain warps do
      const uint32_t ba = smem_u32(&bar[nb - 1]);
      while (!mbar_test(ba, rep & 1)) {
      }
    }
    if (tid == 0) {
      mbar_wait(&bar[nb - 1], rep & 1);
      if (nb > 1)
        for (int i = 0; i < nb - 1; ++i) mbar_wait(&bar[i], rep & 1);
      const long long dt = clock64() - t0;
      best = dt < best ? dt : best;
    }
  }
  __syncthreads();
  if (tid == 0) out[0] = best;
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(t, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 98304);
  const char* names[] = {"fwd 48x(TS128+SS64) K=768", "bwd 4xTS + 2xSS128, 1 commit", "bwd per-block commits",
                         "bwd TS chains only (48)", "bwd SS128 chains only (24)", "bwd K-outer 4TS+2SS (72)",
                         "bwd K-outer 4TS (48)", "one TS chain of 48", "bwd 4x(TS128+SS64), 1 commit",
                         "bwd 4x(TS128+SS64), per-pair commits"};
  for (int threads : {128})
    for (int spin = 0; spin < 2; ++spin)
    for (int rnd = 0; rnd < 2; ++rnd)
    for (int m = 0; m < 10; ++m) {
      if (m != 0 && m != 2 && m != 8 && m != 9) continue;
      bench<<<1, threads, 32768 + 98304>>>(m, spin, rnd, d);
      long long h = 0;
      cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%3d threads spin %d rnd %d  %-32s %6lld cycles  %s\n", threads, spin, rnd, names[m], h, cudaGetErrorString(e));
    }
  return 0;
}
