// mma_cluster_bench.cu -- the backward's per-step MMA mix (4 x (TS M=128 +
// SS M=64), N=16, K=192) in the cluster kernel's launch geometry: 384 threads,
// 218 KB dynamic SMEM (SMEM-A blocks at offset 0, the dg tile at 192 KB),
// 512 TMEM columns, optionally a 16-CTA cluster -- to separate the MMA cost
// from the rest of the kernel.  Per iteration: __syncthreads, warp 0 issues,
// warp 1 waits for the last commit; median cycles over ITERS iterations.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tests/cuda/mma_cluster_bench tests/cuda/mma_cluster_bench.cu
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "../../paper_2412_07752_b200/csrc/sm100.cuh"

using namespace frnn::sm100;

constexpr int N = 16, KB = 192, ITERS = 64, SMEM = 218432 + 256, DGB = 196608, BAROFF = 218432;

__global__ void __launch_bounds__(384, 1) bench(int mode, int gap, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t sbar[8];
  uint64_t* bar = (mode & 128) ? reinterpret_cast<uint64_t*>(sm + BAROFF) : sbar;  // barriers where the kernel has them
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, w = tid >> 5;
  if (w == 0) tmem_alloc(&tb, 512);
  for (int i = tid; i < BAROFF / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  __syncthreads();
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tb;
  const bool per = mode & 1, seq = mode & 2, none = mode & 4, wdg = mode & 8, spin = mode & 16, fen = mode & 32,
             drain = mode & 64, absorb = mode & 256;
  const int last = per ? 3 : 0;
  long long dts[ITERS], iss[ITERS];
  __shared__ uint64_t rbar;
  if (tid == 0) {
    mbar_init(&rbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  float sink = 0.f;
  for (int it = 0; it < ITERS; ++it) {
    if (absorb) {  // like the backward's absorb: local arrive, cluster-scope acquire wait, 16 float2 reads
      if (tid == 0) mbar_arrive_expect_tx(&rbar, 0);
      mbar_wait_cluster(&rbar, it & 1);
      const float* rp = reinterpret_cast<const float*>(sm + 98304) + 2 * tid;
      for (int q = 0; q < 16; ++q) {
        const float2 v = *reinterpret_cast<const float2*>(rp + q * 768);
        sink += v.x + v.y;
      }
      __syncthreads();
    }
    if (gap) {  // idle tensor pipe between bursts, like the rest of a recurrence step
      const long long g0 = clock64();
      while (clock64() - g0 < gap) {
      }
    }
    if (wdg) {  // like the Jacobian phase: every thread rewrites its part of the dg tile
      reinterpret_cast<uint4*>(sm + DGB)[tid] = make_uint4(0x3c003c00u, it, tid, 0x3c003c00u);
      fence_proxy_async_smem();
    }
    if (fen) tc_fence_before();
    __syncthreads();
    if (fen) tc_fence_after();
    const long long t0 = clock64();
    if (w == 0) {
      tc_fence_after();
      const uint32_t LBO = N * 16;
      const uint64_t bd = sdesc_kmajor(smem_u32(sm + DGB), LBO, 128);
      const uint32_t blk64 = 64 * KB * 2, cb = KB / 2;
      for (int i = 0; i < 4; ++i) {
        const uint64_t ad = sdesc_kmajor(smem_u32(sm) + i * blk64, 64 * 16, 128);
        if (none) {
        } else if (seq) {
          mma_chain_ts(t + 384 + i * N, t + i * cb, 8, bd, (2 * LBO) >> 4, idesc_bf16(128, N), KB / 16);
          mma_chain_ss(t + 448 + i * N, ad, (2 * 64 * 16) >> 4, bd, (2 * LBO) >> 4, idesc_bf16(64, N), KB / 16);
        } else {
          mma_chain_ts_ss(t + 384 + i * N, t + i * cb, 8, t + 448 + i * N, ad, (2 * 64 * 16) >> 4, bd,
                          (2 * LBO) >> 4, idesc_bf16(128, N), idesc_bf16(64, N), KB / 16);
        }
        if (per || i == 3) {
          if (elect_one()) mma_commit(&bar[per ? i : 0]);
          __syncwarp();
        }
      }
      iss[it] = clock64() - t0;
    }
    if (w == 1) {
      mbar_wait(&bar[last], it & 1);
      dts[it] = clock64() - t0;
    }
    if (per && w == 2)
      for (int i = 0; i < 3; ++i) mbar_wait(&bar[i], it & 1);
    if (spin && w >= 2)  // like the drain warps: everyone waits on the block barriers
      for (int i = 0; i <= last; ++i) mbar_wait(&bar[i], it & 1);
    if (drain) {  // every warp reads one accumulator block of its lane quadrant, like the drain
      mbar_wait(&bar[last], it & 1);
      tc_fence_after();
      float v[16];
      tmem_ld16(t + ((uint32_t)(32 * (w & 3)) << 16) + 384 + (w >> 2) * N, v);
      float acc = 0.f;
      for (int q = 0; q < 16; ++q) acc += v[q];
      if (acc == 12345.f) out[31] = 1;
    }
  }
  if (sink == 12345.f) out[30] = 1;
  if (tid == 0) {
    for (int i = 1; i < ITERS; ++i)
      for (int j = i; j > 0 && iss[j] < iss[j - 1]; --j) {
        const long long x = iss[j];
        iss[j] = iss[j - 1];
        iss[j - 1] = x;
      }
    out[16 + blockIdx.x] = iss[ITERS / 2];
  }
  if (tid == 32) {
    for (int i = 1; i < ITERS; ++i)  // insertion sort, median
      for (int j = i; j > 0 && dts[j] < dts[j - 1]; --j) {
        const long long x = dts[j];
        dts[j] = dts[j - 1];
        dts[j - 1] = x;
      }
    out[blockIdx.x] = dts[ITERS / 2];
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(t, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 32);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  cudaFuncSetAttribute(bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char* names[] = {"interleaved, 1 commit", "interleaved, per-pair commits", "sequential, 1 commit",
                         "sequential, per-pair commits", "no MMAs, 1 commit", "no MMAs, 4 commits"};
  const int modes[] = {1, 1 | 256, 5 | 256, 1 | 8 | 16 | 32 | 64 | 128 | 256, 5 | 8 | 16 | 32 | 64 | 128 | 256};
  for (int cl : {16})
    for (int gap : {0})
    for (int mode : modes) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cl);
      cfg.blockDim = dim3(384);
      cfg.dynamicSmemBytes = SMEM;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, bench, mode, gap, d);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      std::vector<long long> h(32, 0);
      cudaMemcpy(h.data(), d, 8 * 32, cudaMemcpyDeviceToHost);
      std::sort(h.begin(), h.begin() + cl);
      std::sort(h.begin() + 16, h.begin() + 16 + cl);
      printf("gap %5d cluster %2d mode %2d %-32s median cycles/iter: done %6lld..%6lld  issue %6lld..%6lld  %s\n", gap, cl, mode, names[mode & 7],
             h[0], h[cl - 1], h[16], h[16 + cl - 1], cudaGetErrorString(e));
    }
  return 0;
}
