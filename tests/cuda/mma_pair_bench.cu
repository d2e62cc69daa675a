// mma_pair_bench.cu -- does a CTA pair (tcgen05.mma.cta_group::2, M=256) issue
// the recurrent kernels' small-N MMAs faster than two single CTAs (M=128 each)?
// At N=16 a TMEM-A M=128 MMA costs ~50 cycles regardless of the accumulator
// chain (mma_bwd_bench.cu): if that cost is per instruction, one M=256 pair
// instruction covers twice the rows in the same time.
//   CG=1: both CTAs of a 2-CTA cluster each issue a chain of 48 TS MMAs
//         (M=128, N) on their own TMEM -- the cluster kernels today;
//   CG=2: the leader issues 48 TS MMAs with cta_group::2 (M=256, N; each CTA
//         holds 128 rows of A in TMEM and N/2 rows of B in SMEM).
// clock64 on the leader from the first issue to the commit's mbarrier.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mpb tests/cuda/mma_pair_bench.cu
#include <cuda_bf16.h>

#include <cstdio>

#include "../../paper_2412_07752_b200/csrc/sm100.cuh"

using namespace frnn::sm100;

template <int CG>
__global__ void __cluster_dims__(2, 1, 1) bench(int N, int nmma, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, w = tid >> 5;
  const uint32_t rank = cluster_ctarank();
  if (w == 0) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      tmem_alloc(&tb, 512);
    }
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t t = tb;
  if (w < 4) {  // TMEM A columns 0..383 (K = 768 bf16)
    for (int c0 = 0; c0 < 384; c0 += 16) {
      uint32_t v[16];
      for (int q = 0; q < 16; ++q) v[q] = 0x3c003c00u;
      tmem_st16(t + ((uint32_t)(32 * w) << 16) + c0, v);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const int NB = CG == 2 ? N / 2 : N;  // B rows held by this CTA
  const uint32_t LBO = (uint32_t)NB * 16;  // K-adjacent core matrices
  const uint64_t bd = sdesc_kmajor(smem_u32(sm), LBO, 128), bk = (2 * LBO) >> 4;
  const uint32_t idesc = idesc_bf16(128 * CG, N);
  long long best = 1ll << 60;
  for (int rep = 0; rep < 8; ++rep) {
    __syncthreads();
    cluster_sync_all();
    const long long t0 = clock64();
    if (w == 0 && (CG == 1 || rank == 0)) {
      tc_fence_after();
      if (CG == 1) {
        mma_chain_ts(t + 384, t, 8, bd, bk, idesc, nmma);
        if (elect_one()) mma_commit(&bar);
      } else {
        asm volatile(
            "{\n\t.reg .pred e, p, q;\n\t.reg .b32 k, ta;\n\t.reg .b64 b;\n\t"
            "elect.sync _|e, 0xffffffff;\n\tmov.b32 k, 0;\n\tmov.b32 ta, %1;\n\tmov.b64 b, %2;\n\t"
            "LP%=:\n\tsetp.ne.b32 p, k, 0;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], b, %4, p;\n\t"
            "add.u32 ta, ta, 8;\n\tadd.u64 b, b, %3;\n\tadd.s32 k, k, 1;\n\t"
            "setp.lt.s32 q, k, %5;\n\t@q bra.uni LP%=;\n\t}" ::"r"(t + 384),
            "r"(t), "l"(bd), "l"(bk), "r"(idesc), "r"(nmma)
            : "memory");
        if (elect_one())
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&bar)),
              "h"((uint16_t)3)
              : "memory");
      }
      __syncwarp();
    }
    if (tid == 0) {
      mbar_wait(&bar, rep & 1);
      const long long dt = clock64() - t0;
      best = dt < best ? dt : best;
    }
  }
  __syncthreads();
  if (tid == 0 && rank == 0) out[0] = best;
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (w == 0) {
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(t));
    else
      tmem_dealloc(t, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int N : {16, 32, 64})
    for (int cg = 1; cg <= 2; ++cg) {
      long long h = 0;
      if (cg == 1) bench<1><<<2, 128, 64 * 1024>>>(N, 48, d);
      else bench<2><<<2, 128, 64 * 1024>>>(N, 48, d);
      cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("N=%2d cta_group::%d  48 TS MMAs (M=%d): %6lld cycles (%5.1f / MMA, %5.2f rows/cycle per SM)  %s\n", N, cg,
             128 * cg, h, h / 48.0, 48.0 * 128 / h, cudaGetErrorString(e));
    }
  return 0;
}
