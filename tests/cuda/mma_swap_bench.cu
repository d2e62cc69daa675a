// mma_swap_bench.cu -- which operand should the streamed R be in the
// alternating path's per-step GEMM?  Today R rows are the A operand (M=128)
// and the batch tile h the B operand (N=64), both from SMEM.  Swapped, h is A
// (M=64 batch rows) and R rows are B (N=128 or 256).  48 chained SS MMAs
// (K=16 each) on one CTA, clock64 from the first issue to the commit barrier.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/msb tests/cuda/mma_swap_bench.cu
#include <cuda_bf16.h>

#include <cstdio>

#include "../../paper_2412_07752_b200/csrc/sm100.cuh"

using namespace frnn::sm100;

__global__ void bench(int M, int N, int nmma, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, w = tid >> 5;
  if (w == 0) tmem_alloc(&tb, 512);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tb;
  // A: M rows x K (K-major, no swizzle), B: N rows x K, K = 16 * nmma
  uint8_t* A = sm;
  uint8_t* Bt = sm + 96 * 1024;
  const uint64_t ad = sdesc_kmajor(smem_u32(A), (uint32_t)M * 16, 128), bd = sdesc_kmajor(smem_u32(Bt), (uint32_t)N * 16, 128);
  const uint64_t ak = (2 * M * 16) >> 4, bk = (2 * N * 16) >> 4;
  const uint32_t idesc = idesc_bf16(M, N);
  long long best = 1ll << 60;
  for (int rep = 0; rep < 8; ++rep) {
    __syncthreads();
    const long long t0 = clock64();
    if (w == 0) {
      tc_fence_after();
      // (operands wrap within their buffers: only the issue/execution rate matters)
      mma_chain_ss(t, ad, ak, bd, bk, idesc, nmma);
      if (elect_one()) mma_commit(&bar);
      __syncwarp();
    }
    if (tid == 0) {
      mbar_wait(&bar, rep & 1);
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
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct C { int M, N, nm; const char* what; } cs[] = {
      {128, 16, 24, "R as A (M=128), h as B, N=16"},  {128, 64, 24, "R as A (M=128), h as B, N=64 (today, C5)"},
      {64, 128, 24, "h as A (M=64 batch), R as B (N=128)"}, {64, 256, 12, "h as A (M=64 batch), R as B (N=256)"},
      {128, 128, 24, "M=128, N=128"}, {128, 256, 12, "M=128, N=256"}};
  for (auto c : cs) {
    long long h = 0;
    bench<<<1, 128, 200 * 1024>>>(c.M, c.N, c.nm, d);
    cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / c.nm;
    const int rrows = c.what[0] == 'R' ? c.M : c.N;  // rows of R covered per MMA
    printf("%-44s %3d MMAs: %6lld cycles, %6.1f / MMA, %5.2f R rows x16K per cycle  %s\n", c.what, c.nm, h, per,
           rrows / per, cudaGetErrorString(e));
  }
  return 0;
}
