// pingpong_bench.cu -- cost of the producer/consumer mbarrier handshake of a
// TMA -> MMA ring with no data and no math (the per-stage overhead of the
// alternating path's mainloop): warp 0 = producer (waits `empty`, arrives
// `full`), warp 1 = consumer (waits `full`, releases `empty` with a plain
// arrive or with tcgen05.commit).  clock64 over ITERS stages.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pp tests/cuda/pingpong_bench.cu
#include <cstdio>

#include "../../paper_2412_07752_b200/csrc/sm100.cuh"

using namespace frnn::sm100;
constexpr int ITERS = 1024;

__device__ __forceinline__ void wait_test(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_test(a, phase)) {
  }
}

__global__ void pingpong(int stages, int use_commit, int use_tx, int mode, long long* out) {
  __shared__ uint64_t full[8], empty[8];
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, w = tid >> 5;
  if (w == 2) tmem_alloc(&tb, 32);
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  long long t0 = clock64();
  if (w == 0) {
    if (elect_one()) {
      for (int k = 0; k < ITERS; ++k) {
        const int s = k % stages;
        if (k >= stages) {
          if (mode & 1) wait_test(&empty[s], ((k / stages) - 1) & 1);
          else mbar_wait(&empty[s], ((k / stages) - 1) & 1);
        }
        if (use_tx) mbar_arrive_expect_tx(&full[s], 0);
        else mbar_arrive(&full[s]);
      }
    }
    __syncwarp();
  } else if (w == 1) {
    for (int k = 0; k < ITERS; ++k) {
      const int s = k % stages;
      if (mode & 1) wait_test(&full[s], (k / stages) & 1);
      else mbar_wait(&full[s], (k / stages) & 1);
      if (!(mode & 2)) tc_fence_after();
      if (elect_one()) {
        if (use_commit) mma_commit(&empty[s]);
        else mbar_arrive(&empty[s]);
      }
      __syncwarp();
    }
    if (threadIdx.x == 32) out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (w == 2) tmem_dealloc(tb, 32);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  const char* modes[] = {"try_wait + fence", "test_wait spin + fence", "try_wait, no fence", "test_wait, no fence"};
  for (int st : {4})
    for (int c = 0; c < 2; ++c)
      for (int m = 0; m < 4; ++m) {
        pingpong<<<1, 96>>>(st, c, 1, m, d);
        long long h = 0;
        cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("stages %d release %-16s %-24s: %7.1f cycles/stage  %s\n", st, c ? "tcgen05.commit" : "mbarrier.arrive",
               modes[m], (double)h / ITERS, cudaGetErrorString(e));
      }
  return 0;
}
