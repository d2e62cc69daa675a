// mma_bench.cu -- microbenchmark of the per-step tcgen05 MMA chain used by the
// fused recurrence (K/16 instructions of M x N x 16, bf16 -> fp32) from one CTA:
// clock64 around issue -> commit -> mbarrier wait.  Varies the A source (TMEM
// 'TS' vs SMEM 'SS'), N, and the number of independent accumulators the
// instructions rotate over (dependency latency vs issue/throughput).
#include <cuda_bf16.h>
#include <cstdio>

#include "../../paper_2412_07752_b200/csrc/sm100.cuh"

using namespace frnn::sm100;

template <int M, int N>
__global__ void bench(int ksteps, int ts, int nacc, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;                        // [M x K] K-major, no swizzle
  uint8_t* sB = sm + M * ksteps * 16 * 2;  // [N x K]
  __shared__ uint64_t mbar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, w = tid >> 5;
  if (w == 0) tmem_alloc(&tb, 512);
  if (tid == 0) { mbar_init(&mbar, 1); fence_mbar_init(); }
  for (int i = tid; i < (M + N) * ksteps * 16 * 2 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tb;
  const uint32_t idesc = idesc_bf16(M, N);
  const uint32_t aL = M * 16, aS = 128, bL = N * 16, bS = 128;
  long long best = 1ll << 60;
  for (int rep = 0; rep < 5; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    if (w == 0) {  // warp-uniform issue, one elected lane (no waterfall)
      tc_fence_after();
      const uint32_t tu = __shfl_sync(0xffffffffu, t, 0);
      uint64_t bd = sdesc_kmajor(smem_u32(sB), bL, bS);
      uint64_t ad = sdesc_kmajor(smem_u32(sA), aL, aS);
      uint32_t at = tu;
      const uint32_t acc = tu + 256;
      if (ts) {
        for (int ks = 0; ks < ksteps; ++ks) {
          if (elect_one()) mma_ts(acc, at, bd, idesc, ks > 0 ? 1u : 0u);
          __syncwarp();
          bd += (2 * bL) >> 4;
          at += 8;
        }
      } else {
        for (int ks = 0; ks < ksteps; ++ks) {
          if (elect_one()) mma_ss(acc, ad, bd, idesc, ks > 0 ? 1u : 0u);
          __syncwarp();
          bd += (2 * bL) >> 4;
          ad += (2 * aL) >> 4;
        }
      }
      if (elect_one()) mma_commit(&mbar);
      __syncwarp();
    }
    mbar_wait(&mbar, rep & 1);
    tc_fence_after();
    long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
  }
  if (tid == 0) out[0] = best;
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(t, 512);
}

template <int N, int M = 128>
void run(long long* d, int ks, int ts, int nacc) {
  size_t smem = (size_t)(M + N) * ks * 16 * 2;
  if (smem > 227 * 1024) return;
  cudaFuncSetAttribute(bench<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bench<M, N><<<1, 128, smem>>>(ks, ts, nacc, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = -1;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("M=%3d N=%3d K=%4d %s nacc=%d: %6lld cycles (%5.1f per MMA) %s\n", M, N, ks * 16, ts ? "TS" : "SS", nacc, h,
         (double)h / ks, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int ks : {8, 24, 48, 96}) {
    if (ks <= 48) run<16>(d, ks, 1, 1);
    run<16>(d, ks, 0, 1);
    run<16, 64>(d, ks, 0, 1);
    run<64>(d, ks, 0, 1);
    run<256>(d, ks, 0, 1);
  }
  return 0;
}
