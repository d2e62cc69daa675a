// mma_mix_bench.cu -- tcgen05 issue patterns of the cluster-resident kernels,
// N=16, one CTA, clock64 around issue -> commit -> wait:
//   0: forward, TS M=128 and SS M=64 interleaved per K step (48 + 48)
//   1: forward, TS chain (48) then SS M=64 chain (48)
//   2: forward, SS M=64 chain then TS chain
//   3: backward, 4 TS blocks x 12 then 2 SS M=128 blocks x 12 (6 accumulators)
//   4: backward, SS blocks first then TS blocks
//   5: TS chain only (48), 6: SS M=64 only (48), 7: SS M=128 only (24)
#include <cuda_bf16.h>
#include <cstdio>

#include "../../paper_2412_07752_b200/csrc/sm100.cuh"

using namespace frnn::sm100;
constexpr int N = 16;

__global__ void bench(int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sB = sm;                     // [16 x 768] K-major (24 KB)
  uint8_t* sA64 = sm + 24576;           // [64 x 768] K-major (96 KB)
  uint8_t* sA128 = sA64 + 98304;        // 2 x [128 x 192] K-major (96 KB)
  __shared__ uint64_t mbar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, w = tid >> 5;
  if (w == 0) tmem_alloc(&tb, 512);
  if (tid == 0) { mbar_init(&mbar, 1); fence_mbar_init(); }
  for (int i = tid; i < (24576 + 98304 + 98304) / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = __shfl_sync(0xffffffffu, tb, 0);
  const uint32_t i128 = idesc_bf16(128, N), i64 = idesc_bf16(64, N);
  long long best = 1ll << 60;
  for (int rep = 0; rep < 5; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    if (w == 0) {
      tc_fence_after();
      const uint64_t b0 = sdesc_kmajor(smem_u32(sB), 256, 128);
      const uint64_t a64 = sdesc_kmajor(smem_u32(sA64), 1024, 128);
      if (mode <= 2 || mode == 5 || mode == 6) {
        const bool ts = mode != 6, ss = mode != 5;
        if (mode == 0) {
          for (int ks = 0; ks < 48; ++ks) {
            if (elect_one()) {
              mma_ts(t + 384, t + ks * 8, b0 + ks * 32, i128, ks > 0);
              mma_ss(t + 400, a64 + ks * 128, b0 + ks * 32, i64, ks > 0);
            }
            __syncwarp();
          }
        } else {
          for (int pass = 0; pass < 2; ++pass) {
            const bool do_ts = (mode == 2) ? pass == 1 : pass == 0;
            if (do_ts && !ts) continue;
            if (!do_ts && !ss) continue;
            for (int ks = 0; ks < 48; ++ks) {
              if (elect_one()) {
                if (do_ts) mma_ts(t + 384, t + ks * 8, b0 + ks * 32, i128, ks > 0);
                else mma_ss(t + 400, a64 + ks * 128, b0 + ks * 32, i64, ks > 0);
              }
              __syncwarp();
            }
          }
        }
      } else {
        // backward: dg tile [16 x 192], 6 column blocks
        const uint64_t bd = sdesc_kmajor(smem_u32(sB), 256, 128);
        for (int pass = 0; pass < 2; ++pass) {
          const bool do_ts = (mode == 4) ? pass == 1 : pass == 0;
          if (mode == 7 && do_ts) continue;
          for (int mb = do_ts ? 0 : 4; mb < (do_ts ? 4 : 6); ++mb) {
            const uint64_t ad = sdesc_kmajor(smem_u32(sA128 + (mb - 4) * 49152), 2048, 128);
            for (int ks = 0; ks < 12; ++ks) {
              if (elect_one()) {
                if (do_ts) mma_ts(t + 384 + mb * 16, t + mb * 96 + ks * 8, bd + ks * 32, i128, ks > 0);
                else mma_ss(t + 384 + mb * 16, ad + ks * 256, bd + ks * 32, i128, ks > 0);
              }
              __syncwarp();
            }
          }
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

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  const char* nm[] = {"fwd TS/SS64 interleaved (96)", "fwd TS chain, SS64 chain (96)", "fwd SS64 chain, TS chain (96)",
                      "bwd 4xTS then 2xSS128 (72)",    "bwd 2xSS128 then 4xTS (72)",    "TS chain only (48)",
                      "SS64 chain only (48)",          "SS128 only 2 blocks (24)"};
  const int smem = 24576 + 98304 + 98304;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 8; ++mode) {
    bench<<<1, 128, smem>>>(mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = -1;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %6lld cycles  %s\n", nm[mode], h, cudaGetErrorString(e));
  }
  return 0;
}
