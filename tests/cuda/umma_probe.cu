// umma_probe.cu -- checks the tcgen05 operand conventions the fused kernels rely
// on: A (M=128 x K=32, bf16) resident in TMEM as packed bf16 pairs per lane, B
// (N=16 x K=32) K-major no-swizzle in SMEM with LBO = K-adjacent core-matrix
// stride, SBO = 8-row-group stride; D fp32 in TMEM read with 32x32b loads.
// Prints max |err| for the intended convention and for swapped LBO/SBO.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>

#include "../../paper_2412_07752_b200/csrc/sm100.cuh"

using namespace frnn::sm100;

constexpr int M = 128, N = 16, K = 32;

__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int swap) {
  __shared__ __align__(1024) uint8_t sB[N * K * 2];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  if (w == 0) tmem_alloc(&tb, 64);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  // B tile, K-major core matrices: (k/8, n/8) at ((k/8)*(N/8) + n/8)*128
  for (int i = tid; i < N * K; i += 128) {
    int n = i / K, k = i % K;
    uint32_t off = ((k >> 3) * (N / 8) + (n >> 3)) * 128 + (n & 7) * 16 + (k & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sB + off) = B[n * K + k];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tb;
  {
    int row = 32 * w + l;
    uint32_t v[16];
    for (int c = 0; c < 16; ++c) {
      __nv_bfloat162 p;
      p.x = A[row * K + 2 * c];
      p.y = A[row * K + 2 * c + 1];
      v[c] = *reinterpret_cast<uint32_t*>(&p);
    }
    tmem_st16(t + ((uint32_t)(32 * w) << 16), v);
    tmem_st_wait();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc_fence_after();
    uint32_t LBO = N * 16, SBO = 128;
    if (swap) { uint32_t x = LBO; LBO = SBO; SBO = x; }
    for (int ks = 0; ks < K / 16; ++ks)
      mma_ts(t + 32, t + ks * 8, sdesc_kmajor(smem_u32(sB) + ks * 2 * (N * 16), LBO, SBO),
             idesc_bf16(M, N), ks > 0);
    mma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tc_fence_after();
  float v[16];
  tmem_ld16(t + ((uint32_t)(32 * w) << 16) + 32, v);
  for (int n = 0; n < N; ++n) D[(32 * w + l) * N + n] = v[n];
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(t, 64);
}

int main() {
  __nv_bfloat16 *hA = new __nv_bfloat16[M * K], *hB = new __nv_bfloat16[N * K];
  float* ref = new float[M * N];
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f);
  for (int i = 0; i < N * K; ++i) hB[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < K; ++k) s += __bfloat162float(hA[m * K + k]) * __bfloat162float(hB[n * K + k]);
      ref[m * N + n] = s;
    }
  __nv_bfloat16 *dA, *dB;
  float* dD;
  cudaMalloc(&dA, M * K * 2);
  cudaMalloc(&dB, N * K * 2);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice);
  int rc = 1;
  for (int swap = 0; swap < 2; ++swap) {
    cudaMemset(dD, 0, M * N * 4);
    probe<<<1, 128>>>(dA, dB, dD, swap);
    cudaError_t e = cudaDeviceSynchronize();
    float* hD = new float[M * N];
    cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
    printf("umma_probe swap=%d: %s max_abs_err=%g  D[0][0..3]=%g %g %g %g ref=%g %g %g %g\n", swap,
           cudaGetErrorString(e), err, hD[0], hD[1], hD[2], hD[3], ref[0], ref[1], ref[2], ref[3]);
    if (swap == 0 && err == 0) rc = 0;
  }
  printf("UMMA_PROBE %s\n", rc == 0 ? "PASS" : "FAIL");
  return rc;
}
