// allgather_bench.cu -- per-step all-gather of a hidden-state tile inside one
// thread-block cluster (the h exchange of a cluster-resident recurrence):
// every CTA owns SLICE bytes and needs all CL slices in its own SMEM each step.
//   mode 0: st.async 16-byte pushes into every peer, completion on the peer's
//           mbarrier (complete_tx)
//   mode 1: one cp.async.bulk smem->peer-smem copy per peer (bulk-copy engine)
//   mode 2: slice to global, fence.proxy.async, one multicast bulk load
//           global -> all CTAs of the cluster
// Double-buffered like the recurrence (step t writes buffer t&1); reports
// cycles per step in steady state.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;
constexpr int STEPS = 256;

__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t a, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tW:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(a),
      "r"(ph)
      : "memory");
}

template <int CL, int SLICE>
__global__ void allgather(int mode, uint8_t* gbuf, long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* buf = sm;                         // [2][CL*SLICE]
  uint8_t* stage = sm + 2 * CL * SLICE;      // my slice
  __shared__ __align__(8) uint64_t mbar[2];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t me = cl.block_rank();
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&mbar[i]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < SLICE / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(stage)[i] = me * 1000 + i;
  cl.sync();
  const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(&mbar[0]);
  const uint32_t buf0 = (uint32_t)__cvta_generic_to_shared(buf);
  const uint32_t stg = (uint32_t)__cvta_generic_to_shared(stage);
  if (tid == 0)  // arm step 0
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb0), "r"(CL * SLICE) : "memory");
  __syncthreads();
  long long t0 = 0;
  for (int t = 0; t < STEPS; ++t) {
    if (t == 16) t0 = clock64();
    const int b = t & 1;
    const uint32_t my_mb = mb0 + 8 * b;
    // arm the other buffer for step t+1 before anyone can send it
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb0 + 8 * (b ^ 1)), "r"(CL * SLICE)
                   : "memory");
    __syncthreads();
    const uint32_t dst_off = buf0 + b * CL * SLICE + me * SLICE;
    if (mode == 0) {
      // 16-byte pushes: thread i sends chunk (i % nchunk) to peers i / nchunk, ...
      constexpr int NCH = SLICE / 16;
      for (int w = tid; w < NCH * CL; w += blockDim.x) {
        const int peer = w / NCH, ch = w % NCH;
        uint4 v = reinterpret_cast<const uint4*>(stage)[ch];
        uint32_t ra = mapa(dst_off + ch * 16, peer), rm = mapa(my_mb, peer);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(ra),
                     "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rm)
                     : "memory");
      }
    } else if (mode == 1) {
      if (tid < CL) {
        const uint32_t peer = tid;
        uint32_t ra = mapa(dst_off, peer), rm = mapa(my_mb, peer);
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(ra),
                     "r"(stg), "r"(SLICE), "r"(rm)
                     : "memory");
      }
    } else {
      uint8_t* g = gbuf + ((size_t)(blockIdx.x / CL) * 2 + b) * CL * SLICE + me * SLICE;
      for (int i = tid; i < SLICE / 16; i += blockDim.x) reinterpret_cast<uint4*>(g)[i] = reinterpret_cast<const uint4*>(stage)[i];
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        uint16_t mask = (uint16_t)((1u << CL) - 1);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
                dst_off),
            "l"(g), "r"(SLICE), "r"(my_mb), "h"(mask)
            : "memory");
      }
    }
    mbar_wait_cluster(my_mb, (t >> 1) & 1);
  }
  long long t1 = clock64();
  if (tid == 0 && me == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / (STEPS - 16);
  // check data of the last step
  const int b = (STEPS - 1) & 1;
  int bad = 0;
  for (int q = 0; q < CL; ++q)
    for (int i = tid; i < SLICE / 4; i += blockDim.x)
      bad += reinterpret_cast<uint32_t*>(buf + b * CL * SLICE + q * SLICE)[i] != (uint32_t)(q * 1000 + i);
  if (bad) atomicAdd(reinterpret_cast<unsigned long long*>(out + 1), 1ull);
  cl.sync();
}

template <int CL, int SLICE>
void run(int mode, uint8_t* g, long long* out) {
  size_t smem = 2 * CL * SLICE + SLICE;
  auto k = allgather<CL, SLICE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaMemset(out, 0, 16);
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, mode, g, out);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  long long h[2] = {-1, -1};
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  const char* nm[] = {"st.async push", "bulk smem->smem", "global+multicast TMA"};
  printf("cluster %2d slice %5d B (gather %6d B): %-22s %6lld cycles/step  bad=%lld %s\n", CL, SLICE, CL * SLICE,
         nm[mode], h[0], h[1], cudaGetErrorString(e));
}

int main() {
  uint8_t* g;
  long long* out;
  cudaMalloc(&g, 1 << 22);
  cudaMalloc(&out, 64);
  for (int mode = 0; mode < 3; ++mode) {
    run<16, 1536>(mode, g, out);   // H=768, B=16, 48 units per CTA (bf16)
    run<16, 3072>(mode, g, out);   // backward partials: 48 units x 16 x 4 B
    run<8, 3072>(mode, g, out);    // cluster of 8
    run<6, 1024>(mode, g, out);    // NH=4 DH=192: 32 units
    run<2, 1024>(mode, g, out);    // NH=12 DH=64
  }
  return 0;
}
