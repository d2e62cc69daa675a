// sync_bench.cu -- latency of the inter-CTA primitives a persistent recurrence
// step is built from, measured with clock64 on B200:
//   1. flag ping-pong through L2 between two CTAs (st.release/ld.acquire.gpu),
//   2. the same with relaxed stores + volatile polling (no fences),
//   3. an 8-byte "LL" word (4 B data + 4 B step tag) ping-pong (no fences),
//   4. DSMEM push (st.async + remote mbarrier complete_tx) ping-pong in a cluster,
//   5. time for 128 threads to read a 24 KB tile freshly written by another CTA.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_vol(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_vol(uint32_t* p, uint32_t v) {
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_vol64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_vol64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr int ITERS = 200;

// mode 0: release/acquire flag, 1: volatile flag, 2: LL 8-byte word
__global__ void pingpong(uint32_t* flags, unsigned long long* ll, long long* out, int mode) {
  if (threadIdx.x != 0) return;
  const int me = blockIdx.x;  // 0 or 1
  long long t0 = clock64();
  for (int i = 1; i <= ITERS; ++i) {
    if (me == 0) {
      if (mode == 0) st_rel(flags, i); else if (mode == 1) st_vol(flags, i);
      else st_vol64(ll, ((unsigned long long)i << 32) | 0x1234u);
      if (mode == 0) while (ld_acq(flags + 32) < (uint32_t)i) {}
      else if (mode == 1) while (ld_vol(flags + 32) < (uint32_t)i) {}
      else while ((ld_vol64(ll + 16) >> 32) < (unsigned long long)i) {}
    } else {
      if (mode == 0) while (ld_acq(flags) < (uint32_t)i) {}
      else if (mode == 1) while (ld_vol(flags) < (uint32_t)i) {}
      else while ((ld_vol64(ll) >> 32) < (unsigned long long)i) {}
      if (mode == 0) st_rel(flags + 32, i); else if (mode == 1) st_vol(flags + 32, i);
      else st_vol64(ll + 16, ((unsigned long long)i << 32) | 0x5678u);
    }
  }
  if (me == 0) out[mode] = (clock64() - t0) / ITERS;  // one round trip
}

// 24 KB tile: CTA 1 writes it, releases a flag; CTA 0 acquires and loads it.
__global__ void tile_load(uint4* tile, uint32_t* flags, long long* out) {
  __shared__ uint4 sm[1536];
  __shared__ long long t_load;
  const int me = blockIdx.x;
  for (int it = 1; it <= 20; ++it) {
    if (me == 1) {
      for (int i = threadIdx.x; i < 1536; i += 128) tile[i] = make_uint4(it, it, it, it);
      __syncthreads();
      if (threadIdx.x == 0) st_rel(flags, it);
      if (threadIdx.x == 0) while (ld_acq(flags + 32) < (uint32_t)it) {}
      __syncthreads();
    } else {
      if (threadIdx.x == 0) while (ld_acq(flags) < (uint32_t)it) {}
      __syncthreads();
      long long t0 = clock64();
      uint4 v[12];
#pragma unroll
      for (int q = 0; q < 12; ++q) v[q] = tile[threadIdx.x + 128 * q];
#pragma unroll
      for (int q = 0; q < 12; ++q) sm[threadIdx.x + 128 * q] = v[q];
      __syncthreads();
      if (threadIdx.x == 0) t_load = clock64() - t0;
      if (threadIdx.x == 0) st_rel(flags + 32, it);
    }
  }
  if (me == 0 && threadIdx.x == 0) out[3] = t_load;
}

// DSMEM ping-pong within a cluster of 2: st.async 16 B into the peer's smem,
// completing on the peer's mbarrier; the peer waits on its own mbarrier.
__global__ void __cluster_dims__(2, 1, 1) dsmem_pingpong(long long* out) {
  __shared__ __align__(16) uint4 buf[64];
  __shared__ __align__(8) uint64_t mbar;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned me = cl.block_rank();
  if (threadIdx.x == 0) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  if (threadIdx.x != 0) return;
  uint32_t my_mbar = (uint32_t)__cvta_generic_to_shared(&mbar);
  uint32_t my_buf = (uint32_t)__cvta_generic_to_shared(&buf[0]);
  uint32_t peer_mbar, peer_buf;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer_mbar) : "r"(my_mbar), "r"(me ^ 1));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer_buf) : "r"(my_buf), "r"(me ^ 1));
  long long t0 = clock64();
  uint32_t phase = 0;
  for (int i = 1; i <= ITERS; ++i) {
    auto push = [&]() {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(my_mbar) : "memory");
    };
    auto send = [&]() {
      asm volatile(
          "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%1,%1,%1}, [%2];" ::"r"(peer_buf),
          "r"(i), "r"(peer_mbar)
          : "memory");
    };
    auto wait = [&]() {
      asm volatile(
          "{\n\t.reg .pred P;\n\tW:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(
              my_mbar),
          "r"(phase)
          : "memory");
      phase ^= 1;
    };
    if (me == 0) {
      push();
      send();
      wait();
    } else {
      push();
      wait();
      send();
    }
  }
  if (me == 0) out[4] = (clock64() - t0) / ITERS;
}

int main() {
  uint32_t* flags;
  unsigned long long* ll;
  long long* out;
  uint4* tile;
  cudaMalloc(&flags, 4096);
  cudaMalloc(&ll, 4096);
  cudaMalloc(&out, 64);
  cudaMalloc(&tile, 1536 * 16);
  const char* names[] = {"flag release/acquire round trip", "flag volatile round trip", "LL 8B word round trip"};
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(flags, 0, 4096);
    cudaMemset(ll, 0, 4096);
    pingpong<<<2, 32>>>(flags, ll, out, mode);
    cudaError_t e = cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, out + mode, 8, cudaMemcpyDeviceToHost);
    printf("%-36s: %6lld cycles (%s)\n", names[mode], h, cudaGetErrorString(e));
  }
  cudaMemset(flags, 0, 4096);
  tile_load<<<2, 128>>>(tile, flags, out);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, out + 3, 8, cudaMemcpyDeviceToHost);
  printf("%-36s: %6lld cycles (%s)\n", "24KB tile load after acquire", h, cudaGetErrorString(e));
  dsmem_pingpong<<<2, 32>>>(out);
  e = cudaDeviceSynchronize();
  cudaMemcpy(&h, out + 4, 8, cudaMemcpyDeviceToHost);
  printf("%-36s: %6lld cycles (%s)\n", "DSMEM st.async+mbarrier round trip", h, cudaGetErrorString(e));
  return 0;
}
