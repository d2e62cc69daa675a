// sm100.cuh -- thin inline-PTX wrappers for the sm_100a features the kernels use:
// tcgen05 (TMEM alloc/ld/st, MMA, commit), mbarriers, proxy fences and
// gpu-scope release/acquire flags.  Compiled only for sm_100a.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace frnn::sm100 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- TMEM ----
// Warp-wide: allocates `ncols` (power of two >= 32) columns, writes base to *dst.
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns: thread i <- lane (base+i).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]));
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// ----------------------------------------------------------- descriptors ---
// Shared-memory matrix descriptor, K-major, no swizzle ("interleaved"):
// core matrices of 8 rows x 16 bytes stored contiguously (128 B);
// LBO = byte distance between K-adjacent core matrices, SBO = between
// 8-row groups (cute UMMA::make_umma_desc<K>, SWIZZLE_NONE).
__device__ __forceinline__ uint64_t sdesc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm_100)
  return d;                // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
}

// Instruction descriptor for kind::f16: bf16 x bf16 -> f32, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4)            // c_format = F32
         | (1u << 7)          // a_format = BF16
         | (1u << 10)         // b_format = BF16
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[tmem] . B[smem]   (A 'TS' form: A rows in TMEM lanes)
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// D[tmem] (+)= A[smem] . B[smem]
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// One lane of a converged warp (elect.sync).  Issuing tcgen05 from a full warp
// under this predicate, with warp-uniform operands, lets ptxas keep operands in
// uniform registers -- no per-instruction ELECT/BRA.U.ANY "waterfall" loop.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

// Whole-warp MMA chains in one PTX loop: every lane runs the loop on uniform
// registers (so ptxas keeps them in the uniform datapath) and elect.sync guards
// only the tcgen05.mma.  Iteration k issues
//   D[d] (+)= A . B   with A = a0 + k*a_step (TMEM address or smem descriptor),
//   B desc = b0 + k*b_step, accumulate = (k > 0 || acc_first).
// Must be called by all 32 lanes of one warp.
__device__ __forceinline__ void mma_chain_ts(uint32_t d, uint32_t a0, uint32_t a_step, uint64_t b0, uint64_t b_step,
                                             uint32_t idesc, int n) {
  asm volatile(
      "{\n\t.reg .pred e, p, q;\n\t.reg .b32 k, ta;\n\t.reg .b64 bd;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b32 k, 0;\n\tmov.b32 ta, %1;\n\tmov.b64 bd, %3;\n\t"
      "setp.ge.s32 q, k, %6;\n\t@q bra.uni CHTS_END%=;\n\t"
      "CHTS_LOOP%=:\n\t"
      "setp.ne.b32 p, k, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %5, p;\n\t"
      "add.u32 ta, ta, %2;\n\tadd.u64 bd, bd, %4;\n\tadd.s32 k, k, 1;\n\t"
      "setp.lt.s32 q, k, %6;\n\t@q bra.uni CHTS_LOOP%=;\n\t"
      "CHTS_END%=:\n\t}" ::"r"(d),
      "r"(a0), "r"(a_step), "l"(b0), "l"(b_step), "r"(idesc), "r"(n)
      : "memory");
}
__device__ __forceinline__ void mma_chain_ss(uint32_t d, uint64_t a0, uint64_t a_step, uint64_t b0, uint64_t b_step,
                                             uint32_t idesc, int n) {
  asm volatile(
      "{\n\t.reg .pred e, p, q;\n\t.reg .b32 k;\n\t.reg .b64 ad, bd;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b32 k, 0;\n\tmov.b64 ad, %1;\n\tmov.b64 bd, %3;\n\t"
      "setp.ge.s32 q, k, %6;\n\t@q bra.uni CHSS_END%=;\n\t"
      "CHSS_LOOP%=:\n\t"
      "setp.ne.b32 p, k, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %5, p;\n\t"
      "add.u64 ad, ad, %2;\n\tadd.u64 bd, bd, %4;\n\tadd.s32 k, k, 1;\n\t"
      "setp.lt.s32 q, k, %6;\n\t@q bra.uni CHSS_LOOP%=;\n\t"
      "CHSS_END%=:\n\t}" ::"r"(d),
      "l"(a0), "l"(a_step), "l"(b0), "l"(b_step), "r"(idesc), "r"(n)
      : "memory");
}
// Interleaved pair chain: TS (M=128) into d1 and SS into d2 sharing B.
__device__ __forceinline__ void mma_chain_ts_ss(uint32_t d1, uint32_t a1, uint32_t a1_step, uint32_t d2, uint64_t a2,
                                                uint64_t a2_step, uint64_t b0, uint64_t b_step, uint32_t idesc1,
                                                uint32_t idesc2, int n) {
  asm volatile(
      "{\n\t.reg .pred e, p, q;\n\t.reg .b32 k, ta;\n\t.reg .b64 ad, bd;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b32 k, 0;\n\tmov.b32 ta, %1;\n\tmov.b64 ad, %4;\n\tmov.b64 bd, %6;\n\t"
      "setp.ge.s32 q, k, %10;\n\t@q bra.uni CHP_END%=;\n\t"
      "CHP_LOOP%=:\n\t"
      "setp.ne.b32 p, k, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bd, %8, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%3], ad, bd, %9, p;\n\t"
      "add.u32 ta, ta, %2;\n\tadd.u64 ad, ad, %5;\n\tadd.u64 bd, bd, %7;\n\tadd.s32 k, k, 1;\n\t"
      "setp.lt.s32 q, k, %10;\n\t@q bra.uni CHP_LOOP%=;\n\t"
      "CHP_END%=:\n\t}" ::"r"(d1),
      "r"(a1), "r"(a1_step), "r"(d2), "l"(a2), "l"(a2_step), "l"(b0), "l"(b_step), "r"(idesc1), "r"(idesc2), "r"(n)
      : "memory");
}

// Straight-line MMA runs: the step loop of the chains above costs ~15 SASS
// instructions per MMA (loop counter, vector-predicate branch, re-election),
// which at N=16 is longer than the MMA itself when the issuing warp shares its
// scheduler with busy warps.  These issue 4 steps per asm block (one
// elect.sync, then add + mma per step), and the C++ wrappers below cover any
// step count with 4-step blocks plus single steps.  accumulate = (k > 0 || acc).
#define FRNN_MMA_HEAD(ACC)                                  \
  ".reg .pred e, p, t;\n\t"                                  \
  "elect.sync _|e, 0xffffffff;\n\t"                          \
  "setp.ne.b32 p, " ACC ", 0;\n\tsetp.eq.b32 t, " ACC ", " ACC ";\n\t"
// operands: %0 d, %1 A (tmem address), %2 B desc, %3 B step, %4 idesc, %5 acc
__device__ __forceinline__ void mma4_ts(uint32_t d, uint32_t ta, uint64_t bd, uint64_t bk, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t" FRNN_MMA_HEAD("%5")
      ".reg .b32 a;\n\t.reg .b64 b;\n\tmov.b32 a, %1;\n\tmov.b64 b, %2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, p;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t}" ::"r"(d),
      "r"(ta), "l"(bd), "l"(bk), "r"(idesc), "r"(acc)
      : "memory");
}
// 8 TS steps (operands as mma4_ts).
__device__ __forceinline__ void mma8_ts(uint32_t d, uint32_t ta, uint64_t bd, uint64_t bk, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t" FRNN_MMA_HEAD("%5")
      ".reg .b32 a;\n\t.reg .b64 b;\n\tmov.b32 a, %1;\n\tmov.b64 b, %2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, p;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "}" ::"r"(d),
      "r"(ta), "l"(bd), "l"(bk), "r"(idesc), "r"(acc)
      : "memory");
}
// 3 TS steps (a K=48 block: the single-gate backward at UPC=48).
__device__ __forceinline__ void mma3_ts(uint32_t d, uint32_t ta, uint64_t bd, uint64_t bk, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t" FRNN_MMA_HEAD("%5")
      ".reg .b32 a;\n\t.reg .b64 b;\n\tmov.b32 a, %1;\n\tmov.b64 b, %2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, p;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "}" ::"r"(d),
      "r"(ta), "l"(bd), "l"(bk), "r"(idesc), "r"(acc)
      : "memory");
}
// operands: %0 d, %1 A (tmem address), %2 B desc, %3 idesc, %4 acc
__device__ __forceinline__ void mma1_ts(uint32_t d, uint32_t ta, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t" FRNN_MMA_HEAD("%4")
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(ta), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}
// operands: %0 d, %1 A desc, %2 A step, %3 B desc, %4 B step, %5 idesc, %6 acc
__device__ __forceinline__ void mma4_ss(uint32_t d, uint64_t ad, uint64_t ak, uint64_t bd, uint64_t bk,
                                        uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t" FRNN_MMA_HEAD("%6")
      ".reg .b64 a, b;\n\tmov.b64 a, %1;\n\tmov.b64 b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, p;\n\t"
      "add.u64 a, a, %2;\n\tadd.u64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n\t"
      "add.u64 a, a, %2;\n\tadd.u64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n\t"
      "add.u64 a, a, %2;\n\tadd.u64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n\t}" ::"r"(d),
      "l"(ad), "l"(ak), "l"(bd), "l"(bk), "r"(idesc), "r"(acc)
      : "memory");
}
// operands: %0 d, %1 A desc, %2 B desc, %3 idesc, %4 acc
__device__ __forceinline__ void mma1_ss(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t" FRNN_MMA_HEAD("%4")
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}
// Interleaved TS (M=128, into d1) + SS (into d2) pairs sharing B, 4 steps.
// operands: %0 d1, %1 A1 tmem, %2 d2, %3 A2 desc, %4 A2 step, %5 B desc, %6 B step, %7 idesc1, %8 idesc2, %9 acc
__device__ __forceinline__ void mma4_ts_ss(uint32_t d1, uint32_t ta, uint32_t d2, uint64_t ad, uint64_t ak,
                                           uint64_t bd, uint64_t bk, uint32_t id1, uint32_t id2, uint32_t acc) {
  asm volatile(
      "{\n\t" FRNN_MMA_HEAD("%9")
      ".reg .b32 x;\n\t.reg .b64 a, b;\n\tmov.b32 x, %1;\n\tmov.b64 a, %3;\n\tmov.b64 b, %5;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, p;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t}" ::"r"(d1),
      "r"(ta), "r"(d2), "l"(ad), "l"(ak), "l"(bd), "l"(bk), "r"(id1), "r"(id2), "r"(acc)
      : "memory");
}
// 8 steps of the interleaved pair (same operands as mma4_ts_ss).
__device__ __forceinline__ void mma8_ts_ss(uint32_t d1, uint32_t ta, uint32_t d2, uint64_t ad, uint64_t ak,
                                           uint64_t bd, uint64_t bk, uint32_t id1, uint32_t id2, uint32_t acc) {
  asm volatile(
      "{\n\t" FRNN_MMA_HEAD("%9")
      ".reg .b32 x;\n\t.reg .b64 a, b;\n\tmov.b32 x, %1;\n\tmov.b64 a, %3;\n\tmov.b64 b, %5;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, p;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "}" ::"r"(d1),
      "r"(ta), "r"(d2), "l"(ad), "l"(ak), "l"(bd), "l"(bk), "r"(id1), "r"(id2), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma1_ts_ss(uint32_t d1, uint32_t ta, uint32_t d2, uint64_t ad, uint64_t bd,
                                           uint32_t id1, uint32_t id2, uint32_t acc) {
  asm volatile(
      "{\n\t" FRNN_MMA_HEAD("%7")
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], %3, %4, %6, p;\n\t}" ::"r"(d1),
      "r"(ta), "r"(d2), "l"(ad), "l"(bd), "r"(id1), "r"(id2), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_run_ts_ss(uint32_t d1, uint32_t a1, uint32_t d2, uint64_t a2, uint64_t a2_step,
                                              uint64_t b0, uint64_t b_step, uint32_t id1, uint32_t id2, int n,
                                              bool acc0 = false) {
  int k = 0;
  for (; k + 8 <= n; k += 8)
    mma8_ts_ss(d1, a1 + 8u * k, d2, a2 + (uint64_t)k * a2_step, a2_step, b0 + (uint64_t)k * b_step, b_step, id1,
               id2, k > 0 || acc0);
  for (; k + 4 <= n; k += 4)
    mma4_ts_ss(d1, a1 + 8u * k, d2, a2 + (uint64_t)k * a2_step, a2_step, b0 + (uint64_t)k * b_step, b_step, id1,
               id2, k > 0 || acc0);
  for (; k < n; ++k)
    mma1_ts_ss(d1, a1 + 8u * k, d2, a2 + (uint64_t)k * a2_step, b0 + (uint64_t)k * b_step, id1, id2,
               k > 0 || acc0);
}
// Whole warp, one PTX loop on uniform registers (no per-MMA elect waterfall).
// Interleaves n1 TMEM-A steps  D1 (+)= A_tmem(ta + 8i) . B(b1 + i*bk)
// with        n2 SMEM-A steps  D2 (+)= A_smem(a2 + i*a2k) . B(b2 + i*bk);
// accumulate = (i > 0) || acc1 (resp. acc2); idesc for the TMEM-A, idesc_s for the SMEM-A MMAs.
__device__ __forceinline__ void mma_chain_ksplit(uint32_t d1, uint32_t ta, uint64_t b1, int n1, uint32_t acc1,
                                                 uint32_t d2, uint64_t a2, uint64_t a2k, uint64_t b2, int n2,
                                                 uint32_t acc2, uint64_t bk, uint32_t idesc, uint32_t idesc_s) {
  asm volatile(
      "{\n\t.reg .pred e, q, r, s, g, h, p1, p2, z1, z2;\n\t.reg .b32 k, ta, n;\n\t.reg .b64 bb1, aa2, bb2;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b32 k, 0;\n\tmov.b32 ta, %1;\n\tmov.b64 bb1, %2;\n\tmov.b64 aa2, %6;\n\tmov.b64 bb2, %8;\n\t"
      "max.s32 n, %3, %9;\n\tsetp.ne.b32 z1, %4, 0;\n\tsetp.ne.b32 z2, %10, 0;\n\t"
      "setp.ge.s32 q, k, n;\n\t@q bra.uni KS_END%=;\n\t"
      "KS_LOOP%=:\n\t"
      "setp.lt.s32 r, k, %3;\n\tsetp.lt.s32 s, k, %9;\n\tand.pred g, e, r;\n\tand.pred h, e, s;\n\t"
      "setp.ne.or.b32 p1, k, 0, z1;\n\tsetp.ne.or.b32 p2, k, 0, z2;\n\t"
      "@g tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bb1, %12, p1;\n\t"
      "@h tcgen05.mma.cta_group::1.kind::f16 [%5], aa2, bb2, %13, p2;\n\t"
      "add.u32 ta, ta, 8;\n\tadd.u64 bb1, bb1, %11;\n\tadd.u64 aa2, aa2, %7;\n\tadd.u64 bb2, bb2, %11;\n\t"
      "add.s32 k, k, 1;\n\tsetp.lt.s32 q, k, n;\n\t@q bra.uni KS_LOOP%=;\n\t"
      "KS_END%=:\n\t}" ::"r"(d1),
      "r"(ta), "l"(b1), "r"(n1), "r"(acc1), "r"(d2), "l"(a2), "l"(a2k), "l"(b2), "r"(n2), "r"(acc2), "l"(bk),
      "r"(idesc), "r"(idesc_s)
      : "memory");
}
// 12-step blocks: a whole K=192 backward block (UPC=48, 4-gate cells) per asm.
__device__ __forceinline__ void mma12_ts_ss(uint32_t d1, uint32_t ta, uint32_t d2, uint64_t ad, uint64_t ak,
                                            uint64_t bd, uint64_t bk, uint32_t id1, uint32_t id2, uint32_t acc) {
  asm volatile(
      "{\n\t" FRNN_MMA_HEAD("%9")
      ".reg .b32 x;\n\t.reg .b64 a, b;\n\tmov.b32 x, %1;\n\tmov.b64 a, %3;\n\tmov.b64 b, %5;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, p;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "add.u32 x, x, 8;\n\tadd.u64 a, a, %4;\n\tadd.u64 b, b, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %7, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%2], a, b, %8, t;\n\t"
      "}" ::"r"(d1),
      "r"(ta), "r"(d2), "l"(ad), "l"(ak), "l"(bd), "l"(bk), "r"(id1), "r"(id2), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma12_ts(uint32_t d, uint32_t ta, uint64_t bd, uint64_t bk, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t" FRNN_MMA_HEAD("%5")
      ".reg .b32 a;\n\t.reg .b64 b;\n\tmov.b32 a, %1;\n\tmov.b64 b, %2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, p;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "add.u32 a, a, 8;\n\tadd.u64 b, b, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %4, t;\n\t"
      "}" ::"r"(d),
      "r"(ta), "l"(bd), "l"(bk), "r"(idesc), "r"(acc)
      : "memory");
}
// Whole warp.  D[d] (+)= sum_k A(a0 + k*a_step) . B(b0 + k*b_step), k < n.
// acc0: accumulate onto D from the first step too (a K range continuing a sum).
__device__ __forceinline__ void mma_run_ts(uint32_t d, uint32_t a0, uint32_t a_step, uint64_t b0, uint64_t b_step,
                                           uint32_t idesc, int n, bool acc0 = false) {
  int k = 0;
  if (a_step == 8 && n == 3) {
    mma3_ts(d, a0, b0, b_step, idesc, acc0);
    return;
  }
  if (a_step == 8) {
    for (; k + 8 <= n; k += 8) mma8_ts(d, a0 + 8u * k, b0 + (uint64_t)k * b_step, b_step, idesc, k > 0 || acc0);
    for (; k + 4 <= n; k += 4) mma4_ts(d, a0 + 8u * k, b0 + (uint64_t)k * b_step, b_step, idesc, k > 0 || acc0);
  }
  for (; k < n; ++k) mma1_ts(d, a0 + a_step * k, b0 + (uint64_t)k * b_step, idesc, k > 0 || acc0);
}
__device__ __forceinline__ void mma_run_ss(uint32_t d, uint64_t a0, uint64_t a_step, uint64_t b0, uint64_t b_step,
                                           uint32_t idesc, int n) {
  int k = 0;
  for (; k + 4 <= n; k += 4)
    mma4_ss(d, a0 + (uint64_t)k * a_step, a_step, b0 + (uint64_t)k * b_step, b_step, idesc, k > 0);
  for (; k < n; ++k) mma1_ss(d, a0 + (uint64_t)k * a_step, b0 + (uint64_t)k * b_step, idesc, k > 0);
}

// K-outer / block-inner issue over several independent accumulators, so that
// consecutive MMAs never target the same D (no accumulate-dependency stalls):
//   for k < nk:  for i < nts: D[d0 + i*dstep] (+)= A_tmem[ta0 + i*tblk + 8k] . B(k)
//                for i < nss: D[d0 + (nts+i)*dstep] (+)= A_smem[sa0 + i*sblk + k*sk] . B(k)
// with B(k) = bd0 + k*bk and accumulate = (k > 0).  Whole warp; elect.sync issues.
__device__ __forceinline__ void mma_kloop_multi(uint32_t d0, uint32_t dstep, uint32_t ta0, uint32_t tblk, int nts,
                                                uint64_t sa0, uint64_t sblk, uint64_t sk, int nss, uint64_t bd0,
                                                uint64_t bk, uint32_t idesc, int nk) {
  asm volatile(
      "{\n\t.reg .pred e, p, q;\n\t.reg .b32 k, i, d, ta, tk;\n\t.reg .b64 bd, sa, sak;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b32 k, 0;\n\tmov.b64 bd, %9;\n\tmov.b32 tk, %2;\n\tmov.b64 sak, %5;\n\t"
      "setp.ge.s32 q, k, %12;\n\t@q bra.uni MK_END%=;\n\t"
      "MK_K%=:\n\t"
      "setp.ne.b32 p, k, 0;\n\t"
      "mov.b32 d, %0;\n\tmov.b32 ta, tk;\n\tmov.b32 i, 0;\n\t"
      "setp.ge.s32 q, i, %4;\n\t@q bra.uni MK_TSE%=;\n\t"
      "MK_TS%=:\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [d], [ta], bd, %11, p;\n\t"
      "add.u32 d, d, %1;\n\tadd.u32 ta, ta, %3;\n\tadd.s32 i, i, 1;\n\t"
      "setp.lt.s32 q, i, %4;\n\t@q bra.uni MK_TS%=;\n\t"
      "MK_TSE%=:\n\t"
      "mov.b64 sa, sak;\n\tmov.b32 i, 0;\n\t"
      "setp.ge.s32 q, i, %8;\n\t@q bra.uni MK_SSE%=;\n\t"
      "MK_SS%=:\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [d], sa, bd, %11, p;\n\t"
      "add.u32 d, d, %1;\n\tadd.u64 sa, sa, %6;\n\tadd.s32 i, i, 1;\n\t"
      "setp.lt.s32 q, i, %8;\n\t@q bra.uni MK_SS%=;\n\t"
      "MK_SSE%=:\n\t"
      "add.u32 tk, tk, 8;\n\tadd.u64 sak, sak, %7;\n\tadd.u64 bd, bd, %10;\n\tadd.s32 k, k, 1;\n\t"
      "setp.lt.s32 q, k, %12;\n\t@q bra.uni MK_K%=;\n\t"
      "MK_END%=:\n\t}" ::"r"(d0),
      "r"(dstep), "r"(ta0), "r"(tblk), "r"(nts), "l"(sa0), "l"(sblk), "l"(sk), "r"(nss), "l"(bd0), "l"(bk),
      "r"(idesc), "r"(nk)
      : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05.mma complete.
__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(mbar))
      : "memory");
}

// ------------------------------------------------------------- mbarrier ---
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns();
__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(phase)
      : "memory");
  return ok != 0;
}
// Blocking probe: the thread may be suspended (up to `ns`) until the phase
// completes instead of re-polling -- waiting warps stop competing for issue
// slots with the warps doing the step's work.
__device__ __forceinline__ bool mbar_try_sleep(uint32_t a, uint32_t phase, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(phase), "r"(ns)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_cluster_sleep(uint32_t a, uint32_t phase, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2, %3;\n\tselp.b32 %0, "
      "1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(phase), "r"(ns)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_cluster(uint32_t a, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, "
      "1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(phase)
      : "memory");
  return ok != 0;
}
// try_wait suspends in hardware; after ~4 s without completion the kernel
// traps (a protocol bug must not hang the GPU).
// Non-blocking probes (test_wait never suspends the thread).
__device__ __forceinline__ bool mbar_test(uint32_t a, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_test_cluster(uint32_t a, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 "
      "%0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(phase)
      : "memory");
  return ok != 0;
}
#ifdef FRNN_TRYWAIT  // A/B build: suspend in try_wait instead of spinning on test_wait
constexpr bool g_spin_wait = false;
#else
constexpr bool g_spin_wait = true;
#endif
// Waits are on the per-step critical path: spin with test_wait (a suspended
// try_wait wakes up late, ~0.2-0.5 us); after ~4 s without completion the
// kernel traps (a protocol bug must not hang the GPU).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try(a, phase)) return;
  const uint64_t t0 = globaltimer_ns();
  uint32_t n = 0;
  while (!(g_spin_wait ? mbar_test(a, phase) : mbar_try_sleep(a, phase, 1000000u)))
    if ((++n & 1023u) == 0 && globaltimer_ns() - t0 > 4000000000ull) __trap();
}
// Waits for threads that are NOT on the issue path (the MMA-completion waits of
// the drain / cell warps): mode 1 = mbarrier.try_wait without a time hint (the
// hardware suspends the thread until the phase completes or a system-dependent
// timeout, instead of hammering shared memory with test_wait probes while the
// tensor core streams its operands from SMEM); mode 0 = the test_wait spin.
__device__ __forceinline__ void mbar_wait_idle(uint64_t* bar, uint32_t phase, int mode) {
  if (mode == 0) {
    mbar_wait(bar, phase);
    return;
  }
  const uint32_t a = smem_u32(bar);
  const uint64_t t0 = globaltimer_ns();
  uint32_t n = 0;
  while (!mbar_try(a, phase))
    if ((++n & 1023u) == 0 && globaltimer_ns() - t0 > 4000000000ull) __trap();
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// Generic-proxy smem writes -> visible to the async proxy (tensor core / TMA).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 1-D bulk copy global -> shared, completion on an mbarrier (TMA engine).
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------- gpu-scope step flags ---
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin on a gpu-scope step counter.  A peer that never arrives (a bug, or a
// grid that is not co-resident) traps after ~4 s instead of hanging the GPU.
__device__ __forceinline__ void spin_until_geq(const uint32_t* p, uint32_t target) {
  uint64_t t0 = 0;
  uint32_t n = 0;
  while (ld_acquire(p) < target) {
    if ((++n & 4095u) == 0) {
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 4000000000ull) __trap();
    }
  }
}

// Spin with relaxed loads (no L1 invalidate per probe), then one acquire.
__device__ __forceinline__ void spin_until_geq_relaxed(const uint32_t* p, uint32_t target) {
  uint64_t t0 = 0;
  uint32_t n = 0, v;
  for (;;) {
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    if (v >= target) break;
    if ((++n & 4095u) == 0) {
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 4000000000ull) __trap();
    }
  }
  (void)ld_acquire(p);
}

// L2-only 16-byte load (data written by other SMs during this launch).
__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_cg_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_cg_f4(const void* p) {
  float4 r;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// ------------------------------------------------------------- clusters ---
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
// Full cluster barrier (all threads of all CTAs), release/acquire at cluster scope.
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Address of the same shared-memory location in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ bool mbar_test_relaxed_cluster(uint32_t a, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.relaxed.cluster.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 "
      "%0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void fence_acquire_cluster() { asm volatile("fence.acquire.cluster;" ::: "memory"); }
// Wait on a local mbarrier whose arrivals/transactions come from other CTAs.
// An acquire.cluster probe compiles to PHASECHK + CCTL.IVALL (an L1 invalidate)
// on EVERY poll, which stalls the waiting warps' in-flight loads and those of
// the warps beside them; the spin uses relaxed probes and acquires once
// (fence.acquire.cluster) after the phase is observed complete.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
#ifdef FRNN_ACQ_SPIN  // A/B build: acquire on every probe (round-1 protocol)
  if (mbar_try_cluster(a, phase)) return;
  const uint64_t t0 = globaltimer_ns();
  uint32_t n = 0;
  while (!(g_spin_wait ? mbar_test_cluster(a, phase) : mbar_try_cluster_sleep(a, phase, 1000000u)))
    if ((++n & 1023u) == 0 && globaltimer_ns() - t0 > 4000000000ull) __trap();
#else
  if (!mbar_test_relaxed_cluster(a, phase)) {
    const uint64_t t0 = globaltimer_ns();
    uint32_t n = 0;
    while (!mbar_test_relaxed_cluster(a, phase))
      if ((++n & 1023u) == 0 && globaltimer_ns() - t0 > 4000000000ull) __trap();
  }
  fence_acquire_cluster();
#endif
}
// Arrive (count 1) on the mbarrier at cluster-shared address `remote`.
__device__ __forceinline__ void mbar_arrive_remote(uint32_t remote) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// Generic-proxy global writes -> visible to the async proxy (TMA reads).
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// TMA bulk load global -> the same smem offset in every CTA of ctaMask,
// complete_tx on each destination's mbarrier at the same offset.
__device__ __forceinline__ void bulk_g2s_multicast(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar,
                                                   uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

// ------------------------------------------------------- TMA (tensor maps) ---
// L2 policy: keep (R is re-read every step of the alternating path).
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d(void* smem, const void* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* smem, const void* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_hint(void* smem, const void* map, int c0, int c1, int c2, int c3,
                                                 uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
      "{%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* smem, const void* map, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* smem, const void* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// TMA stores (smem -> global, bulk-group completion; out-of-bounds box rows are clipped).
__device__ __forceinline__ void tma_store_3d(const void* map, int c0, int c1, int c2, const void* smem) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(smem))
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const void* map, int c0, int c1, int c2, int c3, const void* smem) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(map),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(smem))
               : "memory");
}
__device__ __forceinline__ void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Wait until at most N committed bulk groups still READ their shared-memory source.
template <int N>
__device__ __forceinline__ void bulk_wait_group_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// Wait until at most N committed bulk groups are incomplete (writes performed).
template <int N>
__device__ __forceinline__ void bulk_wait_group() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// Ampere-style asynchronous global -> shared copies (per thread, no registers).
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p) : "memory");
}
__device__ __forceinline__ void prefetch_tensormap(const void* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// 128B-swizzled operand descriptors (tiles written by TMA with SWIZZLE_128B).
// K-major: rows of 64 bf16 (128 B), 8-row groups 1 KB apart; +16 K = +32 B.
__device__ __forceinline__ uint64_t sdesc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// MN-major: [64 k rows][64 mn] 8 KB boxes; LBO = stride between 64-wide MN
// chunks, SBO = 8 K-rows (1 KB); +16 K = +2 KB.
__device__ __forceinline__ uint64_t sdesc_mn_sw128_chunk(uint32_t saddr, uint32_t chunk_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((chunk_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// ------------------------------------------- programmatic dependent launch ---
// Let the next kernel in the stream start its prologue (it still waits for
// this grid's memory in griddep_wait before touching dependent data).
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Wait until the preceding grid has completed and its writes are visible.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// 16-byte push into another CTA's shared memory (shared::cluster address),
// completing 16 bytes on that CTA's mbarrier (shared::cluster address).
__device__ __forceinline__ void st_async_v4(uint32_t dst, float a, float b, float c, float d, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(dst),
               "f"(a), "f"(b), "f"(c), "f"(d), "r"(mbar)
               : "memory");
}

__device__ __forceinline__ void st_async_b32(uint32_t dst, float a, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(dst),
               "r"(__float_as_uint(a)), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v4_b32(uint32_t dst, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                                uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(dst),
               "r"(a), "r"(b), "r"(c), "r"(d), "r"(mbar)
               : "memory");
}

// DSMEM load of a float from CTA `rank` at the same smem offset.
__device__ __forceinline__ float ld_dsmem_f32(const void* local, uint32_t rank) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(mapa_shared(smem_u32(local), rank)) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

}  // namespace frnn::sm100
