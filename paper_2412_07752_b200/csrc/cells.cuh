// cells.cuh -- device-side cell functors (Elman / LSTM / GRU / sLSTM).
//
// Restates rnnkit's pointwise maps on the device:
//   forward:  cell.hpp:65-99   (pointwise_forward)
//   backward: cell.hpp:108-201 (pointwise_jacobians) contracted with the state
//             gradient exactly as engine.hpp:275-284 does:
//             dg[j] = sum_i J.d_gate[i][j] * ds[i],  dsp[k] = sum_i J.d_prev[i][k] * ds[i]
// Numerics follow scalar.hpp:58-76: sigma(x) = 1/(1+e^-x), log-sigma split at 0
// with log1p, max_(a,b) = a > b ? a : b, and the sLSTM tie rule of cell.hpp:153
// (ties go to the forget branch in the Jacobian).
//
// Math<false> uses IEEE-accurate libdevice functions (fp32 parity mode, rel 1e-5);
// Math<true> uses the MUFU approximations (bf16 mode, whose tolerance is 2e-2).
#pragma once
#include <cuda_runtime.h>

namespace frnn {

enum Variant { kElman = 0, kLstm = 1, kGru = 2, kSlstm = 3 };

// Raw MUFU approximations with flush-to-zero: no denormal range fix-ups on the
// pointwise critical path (bf16 mode only).
__device__ __forceinline__ float mufu_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float mufu_lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float mufu_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <bool FAST>
struct Math {
  static __device__ __forceinline__ float ex(float x) { return FAST ? mufu_ex2(x * 1.44269504088896341f) : expf(x); }
  static __device__ __forceinline__ float th(float x) {
    if (FAST) {
      float y;
      asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
      return y;
    }
    return tanhf(x);
  }
  static __device__ __forceinline__ float l1p(float x) {
    return FAST ? mufu_lg2(1.0f + x) * 0.693147180559945309f : log1pf(x);
  }
  // bf16 mode: sigma(x) = 0.5 + 0.5 tanh(x/2) -- one MUFU op instead of ex2 + rcp
  // (the pointwise phases are MUFU-throughput bound: 384 threads x 2 elements)
  static __device__ __forceinline__ float sig(float x) {
    if (FAST) return fmaf(0.5f, th(0.5f * x), 0.5f);
    return 1.0f / (1.0f + expf(-x));
  }
  // scalar.hpp:64-70: x >= 0 ? -log1p(e^-x) : x - log1p(e^x).  bf16 mode evaluates
  // the same split branch-free as min(x, 0) - log1p(e^-|x|) (a divergent branch
  // would run both sides' MUFU chains back to back).
  static __device__ __forceinline__ float logsig(float x) {
    if (FAST) return fminf(x, 0.f) - l1p(ex(-fabsf(x)));
    return x >= 0.f ? -l1p(ex(-x)) : x - l1p(ex(x));
  }
  static __device__ __forceinline__ float rcp(float x) { return FAST ? mufu_rcp(x) : 1.0f / x; }
};

// Compile-time cell traits.  NGP = gate rows per hidden unit in the tensor-core
// tiles (all NG gates, padded to a power of two).
//
// Split backward (bf16 cluster kernels): coef<M>(prev, g, k) evaluates every
// transcendental of the Jacobian (cell.hpp:108-201) from the trace alone into
// NK coefficients, and apply(k, ds, dg, dsp) contracts them with the state
// gradient (engine.hpp:275-284) in a few FMAs.  coef does not depend on ds,
// so the kernel forms it for step t-1 while step t's MMAs run; apply is the
// only cell work left between the partial exchange and the next MMA.  The
// contraction is the chain rule through the cell's forward map, algebraically
// equal to J^T ds (reassociated: bf16 mode only; the fp32 paths keep bwd).
template <int V>
struct Cell;

template <>
struct Cell<kElman> {
  static constexpr int NS = 1, NG = 1, NGP = 1;
  static constexpr int NGK = 1;  // backward K rows per unit (gates with R); kgate: their gate index
  static __host__ __device__ constexpr int kgate(int q) { return q; }
  static constexpr bool rec(int) { return true; }
  static constexpr bool inp(int) { return true; }
  template <class M>
  static __device__ __forceinline__ void fwd(const float* p, const float* g, float* n) {
    n[0] = M::th(g[0]);  // cell.hpp:69-72
  }
  template <class M>
  static __device__ __forceinline__ void bwd(const float* p, const float* g, const float* ds,
                                             float* dg, float* dsp) {
    float t = M::th(g[0]);
    dg[0] = (1.f - t * t) * ds[0];  // cell.hpp:114-117
    dsp[0] = 0.f;
  }
  static constexpr int NK = 1;
  template <class M>
  static __device__ __forceinline__ void coef(const float* p, const float* g, float* k) {
    const float t = M::th(g[0]);
    k[0] = 1.f - t * t;
  }
  static __device__ __forceinline__ void apply(const float* k, const float* ds, float* dg, float* dsp) {
    dg[0] = k[0] * ds[0];
    dsp[0] = 0.f;
  }
};

template <>
struct Cell<kLstm> {
  static constexpr int NS = 2, NG = 4, NGP = 4;
  static constexpr int NGK = 4;
  static __host__ __device__ constexpr int kgate(int q) { return q; }
  static constexpr bool rec(int) { return true; }
  static constexpr bool inp(int) { return true; }
  template <class M>
  static __device__ __forceinline__ void fwd(const float* p, const float* g, float* n) {
    // cell.hpp:73-78
    float c = M::sig(g[1]) * p[1] + M::sig(g[2]) * M::th(g[0]);
    n[0] = M::sig(g[3]) * M::th(c);
    n[1] = c;
  }
  template <class M>
  static __device__ __forceinline__ void bwd(const float* p, const float* g, const float* ds,
                                             float* dg, float* dsp) {
    // cell.hpp:119-135
    float sf = M::sig(g[1]), si = M::sig(g[2]), so = M::sig(g[3]);
    float tz = M::th(g[0]);
    float c = sf * p[1] + si * tz;
    float tc = M::th(c);
    float dtc = 1.f - tc * tc;
    float J10 = si * (1.f - tz * tz);
    float J11 = sf * (1.f - sf) * p[1];
    float J12 = si * (1.f - si) * tz;
    float P11 = sf;
    float J00 = so * dtc * J10, J01 = so * dtc * J11, J02 = so * dtc * J12;
    float J03 = so * (1.f - so) * tc;
    float P01 = so * dtc * sf;
    dg[0] = J00 * ds[0] + J10 * ds[1];
    dg[1] = J01 * ds[0] + J11 * ds[1];
    dg[2] = J02 * ds[0] + J12 * ds[1];
    dg[3] = J03 * ds[0];
    dsp[0] = 0.f;
    dsp[1] = P01 * ds[0] + P11 * ds[1];
  }
  // k = {so*(1-tanh^2 c), dc/dz, dc/df, dc/di, dh/do, sf}: dc_tot = ds_c + k0*ds_h
  // carries the whole c path (J0j = so*dtc*J1j, P01 = so*dtc*sf)
  static constexpr int NK = 6;
  template <class M>
  static __device__ __forceinline__ void coef(const float* p, const float* g, float* k) {
    const float sf = M::sig(g[1]), si = M::sig(g[2]), so = M::sig(g[3]);
    const float tz = M::th(g[0]);
    const float tc = M::th(sf * p[1] + si * tz);
    k[0] = so * (1.f - tc * tc);
    k[1] = si * (1.f - tz * tz);
    k[2] = sf * (1.f - sf) * p[1];
    k[3] = si * (1.f - si) * tz;
    k[4] = so * (1.f - so) * tc;
    k[5] = sf;
  }
  static __device__ __forceinline__ void apply(const float* k, const float* ds, float* dg, float* dsp) {
    const float dc = fmaf(k[0], ds[0], ds[1]);
    dg[0] = k[1] * dc;
    dg[1] = k[2] * dc;
    dg[2] = k[3] * dc;
    dg[3] = k[4] * ds[0];
    dsp[0] = 0.f;
    dsp[1] = k[5] * dc;
  }
};

template <>
struct Cell<kGru> {
  static constexpr int NS = 1, NG = 4, NGP = 4;
  // the n gate (j = 2) has no R (cell.hpp:43): the backward's R^T.dg contraction
  // skips its rows -- K = 3 rows per unit instead of the padded 4
  static constexpr int NGK = 3;
  static __host__ __device__ constexpr int kgate(int q) { return q < 2 ? q : 3; }
  static constexpr bool rec(int j) { return j != 2; }  // n skips R   (cell.hpp:43)
  static constexpr bool inp(int j) { return j != 3; }  // g skips x   (cell.hpp:44)
  template <class M>
  static __device__ __forceinline__ void fwd(const float* p, const float* g, float* n) {
    // cell.hpp:79-84
    float sz = M::sig(g[0]);
    float inner = g[2] + M::sig(g[1]) * M::th(g[3]);
    n[0] = sz * p[0] + (1.f - sz) * M::th(inner);
  }
  template <class M>
  static __device__ __forceinline__ void bwd(const float* p, const float* g, const float* ds,
                                             float* dg, float* dsp) {
    // cell.hpp:136-149
    float sz = M::sig(g[0]), sr = M::sig(g[1]);
    float tg = M::th(g[3]);
    float u = g[2] + sr * tg;
    float tu = M::th(u);
    float dtu = 1.f - tu * tu;
    float omz = 1.f - sz;
    dg[0] = sz * (1.f - sz) * (p[0] - tu) * ds[0];
    dg[1] = omz * dtu * sr * (1.f - sr) * tg * ds[0];
    dg[2] = omz * dtu * ds[0];
    dg[3] = omz * dtu * sr * (1.f - tg * tg) * ds[0];
    dsp[0] = sz * ds[0];
  }
  static constexpr int NK = 5;  // every gradient is a multiple of ds_h
  template <class M>
  static __device__ __forceinline__ void coef(const float* p, const float* g, float* k) {
    const float sz = M::sig(g[0]), sr = M::sig(g[1]);
    const float tg = M::th(g[3]);
    const float tu = M::th(g[2] + sr * tg);
    const float od = (1.f - sz) * (1.f - tu * tu);
    k[0] = sz * (1.f - sz) * (p[0] - tu);
    k[1] = od * sr * (1.f - sr) * tg;
    k[2] = od;
    k[3] = od * sr * (1.f - tg * tg);
    k[4] = sz;
  }
  static __device__ __forceinline__ void apply(const float* k, const float* ds, float* dg, float* dsp) {
#pragma unroll
    for (int j = 0; j < 4; ++j) dg[j] = k[j] * ds[0];
    dsp[0] = k[4] * ds[0];
  }
};

template <>
struct Cell<kSlstm> {
  static constexpr int NS = 4, NG = 4, NGP = 4;
  static constexpr int NGK = 4;
  static __host__ __device__ constexpr int kgate(int q) { return q; }
  static constexpr bool rec(int) { return true; }
  static constexpr bool inp(int) { return true; }
  template <class M>
  static __device__ __forceinline__ void fwd(const float* p, const float* g, float* n) {
    // cell.hpp:85-97
    float a = M::logsig(g[1]) + p[3];
    const bool fa = a > g[2];
    float m = fa ? a : g[2];
    // one of exp(a - m), exp(i - m) is exp(0) = 1 exactly: a single MUFU exp
    const float e = M::ex(fa ? g[2] - a : a - g[2]);
    float fexp = fa ? 1.f : e;
    float iexp = fa ? e : 1.f;
    float c = fexp * p[1] + iexp * M::th(g[0]);
    float nn = fexp * p[2] + iexp;
    n[0] = M::sig(g[3]) * (c * M::rcp(nn));
    n[1] = c;
    n[2] = nn;
    n[3] = m;
  }
  template <class M>
  static __device__ __forceinline__ void bwd(const float* p, const float* g, const float* ds,
                                             float* dg, float* dsp) {
    // cell.hpp:150-198
    float sf = M::sig(g[1]), so = M::sig(g[3]);
    float a = M::logsig(g[1]) + p[3];
    bool use_a = !(a < g[2]);  // ties -> forget branch (cell.hpp:153)
    float m = use_a ? a : g[2];
    const float e = M::ex(use_a ? g[2] - a : a - g[2]);  // the other exponent is exp(0) = 1
    float fexp = use_a ? 1.f : e;
    float iexp = use_a ? e : 1.f;
    float tz = M::th(g[0]);
    float c = fexp * p[1] + iexp * tz;
    float n = fexp * p[2] + iexp;
    float da_df = 1.f - sf;
    float dm_df = use_a ? da_df : 0.f;
    float dm_di = use_a ? 0.f : 1.f;
    float dm_dmp = use_a ? 1.f : 0.f;
    float dfexp_df = fexp * (da_df - dm_df);
    float diexp_df = -iexp * dm_df;
    float dfexp_di = -fexp * dm_di;
    float diexp_di = iexp * (1.f - dm_di);
    float dfexp_dmp = fexp * (1.f - dm_dmp);
    float diexp_dmp = -iexp * dm_dmp;
    float J10 = iexp * (1.f - tz * tz);
    float J11 = dfexp_df * p[1] + diexp_df * tz;
    float J12 = dfexp_di * p[1] + diexp_di * tz;
    float P11 = fexp;
    float P13 = dfexp_dmp * p[1] + diexp_dmp * tz;
    float J21 = dfexp_df * p[2] + diexp_df;
    float J22 = dfexp_di * p[2] + diexp_di;
    float P22 = fexp;
    float P23 = dfexp_dmp * p[2] + diexp_dmp;
    float J31 = dm_df, J32 = dm_di, P33 = dm_dmp;
    float inv_n = M::rcp(n);
    float h_over = c * inv_n;
    float J00 = so * J10 * inv_n;                      // J20 = 0
    float J01 = so * (J11 - h_over * J21) * inv_n;
    float J02 = so * (J12 - h_over * J22) * inv_n;
    float J03 = so * (1.f - so) * h_over;               // J13 = J23 = 0
    float P01 = so * P11 * inv_n;                       // P21 = 0
    float P02 = so * (-h_over * P22) * inv_n;           // P12 = 0
    float P03 = so * (P13 - h_over * P23) * inv_n;
    dg[0] = J00 * ds[0] + J10 * ds[1];
    dg[1] = J01 * ds[0] + J11 * ds[1] + J21 * ds[2] + J31 * ds[3];
    dg[2] = J02 * ds[0] + J12 * ds[1] + J22 * ds[2] + J32 * ds[3];
    dg[3] = J03 * ds[0];
    dsp[0] = 0.f;
    dsp[1] = P01 * ds[0] + P11 * ds[1];
    dsp[2] = P02 * ds[0] + P22 * ds[2];
    dsp[3] = P03 * ds[0] + P13 * ds[1] + P23 * ds[2] + P33 * ds[3];
  }
  // Chain rule through h = so*c/n, c = fe*c' + ie*tz, n = fe*n' + ie, fe = e^(a-m),
  // ie = e^(i-m), m = max(a, i) (ties -> a, cell.hpp:153), a = logsig(f) + m':
  // dc = ds_c + ds_h*so/n, dn = ds_n - ds_h*so*c/n^2, dm = ds_m - fe*dfe - ie*die,
  // da = fe*dfe + [a wins]*dm = dm', df = (1-sf)*da, di = ds_m - da.  Equal to
  // the J^T ds of cell.hpp:150-198 (J11 = (1-sf)*P13, J12 = -P13, J01 = (1-sf)*P03 ...).
  // k = {so/n, c/n, c', n', tz, fe, ie, ie*(1-tz^2), [a wins], 1-sf, so*(1-so)*c/n}
  static constexpr int NK = 11;
  template <class M>
  static __device__ __forceinline__ void coef(const float* p, const float* g, float* k) {
    const float sf = M::sig(g[1]), so = M::sig(g[3]);
    const float a = M::logsig(g[1]) + p[3];
    const bool use_a = !(a < g[2]);
    const float e = M::ex(use_a ? g[2] - a : a - g[2]);
    const float fexp = use_a ? 1.f : e, iexp = use_a ? e : 1.f;
    const float tz = M::th(g[0]);
    const float c = fexp * p[1] + iexp * tz;
    const float inv_n = M::rcp(fexp * p[2] + iexp);
    const float hov = c * inv_n;
    k[0] = so * inv_n;
    k[1] = hov;
    k[2] = p[1];
    k[3] = p[2];
    k[4] = tz;
    k[5] = fexp;
    k[6] = iexp;
    k[7] = iexp * (1.f - tz * tz);
    k[8] = use_a ? 1.f : 0.f;
    k[9] = 1.f - sf;
    k[10] = so * (1.f - so) * hov;
  }
  static __device__ __forceinline__ void apply(const float* k, const float* ds, float* dg, float* dsp) {
    const float q = ds[0] * k[0];
    const float dc = ds[1] + q;
    const float dn = fmaf(-q, k[1], ds[2]);
    const float ef = (dc * k[2] + dn * k[3]) * k[5];
    const float ei = (dc * k[4] + dn) * k[6];
    const float dm = ds[3] - ef - ei;
    const float da = fmaf(dm, k[8], ef);
    dg[0] = dc * k[7];
    dg[1] = da * k[9];
    dg[2] = ds[3] - da;
    dg[3] = ds[0] * k[10];
    dsp[0] = 0.f;
    dsp[1] = dc * k[5];
    dsp[2] = dn * k[5];
    dsp[3] = da;
  }
};

}  // namespace frnn
