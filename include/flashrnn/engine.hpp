// flashrnn/engine.hpp -- C++ drop-in for rnnkit's operator API, backed by the
// B200 kernels through the C ABI (flashrnn.h).  Header-only; link with
// -lflashrnn -lcudart.
//
// Same types, members, layouts and signatures as the reference
//   rnnkit::rnn::forward   (/root/reference/proj/core/include/rnnkit/rnn/engine.hpp:143-144)
//   rnnkit::rnn::backward  (engine.hpp:221-225)
// in namespace flashrnn::rnn, so a caller switches engines by changing the
// namespace.  Value semantics: host std::vectors in, host
// std::vectors out; the shim owns the device staging.  Errors: the reference's
// std::invalid_argument cases (engine.hpp:107, :119-134, :231-236) throw
// std::invalid_argument; device/runtime failures throw std::runtime_error.
// Element types: float (fp32 mode, FFMA kernels) and BFloat16 (bf16 mode,
// tcgen05 kernels); double is rejected (there is no CPU fallback).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../flashrnn.h"

namespace flashrnn::rnn {

// ---- cell.hpp:11-53 ----
enum class Variant { Elman, Lstm, Gru, Slstm };

struct CellSpec {
  Variant variant = Variant::Elman;
  std::string name;
  int num_states = 1;
  int num_gates = 1;
  std::array<bool, 4> gate_uses_recurrent{true, true, true, true};
  std::array<bool, 4> gate_uses_input{true, true, true, true};
};

inline CellSpec cell_spec(Variant v) {
  frnn_cell c{};
  frnn_cell_spec(static_cast<int32_t>(v), &c);
  CellSpec s;
  s.variant = v;
  static const char* names[] = {"elman", "lstm", "gru", "slstm"};
  s.name = names[static_cast<int>(v)];
  s.num_states = c.num_states;
  s.num_gates = c.num_gates;
  for (int j = 0; j < 4; ++j) {
    s.gate_uses_recurrent[j] = c.uses_recurrent[j] != 0;
    s.gate_uses_input[j] = c.uses_input[j] != 0;
  }
  return s;
}

inline std::optional<Variant> variant_from_name(const std::string& n) {
  if (n == "elman") return Variant::Elman;
  if (n == "lstm") return Variant::Lstm;
  if (n == "gru") return Variant::Gru;
  if (n == "slstm") return Variant::Slstm;
  return std::nullopt;
}

// ---- scalar.hpp:12-43: bf16 value type (float storage, RNE rounding) ----
struct BFloat16 {
  float v = 0.0f;
  BFloat16() = default;
  explicit BFloat16(double x) : v(round(static_cast<float>(x))) {}
  explicit BFloat16(float x) : v(round(x)) {}
  explicit BFloat16(int x) : v(round(static_cast<float>(x))) {}
  static float round(float x) {
    if (!std::isfinite(x)) return x;
    uint32_t bits;
    std::memcpy(&bits, &x, 4);
    bits += 0x7FFFu + ((bits >> 16) & 1u);
    bits &= 0xFFFF0000u;
    std::memcpy(&x, &bits, 4);
    return x;
  }
  explicit operator double() const { return v; }
  explicit operator float() const { return v; }
  uint16_t bits() const {
    uint32_t b;
    std::memcpy(&b, &v, 4);
    return static_cast<uint16_t>(b >> 16);
  }
  static BFloat16 from_bits(uint16_t h) {
    BFloat16 r;
    uint32_t b = static_cast<uint32_t>(h) << 16;
    std::memcpy(&r.v, &b, 4);
    return r;
  }
};

// ---- engine.hpp:15-111 ----
template <class S>
struct Params {
  int num_heads = 1;
  int head_dim = 0;
  int num_gates = 1;
  std::vector<S> recurrent;  // [head][gate][row][col]
  std::vector<S> bias;       // [gate][dim]
  int dim() const { return num_heads * head_dim; }
  std::size_t r_index(int head, int gate, int row, int col) const {
    return ((static_cast<std::size_t>(head) * num_gates + gate) * head_dim + row) * head_dim + col;
  }
  std::size_t b_index(int gate, int e) const { return static_cast<std::size_t>(gate) * dim() + e; }
  static Params zeros(int num_heads, int head_dim, int num_gates) {
    Params p;
    p.num_heads = num_heads;
    p.head_dim = head_dim;
    p.num_gates = num_gates;
    p.recurrent.assign(static_cast<std::size_t>(num_heads) * num_gates * head_dim * head_dim, S(0));
    p.bias.assign(static_cast<std::size_t>(num_gates) * num_heads * head_dim, S(0));
    return p;
  }
};

template <class S>
struct SequenceBatch {
  int seq_len = 0, batch = 0, num_gates = 1, num_states = 1, dim = 0;
  std::vector<S> inputs;       // [T][batch][gate][dim]
  std::vector<S> init_states;  // [state][batch][dim]
  std::size_t x_index(int t, int b, int gate, int e) const {
    return ((static_cast<std::size_t>(t) * batch + b) * num_gates + gate) * dim + e;
  }
  std::size_t s_index(int state, int b, int e) const {
    return (static_cast<std::size_t>(state) * batch + b) * dim + e;
  }
  static SequenceBatch zeros(int seq_len, int batch, int num_gates, int num_states, int dim) {
    SequenceBatch sb;
    sb.seq_len = seq_len;
    sb.batch = batch;
    sb.num_gates = num_gates;
    sb.num_states = num_states;
    sb.dim = dim;
    sb.inputs.assign(static_cast<std::size_t>(seq_len) * batch * num_gates * dim, S(0));
    sb.init_states.assign(static_cast<std::size_t>(num_states) * batch * dim, S(0));
    return sb;
  }
};

template <class S>
struct ForwardTrace {
  int seq_len = 0, batch = 0, num_states = 1, num_gates = 1, dim = 0;
  std::vector<S> states;  // [T+1][state][batch][dim]
  std::vector<S> gates;   // [T][gate][batch][dim]
  std::size_t s_index(int t, int state, int b, int e) const {
    return ((static_cast<std::size_t>(t) * num_states + state) * batch + b) * dim + e;
  }
  std::size_t g_index(int t, int gate, int b, int e) const {
    return ((static_cast<std::size_t>(t) * num_gates + gate) * batch + b) * dim + e;
  }
};

template <class S>
struct Gradients {
  std::vector<S> d_inputs, d_bias, d_recurrent, d_init_states;
};

struct ClipPolicy {
  enum class Mode { Off, ClipValue, Zero };
  Mode mode = Mode::Off;
  double magnitude = 0.0;
  static ClipPolicy off() { return {Mode::Off, 0.0}; }
  static ClipPolicy value(double m) {
    if (m <= 0) throw std::invalid_argument("clip magnitude must be positive");  // engine.hpp:107
    return {Mode::ClipValue, m};
  }
  static ClipPolicy zero() { return {Mode::Zero, 0.0}; }
};

template <class S>
struct StepGradients {
  std::vector<S> hidden;  // [T][batch][dim]; empty means none
};

namespace detail {

template <class S>
constexpr int32_t dtype_of() {
  static_assert(std::is_same_v<S, float> || std::is_same_v<S, BFloat16>,
                "flashrnn GPU engine supports float and BFloat16 (no fp64, no CPU fallback)");
  return std::is_same_v<S, float> ? FRNN_F32 : FRNN_BF16;
}

[[noreturn]] inline void raise(int rc) {
  const std::string msg = frnn_last_error();
  if (rc == FRNN_EINVAL_SHAPE || rc == FRNN_ENONFINITE || rc == FRNN_EINVAL_ARG) throw std::invalid_argument(msg);
  throw std::runtime_error("flashrnn: " + msg);
}
inline void check(int rc) {
  if (rc != FRNN_OK) raise(rc);
}
inline void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("flashrnn: ") + what + ": " + cudaGetErrorString(e));
}

// Device buffer of element type S (float or bf16 bits).
template <class S>
struct DevBuf {
  void* ptr = nullptr;
  std::size_t n = 0;
  static constexpr std::size_t esz = std::is_same_v<S, float> ? 4 : 2;
  explicit DevBuf(std::size_t count) : n(count) {
    if (n) cuda(cudaMalloc(&ptr, n * esz), "cudaMalloc");
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (ptr) cudaFree(ptr);
  }
  void upload(const std::vector<S>& v) {
    if (v.size() != n) throw std::invalid_argument("tensor storage size mismatch");  // engine.hpp:128
    if (!n) return;
    if constexpr (std::is_same_v<S, float>) {
      cuda(cudaMemcpy(ptr, v.data(), n * 4, cudaMemcpyHostToDevice), "H2D");
    } else {
      std::vector<uint16_t> h(n);
      for (std::size_t i = 0; i < n; ++i) h[i] = v[i].bits();
      cuda(cudaMemcpy(ptr, h.data(), n * 2, cudaMemcpyHostToDevice), "H2D");
    }
  }
  std::vector<S> download() const {
    std::vector<S> v(n);
    if (!n) return v;
    if constexpr (std::is_same_v<S, float>) {
      cuda(cudaMemcpy(v.data(), ptr, n * 4, cudaMemcpyDeviceToHost), "D2H");
    } else {
      std::vector<uint16_t> h(n);
      cuda(cudaMemcpy(h.data(), ptr, n * 2, cudaMemcpyDeviceToHost), "D2H");
      for (std::size_t i = 0; i < n; ++i) v[i] = BFloat16::from_bits(h[i]);
    }
    return v;
  }
};

inline frnn_cell to_c(const CellSpec& c) {
  frnn_cell r{};
  r.variant = static_cast<int32_t>(c.variant);
  r.num_states = c.num_states;
  r.num_gates = c.num_gates;
  for (int j = 0; j < 4; ++j) {
    r.uses_recurrent[j] = c.gate_uses_recurrent[j];
    r.uses_input[j] = c.gate_uses_input[j];
  }
  return r;
}

template <class S>
void check_counts(const CellSpec& cell, const Params<S>& p, const SequenceBatch<S>& sb) {  // engine.hpp:116-122
  if (p.num_gates != cell.num_gates || sb.num_gates != cell.num_gates || sb.num_states != cell.num_states)
    throw std::invalid_argument("cell/params/batch gate or state counts disagree");
  if (sb.dim != p.dim()) throw std::invalid_argument("batch dim != params dim");
}

}  // namespace detail

/// engine.hpp:143-203 on the GPU.
template <class S>
ForwardTrace<S> forward(const CellSpec& cell, const Params<S>& p, const SequenceBatch<S>& sb) {
  detail::check_counts(cell, p, sb);
  const frnn_cell c = detail::to_c(cell);
  const frnn_shape sh{sb.seq_len, sb.batch, p.num_heads, p.head_dim};
  const int32_t dt = detail::dtype_of<S>();
  const int NS = cell.num_states, NG = cell.num_gates, D = sb.dim, T = sb.seq_len, B = sb.batch;
  frnn_options opt{FRNN_FLAG_CHECK_FINITE, FRNN_ALGO_AUTO};  // engine.hpp:146-147
  std::size_t wsb = 0;
  detail::check(frnn_workspace_size(&c, sh, dt, FRNN_PASS_FORWARD, &opt, &wsb));
  detail::DevBuf<S> R(p.recurrent.size()), bias(p.bias.size()), x(sb.inputs.size()), s0(sb.init_states.size()),
      st((std::size_t)(T + 1) * NS * B * D), ga((std::size_t)T * NG * B * D);
  void* ws = nullptr;
  detail::cuda(cudaMalloc(&ws, wsb), "cudaMalloc workspace");
  struct Free {
    void* p;
    ~Free() { cudaFree(p); }
  } fws{ws};
  if (p.recurrent.size() != (std::size_t)p.num_heads * NG * p.head_dim * p.head_dim ||
      p.bias.size() != (std::size_t)NG * p.dim() || sb.inputs.size() != (std::size_t)T * B * NG * D ||
      sb.init_states.size() != (std::size_t)NS * B * D)
    throw std::invalid_argument("tensor storage size mismatch");
  R.upload(p.recurrent);
  bias.upload(p.bias);
  x.upload(sb.inputs);
  s0.upload(sb.init_states);
  detail::check(frnn_forward(&c, sh, dt, R.ptr, bias.ptr, x.ptr, s0.ptr, st.ptr, ga.ptr, ws, wsb, &opt, nullptr));
  detail::cuda(cudaDeviceSynchronize(), "forward");
  ForwardTrace<S> tr;
  tr.seq_len = T;
  tr.batch = B;
  tr.num_states = NS;
  tr.num_gates = NG;
  tr.dim = D;
  tr.states = st.download();
  tr.gates = ga.download();
  return tr;
}

/// engine.hpp:221-339 on the GPU.
template <class S>
Gradients<S> backward(const CellSpec& cell, const Params<S>& p, const SequenceBatch<S>& sb,
                      const ForwardTrace<S>& tr, const std::vector<S>& d_states_final,
                      const ClipPolicy& clip = ClipPolicy::off(), const StepGradients<S>* extra = nullptr) {
  detail::check_counts(cell, p, sb);
  const int NS = cell.num_states, NG = cell.num_gates, D = sb.dim, T = sb.seq_len, B = sb.batch;
  if (tr.seq_len != T || tr.batch != B || tr.dim != D || tr.num_states != NS || tr.num_gates != NG)
    throw std::invalid_argument("trace does not match batch");  // engine.hpp:229-231
  if (d_states_final.size() != (std::size_t)NS * B * D)
    throw std::invalid_argument("terminal state gradient has wrong size");
  const bool has_dh = extra && !extra->hidden.empty();
  if (has_dh && extra->hidden.size() != (std::size_t)T * B * D)
    throw std::invalid_argument("per-step hidden gradients have wrong size");
  const frnn_cell c = detail::to_c(cell);
  const frnn_shape sh{T, B, p.num_heads, p.head_dim};
  const int32_t dt = detail::dtype_of<S>();
  std::size_t wsb = 0;
  detail::check(frnn_workspace_size(&c, sh, dt, FRNN_PASS_BACKWARD, nullptr, &wsb));
  detail::DevBuf<S> R(p.recurrent.size()), bias(p.bias.size()), st(tr.states.size()), ga(tr.gates.size()),
      dsf(d_states_final.size()), dh(has_dh ? extra->hidden.size() : 0), dx(sb.inputs.size()), db(p.bias.size()),
      dR(p.recurrent.size()), ds0(d_states_final.size());
  void* ws = nullptr;
  detail::cuda(cudaMalloc(&ws, wsb), "cudaMalloc workspace");
  struct Free {
    void* p;
    ~Free() { cudaFree(p); }
  } fws{ws};
  R.upload(p.recurrent);
  bias.upload(p.bias);
  st.upload(tr.states);
  ga.upload(tr.gates);
  dsf.upload(d_states_final);
  if (has_dh) dh.upload(extra->hidden);
  const frnn_clip cl{static_cast<int32_t>(clip.mode), clip.magnitude};
  detail::check(frnn_backward(&c, sh, dt, R.ptr, bias.ptr, st.ptr, ga.ptr, dsf.ptr, has_dh ? dh.ptr : nullptr, cl,
                              dx.ptr, db.ptr, dR.ptr, ds0.ptr, ws, wsb, nullptr, nullptr));
  detail::cuda(cudaDeviceSynchronize(), "backward");
  Gradients<S> g;
  g.d_inputs = dx.download();
  g.d_bias = db.download();
  g.d_recurrent = dR.download();
  g.d_init_states = ds0.download();
  return g;
}

}  // namespace flashrnn::rnn
