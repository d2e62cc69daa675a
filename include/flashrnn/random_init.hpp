// flashrnn/random_init.hpp -- the reference's deterministic synthetic inputs
// (rng.hpp:12-50, random_init.hpp:10-40) for callers of the GPU engine:
// std::mt19937_64 (specified bit-exactly by the standard) with an explicit
// Box-Muller transform, Gaussian parameters and inputs, sLSTM normaliser /
// stabiliser initial states.  Header-only.
#pragma once
#include <cmath>
#include <cstdint>
#include <random>

#include "flashrnn/engine.hpp"

namespace flashrnn::rnn {

// rng.hpp:12-50: deterministic stream (std::mt19937_64 is specified bit-exactly
// by the standard; gaussians by an explicit Box-Muller transform).
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : gen_(seed) {}
  std::uint64_t next_u64() { return gen_(); }
  double uniform() { return std::ldexp(static_cast<double>(gen_() >> 11), -53); }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * M_PI * u2;
    spare_ = r * std::sin(th);
    spare_ok_ = true;
    return r * std::cos(th);
  }
  int bit() { return static_cast<int>(gen_() >> 63); }
  std::int64_t uniform_int(std::int64_t lo, std::int64_t hi) {
    return lo + static_cast<std::int64_t>(gen_() % static_cast<std::uint64_t>(hi - lo + 1));
  }

 private:
  std::mt19937_64 gen_;
  bool spare_ok_ = false;
  double spare_ = 0.0;
};

// random_init.hpp:10-18
inline Params<double> random_params(const CellSpec& cell, int num_heads, int head_dim, Rng& rng,
                                    double r_scale = 1.0, double bias_scale = 0.1) {
  Params<double> p = Params<double>::zeros(num_heads, head_dim, cell.num_gates);
  const double rs = r_scale / std::sqrt(static_cast<double>(head_dim));
  for (auto& v : p.recurrent) v = rs * rng.normal();
  for (auto& v : p.bias) v = bias_scale * rng.normal();
  return p;
}

// random_init.hpp:22-40
inline SequenceBatch<double> random_batch(const CellSpec& cell, int seq_len, int batch, int num_heads, int head_dim,
                                          Rng& rng, double input_scale = 1.0, double state_scale = 0.5) {
  auto sb = SequenceBatch<double>::zeros(seq_len, batch, cell.num_gates, cell.num_states, num_heads * head_dim);
  for (auto& v : sb.inputs) v = input_scale * rng.normal();
  for (int i = 0; i < cell.num_states; ++i)
    for (int b = 0; b < batch; ++b)
      for (int e = 0; e < sb.dim; ++e) {
        double v = state_scale * rng.normal();
        if (cell.variant == Variant::Slstm && i == 2) v = 1.0 + 0.1 * std::abs(v);
        if (cell.variant == Variant::Slstm && i == 3) v = 0.0;
        sb.init_states[sb.s_index(i, b, e)] = v;
      }
  return sb;
}

}  // namespace flashrnn::rnn

