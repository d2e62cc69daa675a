// e2e_bench.cpp -- end-to-end throughput through the C++ drop-in exactly as an
// rnnkit caller uses it: host std::vectors in, host std::vectors out,
//   tr = flashrnn::rnn::forward(cell, params, batch)            (engine.hpp:144)
//   g  = flashrnn::rnn::backward(cell, params, batch, tr, dsf)  (engine.hpp:222)
// per step, timed on the host wall clock around the two calls (every staging
// conversion, H2D/D2H copy and kernel inside).  Inputs are the reference
// generator's (random_init.hpp:10-40, seed 0), cast to the element type once.
// Prints one JSON line.
//
//   e2e_bench [--variant slstm] [--hidden 768] [--heads 1] [--batch 16] [--seq 1024]
//             [--dtype bf16|f32] [--steps 5] [--warmup 2]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "flashrnn/engine.hpp"
#include "flashrnn/random_init.hpp"

using namespace flashrnn::rnn;

template <class S>
int run(const CellSpec& cell, int T, int B, int NH, int DH, int steps, int warmup, const char* dtype) {
  Rng rng(0);
  const Params<double> pd = random_params(cell, NH, DH, rng);
  const SequenceBatch<double> bd = random_batch(cell, T, B, NH, DH, rng);
  std::vector<double> dsfd((size_t)cell.num_states * B * NH * DH);
  for (auto& v : dsfd) v = rng.normal();
  auto cast = [](const std::vector<double>& a) {
    std::vector<S> o(a.size());
    for (size_t i = 0; i < a.size(); ++i) o[i] = S(a[i]);
    return o;
  };
  Params<S> p = Params<S>::zeros(NH, DH, cell.num_gates);
  p.recurrent = cast(pd.recurrent);
  p.bias = cast(pd.bias);
  SequenceBatch<S> sb = SequenceBatch<S>::zeros(T, B, cell.num_gates, cell.num_states, NH * DH);
  sb.inputs = cast(bd.inputs);
  sb.init_states = cast(bd.init_states);
  const std::vector<S> dsf = cast(dsfd);
  using clk = std::chrono::steady_clock;
  std::vector<double> ms;
  double sum = 0;
  for (int i = 0; i < warmup + steps; ++i) {
    const auto t0 = clk::now();
    ForwardTrace<S> tr = forward(cell, p, sb);
    Gradients<S> g = backward(cell, p, sb, tr, dsf);
    const auto t1 = clk::now();
    if (i >= warmup) {
      ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
      sum += ms.back();
    }
    if (g.d_inputs.size() != sb.inputs.size()) return 1;
  }
  const size_t E = std::is_same_v<S, float> ? 4 : 2, D = (size_t)NH * DH;
  const size_t NG = cell.num_gates, NS = cell.num_states;
  const size_t h2d = E * (2 * p.recurrent.size() + 2 * p.bias.size() + sb.inputs.size() + sb.init_states.size() +
                          dsf.size());
  const size_t d2h = E * ((size_t)(T + 1) * NS * B * D + (size_t)T * NG * B * D + sb.inputs.size() +
                          p.bias.size() + p.recurrent.size() + dsf.size());
  const double per = sum / steps;
  std::printf(
      "{\"metric\": \"fwd+bwd batch*timesteps/s through flashrnn::rnn::forward/backward (host vectors)\", "
      "\"value\": %.3f, \"unit\": \"batch*timesteps/s\", \"ms_per_step\": %.4f, \"steps\": %d, \"warmup\": %d, "
      "\"variant\": \"%s\", \"dtype\": \"%s\", \"T\": %d, \"B\": %d, \"NH\": %d, \"DH\": %d, "
      "\"h2d_bytes_per_step\": %zu, \"d2h_bytes_per_step\": %zu, \"host_threads\": %u}\n",
      1e3 * (double)B * T / per, per, steps, warmup, cell.name.c_str(), dtype, T, B, NH, DH, h2d, d2h,
      std::thread::hardware_concurrency());
  return 0;
}

int main(int argc, char** argv) {
  std::string variant = "slstm", dtype = "bf16";
  int H = 768, NH = 1, B = 16, T = 1024, steps = 5, warmup = 2;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--variant") variant = v;
    else if (k == "--dtype") dtype = v;
    else if (k == "--hidden") H = std::atoi(v.c_str());
    else if (k == "--heads") NH = std::atoi(v.c_str());
    else if (k == "--batch") B = std::atoi(v.c_str());
    else if (k == "--seq") T = std::atoi(v.c_str());
    else if (k == "--steps") steps = std::atoi(v.c_str());
    else if (k == "--warmup") warmup = std::atoi(v.c_str());
    else {
      std::fprintf(stderr, "unknown option %s\n", k.c_str());
      return 2;
    }
  }
  const auto vv = variant_from_name(variant);
  if (!vv || H % NH || steps < 1 || (dtype != "bf16" && dtype != "f32")) {
    std::fprintf(stderr, "usage: e2e_bench [--variant elman|lstm|gru|slstm] [--dtype bf16|f32] ...\n");
    return 2;
  }
  const CellSpec cell = cell_spec(*vv);
  try {
    return dtype == "bf16" ? run<BFloat16>(cell, T, B, NH, H / NH, steps, warmup, "bf16")
                           : run<float>(cell, T, B, NH, H / NH, steps, warmup, "f32");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "e2e_bench: %s\n", e.what());
    return 1;
  }
}
