// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Thin extern "C" harness around the UNMODIFIED reference engine
// (/root/reference/proj/core/include/rnnkit/rnn/engine.hpp, included in place,
// never copied).  Built by oracle/Makefile into oracle/_ref/libref.so, which is
// git-ignored but travels to the GPU box with the snapshot.  It pins the C
// restatement in oracle/rnn_oracle.c and generates tests/golden/ fixtures; it
// is also the "reference" CPU baseline timed by bench.py --impl reference.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "rnnkit/rnn/engine.hpp"
#include "rnnkit/rnn/gradcheck.hpp"
#include "rnnkit/rnn/random_init.hpp"
#include "rnnkit/rnn/tensor_io.hpp"
#include "rnnkit/tasks/parity.hpp"

using namespace rnnkit::rnn;

namespace {

CellSpec spec(int v) { return cell_spec(static_cast<Variant>(v)); }

template <class S>
Params<S> make_params(const CellSpec& c, int NH, int DH, const S* R, const S* bias) {
  Params<S> p = Params<S>::zeros(NH, DH, c.num_gates);
  std::memcpy(p.recurrent.data(), R, sizeof(S) * p.recurrent.size());
  std::memcpy(p.bias.data(), bias, sizeof(S) * p.bias.size());
  return p;
}

template <class S>
SequenceBatch<S> make_batch(const CellSpec& c, int T, int B, int D, const S* x, const S* s0) {
  SequenceBatch<S> sb = SequenceBatch<S>::zeros(T, B, c.num_gates, c.num_states, D);
  std::memcpy(sb.inputs.data(), x, sizeof(S) * sb.inputs.size());
  std::memcpy(sb.init_states.data(), s0, sizeof(S) * sb.init_states.size());
  return sb;
}

template <class S>
int fwd(int v, int T, int B, int NH, int DH, const S* R, const S* bias, const S* x, const S* s0,
        S* states, S* gates) {
  try {
    CellSpec c = spec(v);
    auto p = make_params<S>(c, NH, DH, R, bias);
    auto sb = make_batch<S>(c, T, B, NH * DH, x, s0);
    ForwardTrace<S> tr = forward(c, p, sb);
    std::memcpy(states, tr.states.data(), sizeof(S) * tr.states.size());
    std::memcpy(gates, tr.gates.data(), sizeof(S) * tr.gates.size());
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

template <class S>
int bwd(int v, int T, int B, int NH, int DH, const S* R, const S* bias, const S* x, const S* s0,
        const S* states, const S* gates, const S* dsf, int clip_mode, double clip_mag,
        const S* d_hidden, S* dx, S* db, S* dR, S* ds0) {
  try {
    CellSpec c = spec(v);
    auto p = make_params<S>(c, NH, DH, R, bias);
    auto sb = make_batch<S>(c, T, B, NH * DH, x, s0);
    const int NS = c.num_states, NG = c.num_gates, D = NH * DH;
    ForwardTrace<S> tr;
    tr.seq_len = T; tr.batch = B; tr.num_states = NS; tr.num_gates = NG; tr.dim = D;
    tr.states.assign(states, states + (size_t)(T + 1) * NS * B * D);
    tr.gates.assign(gates, gates + (size_t)T * NG * B * D);
    std::vector<S> d_final(dsf, dsf + (size_t)NS * B * D);
    ClipPolicy clip = clip_mode == 1 ? ClipPolicy::value(clip_mag)
                      : clip_mode == 2 ? ClipPolicy::zero() : ClipPolicy::off();
    StepGradients<S> extra;
    if (d_hidden) extra.hidden.assign(d_hidden, d_hidden + (size_t)T * B * D);
    Gradients<S> g = backward(c, p, sb, tr, d_final, clip, d_hidden ? &extra : nullptr);
    std::memcpy(dx, g.d_inputs.data(), sizeof(S) * g.d_inputs.size());
    std::memcpy(db, g.d_bias.data(), sizeof(S) * g.d_bias.size());
    std::memcpy(dR, g.d_recurrent.data(), sizeof(S) * g.d_recurrent.size());
    std::memcpy(ds0, g.d_init_states.data(), sizeof(S) * g.d_init_states.size());
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

}  // namespace

extern "C" {

// Reference input generator exactly as gradient_check seeds it
// (gradcheck.cpp:20-27): Rng(seed*7919+13) -> random_params -> random_batch
// -> d_states_final ~ N(0,1).
void ref_generate(int v, int T, int B, int NH, int DH, uint64_t seed, double* R, double* bias,
                  double* x, double* s0, double* dsf) {
  CellSpec c = spec(v);
  Rng rng(seed * 7919 + 13);
  Params<double> p = random_params(c, NH, DH, rng);
  SequenceBatch<double> sb = random_batch(c, T, B, NH, DH, rng);
  std::memcpy(R, p.recurrent.data(), sizeof(double) * p.recurrent.size());
  std::memcpy(bias, p.bias.data(), sizeof(double) * p.bias.size());
  std::memcpy(x, sb.inputs.data(), sizeof(double) * sb.inputs.size());
  std::memcpy(s0, sb.init_states.data(), sizeof(double) * sb.init_states.size());
  size_t n = (size_t)c.num_states * B * NH * DH;
  for (size_t i = 0; i < n; ++i) dsf[i] = rng.normal();
}

int ref_forward_f64(int v, int T, int B, int NH, int DH, const double* R, const double* bias,
                    const double* x, const double* s0, double* states, double* gates) {
  return fwd<double>(v, T, B, NH, DH, R, bias, x, s0, states, gates);
}
int ref_forward_f32(int v, int T, int B, int NH, int DH, const float* R, const float* bias,
                    const float* x, const float* s0, float* states, float* gates) {
  return fwd<float>(v, T, B, NH, DH, R, bias, x, s0, states, gates);
}
int ref_backward_f64(int v, int T, int B, int NH, int DH, const double* R, const double* bias,
                     const double* x, const double* s0, const double* states,
                     const double* gates, const double* dsf, int clip_mode, double clip_mag,
                     const double* d_hidden, double* dx, double* db, double* dR, double* ds0) {
  return bwd<double>(v, T, B, NH, DH, R, bias, x, s0, states, gates, dsf, clip_mode, clip_mag,
                     d_hidden, dx, db, dR, ds0);
}
int ref_backward_f32(int v, int T, int B, int NH, int DH, const float* R, const float* bias,
                     const float* x, const float* s0, const float* states, const float* gates,
                     const float* dsf, int clip_mode, double clip_mag, const float* d_hidden,
                     float* dx, float* db, float* dR, float* ds0) {
  return bwd<float>(v, T, B, NH, DH, R, bias, x, s0, states, gates, dsf, clip_mode, clip_mag,
                    d_hidden, dx, db, dR, ds0);
}

// engine.cpp:75-93
double ref_blockdiag_check(int v, int T, int B, int NH, int DH, const double* R,
                           const double* bias, const double* x, const double* s0) {
  CellSpec c = spec(v);
  auto p = make_params<double>(c, NH, DH, R, bias);
  auto sb = make_batch<double>(c, T, B, NH * DH, x, s0);
  return forward_blockdiag_equivalence_check(c, p, sb);
}

// gradcheck.cpp:18-75 (FD sanity check; fills 4 maxima).
void ref_gradient_check(int v, int T, int DH, int NH, int B, uint64_t seed, double step,
                        double floor, double* out4) {
  GradCheckConfig cfg;
  cfg.variant = static_cast<Variant>(v);
  cfg.seq_len = T; cfg.head_dim = DH; cfg.num_heads = NH; cfg.batch = B; cfg.seed = seed;
  cfg.fd_step = step; cfg.rel_floor = floor;
  GradCheckReport r = gradient_check(cfg);
  out4[0] = r.max_rel_inputs; out4[1] = r.max_rel_bias;
  out4[2] = r.max_rel_recurrent; out4[3] = r.max_rel_init_states;
}

// A complete reference case as an RTN1 file written by the reference's own
// save_tensors (tensor_io.cpp:28-47): generator inputs (seeded as
// ref_generate), the f64 forward trace and the f64 backward (clip off).
int ref_save_case(const char* path, int v, int T, int B, int NH, int DH, uint64_t seed) {
  try {
    CellSpec c = spec(v);
    Rng rng(seed * 7919 + 13);
    Params<double> p = random_params(c, NH, DH, rng);
    SequenceBatch<double> sb = random_batch(c, T, B, NH, DH, rng);
    std::vector<double> dsf((size_t)c.num_states * B * NH * DH);
    for (auto& d : dsf) d = rng.normal();
    ForwardTrace<double> tr = forward(c, p, sb);
    Gradients<double> g = backward(c, p, sb, tr, dsf);
    const uint64_t D = (uint64_t)NH * DH, NS = c.num_states, NG = c.num_gates;
    TensorMap t = params_to_tensors(p);
    t["inputs"] = NamedTensor{{(uint64_t)T, (uint64_t)B, NG, D}, sb.inputs};
    t["init_states"] = NamedTensor{{NS, (uint64_t)B, D}, sb.init_states};
    t["d_states_final"] = NamedTensor{{NS, (uint64_t)B, D}, dsf};
    t["states"] = NamedTensor{{(uint64_t)T + 1, NS, (uint64_t)B, D}, tr.states};
    t["gates"] = NamedTensor{{(uint64_t)T, NG, (uint64_t)B, D}, tr.gates};
    t["d_inputs"] = NamedTensor{{(uint64_t)T, (uint64_t)B, NG, D}, g.d_inputs};
    t["d_bias"] = NamedTensor{{NG, D}, g.d_bias};
    t["d_recurrent"] = NamedTensor{{(uint64_t)NH, NG, (uint64_t)DH, (uint64_t)DH}, g.d_recurrent};
    t["d_init_states"] = NamedTensor{{NS, (uint64_t)B, D}, g.d_init_states};
    save_tensors(path, t);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// The reference parity-task trainer (parity.cpp:142-245), in double on the CPU.
int ref_train_parity(int v, int dh, int nh, int steps, int batch, int len_max, int warmup, double lr, uint64_t seed,
                     int eval_sequences, int eval_len_min, int eval_len_max, double* losses, int* steps_run,
                     double* final_acc) {
  try {
    rnnkit::tasks::ParityConfig cfg;
    cfg.steps = steps;
    cfg.batch_size = batch;
    cfg.train_len_max = len_max;
    cfg.warmup_steps = warmup;
    cfg.eval_every = 0;
    cfg.eval_sequences = eval_sequences;
    cfg.eval_len_min = eval_len_min;
    cfg.eval_len_max = eval_len_max;
    auto run = rnnkit::tasks::train_parity_run(static_cast<Variant>(v), dh, nh, cfg, lr, seed);
    for (size_t i = 0; i < run.losses.size(); ++i) losses[i] = run.losses[i];
    *steps_run = run.steps_run;
    *final_acc = run.final_accuracy;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// Round trip through the reference reader + writer (load_tensors, save_tensors).
int ref_rewrite_tensors(const char* in, const char* out) {
  try {
    save_tensors(out, load_tensors(in));
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
