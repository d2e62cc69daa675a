// shim_test.cpp -- the C++ drop-in (flashrnn/engine.hpp) used exactly like
// rnnkit::rnn::forward/backward, checked against the CPU oracle
// (oracle/liboracle.so, test infrastructure) and for the reference's
// std::invalid_argument behaviour.  Exit code 0 = pass.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "flashrnn/engine.hpp"

extern "C" {
struct orc_cell {
  int variant, num_states, num_gates, uses_rec[4], uses_in[4];
};
orc_cell orc_cell_spec(int v);
void* orc_rng_new(uint64_t seed);
void orc_rng_free(void*);
void orc_random_params(void*, const orc_cell*, int NH, int DH, double rs, double bs, double* R, double* b);
void orc_random_batch(void*, const orc_cell*, int T, int B, int NH, int DH, double is, double ss, double* x, double* s0);
void orc_rng_fill_normal(void*, double scale, size_t n, double* out);
void orc_round_bf16(size_t n, const double* in, double* out);
void orc_forward_f64(const orc_cell*, int T, int B, int NH, int DH, const double* R, const double* b, const double* x,
                     const double* s0, double* states, double* gates);
void orc_backward_f64(const orc_cell*, int T, int B, int NH, int DH, const double* R, const double* st,
                      const double* ga, const double* dsf, int clip, double mag, const double* dh, double* dx,
                      double* db, double* dR, double* ds0);
}

using namespace flashrnn::rnn;

template <class S>
double to_d(S v) {
  return static_cast<double>(v);
}

template <class S>
double normwise(const std::vector<S>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < b.size(); ++i) {
    const double d = to_d(a[i]) - b[i];
    num += d * d;
    den += b[i] * b[i];
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

template <class S>
int run(Variant v, int T, int B, int NH, int DH, double tol, bool bf) {
  const CellSpec cell = cell_spec(v);
  const orc_cell oc = orc_cell_spec(static_cast<int>(v));
  const int NG = cell.num_gates, NS = cell.num_states, D = NH * DH;
  std::vector<double> R((size_t)NH * NG * DH * DH), b((size_t)NG * D), x((size_t)T * B * NG * D),
      s0((size_t)NS * B * D), dsf((size_t)NS * B * D);
  void* rng = orc_rng_new(42 + static_cast<int>(v));
  orc_random_params(rng, &oc, NH, DH, 1.0, 0.1, R.data(), b.data());
  orc_random_batch(rng, &oc, T, B, NH, DH, 1.0, 0.5, x.data(), s0.data());
  orc_rng_fill_normal(rng, 1.0, dsf.size(), dsf.data());
  orc_rng_free(rng);
  if (bf)
    for (auto* vec : {&R, &b, &x, &s0, &dsf}) orc_round_bf16(vec->size(), vec->data(), vec->data());
  auto cast = [](const std::vector<double>& a) {
    std::vector<S> o(a.size());
    for (size_t i = 0; i < a.size(); ++i) o[i] = S(a[i]);
    return o;
  };
  Params<S> p = Params<S>::zeros(NH, DH, NG);
  p.recurrent = cast(R);
  p.bias = cast(b);
  SequenceBatch<S> sb = SequenceBatch<S>::zeros(T, B, NG, NS, D);
  sb.inputs = cast(x);
  sb.init_states = cast(s0);
  ForwardTrace<S> tr = forward(cell, p, sb);                           // engine.hpp:144 signature
  Gradients<S> g = backward(cell, p, sb, tr, cast(dsf), ClipPolicy::value(0.5));  // engine.hpp:222 signature
  std::vector<double> st((size_t)(T + 1) * NS * B * D), ga((size_t)T * NG * B * D);
  orc_forward_f64(&oc, T, B, NH, DH, R.data(), b.data(), x.data(), s0.data(), st.data(), ga.data());
  // backward oracle on the GPU's own trace (rnnkit's backward takes the trace)
  std::vector<double> gst(tr.states.size()), gga(tr.gates.size());
  for (size_t i = 0; i < gst.size(); ++i) gst[i] = to_d(tr.states[i]);
  for (size_t i = 0; i < gga.size(); ++i) gga[i] = to_d(tr.gates[i]);
  std::vector<double> dx(x.size()), db(b.size()), dR(R.size()), ds0(s0.size());
  orc_backward_f64(&oc, T, B, NH, DH, R.data(), gst.data(), gga.data(), dsf.data(), 1, 0.5, nullptr, dx.data(),
                   db.data(), dR.data(), ds0.data());
  const double e[6] = {normwise(tr.states, st), normwise(tr.gates, ga), normwise(g.d_inputs, dx),
                       normwise(g.d_bias, db), normwise(g.d_recurrent, dR), normwise(g.d_init_states, ds0)};
  int bad = 0;
  for (double v_ : e) bad += !(v_ <= tol);
  std::printf("%-6s %s T=%d B=%d NH=%d DH=%d: states %.2e gates %.2e dx %.2e db %.2e dR %.2e ds0 %.2e %s\n",
              cell.name.c_str(), bf ? "bf16" : "f32 ", T, B, NH, DH, e[0], e[1], e[2], e[3], e[4], e[5],
              bad ? "FAIL" : "ok");
  return bad;
}

int expect_invalid(const char* what, void (*fn)()) {
  try {
    fn();
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument as expected (%s): %s\n", what, e.what());
    return 0;
  } catch (const std::exception& e) {
    std::printf("FAIL %s: wrong exception %s\n", what, e.what());
    return 1;
  }
  std::printf("FAIL %s: no exception\n", what);
  return 1;
}

int main() {
  int bad = 0;
  for (Variant v : {Variant::Elman, Variant::Lstm, Variant::Gru, Variant::Slstm}) {
    bad += run<float>(v, 10, 5, 2, 32, 1e-5, false);
    bad += run<BFloat16>(v, 12, 16, 2, 64, 2e-2, true);
  }
  bad += expect_invalid("count mismatch", [] {
    CellSpec c = cell_spec(Variant::Lstm);
    Params<float> p = Params<float>::zeros(1, 8, 4);
    SequenceBatch<float> sb = SequenceBatch<float>::zeros(3, 2, 4, 3, 8);  // wrong state count
    forward(c, p, sb);
  });
  bad += expect_invalid("non-finite input", [] {
    CellSpec c = cell_spec(Variant::Lstm);
    Params<float> p = Params<float>::zeros(1, 8, 4);
    SequenceBatch<float> sb = SequenceBatch<float>::zeros(3, 2, 4, 2, 8);
    sb.inputs[5] = NAN;
    forward(c, p, sb);
  });
  bad += expect_invalid("clip magnitude", [] { ClipPolicy::value(0.0); });
  bad += expect_invalid("terminal gradient size", [] {
    CellSpec c = cell_spec(Variant::Gru);
    Params<float> p = Params<float>::zeros(1, 8, 4);
    SequenceBatch<float> sb = SequenceBatch<float>::zeros(3, 2, 4, 1, 8);
    ForwardTrace<float> tr = forward(c, p, sb);
    backward(c, p, sb, tr, std::vector<float>(3));
  });
  std::printf("SHIM_TEST %s\n", bad ? "FAIL" : "PASS");
  return bad ? 1 : 0;
}
