// tools/frnn.cpp -- GPU-backed command-line front end: the
// reference CLI's subcommands (proj/tools/main.cpp:239-362) on the B200 engine,
// with a small built-in option parser instead of CLI11.
//
//   frnn plan            --variant V --head-dim D --heads H --batch B [--seq T] [--pass forward|backward|both]
//   frnn feasible-heads  --variant V [--min 16 --max 1024 --step 16 --heads 1 --batch 16 --pass both]
//   frnn solve-csp       <problem.txt>          (text form of include/flashrnn_csp.h)
//   frnn gradcheck       --variant V [--t 8 --dh 16 --heads 2 --batch 4 --seeds 1 --h 1e-2 --floor 0.1 --tol 1e-2]
//   frnn precision-drift --variant V [--t 512 --dh 768 --heads 1 --batch 1]
//   frnn train-parity    --variant V [--dh 16 --heads 1 --steps N --batch 64 --train-len-max 40
//                         --warmup W --eval-every E --eval-sequences S --lrs a,b --seeds 1,2]
//   common: --seed S, --json, --out FILE
//
// Exit codes as main.cpp:4-5: 0 success, 1 infeasible / tolerance failure, 2 usage or input error.
//
// gradcheck runs central finite differences through the GPU forward in fp32
// mode (the reference does it in double, gradcheck.cpp:18-75).  fp32 rounding
// noise in the loss (~1e-6 absolute over the final states) divided by 2h sets
// the resolution, so h defaults to 1e-2 and the relative-error floor to 0.1
// (|a-b| / max(|a|, |b|, floor), gradcheck.cpp:11-14); the backward itself is
// pinned against the f64 oracle to 1e-5 normwise by tests/test_gpu_parity.py.
// precision-drift compares the GPU bf16 forward with the GPU fp32 forward of
// the same inputs (engine.cpp:45-71 uses the double engine as the
// high-precision side; fp32 is within 1e-6 of it).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "flashrnn.h"
#include "flashrnn/engine.hpp"
#include "flashrnn/parity.hpp"
#include "flashrnn/random_init.hpp"
#include "flashrnn_csp.h"

namespace {

constexpr int kOk = 0, kFail = 1, kUsage = 2;
namespace rnn = flashrnn::rnn;

struct Args {
  std::string cmd;
  std::vector<std::string> pos;
  std::map<std::string, std::string> kv;
  bool flag(const std::string& k) const { return kv.count(k) != 0; }
  std::string str(const std::string& k, const std::string& d) const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
  long long num(const std::string& k, long long d) const { return flag(k) ? std::stoll(kv.at(k)) : d; }
  double real(const std::string& k, double d) const { return flag(k) ? std::stod(kv.at(k)) : d; }
};

Args parse(int argc, char** argv) {
  Args a;
  for (int i = 1; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) == 0) {
      const std::string key = s.substr(2);
      if (key == "json") {
        a.kv[key] = "1";
      } else {
        if (i + 1 >= argc) throw std::invalid_argument("missing value for --" + key);
        a.kv[key] = argv[++i];
      }
    } else if (a.cmd.empty()) {
      a.cmd = s;
    } else {
      a.pos.push_back(s);
    }
  }
  if (a.cmd.empty()) throw std::invalid_argument("missing subcommand");
  return a;
}

void emit(const Args& a, const std::string& text) {
  const std::string out = a.str("out", "");
  if (out.empty()) {
    std::cout << text;
    if (!text.empty() && text.back() != '\n') std::cout << '\n';
    return;
  }
  std::ofstream f(out);
  if (!f) throw std::invalid_argument("cannot open output file: " + out);
  f << text;
}

rnn::Variant variant_of(const Args& a) {
  auto v = rnn::variant_from_name(a.str("variant", "lstm"));
  if (!v) throw std::invalid_argument("unknown variant (elman|lstm|gru|slstm)");
  return *v;
}

frnn_cell cell_c(rnn::Variant v) {
  frnn_cell c{};
  frnn_cell_spec(static_cast<int32_t>(v), &c);
  return c;
}

// ------------------------------------------------------------------ plan --
int cmd_plan(const Args& a) {
  const frnn_cell c = cell_c(variant_of(a));
  const frnn_shape sh{(int32_t)a.num("seq", 1024), (int32_t)a.num("batch", 16), (int32_t)a.num("heads", 1),
                      (int32_t)a.num("head-dim", 768)};
  const std::string ds = a.str("dtype", "bf16"), pass = a.str("pass", "both");
  if (ds != "bf16" && ds != "fp32") throw std::invalid_argument("--dtype must be bf16 or fp32");  // exit 2
  if (pass != "both" && pass != "forward" && pass != "backward")
    throw std::invalid_argument("--pass must be forward, backward or both");
  const int dtype = ds == "fp32" ? FRNN_F32 : FRNN_BF16;
  std::string out = "{";
  bool ok = true;
  for (int p : {0, 1}) {
    if ((pass == "forward" && p == 1) || (pass == "backward" && p == 0)) continue;
    char buf[4096];
    const int rc = frnn_plan_json(&c, sh, dtype, p, nullptr, buf, sizeof buf);
    out += std::string(out.size() > 1 ? ",\n" : "\n") + (p ? "\"backward\": " : "\"forward\": ");
    if (rc == FRNN_OK) {
      out += buf;
    } else {
      ok = false;
      out += std::string("{\"status\": \"infeasible\", \"why\": \"") + frnn_last_error() + "\"}";
    }
  }
  emit(a, out + "\n}\n");
  return ok ? kOk : kFail;
}

int cmd_feasible_heads(const Args& a) {
  const frnn_cell c = cell_c(variant_of(a));
  const int lo = (int)a.num("min", 16), hi = (int)a.num("max", 1024), st = (int)a.num("step", 16);
  frnn_options o{0, FRNN_ALGO_FUSED};  // R resident on-chip (the paper's "max fused head dim")
  const std::string pass = a.str("pass", "both");  // forward | backward | both
  if (pass != "forward" && pass != "backward" && pass != "both")
    throw std::invalid_argument("--pass must be forward, backward or both");
  std::ostringstream os;
  for (int dh = lo; dh <= hi; dh += st) {
    const frnn_shape sh{1024, (int32_t)a.num("batch", 16), (int32_t)a.num("heads", 1), dh};
    frnn_plan_info f{}, b{};
    const bool fw = pass != "backward" ? frnn_plan(&c, sh, FRNN_BF16, 0, &o, &f) == FRNN_OK : true;
    const bool bw = pass != "forward" ? frnn_plan(&c, sh, FRNN_BF16, 1, &o, &b) == FRNN_OK : true;
    if (fw && bw) os << dh << "\n";
  }
  emit(a, os.str());
  return kOk;
}

int cmd_solve_csp(const Args& a) {
  if (a.pos.empty()) throw std::invalid_argument("solve-csp needs a problem file");
  std::ifstream f(a.pos[0]);
  if (!f) throw std::invalid_argument("cannot open problem file: " + a.pos[0]);
  std::stringstream ss;
  ss << f.rdbuf();
  std::vector<char> out(1 << 20);
  int64_t stats[3] = {0, 0, 0};
  const int rc = frnn_csp_solve(ss.str().c_str(), out.data(), out.size(), stats);
  if (rc == FRNN_EINVAL_ARG) throw std::invalid_argument("malformed problem");
  emit(a, rc == FRNN_OK ? std::string(out.data()) : "infeasible\n");
  return rc == FRNN_OK ? kOk : kFail;
}

// ------------------------------------------------------------- gradcheck --
// gradcheck.cpp:18-75 on the GPU: loss = sum w * states[T], w ~ N(0,1).
double loss_of(const rnn::CellSpec& cell, const rnn::Params<float>& p, const rnn::SequenceBatch<float>& sb,
               const std::vector<double>& w) {
  const auto tr = rnn::forward(cell, p, sb);
  const std::size_t n = w.size(), off = tr.states.size() - n;
  double l = 0;
  for (std::size_t i = 0; i < n; ++i) l += w[i] * tr.states[off + i];
  return l;
}

int cmd_gradcheck(const Args& a) {
  const auto v = variant_of(a);
  const auto cell = rnn::cell_spec(v);
  const int T = (int)a.num("t", 8), dh = (int)a.num("dh", 16), nh = (int)a.num("heads", 2),
            B = (int)a.num("batch", 4), seeds = (int)a.num("seeds", 1);
  const double h = a.real("h", 1e-2), floor = a.real("floor", 0.1), tol = a.real("tol", 1e-2);
  double worst = 0;
  std::ostringstream os;
  os << "variant seed  d_inputs      d_bias        d_R           d_init\n";
  for (int k = 0; k < seeds; ++k) {
    const std::uint64_t seed = (std::uint64_t)a.num("seed", 0) + k;
    rnn::Rng rng(seed * 7919 + 13);
    const auto pd = rnn::random_params(cell, nh, dh, rng);
    const auto sd = rnn::random_batch(cell, T, B, nh, dh, rng);
    std::vector<double> w((std::size_t)cell.num_states * B * nh * dh);
    for (auto& x : w) x = rng.normal();
    auto p = flashrnn::tasks::detail::cast_params<float>(pd);
    auto sb = rnn::SequenceBatch<float>::zeros(T, B, cell.num_gates, cell.num_states, nh * dh);
    for (std::size_t i = 0; i < sb.inputs.size(); ++i) sb.inputs[i] = (float)sd.inputs[i];
    for (std::size_t i = 0; i < sb.init_states.size(); ++i) sb.init_states[i] = (float)sd.init_states[i];
    const auto tr = rnn::forward(cell, p, sb);
    std::vector<float> dsf(w.begin(), w.end());
    const auto g = rnn::backward(cell, p, sb, tr, dsf);
    auto check = [&](std::vector<float>& x, const std::vector<float>& analytic, const std::vector<bool>* skip) {
      double m = 0;
      for (std::size_t i = 0; i < x.size(); ++i) {
        if (skip && (*skip)[i]) continue;
        const float x0 = x[i];
        x[i] = x0 + (float)h;
        const double lp = loss_of(cell, p, sb, w);
        x[i] = x0 - (float)h;
        const double lm = loss_of(cell, p, sb, w);
        x[i] = x0;
        const double fd = (lp - lm) / (2 * h), an = analytic[i];
        m = std::max(m, std::abs(fd - an) / std::max({std::abs(fd), std::abs(an), floor}));
      }
      return m;
    };
    // inputs of gates without input wiring carry no gradient (engine.hpp:311-316)
    std::vector<bool> skip_x(sb.inputs.size(), false);
    for (int t = 0; t < T; ++t)
      for (int b = 0; b < B; ++b)
        for (int j = 0; j < cell.num_gates; ++j)
          for (int e = 0; e < nh * dh; ++e) skip_x[sb.x_index(t, b, j, e)] = !cell.gate_uses_input[j];
    const double ex = check(sb.inputs, g.d_inputs, &skip_x);
    const double eb = check(p.bias, g.d_bias, nullptr);
    std::vector<bool> skip_r(p.recurrent.size(), false);
    for (int hd = 0; hd < nh; ++hd)
      for (int j = 0; j < cell.num_gates; ++j)
        for (int r = 0; r < dh; ++r)
          for (int c = 0; c < dh; ++c) skip_r[p.r_index(hd, j, r, c)] = !cell.gate_uses_recurrent[j];
    const double er = check(p.recurrent, g.d_recurrent, &skip_r);
    const double es = check(sb.init_states, g.d_init_states, nullptr);
    worst = std::max({worst, ex, eb, er, es});
    char buf[200];
    std::snprintf(buf, sizeof buf, "%-7s %4llu %.3e    %.3e    %.3e    %.3e\n", a.str("variant", "lstm").c_str(),
                  (unsigned long long)seed, ex, eb, er, es);
    os << buf;
  }
  os << "max relative error: " << worst << " (tolerance " << tol << ", fp32 GPU, h " << h << ", floor " << floor
     << ")\n";
  emit(a, os.str());
  return worst < tol ? kOk : kFail;
}

// ------------------------------------------------------- precision drift --
int cmd_precision_drift(const Args& a) {
  const auto cell = rnn::cell_spec(variant_of(a));
  const int T = (int)a.num("t", 512), dh = (int)a.num("dh", 768), nh = (int)a.num("heads", 1),
            B = (int)a.num("batch", 1);
  rnn::Rng rng((std::uint64_t)a.num("seed", 0));
  const auto pd = rnn::random_params(cell, nh, dh, rng);
  const auto sd = rnn::random_batch(cell, T, B, nh, dh, rng);
  auto hi_p = flashrnn::tasks::detail::cast_params<float>(pd);
  auto lo_p = flashrnn::tasks::detail::cast_params<rnn::BFloat16>(pd);
  auto hi_b = rnn::SequenceBatch<float>::zeros(T, B, cell.num_gates, cell.num_states, nh * dh);
  auto lo_b = rnn::SequenceBatch<rnn::BFloat16>::zeros(T, B, cell.num_gates, cell.num_states, nh * dh);
  for (std::size_t i = 0; i < sd.inputs.size(); ++i) {
    lo_b.inputs[i] = rnn::BFloat16(sd.inputs[i]);
    hi_b.inputs[i] = (float)lo_b.inputs[i];  // the same (bf16-representable) inputs on both sides
  }
  for (std::size_t i = 0; i < sd.init_states.size(); ++i) {
    lo_b.init_states[i] = rnn::BFloat16(sd.init_states[i]);
    hi_b.init_states[i] = (float)lo_b.init_states[i];
  }
  for (std::size_t i = 0; i < pd.recurrent.size(); ++i) hi_p.recurrent[i] = (float)lo_p.recurrent[i];
  for (std::size_t i = 0; i < pd.bias.size(); ++i) hi_p.bias[i] = (float)lo_p.bias[i];
  const auto hi = rnn::forward(cell, hi_p, hi_b);
  const auto lo = rnn::forward(cell, lo_p, lo_b);
  std::ostringstream os;
  os << "step,p50,p90,p100\n";  // engine.cpp:104-113 drift_to_csv columns
  std::vector<double> err((std::size_t)B * nh * dh);
  for (int t = 1; t <= T; ++t) {
    std::size_t k = 0;
    for (int b = 0; b < B; ++b)
      for (int e = 0; e < nh * dh; ++e, ++k)
        err[k] = std::abs((double)(float)lo.states[lo.s_index(t, 0, b, e)] - hi.states[hi.s_index(t, 0, b, e)]);
    std::sort(err.begin(), err.end());
    auto rank = [&](double pct) {  // nearest rank (engine.cpp:38-43)
      const std::size_t n = err.size(), r = (std::size_t)std::max(1.0, std::ceil(pct / 100.0 * n));
      return err[std::min(r, n) - 1];
    };
    os << t << "," << rank(50) << "," << rank(90) << "," << rank(100) << "\n";
  }
  emit(a, os.str());
  return kOk;
}

// ---------------------------------------------------------- train-parity --
std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  for (std::string tok; std::getline(ss, tok, ',');)
    if (!tok.empty()) out.push_back(tok);
  return out;
}

int cmd_train_parity(const Args& a) {
  namespace T = flashrnn::tasks;
  T::ParityConfig cfg;
  cfg.steps = (int)a.num("steps", cfg.steps);
  cfg.batch_size = (int)a.num("batch", cfg.batch_size);
  cfg.train_len_max = (int)a.num("train-len-max", cfg.train_len_max);
  cfg.warmup_steps = (int)a.num("warmup", cfg.warmup_steps);
  cfg.eval_every = (int)a.num("eval-every", cfg.eval_every);
  cfg.eval_sequences = (int)a.num("eval-sequences", cfg.eval_sequences);
  cfg.eval_len_min = (int)a.num("eval-len-min", cfg.eval_len_min);
  cfg.eval_len_max = (int)a.num("eval-len-max", cfg.eval_len_max);
  const int dh = (int)a.num("dh", 16), nh = (int)a.num("heads", 1);
  std::ostringstream os;
  os << "{\n  \"config\": {\"variant\": \"" << a.str("variant", "lstm") << "\", \"head_dim\": " << dh
     << ", \"num_heads\": " << nh << ", \"steps\": " << cfg.steps << ", \"batch_size\": " << cfg.batch_size
     << ", \"train_len_max\": " << cfg.train_len_max << ", \"engine\": \"B200 fp32\"},\n  \"runs\": [";
  double best_acc = -1, best_lr = 0;
  bool first = true;
  for (const auto& lr_s : split(a.str("lrs", "1e-2,1e-3"))) {
    double acc_sum = 0;
    int n = 0;
    for (const auto& seed_s : split(a.str("seeds", "1"))) {
      const double lr = std::stod(lr_s);
      const auto r = T::train_parity_run<float>(variant_of(a), dh, nh, cfg, lr, std::stoull(seed_s));
      os << (first ? "\n" : ",\n") << "    {\"lr\": " << lr << ", \"seed\": " << seed_s << ", \"steps_run\": "
         << r.steps_run << ", \"diverged\": " << (r.diverged ? "true" : "false")
         << ", \"final_extrapolation_accuracy\": " << r.final_accuracy << ", \"last_loss\": "
         << (r.losses.empty() ? 0.0 : r.losses.back()) << "}";
      first = false;
      acc_sum += r.final_accuracy;
      ++n;
    }
    if (n && acc_sum / n > best_acc) {
      best_acc = acc_sum / n;
      best_lr = std::stod(lr_s);
    }
  }
  os << "\n  ],\n  \"best_lr\": " << best_lr << ",\n  \"best_extrapolation_accuracy\": " << best_acc << "\n}\n";
  emit(a, os.str());
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.cmd == "plan") return cmd_plan(a);
    if (a.cmd == "feasible-heads") return cmd_feasible_heads(a);
    if (a.cmd == "solve-csp") return cmd_solve_csp(a);
    if (a.cmd == "gradcheck") return cmd_gradcheck(a);
    if (a.cmd == "precision-drift") return cmd_precision_drift(a);
    if (a.cmd == "train-parity") return cmd_train_parity(a);
    throw std::invalid_argument("unknown subcommand " + a.cmd +
                                " (plan|feasible-heads|solve-csp|gradcheck|precision-drift|train-parity)");
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kUsage;
  } catch (const std::exception& e) {
    std::cerr << "internal error: " << e.what() << "\n";
    return kUsage;
  }
}
