// oracle/ref_csp_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" harness around the UNMODIFIED reference ConstrINT core and tiling
// planner (/root/reference/proj/core/src/csp/*.cpp, src/plan/planner.cpp,
// src/hw/gpu_spec.cpp -- compiled in place by oracle/Makefile into
// oracle/_ref/libref_csp.so, never copied).  It lets tests/test_csp.py pin
// the repo's own solver (paper_2412_07752_b200/csrc/csp.cpp) against the
// reference: the same problems, in the text form of include/flashrnn_csp.h,
// must give the same first solution.
#include <cstdint>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "rnnkit/csp/solver.hpp"
#include "rnnkit/plan/planner.hpp"

using namespace rnnkit;

namespace {

int put(const std::string& s, char* out, size_t cap) {
  if (!out || s.size() + 1 > cap) return -2;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}

csp::CspProblem parse(const std::string& text) {
  csp::CspProblem p;
  std::istringstream in(text);
  std::string line;
  while (std::getline(in, line)) {
    std::istringstream ls(line);
    std::string tag;
    if (!(ls >> tag) || tag[0] == '#') continue;
    if (tag == "v") {
      std::string id, kind, form;
      ls >> id >> kind >> form;
      csp::Domain d;
      if (form == "r") {
        csp::Int lo, hi;
        ls >> lo >> hi;
        d = csp::Domain::range(lo, hi);
      } else if (form == "s") {
        csp::Int lo, hi, st;
        ls >> lo >> hi >> st;
        d = csp::Domain::strided(lo, hi, st);
      } else {
        std::vector<csp::Int> v;
        csp::Int x;
        while (ls >> x) v.push_back(x);
        d = csp::Domain::of(v);
      }
      p.add_variable(id, d,
                     kind == "C" ? csp::VarKind::Constant
                                 : kind == "R" ? csp::VarKind::Resolution : csp::VarKind::Intermediate);
    } else if (tag == "n") {
      std::string op;
      int a, b = 0;
      ls >> op >> a;
      if (op == "v") p.leaf(a);
      else {
        ls >> b;
        p.node(op == "+" ? csp::ExprOp::Add : csp::ExprOp::Mul, a, b);
      }
    } else if (tag == "c") {
      std::string rel;
      int a, b;
      ls >> rel >> a >> b;
      p.add_constraint(rel == "=" ? csp::Relation::Equal
                                  : rel == "<" ? csp::Relation::LessEqual : csp::Relation::Divides,
                       a, b);
    } else if (tag == "h") {
      int v;
      std::string pref;
      ls >> v >> pref;
      p.heuristic().order.push_back(v);
      p.heuristic().value_preference[v] = pref == "L" ? csp::Prefer::Largest : csp::Prefer::Smallest;
    }
  }
  return p;
}

std::string format(const csp::CspProblem& p) {
  std::ostringstream s;
  for (const auto& v : p.variables()) {
    s << "v " << v.id << ' '
      << (v.kind == csp::VarKind::Constant ? 'C' : v.kind == csp::VarKind::Resolution ? 'R' : 'I');
    const auto& d = v.domain;
    bool prog = d.size() == 1 || d.stride() > 1 || d.max() - d.min() + 1 == d.size();
    if (prog && d.stride() > 1) s << " s " << d.min() << ' ' << d.max() << ' ' << d.stride();
    else if (prog) s << " r " << d.min() << ' ' << d.max();
    else {
      s << " e";
      for (csp::Int x : d.values()) s << ' ' << x;
    }
    s << '\n';
  }
  for (const auto& n : p.nodes()) {
    if (n.op == csp::ExprOp::Var) s << "n v " << n.var << '\n';
    else s << "n " << (n.op == csp::ExprOp::Add ? '+' : '*') << ' ' << n.lhs << ' ' << n.rhs << '\n';
  }
  for (const auto& c : p.constraints())
    s << "c " << (c.relation == csp::Relation::Equal ? '=' : c.relation == csp::Relation::LessEqual ? '<' : '|') << ' '
      << c.lhs << ' ' << c.rhs << '\n';
  for (int v : p.heuristic().order)
    s << "h " << v << ' ' << (p.heuristic().preference_of(v) == csp::Prefer::Largest ? 'L' : 'S') << '\n';
  return s.str();
}

}  // namespace

extern "C" {

// 1: solution written as id=value lines; 0: infeasible; <0: error.
int ref_csp_solve(const char* text, char* out, size_t cap, int64_t* nodes) {
  try {
    csp::SolverStats st;
    auto sol = csp::solve(parse(text), {}, &st);
    if (nodes) *nodes = st.nodes;
    if (!sol) return 0;
    std::string s;
    for (const auto& [id, v] : sol->assignment) s += id + "=" + std::to_string(v) + "\n";
    return put(s, out, cap) == 0 ? 1 : -2;
  } catch (const std::exception&) {
    return -1;
  }
}

// Number of solutions by the reference brute force (or <0 on error).
int64_t ref_csp_brute_count(const char* text, int64_t cap) {
  try {
    return (int64_t)csp::brute_force_solve(parse(text), cap).size();
  } catch (const std::exception&) {
    return -1;
  }
}

// The reference planner's CSP (plan::build_csp, planner.cpp:100-231) for a
// preset GPU, in the text form.  pass 0 fwd / 1 bwd; budget < 0 -> register file.
int ref_build_csp(const char* gpu, int ns, int ng, int dh, int nh, int batch, const char* dtype, int pass,
                  int64_t budget, char* out, size_t cap) {
  try {
    hw::GpuSpec g = hw::preset(gpu);
    plan::RnnShape s;
    s.num_states = ns;
    s.num_gates = ng;
    s.head_dim = dh;
    s.num_heads = nh;
    s.batch = batch;
    s.dtype = hw::dtype(dtype);
    auto p = plan::build_csp(s, g, pass ? plan::Pass::Backward : plan::Pass::Forward,
                             budget < 0 ? g.register_file_per_sm_bytes : budget);
    return put(format(p), out, cap);
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
