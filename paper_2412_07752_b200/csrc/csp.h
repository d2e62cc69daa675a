// csp.h -- ConstrINT-style integer constraint solver (host C++), the engine
// behind the B200 tiling planner.
//
// Restates the semantics of the reference's CSP core (SPEC.md csp_core;
// /root/reference/proj/core/include/rnnkit/csp/{domain,problem,propagation,
// solver}.hpp) with its own data structures:
//   * domains are finite sets of positive int64 values, stored either as an
//     arithmetic progression (first, step, count) or as an explicit sorted set
//     (domain.hpp:17-72); progressions intersect by CRT without enumeration;
//   * problems are variables (constant / resolution / intermediate), binary
//     Add/Mul expression trees and Equal / LessEqual / Divides constraints
//     (problem.hpp:13-45); compound terms are flattened onto intermediates
//     (propagation.cpp normalize_problem) with shared sub-terms;
//   * propagation is an AC-3 worklist over parent = x op y bindings and
//     leaf relations, with exact set arithmetic for small domains and
//     lattice hulls otherwise (propagation.cpp revise_binding/revise_relation);
//   * search is depth-first over the resolution variables in heuristic order,
//     values in each variable's preference direction, fixpoint propagation
//     after every assignment (solver.cpp:22-73) -- here with an undo trail
//     instead of whole-store snapshots.
// Propagation is sound (it never removes a value that belongs to a solution),
// so the first solution found is the lexicographically extremal one under the
// heuristic, independent of how strong the propagation is: the same answer
// the reference returns (tests/test_csp.py checks this against the reference
// solver compiled in place).
#pragma once
#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

namespace frnn::csp {

using Int = std::int64_t;
constexpr Int kCap = Int{1} << 62;  // saturation bound (domain.hpp:14)

inline Int sadd(Int a, Int b) {
  Int r;
  return (__builtin_add_overflow(a, b, &r) || r > kCap) ? kCap : r;
}
inline Int smul(Int a, Int b) {
  Int r;
  return (__builtin_mul_overflow(a, b, &r) || r > kCap) ? kCap : r;
}

class Domain {
 public:
  Domain() = default;  // empty
  static Domain single(Int v);
  static Domain span(Int lo, Int hi);              // {lo..hi}
  static Domain grid(Int lo, Int hi, Int step);    // {lo, lo+step, .. <= hi}, values >= 1
  static Domain set(std::vector<Int> values);      // sorted, deduplicated

  bool empty() const { return n_ == 0; }
  Int size() const { return n_; }
  bool is_single() const { return n_ == 1; }
  Int lo() const { return vals_.empty() ? first_ : vals_.front(); }
  Int hi() const { return vals_.empty() ? first_ + step_ * (n_ - 1) : vals_.back(); }
  Int step() const { return vals_.empty() ? step_ : 1; }
  Int at(Int i) const { return vals_.empty() ? first_ + step_ * i : vals_[(size_t)i]; }
  bool has(Int v) const;
  Int lower_index(Int x) const;  // index of the first value >= x (size() if none)
  bool small(Int limit) const { return n_ <= limit; }

  Domain meet(const Domain& o) const;      // intersection
  bool intersects(const Domain& o) const;  // meet(o) non-empty, without building it
  Domain within(Int lo, Int hi) const;     // clamp to [lo, hi]
  Domain multiples(Int m) const;           // values divisible by m
  template <class F>
  Domain where(F keep) const {
    std::vector<Int> out;
    for (Int i = 0; i < n_; ++i)
      if (keep(at(i))) out.push_back(at(i));
    return set(std::move(out));
  }
  bool operator==(const Domain& o) const;
  bool operator!=(const Domain& o) const { return !(*this == o); }
  std::string str() const;

 private:
  Int first_ = 0, step_ = 1, n_ = 0;
  std::vector<Int> vals_;  // non-empty: explicit set
  static Domain prog(Int first, Int step, Int n);
};

enum class Kind { Constant, Resolution, Intermediate };
enum class Op { Leaf, Add, Mul };
enum class Rel { Eq, Le, Div };  // Div: lhs divides rhs
enum class Pref { Smallest, Largest };

struct Var {
  std::string id;
  Domain dom;
  Kind kind;
};
struct Node {
  Op op;
  int var, l, r;
};
struct Con {
  Rel rel;
  int l, r;  // node indices
};

class Problem {
 public:
  int add_var(const std::string& id, Domain d, Kind k = Kind::Resolution);
  int constant(Int v);  // shared singleton constants
  int leaf(int var);
  int add(int l, int r);
  int mul(int l, int r);
  void require(Rel rel, int l, int r);
  void prefer(int var, Pref p);  // appends to the heuristic order

  std::vector<Var> vars;
  std::vector<Node> nodes;
  std::vector<Con> cons;
  std::vector<std::pair<int, Pref>> order;

 private:
  std::map<Int, int> consts_;
};

struct Options {
  Int enum_limit = 4096;    // per-value scans below this domain size
  Int pair_limit = 1 << 16; // exact sum/product sets below this many pairs
  Int divisor_limit = 512;  // divisor enumeration of small parent domains
};

struct Solution {
  std::map<std::string, Int> values;  // resolution variables
  long long nodes = 0, backtracks = 0;
};

// First solution in heuristic order (nullopt: infeasible).  Throws
// std::invalid_argument on malformed problems.
std::optional<Solution> solve(const Problem& p, const Options& o = {});

// Every solution by exhaustive enumeration of the resolution domains with
// direct constraint evaluation (the test oracle; problem must have no
// intermediates).  Throws when the search space exceeds `cap`.
std::vector<std::map<std::string, Int>> brute_force(const Problem& p, Int cap);

// Saturating evaluation of node n under per-variable values.
Int eval(const Problem& p, int n, const std::vector<Int>& values);
bool satisfied(const Problem& p, const std::vector<Int>& values);

// Text form (one item per line; indices refer to declaration order):
//   v <id> <C|R|I> r <lo> <hi> | s <lo> <hi> <step> | e <v1> <v2> ...
//   n v <var> | n + <node> <node> | n * <node> <node>
//   c = <node> <node> | c < <node> <node> (<=) | c | <node> <node> (divides)
//   h <var> <S|L>
Problem parse(const std::string& text);
std::string format(const Problem& p);

}  // namespace frnn::csp
