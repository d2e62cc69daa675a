// csp.cpp -- the ConstrINT-style CSP engine (see csp.h for the contract and
// the reference sections each part restates).
#include "csp.h"

#include <algorithm>
#include <cmath>
#include <deque>
#include <functional>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <tuple>

namespace frnn::csp {

// ================================================================ Domain ===
Domain Domain::prog(Int first, Int step, Int n) {
  Domain d;
  if (n <= 0) return d;
  d.first_ = first;
  d.step_ = n == 1 ? 1 : step;
  d.n_ = n;
  return d;
}

Domain Domain::single(Int v) {
  if (v < 1) throw std::invalid_argument("domain values must be >= 1");
  return prog(v, 1, 1);
}

Domain Domain::span(Int lo, Int hi) { return grid(lo, hi, 1); }

Domain Domain::grid(Int lo, Int hi, Int step) {
  if (step < 1) throw std::invalid_argument("domain step must be >= 1");
  if (lo < 1) lo += (1 - lo + step - 1) / step * step;
  if (lo > hi) return Domain{};
  return prog(lo, step, (hi - lo) / step + 1);
}

Domain Domain::set(std::vector<Int> v) {
  v.erase(std::remove_if(v.begin(), v.end(), [](Int x) { return x < 1; }), v.end());
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
  if (v.empty()) return Domain{};
  if (v.size() == 1) return prog(v[0], 1, 1);
  const Int st = v[1] - v[0];
  bool regular = true;
  for (size_t i = 2; i < v.size() && regular; ++i) regular = v[i] - v[i - 1] == st;
  if (regular) return prog(v[0], st, (Int)v.size());
  Domain d;
  d.n_ = (Int)v.size();
  d.vals_ = std::move(v);
  return d;
}

bool Domain::has(Int v) const {
  if (n_ == 0) return false;
  if (!vals_.empty()) return std::binary_search(vals_.begin(), vals_.end(), v);
  return v >= first_ && v <= hi() && (v - first_) % step_ == 0;
}

Int Domain::lower_index(Int x) const {
  if (n_ == 0 || x <= lo()) return 0;
  if (x > hi()) return n_;
  if (!vals_.empty()) return (Int)(std::lower_bound(vals_.begin(), vals_.end(), x) - vals_.begin());
  return (x - first_ + step_ - 1) / step_;
}

namespace {
using I128 = __int128;

I128 floor_div(I128 a, I128 b) {  // b > 0
  I128 q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return q;
}

// inverse of a modulo m (gcd(a, m) == 1), extended Euclid
Int inverse_mod(Int a, Int m) {
  I128 r0 = m, r1 = ((a % m) + m) % m, t0 = 0, t1 = 1;
  while (r1 != 0) {
    const I128 q = r0 / r1;
    std::tie(r0, r1) = std::make_tuple(r1, r0 - q * r1);
    std::tie(t0, t1) = std::make_tuple(t1, t0 - q * t1);
  }
  I128 inv = t0 % m;
  if (inv < 0) inv += m;
  return (Int)inv;
}
}  // namespace

Domain Domain::meet(const Domain& o) const {
  if (empty() || o.empty()) return Domain{};
  if (!vals_.empty() || !o.vals_.empty()) {
    // iterate the explicit side's values inside the common range (the smaller
    // explicit side when both are sets), testing membership in the other
    const bool mine = !vals_.empty() && (o.vals_.empty() || n_ <= o.n_);
    const Domain& ex = mine ? *this : o;
    const Domain& other = mine ? o : *this;
    const Int lo = std::max(this->lo(), o.lo()), hi = std::min(this->hi(), o.hi());
    std::vector<Int> out;
    for (auto it = std::lower_bound(ex.vals_.begin(), ex.vals_.end(), lo); it != ex.vals_.end() && *it <= hi; ++it)
      if (other.has(*it)) out.push_back(*it);
    return set(std::move(out));
  }
  const Int lo = std::max(first_, o.first_), hi = std::min(this->hi(), o.hi());
  if (lo > hi) return Domain{};
  // x = first_ (mod step_) and x = o.first_ (mod o.step_)
  const Int s1 = step_, s2 = o.step_;
  const Int g = std::gcd(s1, s2);
  const I128 diff = (I128)o.first_ - first_;
  if (diff % g != 0) return Domain{};
  const Int m = s2 / g;
  I128 k = 0;
  if (m > 1) {
    I128 rhs = (diff / g) % m;
    if (rhs < 0) rhs += m;
    k = rhs * inverse_mod((s1 / g) % m, m) % m;
  }
  const I128 x0 = (I128)first_ + (I128)s1 * k;
  const I128 lcm = (I128)(s1 / g) * s2;
  const I128 first = x0 + (floor_div((I128)lo - x0 + lcm - 1, lcm)) * lcm;
  if (first > hi) return Domain{};
  const I128 n = ((I128)hi - first) / lcm + 1;
  return prog((Int)first, lcm > kCap ? kCap : (Int)lcm, (Int)n);
}

bool Domain::intersects(const Domain& o) const {
  if (empty() || o.empty()) return false;
  const Int lo = std::max(this->lo(), o.lo()), hi = std::min(this->hi(), o.hi());
  if (lo > hi) return false;
  if (vals_.empty() && o.vals_.empty()) return !meet(o).empty();
  const bool mine = !vals_.empty() && (o.vals_.empty() || n_ <= o.n_);
  const Domain& ex = mine ? *this : o;
  const Domain& other = mine ? o : *this;
  if (other.vals_.empty()) {  // progression: count of its values in range may be far smaller
    const Int first = other.first_ + (lo - other.first_ + other.step_ - 1) / other.step_ * other.step_;
    const Int cnt = first > hi ? 0 : (hi - first) / other.step_ + 1;
    auto b = std::lower_bound(ex.vals_.begin(), ex.vals_.end(), lo);
    auto e = std::upper_bound(b, ex.vals_.end(), hi);
    if (cnt < e - b) {
      for (Int v = first; v <= hi; v += other.step_)
        if (std::binary_search(b, e, v)) return true;
      return false;
    }
    for (auto it = b; it != e; ++it)
      if ((*it - other.first_) % other.step_ == 0) return true;
    return false;
  }
  for (auto it = std::lower_bound(ex.vals_.begin(), ex.vals_.end(), lo); it != ex.vals_.end() && *it <= hi; ++it)
    if (other.has(*it)) return true;
  return false;
}

Domain Domain::within(Int lo, Int hi) const {
  if (empty()) return Domain{};
  lo = std::max(lo, this->lo());
  hi = std::min(hi, this->hi());
  if (lo > hi) return Domain{};
  if (!vals_.empty()) {
    auto b = std::lower_bound(vals_.begin(), vals_.end(), lo);
    auto e = std::upper_bound(vals_.begin(), vals_.end(), hi);
    return set(std::vector<Int>(b, e));
  }
  const Int first = first_ + (lo - first_ + step_ - 1) / step_ * step_;
  if (first > hi) return Domain{};
  return prog(first, step_, (hi - first) / step_ + 1);
}

Domain Domain::multiples(Int m) const {
  if (m < 1) throw std::invalid_argument("divisor must be >= 1");
  if (m == 1 || empty()) return *this;
  if (!vals_.empty()) return where([m](Int v) { return v % m == 0; });
  return meet(grid(m, hi(), m));
}

bool Domain::operator==(const Domain& o) const {
  if (n_ != o.n_) return false;
  if (vals_.empty() && o.vals_.empty()) return n_ == 0 || (first_ == o.first_ && step_ == o.step_);
  for (Int i = 0; i < n_; ++i)
    if (at(i) != o.at(i)) return false;
  return true;
}

std::string Domain::str() const {
  std::ostringstream s;
  if (empty()) return "{}";
  if (vals_.empty()) {
    s << "{" << first_;
    if (n_ > 1) s << ".." << hi() << (step_ > 1 ? " step " + std::to_string(step_) : "");
    s << "}";
    return s.str();
  }
  s << "{";
  for (size_t i = 0; i < vals_.size(); ++i) s << (i ? "," : "") << vals_[i];
  s << "}";
  return s.str();
}

// =============================================================== Problem ===
int Problem::add_var(const std::string& id, Domain d, Kind k) {
  for (const Var& v : vars)
    if (v.id == id) throw std::invalid_argument("duplicate variable id: " + id);
  if (k == Kind::Constant && !d.is_single()) throw std::invalid_argument("constant needs a singleton: " + id);
  vars.push_back({id, std::move(d), k});
  return (int)vars.size() - 1;
}

int Problem::constant(Int v) {
  auto it = consts_.find(v);
  if (it == consts_.end()) it = consts_.emplace(v, add_var("_k" + std::to_string(v), Domain::single(v), Kind::Constant)).first;
  return leaf(it->second);
}

int Problem::leaf(int var) {
  if (var < 0 || var >= (int)vars.size()) throw std::invalid_argument("leaf of unknown variable");
  nodes.push_back({Op::Leaf, var, -1, -1});
  return (int)nodes.size() - 1;
}

int Problem::add(int l, int r) {
  if (l < 0 || r < 0 || l >= (int)nodes.size() || r >= (int)nodes.size())
    throw std::invalid_argument("expression child out of range");
  nodes.push_back({Op::Add, -1, l, r});
  return (int)nodes.size() - 1;
}

int Problem::mul(int l, int r) {
  if (l < 0 || r < 0 || l >= (int)nodes.size() || r >= (int)nodes.size())
    throw std::invalid_argument("expression child out of range");
  nodes.push_back({Op::Mul, -1, l, r});
  return (int)nodes.size() - 1;
}

void Problem::require(Rel rel, int l, int r) {
  if (l < 0 || r < 0 || l >= (int)nodes.size() || r >= (int)nodes.size())
    throw std::invalid_argument("constraint references an unknown node");
  cons.push_back({rel, l, r});
}

void Problem::prefer(int var, Pref p) { order.emplace_back(var, p); }

Int eval(const Problem& p, int n, const std::vector<Int>& values) {
  const Node& e = p.nodes[(size_t)n];
  switch (e.op) {
    case Op::Leaf: return values[(size_t)e.var];
    case Op::Add: return sadd(eval(p, e.l, values), eval(p, e.r, values));
    case Op::Mul: return smul(eval(p, e.l, values), eval(p, e.r, values));
  }
  return 0;
}

bool satisfied(const Problem& p, const std::vector<Int>& values) {
  for (const Con& c : p.cons) {
    const Int a = eval(p, c.l, values), b = eval(p, c.r, values);
    if ((c.rel == Rel::Eq && a != b) || (c.rel == Rel::Le && a > b) || (c.rel == Rel::Div && b % a != 0)) return false;
  }
  return true;
}

// ============================================================ propagation ===
namespace {

struct Bind {
  int p, x, y;
  Op op;
};
struct RelC {
  Rel rel;
  int a, b;
};

bool is_prog(const Domain& d) { return d.step() > 1 || d.size() <= 2 || d.hi() - d.lo() + 1 == d.size(); }

// Superset of {x op y}: exact below the pair limit, lattice hull above.
Domain combine(const Domain& x, const Domain& y, Op op, const Options& o) {
  if (x.empty() || y.empty()) return Domain{};
  // exact progression forms: a singleton operand, or sums of equal-step progressions
  if (y.is_single() && is_prog(x) && smul(x.hi(), y.lo()) < kCap && sadd(x.hi(), y.lo()) < kCap)
    return op == Op::Add ? Domain::grid(x.lo() + y.lo(), x.hi() + y.lo(), x.step())
                         : Domain::grid(x.lo() * y.lo(), x.hi() * y.lo(), x.step() * y.lo());
  if (x.is_single() && is_prog(y) && smul(y.hi(), x.lo()) < kCap && sadd(y.hi(), x.lo()) < kCap)
    return op == Op::Add ? Domain::grid(y.lo() + x.lo(), y.hi() + x.lo(), y.step())
                         : Domain::grid(y.lo() * x.lo(), y.hi() * x.lo(), y.step() * x.lo());
  if (op == Op::Add && is_prog(x) && is_prog(y) && x.step() == y.step() && sadd(x.hi(), y.hi()) < kCap)
    return Domain::grid(x.lo() + y.lo(), x.hi() + y.hi(), x.step());
  if (smul(x.size(), y.size()) <= o.pair_limit) {
    std::vector<Int> out;
    out.reserve((size_t)(x.size() * y.size()));
    for (Int i = 0; i < x.size(); ++i)
      for (Int j = 0; j < y.size(); ++j) out.push_back(op == Op::Add ? sadd(x.at(i), y.at(j)) : smul(x.at(i), y.at(j)));
    return Domain::set(std::move(out));
  }
  if (op == Op::Add) {
    const Int lo = sadd(x.lo(), y.lo());
    if (lo >= kCap) return Domain::single(kCap);
    return Domain::grid(lo, sadd(x.hi(), y.hi()), std::max<Int>(1, std::gcd(x.step(), y.step())));
  }
  // (x0 + i sx)(y0 + j sy) = x0 y0 + multiples of gcd(x0 sy, y0 sx, sx sy)
  Int g = std::gcd(std::gcd(smul(x.lo(), y.step()), smul(y.lo(), x.step())), smul(x.step(), y.step()));
  if (g < 1 || g >= kCap) g = 1;
  const Int lo = smul(x.lo(), y.lo());
  if (lo >= kCap) return Domain::single(kCap);
  return Domain::grid(lo, smul(x.hi(), y.hi()), g);
}

// {v + w : w in s} / {v * w : w in s} as a domain (exact for progressions;
// a superset for explicit sets under *).
Domain shifted(const Domain& s, Int v) {
  if (is_prog(s)) return Domain::grid(sadd(s.lo(), v), sadd(s.hi(), v), s.step());
  std::vector<Int> out;
  for (Int i = 0; i < s.size(); ++i) out.push_back(sadd(s.at(i), v));
  return Domain::set(std::move(out));
}
Domain scaled_hull(const Domain& s, Int v) {
  return Domain::grid(smul(s.lo(), v), smul(s.hi(), v), std::max<Int>(1, smul(s.step(), v)));
}

// Is there a w in s with (v op w) in p?  Allocation-free.
bool hits(const Domain& p, const Domain& s, Int v, Op op) {
  if (op == Op::Add) {
    if (is_prog(s)) return p.intersects(shifted(s, v));
    for (Int i = s.lower_index(p.lo() - v); i < s.size() && s.at(i) <= p.hi() - v; ++i)
      if (p.has(s.at(i) + v)) return true;
    return false;
  }
  if (is_prog(s) && smul(s.hi(), v) < kCap) return p.intersects(scaled_hull(s, v));
  for (Int i = s.lower_index((p.lo() + v - 1) / v); i < s.size() && s.at(i) <= p.hi() / v; ++i)
    if (p.has(smul(s.at(i), v))) return true;
  return false;
}

void divisors(Int n, std::vector<Int>& out) {
  for (Int d = 1; d * d <= n; ++d)
    if (n % d == 0) {
      out.push_back(d);
      if (d != n / d) out.push_back(n / d);
    }
}

// Values v of c with some w in s such that v op w lies in p.
Domain support(const Domain& c, const Domain& p, const Domain& s, Op op, const Options& o) {
  if (c.empty() || p.empty() || s.empty()) return Domain{};
  if (op == Op::Add) {
    if (c.small(o.enum_limit)) return c.where([&](Int v) { return hits(p, s, v, Op::Add); });
    if (smul(p.size(), s.size()) <= o.pair_limit) {
      std::vector<Int> keep;
      for (Int i = 0; i < p.size(); ++i)
        for (Int j = 0; j < s.size(); ++j) keep.push_back(p.at(i) - s.at(j));
      return c.meet(Domain::set(std::move(keep)));
    }
    const Int g = std::max<Int>(1, std::gcd(p.step(), s.step()));
    const Int hi = p.hi() - s.lo();
    if (hi < 1) return Domain{};
    const Int lo = std::max<Int>(1, p.lo() - s.hi());
    const Int first = hi - (hi - lo) / g * g;  // on the lattice of p.hi - s.lo
    return c.meet(Domain::grid(first, hi, g));
  }
  if (c.small(o.enum_limit)) return c.where([&](Int v) { return hits(p, s, v, Op::Mul); });
  if (p.small(o.divisor_limit) && p.hi() <= (Int{1} << 32)) {
    std::vector<Int> keep, ds;
    for (Int i = 0; i < p.size(); ++i) {
      ds.clear();
      divisors(p.at(i), ds);
      for (Int d : ds)
        if (s.has(p.at(i) / d)) keep.push_back(d);
    }
    return c.meet(Domain::set(std::move(keep)));
  }
  const Int lo = (p.lo() + s.hi() - 1) / s.hi(), hi = p.hi() / s.lo();
  return lo > hi ? Domain{} : c.within(lo, hi);
}

Int isqrt(Int n) {
  Int r = (Int)std::sqrt((long double)n);
  while (r > 0 && (I128)r * r > n) --r;
  while ((I128)(r + 1) * (r + 1) <= n) ++r;
  return r;
}

struct Engine {
  const Options& o;
  std::vector<Domain> dom;
  std::vector<RelC> rels;
  std::vector<Bind> binds;
  std::vector<std::vector<int>> adj;  // var -> constraint ids (rels, then binds)
  std::vector<std::pair<int, Domain>> trail;
  std::vector<int> changed;

  explicit Engine(const Options& opt) : o(opt) {}

  void set(int v, Domain d) {
    if (d == dom[(size_t)v]) return;
    trail.emplace_back(v, std::move(dom[(size_t)v]));
    dom[(size_t)v] = std::move(d);
    changed.push_back(v);
  }
  void undo(size_t mark) {
    while (trail.size() > mark) {
      dom[(size_t)trail.back().first] = std::move(trail.back().second);
      trail.pop_back();
    }
  }

  bool revise_rel(const RelC& r) {
    if (r.a == r.b) return true;
    const Domain &A = dom[(size_t)r.a], &B = dom[(size_t)r.b];
    switch (r.rel) {
      case Rel::Eq: {
        Domain m = A.meet(B);
        set(r.a, m);
        set(r.b, std::move(m));
        break;
      }
      case Rel::Le:
        set(r.a, A.within(1, B.hi()));
        if (dom[(size_t)r.a].empty()) return false;
        set(r.b, dom[(size_t)r.b].within(dom[(size_t)r.a].lo(), kCap));
        break;
      case Rel::Div: {
        const Domain Bv = B;
        set(r.a, A.small(o.enum_limit) ? A.where([&](Int v) { return Bv.intersects(Domain::grid(v, Bv.hi(), v)); })
                                        : A.within(1, Bv.hi()));
        const Domain& A2 = dom[(size_t)r.a];
        if (A2.empty()) return false;
        if (A2.is_single()) {
          set(r.b, Bv.multiples(A2.lo()));
        } else if (A2.small(o.enum_limit) && Bv.small(o.enum_limit)) {
          const Domain Ad = A2;
          set(r.b, Bv.where([&](Int u) {
            for (Int i = 0; i < Ad.size(); ++i)
              if (u % Ad.at(i) == 0) return true;
            return false;
          }));
        } else if (A2.small(o.enum_limit)) {
          std::vector<Int> u;
          bool exact = true;
          for (Int i = 0; i < A2.size() && exact; ++i) {
            const Domain m = Bv.multiples(A2.at(i));
            if ((Int)u.size() + m.size() > o.pair_limit) exact = false;
            for (Int j = 0; exact && j < m.size(); ++j) u.push_back(m.at(j));
          }
          set(r.b, exact ? Domain::set(std::move(u)) : Bv.within(A2.lo(), kCap));
        } else {
          set(r.b, Bv.within(A2.lo(), kCap));
        }
        break;
      }
    }
    return !dom[(size_t)r.a].empty() && !dom[(size_t)r.b].empty();
  }

  bool revise_bind(const Bind& b) {
    if (b.x == b.y) {
      const Domain X = dom[(size_t)b.x];
      Domain sq;
      if (X.small(o.enum_limit)) {
        std::vector<Int> v;
        for (Int i = 0; i < X.size(); ++i) v.push_back(b.op == Op::Add ? sadd(X.at(i), X.at(i)) : smul(X.at(i), X.at(i)));
        sq = Domain::set(std::move(v));
      } else {
        sq = combine(X, X, b.op, o);
      }
      set(b.p, dom[(size_t)b.p].meet(sq));
      const Domain P = dom[(size_t)b.p];
      if (P.empty()) return false;
      if (X.small(o.enum_limit))
        set(b.x, X.where([&](Int v) { return P.has(b.op == Op::Add ? sadd(v, v) : smul(v, v)); }));
      else if (b.op == Op::Add)
        set(b.x, X.within((P.lo() + 1) / 2, P.hi() / 2));
      else
        set(b.x, X.within(isqrt(P.lo() - 1) + 1, isqrt(P.hi())));
      return !dom[(size_t)b.x].empty();
    }
    set(b.p, dom[(size_t)b.p].meet(combine(dom[(size_t)b.x], dom[(size_t)b.y], b.op, o)));
    if (dom[(size_t)b.p].empty()) return false;
    set(b.x, support(dom[(size_t)b.x], dom[(size_t)b.p], dom[(size_t)b.y], b.op, o));
    if (dom[(size_t)b.x].empty()) return false;
    set(b.y, support(dom[(size_t)b.y], dom[(size_t)b.p], dom[(size_t)b.x], b.op, o));
    return !dom[(size_t)b.y].empty();
  }

  // AC-3 worklist to fixpoint.  false: some domain emptied.
  bool propagate(const std::vector<int>& seeds) {
    const int nc = (int)(rels.size() + binds.size());
    std::vector<char> queued((size_t)nc, 0);
    std::deque<int> q;
    for (int c : seeds)
      if (!queued[(size_t)c]) {
        queued[(size_t)c] = 1;
        q.push_back(c);
      }
    while (!q.empty()) {
      const int c = q.front();
      q.pop_front();
      queued[(size_t)c] = 0;
      changed.clear();
      const bool ok = c < (int)rels.size() ? revise_rel(rels[(size_t)c]) : revise_bind(binds[(size_t)c - rels.size()]);
      if (!ok) return false;
      for (int v : changed)
        for (int a : adj[(size_t)v])
          if (!queued[(size_t)a]) {
            queued[(size_t)a] = 1;
            q.push_back(a);
          }
    }
    return true;
  }
};

void validate(const Problem& p) {
  std::vector<char> seen(p.vars.size(), 0);
  for (const auto& [v, pref] : p.order) {
    if (v < 0 || v >= (int)p.vars.size() || p.vars[(size_t)v].kind != Kind::Resolution)
      throw std::invalid_argument("heuristic order must list resolution variables");
    if (seen[(size_t)v]++) throw std::invalid_argument("heuristic order lists a variable twice");
  }
  for (const Var& v : p.vars)
    if (v.dom.empty() && v.kind == Kind::Constant) throw std::invalid_argument("empty constant " + v.id);
}

}  // namespace

// ================================================================ search ===
std::optional<Solution> solve(const Problem& p, const Options& o) {
  validate(p);
  Engine E(o);
  for (const Var& v : p.vars) E.dom.push_back(v.dom);
  // Flatten compound terms onto intermediates; identical (op, a, b) terms share one.
  std::map<std::tuple<int, int, int>, int> memo;
  std::vector<Domain>& dom = E.dom;
  std::function<int(int)> flat = [&](int n) -> int {
    const Node& e = p.nodes[(size_t)n];
    if (e.op == Op::Leaf) return e.var;
    int a = flat(e.l), b = flat(e.r);
    if (a > b) std::swap(a, b);
    const auto key = std::make_tuple((int)e.op, a, b);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    Options hull = o;
    hull.pair_limit = 0;
    dom.push_back(combine(dom[(size_t)a], dom[(size_t)b], e.op, hull));
    const int t = (int)dom.size() - 1;
    E.binds.push_back({t, a, b, e.op});
    memo.emplace(key, t);
    return t;
  };
  for (const Con& c : p.cons) {
    const int a = flat(c.l), b = flat(c.r);
    E.rels.push_back({c.rel, a, b});
  }
  E.adj.assign(dom.size(), {});
  for (int i = 0; i < (int)E.rels.size(); ++i) {
    E.adj[(size_t)E.rels[(size_t)i].a].push_back(i);
    E.adj[(size_t)E.rels[(size_t)i].b].push_back(i);
  }
  const int base = (int)E.rels.size();
  for (int i = 0; i < (int)E.binds.size(); ++i)
    for (int v : {E.binds[(size_t)i].p, E.binds[(size_t)i].x, E.binds[(size_t)i].y}) E.adj[(size_t)v].push_back(base + i);
  for (auto& l : E.adj) {
    std::sort(l.begin(), l.end());
    l.erase(std::unique(l.begin(), l.end()), l.end());
  }
  // Heuristic order, completed with the unlisted resolution variables in
  // declaration order (smallest first).
  std::vector<std::pair<int, Pref>> ord = p.order;
  {
    std::vector<char> listed(p.vars.size(), 0);
    for (const auto& e : ord) listed[(size_t)e.first] = 1;
    for (int v = 0; v < (int)p.vars.size(); ++v)
      if (p.vars[(size_t)v].kind == Kind::Resolution && !listed[(size_t)v]) ord.emplace_back(v, Pref::Smallest);
  }
  std::vector<int> all(E.rels.size() + E.binds.size());
  std::iota(all.begin(), all.end(), 0);
  Solution sol;
  if (!E.propagate(all)) return std::nullopt;

  struct Frame {
    Domain entry;
    Int k;
    size_t mark;
  };
  const size_t n = ord.size();
  std::vector<Frame> fr(n);
  bool found = n == 0;
  size_t depth = 0;
  if (n) fr[0] = {dom[(size_t)ord[0].first], 0, E.trail.size()};
  while (!found) {
    Frame& f = fr[depth];
    const int v = ord[depth].first;
    E.undo(f.mark);
    if (f.k >= f.entry.size()) {
      if (depth == 0) return std::nullopt;
      --depth;
      ++sol.backtracks;
      continue;
    }
    const Int idx = ord[depth].second == Pref::Largest ? f.entry.size() - 1 - f.k : f.k;
    const Int val = f.entry.at(idx);
    ++f.k;
    if (!dom[(size_t)v].has(val)) continue;
    ++sol.nodes;
    E.changed.clear();
    E.set(v, Domain::single(val));
    if (E.propagate(E.adj[(size_t)v])) {
      if (depth + 1 == n) {
        found = true;
      } else {
        ++depth;
        fr[depth] = {dom[(size_t)ord[depth].first], 0, E.trail.size()};
      }
    } else {
      ++sol.backtracks;
    }
  }
  std::vector<Int> values(p.vars.size(), 0);
  for (size_t v = 0; v < p.vars.size(); ++v) values[v] = dom[v].empty() ? 0 : dom[v].lo();
  bool determined = true;
  for (size_t v = 0; v < p.vars.size(); ++v) determined = determined && dom[v].is_single();
  if (determined && !satisfied(p, values))
    throw std::logic_error("csp: assignment violates a constraint (propagation bug)");
  for (const auto& e : ord) sol.values[p.vars[(size_t)e.first].id] = dom[(size_t)e.first].lo();
  return sol;
}

std::vector<std::map<std::string, Int>> brute_force(const Problem& p, Int cap) {
  validate(p);
  std::vector<int> res;
  Int space = 1;
  std::vector<Int> values(p.vars.size(), 0);
  for (int v = 0; v < (int)p.vars.size(); ++v) {
    const Var& x = p.vars[(size_t)v];
    if (x.kind == Kind::Intermediate) throw std::invalid_argument("brute_force: problem has intermediates");
    if (x.kind == Kind::Constant) values[(size_t)v] = x.dom.lo();
    if (x.kind == Kind::Resolution) {
      res.push_back(v);
      space = smul(space, x.dom.size());
    }
  }
  if (space > cap) throw std::invalid_argument("brute_force: search space exceeds cap");
  std::vector<std::map<std::string, Int>> out;
  if (space == 0) return out;
  std::vector<Int> idx(res.size(), 0);
  while (true) {
    for (size_t i = 0; i < res.size(); ++i) values[(size_t)res[i]] = p.vars[(size_t)res[i]].dom.at(idx[i]);
    if (satisfied(p, values)) {
      std::map<std::string, Int> m;
      for (int v : res) m[p.vars[(size_t)v].id] = values[(size_t)v];
      out.push_back(std::move(m));
    }
    size_t i = res.size();
    while (i > 0) {
      --i;
      if (++idx[i] < p.vars[(size_t)res[i]].dom.size()) break;
      idx[i] = 0;
      if (i == 0) return out;
    }
    if (res.empty()) return out;
  }
}

// =========================================================== text format ===
Problem parse(const std::string& text) {
  Problem p;
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    std::istringstream ls(line);
    std::string tag;
    if (!(ls >> tag) || tag[0] == '#') continue;
    auto bad = [&](const std::string& why) {
      return std::invalid_argument("csp text line " + std::to_string(lineno) + ": " + why);
    };
    if (tag == "v") {
      std::string id, kind, form;
      if (!(ls >> id >> kind >> form)) throw bad("variable needs id kind form");
      const Kind k = kind == "C" ? Kind::Constant : kind == "R" ? Kind::Resolution : kind == "I" ? Kind::Intermediate
                                                                                               : throw bad("kind");
      Domain d;
      if (form == "r") {
        Int lo, hi;
        if (!(ls >> lo >> hi) || lo < 1) throw bad("range lo hi (lo >= 1)");
        d = Domain::span(lo, hi);
      } else if (form == "s") {
        Int lo, hi, st;
        if (!(ls >> lo >> hi >> st) || lo < 1 || st < 1) throw bad("strided lo hi step");
        d = Domain::grid(lo, hi, st);
      } else if (form == "e") {
        std::vector<Int> v;
        Int x;
        while (ls >> x) {
          if (x < 1) throw bad("values must be >= 1");
          v.push_back(x);
        }
        d = Domain::set(std::move(v));
      } else {
        throw bad("domain form r|s|e");
      }
      p.add_var(id, std::move(d), k);
    } else if (tag == "n") {
      std::string op;
      int a, b;
      if (!(ls >> op >> a)) throw bad("node");
      if (op == "v") p.leaf(a);
      else if (op == "+" && (ls >> b)) p.add(a, b);
      else if (op == "*" && (ls >> b)) p.mul(a, b);
      else throw bad("node op v|+|*");
    } else if (tag == "c") {
      std::string rel;
      int a, b;
      if (!(ls >> rel >> a >> b)) throw bad("constraint");
      p.require(rel == "=" ? Rel::Eq : rel == "<" ? Rel::Le : rel == "|" ? Rel::Div : throw bad("relation =|<||"), a, b);
    } else if (tag == "h") {
      int v;
      std::string pref;
      if (!(ls >> v >> pref)) throw bad("heuristic");
      p.prefer(v, pref == "L" ? Pref::Largest : Pref::Smallest);
    } else {
      throw bad("unknown tag " + tag);
    }
  }
  return p;
}

std::string format(const Problem& p) {
  std::ostringstream s;
  for (const Var& v : p.vars) {
    s << "v " << v.id << ' ' << (v.kind == Kind::Constant ? 'C' : v.kind == Kind::Resolution ? 'R' : 'I');
    const Domain& d = v.dom;
    if (d.step() > 1 || d.size() == 1 || d.hi() - d.lo() + 1 == d.size()) {
      if (d.step() > 1) s << " s " << d.lo() << ' ' << d.hi() << ' ' << d.step();
      else s << " r " << d.lo() << ' ' << d.hi();
    } else {
      s << " e";
      for (Int i = 0; i < d.size(); ++i) s << ' ' << d.at(i);
    }
    s << '\n';
  }
  for (const Node& n : p.nodes) {
    if (n.op == Op::Leaf) s << "n v " << n.var << '\n';
    else s << "n " << (n.op == Op::Add ? '+' : '*') << ' ' << n.l << ' ' << n.r << '\n';
  }
  for (const Con& c : p.cons) s << "c " << (c.rel == Rel::Eq ? '=' : c.rel == Rel::Le ? '<' : '|') << ' ' << c.l << ' ' << c.r << '\n';
  for (const auto& [v, pr] : p.order) s << "h " << v << ' ' << (pr == Pref::Largest ? 'L' : 'S') << '\n';
  return s.str();
}

}  // namespace frnn::csp
