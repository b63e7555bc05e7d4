#include "host/ilp.hpp"

#include <algorithm>
#include <memory>
#include <queue>
#include <sstream>
#include <stdexcept>

namespace lynx::host {

const char* status_text(SolveStatus s) {
  switch (s) {
    case SolveStatus::Optimal: return "optimal";
    case SolveStatus::Feasible: return "feasible";
    case SolveStatus::Infeasible: return "infeasible";
    case SolveStatus::TimedOut: return "timed_out";
  }
  return "?";
}

Linear& Linear::add(const Rat& c, int var) {
  if (c.sign() == 0) return *this;
  auto it = coef.find(var);
  if (it == coef.end()) {
    coef.emplace(var, c);
  } else {
    it->second += c;
    if (it->second.sign() == 0) coef.erase(it);
  }
  return *this;
}

int Program::new_bool(std::string name) {
  type_.push_back(VarType::Bool);
  name_.push_back(std::move(name));
  lo_.push_back(Rat(0));
  hi_.push_back(Rat(1));
  return size() - 1;
}

int Program::new_cont(std::string name, Rat lo, Rat hi) {
  type_.push_back(VarType::Cont);
  name_.push_back(std::move(name));
  lo_.push_back(std::move(lo));
  hi_.push_back(std::move(hi));
  return size() - 1;
}

void Program::pin(int v, const Rat& value) {
  lo_[v] = value;
  hi_[v] = value;
}

void Program::add_row(Linear lhs, Sense s, Rat rhs, std::string name) {
  rows_.push_back(Row{std::move(lhs), s, std::move(rhs), std::move(name)});
}

int Program::land(int a, int b) {
  const int z = new_bool("and_" + std::to_string(size()));
  add_row(Linear().add(1, z).add(-1, a), Sense::Le, 0);
  add_row(Linear().add(1, z).add(-1, b), Sense::Le, 0);
  add_row(Linear().add(1, z).add(-1, a).add(-1, b), Sense::Ge, -1);
  return z;
}

int Program::lnot(int a) {
  auto it = not_of_.find(a);
  if (it != not_of_.end()) return it->second;
  const int n = new_bool("not_" + name_[a]);
  add_row(Linear().add(1, n).add(1, a), Sense::Eq, 1);
  not_of_.emplace(a, n);
  return n;
}

int Program::bool_count() const {
  return static_cast<int>(std::count(type_.begin(), type_.end(), VarType::Bool));
}

std::vector<std::string> violations(const Program& p, const std::vector<Rat>& x) {
  std::vector<std::string> out;
  if (static_cast<int>(x.size()) != p.size()) {
    out.push_back("assignment size mismatch");
    return out;
  }
  for (int v = 0; v < p.size(); ++v) {
    if (x[v] < p.lo(v) || x[v] > p.hi(v)) out.push_back("bound violated for " + p.name(v));
    if (p.type(v) == VarType::Bool && x[v] != Rat(0) && x[v] != Rat(1))
      out.push_back("non-binary value for " + p.name(v));
  }
  int idx = 0;
  for (const Row& r : p.rows()) {
    Rat lhs = r.lhs.constant;
    for (const auto& [v, c] : r.lhs.coef) lhs += c * x[v];
    const bool ok = r.sense == Sense::Le ? lhs <= r.rhs : (r.sense == Sense::Ge ? lhs >= r.rhs : lhs == r.rhs);
    if (!ok) out.push_back("constraint " + (r.name.empty() ? "#" + std::to_string(idx) : r.name) + " violated");
    ++idx;
  }
  return out;
}

namespace {

struct Box {
  std::vector<Rat> lo, hi;
};

// Interval propagation over the row list in order (see header).
class Propagate {
 public:
  explicit Propagate(const Program& p) : p_(p) {}

  bool operator()(Box& b, bool leaf) const {
    const int passes = leaf ? p_.size() + 2 : 8;
    for (int it = 0; it < passes; ++it) {
      bool moved = false;
      for (const Row& r : p_.rows())
        if (!row(r, b, moved)) return false;
      if (!moved) return true;
    }
    return true;
  }

 private:
  bool lower_hi(Box& b, int v, Rat val, bool& moved) const {
    if (p_.type(v) == VarType::Bool && val.sign() > 0 && val < Rat(1)) val = Rat(0);
    if (val < b.hi[v]) {
      if (val < b.lo[v]) return false;
      b.hi[v] = std::move(val);
      moved = true;
    }
    return true;
  }
  bool raise_lo(Box& b, int v, Rat val, bool& moved) const {
    if (p_.type(v) == VarType::Bool && val.sign() > 0 && val < Rat(1)) val = Rat(1);
    if (val > b.lo[v]) {
      if (val > b.hi[v]) return false;
      b.lo[v] = std::move(val);
      moved = true;
    }
    return true;
  }
  bool row(const Row& r, Box& b, bool& moved) const {
    Rat act_min = r.lhs.constant, act_max = r.lhs.constant;
    for (const auto& [v, c] : r.lhs.coef) {
      if (c.sign() > 0) {
        act_min += c * b.lo[v];
        act_max += c * b.hi[v];
      } else {
        act_min += c * b.hi[v];
        act_max += c * b.lo[v];
      }
    }
    const bool upper = r.sense != Sense::Ge, lower = r.sense != Sense::Le;
    if (upper && act_min > r.rhs) return false;
    if (lower && act_max < r.rhs) return false;
    for (const auto& [v, c] : r.lhs.coef) {
      if (b.lo[v] == b.hi[v]) continue;
      const bool pos = c.sign() > 0;
      if (upper) {
        const Rat rest = act_min - c * (pos ? b.lo[v] : b.hi[v]);
        const Rat bound = (r.rhs - rest) / c;
        if (!(pos ? lower_hi(b, v, bound, moved) : raise_lo(b, v, bound, moved))) return false;
      }
      if (lower) {
        const Rat rest = act_max - c * (pos ? b.hi[v] : b.lo[v]);
        const Rat bound = (r.rhs - rest) / c;
        if (!(pos ? raise_lo(b, v, bound, moved) : lower_hi(b, v, bound, moved))) return false;
      }
    }
    return true;
  }
  const Program& p_;
};

Rat bound_of(const Program& p, const Box& b) {
  Rat s = p.objective().constant;
  for (const auto& [v, c] : p.objective().coef) s += c * (c.sign() > 0 ? b.lo[v] : b.hi[v]);
  return s;
}

int first_free_bool(const Program& p, const Box& b) {
  for (int v = 0; v < p.size(); ++v)
    if (p.type(v) == VarType::Bool && b.lo[v] != b.hi[v]) return v;
  return -1;
}

struct Node {
  Box box;
  Rat bound;
  int64_t seq = 0;
};
using NodeRef = std::shared_ptr<Node>;
struct WorseFirst {  // priority_queue top = smallest bound, then largest seq
  bool operator()(const NodeRef& a, const NodeRef& b) const {
    const int c = cmp(a->bound, b->bound);
    if (c != 0) return c > 0;
    return a->seq < b->seq;
  }
};

}  // namespace

Solution branch_and_bound(const Program& p, int64_t time_limit_ms) {
  const Propagate propagate(p);
  const int64_t budget = time_limit_ms <= 0 ? 1 : std::max<int64_t>(64, time_limit_ms * 25);
  Solution out;
  auto root = std::make_shared<Node>();
  for (int v = 0; v < p.size(); ++v) {
    root->box.lo.push_back(p.lo(v));
    root->box.hi.push_back(p.hi(v));
  }
  if (!propagate(root->box, false)) return out;
  root->bound = bound_of(p, root->box);

  std::priority_queue<NodeRef, std::vector<NodeRef>, WorseFirst> open;
  open.push(root);
  int64_t seq = 1, expanded = 0;
  bool have = false, out_of_budget = false;
  Rat best;
  std::vector<Rat> best_x;

  while (!open.empty()) {
    if (expanded >= budget) {
      out_of_budget = true;
      break;
    }
    NodeRef node = open.top();
    open.pop();
    ++expanded;
    if (have && node->bound >= best) continue;
    const int v = first_free_bool(p, node->box);
    if (v < 0) {
      Box leaf = node->box;
      if (!propagate(leaf, true)) continue;
      for (int i = 0; i < p.size(); ++i)
        if (leaf.lo[i] != leaf.hi[i])
          throw std::logic_error("continuous variables are not determined by the boolean assignment");
      if (!violations(p, leaf.lo).empty()) continue;
      Rat obj = p.objective().constant;
      for (const auto& [i, c] : p.objective().coef) obj += c * leaf.lo[i];
      if (!have || obj < best) {
        have = true;
        best = obj;
        best_x = std::move(leaf.lo);
      }
      continue;
    }
    for (int val = 0; val <= 1; ++val) {
      auto child = std::make_shared<Node>(*node);
      child->box.lo[v] = Rat(val);
      child->box.hi[v] = Rat(val);
      child->seq = seq++;
      if (!propagate(child->box, false)) continue;
      child->bound = bound_of(p, child->box);
      if (have && child->bound >= best) continue;
      open.push(std::move(child));
    }
  }

  if (!out_of_budget) {
    if (have) {
      out.status = SolveStatus::Optimal;
      out.objective = best;
      out.x = std::move(best_x);
    }
    return out;
  }
  Rat lb = have ? best : Rat(0);
  if (!open.empty()) lb = open.top()->bound;
  if (have) {
    out.status = SolveStatus::Feasible;
    out.objective = best;
    out.x = std::move(best_x);
    out.gap = best - rmin(lb, best);
  } else {
    out.status = SolveStatus::TimedOut;
  }
  return out;
}

std::string to_lp_text(const Program& p, const std::string& problem_name) {
  std::ostringstream os;
  os << "\\ Problem: " << problem_name << "\n";
  auto num = [](const Rat& r) {
    if (r.is_integer()) return r.num().str();
    const std::string s = to_canonical(r);
    return s.find('/') == std::string::npos ? s : to_fixed(r, 18);
  };
  auto expr = [&](const Linear& e) {
    bool first = true;
    for (const auto& [v, c0] : e.coef) {
      Rat c = c0;
      if (first) {
        if (c.sign() < 0) {
          os << "- ";
          c = -c;
        }
        first = false;
      } else {
        os << (c.sign() < 0 ? " - " : " + ");
        if (c.sign() < 0) c = -c;
      }
      if (c != Rat(1)) os << num(c) << " ";
      os << p.name(v);
    }
    if (first) os << "0 " << (p.size() > 0 ? p.name(0) : "x");
  };
  os << "Minimize\n obj: ";
  expr(p.objective());
  os << "\nSubject To\n";
  int idx = 0;
  for (const Row& r : p.rows()) {
    os << " " << (r.name.empty() ? "c" + std::to_string(idx) : r.name) << ": ";
    expr(r.lhs);
    os << (r.sense == Sense::Le ? " <= " : (r.sense == Sense::Ge ? " >= " : " = "));
    os << num(r.rhs - r.lhs.constant) << "\n";
    ++idx;
  }
  os << "Bounds\n";
  for (int v = 0; v < p.size(); ++v)
    if (p.type(v) == VarType::Cont || p.lo(v) == p.hi(v))
      os << " " << num(p.lo(v)) << " <= " << p.name(v) << " <= " << num(p.hi(v)) << "\n";
  os << "Binaries\n";
  for (int v = 0; v < p.size(); ++v)
    if (p.type(v) == VarType::Bool && p.lo(v) != p.hi(v)) os << " " << p.name(v) << "\n";
  os << "End\n";
  return os.str();
}

}  // namespace lynx::host
