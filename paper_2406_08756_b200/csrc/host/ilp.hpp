// Exact 0/1 integer programs and a deterministic branch-and-bound.
//
// The HEU plan bits depend on the exact exploration order of the reference
// solver (proj/src/ilp_bnb.cpp:29-244; model encodings proj/src/ilp_model.cpp:36-87):
// variables branch in issue order, 0 before 1; nodes are explored best-first
// on their objective lower bound with the newest node first among ties;
// bounds are tightened by interval propagation (<= 8 passes, var_count + 2 at
// leaves); the first strictly better leaf wins; the "time limit" is a node
// budget of max(64, 25 * ms). This restatement keeps those rules, so plans are
// bit-identical to the reference's.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "host/rational.hpp"

namespace lynx::host {

enum class VarType { Bool, Cont };
enum class Sense { Le, Eq, Ge };
enum class SolveStatus { Optimal, Feasible, Infeasible, TimedOut };
const char* status_text(SolveStatus s);

// Canonical linear form: one coefficient per variable index, zeros dropped.
struct Linear {
  std::map<int, Rat> coef;
  Rat constant;
  Linear& add(const Rat& c, int var);
};

struct Row {
  Linear lhs;
  Sense sense = Sense::Le;
  Rat rhs;
  std::string name;
};

class Program {
 public:
  int new_bool(std::string name);
  int new_cont(std::string name, Rat lo, Rat hi);
  void pin(int var, const Rat& value);
  void add_row(Linear lhs, Sense s, Rat rhs, std::string name = "");
  int land(int a, int b);   // z = a AND b  (z<=a, z<=b, z>=a+b-1)
  int lnot(int a);          // n = 1 - a, cached per variable
  void minimize(Linear obj) { objective_ = std::move(obj); }

  int size() const { return static_cast<int>(type_.size()); }
  int bool_count() const;
  VarType type(int v) const { return type_[v]; }
  const std::string& name(int v) const { return name_[v]; }
  const Rat& lo(int v) const { return lo_[v]; }
  const Rat& hi(int v) const { return hi_[v]; }
  const std::vector<Row>& rows() const { return rows_; }
  const Linear& objective() const { return objective_; }

 private:
  std::vector<VarType> type_;
  std::vector<std::string> name_;
  std::vector<Rat> lo_, hi_;
  std::vector<Row> rows_;
  Linear objective_;
  std::map<int, int> not_of_;
};

struct Solution {
  SolveStatus status = SolveStatus::Infeasible;
  std::vector<Rat> x;
  Rat objective;
  Rat gap;
};

Solution branch_and_bound(const Program& p, int64_t time_limit_ms);
std::vector<std::string> violations(const Program& p, const std::vector<Rat>& x);
std::string to_lp_text(const Program& p, const std::string& problem_name);

}  // namespace lynx::host
