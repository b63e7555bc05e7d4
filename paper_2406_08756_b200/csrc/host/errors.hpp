// Error taxonomy of the host planner. Mirrors the reference's exception types
// (proj/include/lynx/errors.hpp:22-64) and their mapping onto exit/status codes
// (proj/tools/lynx_main.cpp:30-35, :280-301); the C-ABI converts them to
// LYNX_E_* codes, so no exception ever crosses the boundary.
#pragma once

#include <stdexcept>
#include <string>

namespace lynx::host {

struct PlanError : std::runtime_error {
  PlanError(const std::string& what, int code) : std::runtime_error(what), status(code) {}
  int status;
};

// status codes (include/lynx_b200.h)
constexpr int kStValidation = 1, kStParse = 2, kStTimedOut = 3, kStInfeasible = 4, kStNoPartition = 5;

struct ParseError : PlanError {
  explicit ParseError(const std::string& w) : PlanError(w, kStParse) {}
};
struct ValidationError : PlanError {
  explicit ValidationError(const std::string& w) : PlanError(w, kStValidation) {}
};
struct BudgetInfeasible : PlanError {
  explicit BudgetInfeasible(const std::string& w) : PlanError(w, kStInfeasible) {}
};
struct BudgetTooSmall : PlanError {
  explicit BudgetTooSmall(const std::string& w) : PlanError(w, kStInfeasible) {}
};
struct TooLarge : PlanError {
  explicit TooLarge(const std::string& w) : PlanError(w, kStTimedOut) {}
};
struct NoValidPartition : PlanError {
  explicit NoValidPartition(const std::string& w) : PlanError(w, kStNoPartition) {}
};
// Logic errors of the reference (ModelMismatch, RoleMismatch) and the
// simulator's InconsistentPlan / WindowConfigError / EmptyGraph surface as
// generic failures (exit 2 in the reference CLI's catch-all).
struct InconsistentPlan : PlanError {
  explicit InconsistentPlan(const std::string& w) : PlanError(w, kStParse) {}
};
struct WindowConfigError : PlanError {
  explicit WindowConfigError(const std::string& w) : PlanError(w, kStParse) {}
};
struct RoleMismatch : PlanError {
  explicit RoleMismatch(const std::string& w) : PlanError(w, kStParse) {}
};
struct EmptyGraph : PlanError {
  explicit EmptyGraph(const std::string& w) : PlanError(w, kStParse) {}
};

}  // namespace lynx::host
