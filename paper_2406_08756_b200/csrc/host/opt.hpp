// OPT: the global phase-grid MILP over one stage's unrolled 1F1B operator
// sequence (paper Eqs. 1-10), its independent checker, and the conversion of
// an optimal schedule into executor placements. Restates
// proj/src/optsched.cpp:54-399 and proj/src/report_io.cpp:187-294.
// Tractable for small/coarse graphs only (Θ(n²) booleans); at GPT scale the
// LP text (to_lp_text) is the escape hatch to an external MILP solver.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "host/heu.hpp"

namespace lynx::host {

struct OptModel {
  StageGraph graph;
  int64_t budget = 0, static_bytes = 0;
  std::vector<Rat> cost;
  Program prog;
  std::vector<std::vector<int>> R, S;  // R[t][i] (i <= t), S[t][i] (i < t)
};

struct PhaseSchedule {
  SolveStatus status = SolveStatus::Infeasible;
  std::vector<std::pair<int, int>> keep, recompute, overlapped;
  Rat cost_us, gap;
};

struct PhaseOrigin {
  int microbatch = 0;
  bool backward = false;
  int local = 0;
};

struct UnrolledStage {
  StageGraph graph;
  std::vector<PhaseOrigin> origin;
  int fwd_ops = 0, bwd_ops = 0;
};

OptModel opt_model(const StageGraph& g, const HardwareProfile& hw, int64_t static_bytes);
PhaseSchedule opt_solve(const OptModel& m, int64_t time_limit_ms = 10000);
std::string schedule_issues(const PhaseSchedule& s, const OptModel& m);  // "" when valid
UnrolledStage unroll(const StageGraph& single, int n_microbatches, int n_batch);
UnrolledStage stage_phase_graph(const Profile& p, int stage, int stage_layers);
int64_t static_share_ceil(const Profile& p, int stage_layers);
// host_in_layer (optional): per emitted item, whether its host phase lies inside the stage's layers
// (false: the embedding / head phases, emitted as CriticalPath at layer 0, elem 0).
StageTimeline timeline_from_schedule(const Profile& p, int stage, int stage_layers, const PhaseSchedule& s,
                                     const UnrolledStage& u, std::vector<bool>* host_in_layer = nullptr);

}  // namespace lynx::host
