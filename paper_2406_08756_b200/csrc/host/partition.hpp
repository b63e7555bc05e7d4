// Stage planning (two reservation policies, keep the shorter steady period),
// the plan cache, the OOM check, the initial split and Algorithm 1's greedy
// partition search — restating proj/src/partition.cpp:26-215.
#pragma once

#include <map>
#include <tuple>
#include <vector>

#include "host/pipeline.hpp"

namespace lynx::host {

enum class PlanMode { Opt, Heu };

struct StagePlan {
  StageTimeline timeline;
  Rat period_us;
};

struct Move {
  int from = 0, to = 0;
  bool accepted = true;
};

struct Partition {
  std::vector<int> layers;
  std::vector<StageTimeline> timelines;
  std::vector<Rat> durations;
  PlanMode mode = PlanMode::Heu;
  int iterations = 0;
  std::vector<Move> moves;
};

class StagePlanner {
 public:
  explicit StagePlanner(const Profile& p) : p_(p) {}
  const StagePlan& plan(int stage, int stage_layers, PlanMode mode, int64_t time_limit_ms = 10000);

 private:
  const Profile& p_;
  std::map<std::tuple<int, int, int>, StagePlan> memo_;
};

bool stage_oom(const ModelProfile& m, int stage_layers, int stage, const PipelineConfig& pipe,
               const HardwareProfile& hw);
Partition even_partition(const Profile& p, PlanMode mode = PlanMode::Heu);
Partition greedy_partition(const Profile& p, PlanMode mode = PlanMode::Heu, int64_t time_limit_ms = 10000);

// OPT (global phase-grid MILP) stage plan; implemented in opt.cpp.
StagePlan plan_stage_opt(const Profile& p, int stage, int stage_layers, int64_t time_limit_ms);

}  // namespace lynx::host
