// HEU per-layer recomputation planner and its expansion into the per-
// microbatch placements the GPU executor replays.
//
// Restates, bit-exactly, the reference's 5-phase per-layer ILP
// (Eqs. 11-18 of the paper; proj/src/heusched.cpp:53-258), the plan peak-memory
// formula (:260-277), the independent plan checker (:279-311), the fixed
// baselines (:313-341) and expand_plan_to_stage (:343-427).
#pragma once

#include <array>
#include <string>
#include <vector>

#include "host/ilp.hpp"
#include "host/profile.hpp"

namespace lynx::host {

enum class Role { Interior, Last };
enum class Reserve { FixedBytes, Unretained };

struct HeuCtx {
  int layers = 1;
  int n_batch = 1;
  std::array<Rat, 4> ctime{};  // CTime_1..4: the layer's two fwd and two bwd all-reduce windows
  Rat static_bytes, budget, delta, comm_scale = 1;
  Reserve policy = Reserve::FixedBytes;
  Role role = Role::Interior;
};

struct LayerPlan {
  SolveStatus status = SolveStatus::Infeasible;
  std::vector<bool> retained;  // S_i over the forward template positions
  std::vector<int> phase;      // 1..5
  Rat critical_us, peak_bytes, delta_bytes;
  Role role = Role::Interior;
};

struct HeuModel {
  Program prog;
  int n = 0;
  std::vector<int> S;
  std::vector<std::vector<int>> R;  // R[t-1][i], empty rows for absent phases
  std::vector<int> phases;
  std::vector<Rat> cost;
  std::vector<int64_t> bytes;
  std::vector<bool> comm;
  HeuCtx ctx;
};

// Where one regeneration of a discarded forward tensor runs.
struct Recompute {
  enum class Host { Window, Critical, Stall };
  int owner_mb = 0, owner_layer = 0, op = 0;
  Host host = Host::Critical;
  int host_mb = 0;
  bool host_bwd = false;
  int host_layer = 0, host_window = 0, host_elem = 0;
};

struct StageTimeline {
  int stage = 0;
  Role role = Role::Interior;
  LayerPlan plan;
  std::vector<Recompute> items;
  bool strict_deps = true;
};

HeuCtx heu_context(const Profile& p, int stage, int stage_layers, Reserve policy = Reserve::FixedBytes,
                   Rat delta = Rat(0));
HeuModel heu_model(const LayerTemplate& layer, const HeuCtx& ctx);
LayerPlan heu_solve(const HeuModel& m, int64_t time_limit_ms = 10000);
Rat plan_peak(const LayerPlan& plan, const HeuCtx& ctx, const LayerTemplate& layer);
std::vector<std::string> plan_violations(const LayerPlan& plan, const HeuCtx& ctx, const LayerTemplate& layer);
LayerPlan full_recompute(const LayerTemplate& layer, const HeuCtx& ctx);
LayerPlan retain_all(const LayerTemplate& layer, const HeuCtx& ctx);
LayerPlan selective_recompute(const LayerTemplate& layer, const HeuCtx& ctx);
StageTimeline expand_to_stage(const LayerPlan& plan, const HeuCtx& ctx, const PipelineConfig& pipe, int stage);

}  // namespace lynx::host
