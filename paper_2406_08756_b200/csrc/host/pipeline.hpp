// Exact 1F1B timing / liveness model of a stage set executing recompute
// timelines — the planner-side model of the executor.
//
// This restates the reference's CPU executor `simulate()` and
// `stage_period_us()` (proj/src/pipesim.cpp:28-779) with identical semantics:
// per-stage pass order (warm-up forwards, 1F1B pairs, cool-down backwards),
// compute runs merged into elements, window recomputation packed from the
// all-reduce start with spill, critical-path items before their element,
// cool-down stall fill under the budget, and the element-granular memory
// ledger whose peaks are sampled after netting equal-timestamp deltas.
// The GPU runtime replays the same timelines for real; this model supplies
// the plan-time ledger and the predicted schedule it is checked against, and
// the stage period the partitioner and plan selection minimise.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "host/heu.hpp"

namespace lynx::host {

enum class EvKind { Fwd, Bwd, CommFwd, CommBwd, Recompute, StallRecompute, P2P, Stall };
const char* ev_kind_name(EvKind k);

struct Event {
  int stage = 0, microbatch = -1;
  EvKind kind = EvKind::Fwd;
  int op = -1;
  Rat start, end;
  bool overlapped = false;
};

struct StageSummary {
  Rat busy, comm, stall, on_demand, overlapped;
};

struct Breakdown {
  Rat no_recompute, overlapped, on_demand;
};

struct PipeResult {
  Rat iteration_us;
  std::vector<StageSummary> stages;
  std::vector<Breakdown> breakdown;
  std::vector<Rat> peaks;
  std::vector<std::vector<std::pair<Rat, Rat>>> traces;
  std::vector<Event> events;
  std::vector<std::vector<Rat>> pass_starts;  // per stage: start of each pass, in pass order
};

PipeResult run_pipeline(const Profile& p, const std::vector<int>& layers, const std::vector<StageTimeline>& tls,
                        const Rat& p2p_us = Rat(0));
Rat steady_period(const Profile& p, int stage, int stage_layers, const StageTimeline& tl);

// Element structure of one layer pass (shared with the GPU runtime).
struct Element {
  bool comm = false;
  std::vector<int> ops;  // template positions (compute run)
  int op = -1;           // comm op position
  int window = -1;       // window index within the pass kind
  Rat dur;
};
std::vector<Element> layer_elements(const LayerTemplate& layer, const HardwareProfile& hw, bool backward);

// (backward?, microbatch) pass sequence of one stage under 1F1B.
std::vector<std::pair<bool, int>> stage_passes(int n_stages, int stage, int n_microbatches);

std::string trace_csv(const PipeResult& r);
std::string trace_chrome(const PipeResult& r);

}  // namespace lynx::host
