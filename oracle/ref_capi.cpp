// TEST INFRASTRUCTURE ONLY — C-ABI wrapper over the reference's own lynx_core,
// compiled from the unmodified sources in /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/liblynx_ref.so. Only tests/, bench.py's
// cpu_baseline / --impl reference legs and __graft_entry__.smoke() load it, as
// the checker. Every entry point returns a malloc'd JSON string (free with
// lynx_ref_free) or NULL, with the exception text in lynx_ref_last_error().
//
// The functions mirror the reference's front-ends:
//   lynx_ref_schedule   ~ cmd_schedule / _lynx.schedule   (lynx_main.cpp:117-157, module.cpp:18-33)
//   lynx_ref_partition  ~ cmd_partition / _lynx.partition (lynx_main.cpp:159-171)
//   lynx_ref_simulate   ~ cmd_simulate (HEU branch)        (lynx_main.cpp:200-226)
//   lynx_ref_stage_plan ~ PlanCache::stage_plan + the expanded RecomputeItem list
//   lynx_ref_simulate_timelines ~ simulate() on caller-provided timelines
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include <nlohmann/json.hpp>

#include "lynx/heusched.hpp"
#include "lynx/optsched.hpp"
#include "lynx/partition.hpp"
#include "lynx/pipesim.hpp"
#include "lynx/profile.hpp"
#include "lynx/report_io.hpp"

using nlohmann::ordered_json;
using namespace lynx;

namespace {

thread_local std::string g_err;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

const char* host_name(RecomputeItem::Host h) {
  switch (h) {
    case RecomputeItem::Host::Window: return "window";
    case RecomputeItem::Host::CriticalPath: return "critical";
    case RecomputeItem::Host::StallFill: return "stall";
  }
  return "?";
}

const char* status_name(SolStatus s) {
  switch (s) {
    case SolStatus::Optimal: return "optimal";
    case SolStatus::Feasible: return "feasible";
    case SolStatus::Infeasible: return "infeasible";
    case SolStatus::TimedOut: return "timed_out";
  }
  return "?";
}

SolStatus status_of(const std::string& s) {
  if (s == "optimal") return SolStatus::Optimal;
  if (s == "feasible") return SolStatus::Feasible;
  if (s == "timed_out") return SolStatus::TimedOut;
  return SolStatus::Infeasible;
}

ordered_json timeline_to_json(const StageRecomputeTimeline& tl) {
  ordered_json j;
  j["stage"] = tl.stage;
  j["role"] = tl.role == StageRole::LastStage ? "last" : "interior";
  j["strict_deps"] = tl.strict_deps;
  ordered_json p;
  p["status"] = status_name(tl.plan.status);
  p["retained"] = ordered_json::array();
  for (bool b : tl.plan.retained) p["retained"].push_back(b);
  p["phase"] = tl.plan.phase;
  p["critical_path_us"] = rat_to_string(tl.plan.critical_path_us);
  p["peak_bytes"] = rat_to_string(tl.plan.peak_bytes);
  p["delta_bytes"] = rat_to_string(tl.plan.delta_bytes);
  p["role"] = tl.plan.role == StageRole::LastStage ? "last" : "interior";
  j["plan"] = p;
  ordered_json items = ordered_json::array();
  for (const auto& it : tl.items) {
    ordered_json i;
    i["owner_mb"] = it.owner_mb;
    i["owner_layer"] = it.owner_layer;
    i["op"] = it.op;
    i["host"] = host_name(it.host);
    i["host_mb"] = it.host_mb;
    i["host_backward"] = it.host_backward;
    i["host_layer"] = it.host_layer;
    i["host_window"] = it.host_window;
    i["host_elem"] = it.host_elem;
    items.push_back(i);
  }
  j["items"] = items;
  return j;
}

StageRecomputeTimeline timeline_from_json(const ordered_json& j) {
  StageRecomputeTimeline tl;
  tl.stage = j.at("stage").get<int>();
  tl.role = j.at("role").get<std::string>() == "last" ? StageRole::LastStage : StageRole::Interior;
  tl.strict_deps = j.value("strict_deps", true);
  const auto& p = j.at("plan");
  tl.plan.status = status_of(p.value("status", std::string("optimal")));
  for (const auto& b : p.at("retained")) tl.plan.retained.push_back(b.get<bool>());
  tl.plan.phase = p.at("phase").get<std::vector<int>>();
  tl.plan.critical_path_us = *rat_parse(p.value("critical_path_us", std::string("0")));
  tl.plan.peak_bytes = *rat_parse(p.value("peak_bytes", std::string("0")));
  tl.plan.delta_bytes = *rat_parse(p.value("delta_bytes", std::string("0")));
  tl.plan.role = tl.role;
  for (const auto& i : j.at("items")) {
    RecomputeItem it;
    it.owner_mb = i.at("owner_mb");
    it.owner_layer = i.at("owner_layer");
    it.op = i.at("op");
    std::string h = i.at("host");
    it.host = h == "window" ? RecomputeItem::Host::Window
                            : (h == "stall" ? RecomputeItem::Host::StallFill
                                            : RecomputeItem::Host::CriticalPath);
    it.host_mb = i.at("host_mb");
    it.host_backward = i.at("host_backward");
    it.host_layer = i.at("host_layer");
    it.host_window = i.at("host_window");
    it.host_elem = i.at("host_elem");
    tl.items.push_back(it);
  }
  return tl;
}

std::vector<int> layers_or_initial(const Profile& p, const int* layers, int n) {
  if (layers && n > 0) return std::vector<int>(layers, layers + n);
  return initial_partition(p).layers_per_stage;
}

template <class F>
char* guard(F&& f) {
  try {
    g_err.clear();
    return dup(f());
  } catch (const std::exception& e) {
    g_err = std::string(typeid(e).name()) + ": " + e.what();
    return nullptr;
  }
}

}  // namespace

extern "C" {

const char* lynx_ref_last_error() { return g_err.c_str(); }
void lynx_ref_free(char* p) { std::free(p); }

char* lynx_ref_serialize_profile(const char* profile_json, int lenient) {
  return guard([&] { return serialize_profile(load_profile_string(profile_json, lenient != 0)); });
}

// HEU stage plan exactly as `lynx schedule --mode heu` prints it, plus the
// expanded timeline and the simulated stage period.
char* lynx_ref_stage_plan(const char* profile_json, int stage, const int* layers, int n_layers,
                          long long time_limit_ms) {
  return guard([&] {
    Profile p = load_profile_string(profile_json);
    std::vector<int> ls = layers_or_initial(p, layers, n_layers);
    PlanCache cache(p);
    const StagePlan& sp = cache.stage_plan(stage, ls[stage], PlanMode::Heu, time_limit_ms);
    ordered_json j;
    j["plan_json"] = plan_to_json(sp.timeline.plan, stage);
    j["timeline"] = timeline_to_json(sp.timeline);
    j["period_us"] = rat_to_string(sp.duration_us);
    j["layers_per_stage"] = ls;
    return j.dump();
  });
}

// Fixed baseline plans (heusched.cpp:313-341) expanded for a stage.
char* lynx_ref_fixed_plan(const char* profile_json, int stage, const int* layers, int n_layers,
                          int retain_all) {
  return guard([&] {
    Profile p = load_profile_string(profile_json);
    std::vector<int> ls = layers_or_initial(p, layers, n_layers);
    HeuContext ctx = make_heu_context(p, stage, ls[stage]);
    LayerPhasePlan plan = retain_all ? retain_all_plan(p.model.layer, ctx)
                                     : full_recompute_plan(p.model.layer, ctx);
    StageRecomputeTimeline tl = expand_plan_to_stage(plan, ctx, p.pipeline, stage);
    ordered_json j;
    j["plan_json"] = plan_to_json(plan, stage);
    j["timeline"] = timeline_to_json(tl);
    j["period_us"] = rat_to_string(stage_period_us(p, stage, ls[stage], tl));
    return j.dump();
  });
}

// Solve HEU for an explicit context (policy 0 = FixedBytes, 1 = ReserveUnretained).
char* lynx_ref_solve_heu(const char* profile_json, int stage, int stage_layers, int policy,
                         const char* delta_bytes, long long time_limit_ms) {
  return guard([&] {
    Profile p = load_profile_string(profile_json);
    HeuContext ctx = make_heu_context(p, stage, stage_layers,
                                      policy ? DeltaPolicy::ReserveUnretained : DeltaPolicy::FixedBytes,
                                      *rat_parse(delta_bytes));
    HeuModelInstance inst = build_heu_model(p.model.layer, ctx);
    LayerPhasePlan plan = solve_heu(inst, time_limit_ms);
    plan.peak_bytes = plan_peak_bytes(plan, ctx, p.model.layer);
    ordered_json j;
    j["plan_json"] = plan_to_json(plan, stage);
    j["n_vars"] = inst.model.var_count();
    j["n_cons"] = static_cast<int>(inst.model.constraints().size());
    j["lp"] = write_lp(inst.model, "heu_stage_" + std::to_string(stage));
    j["check"] = check_plan(plan, ctx, p.model.layer);
    j["timeline"] = timeline_to_json(expand_plan_to_stage(plan, ctx, p.pipeline, stage));
    return j.dump();
  });
}

char* lynx_ref_partition(const char* profile_json, long long time_limit_ms) {
  return guard([&] {
    Profile p = load_profile_string(profile_json);
    return partition_to_json(search_partition(p, PlanMode::Heu, time_limit_ms));
  });
}

// `lynx simulate --mode heu` (format 0 json, 1 csv, 2 chrome-trace, 3 report table).
char* lynx_ref_simulate(const char* profile_json, const int* layers, int n_layers,
                        const char* p2p_us, int format, long long time_limit_ms) {
  return guard([&] {
    Profile p = load_profile_string(profile_json);
    std::vector<int> ls = layers_or_initial(p, layers, n_layers);
    PlanCache cache(p);
    std::vector<StageRecomputeTimeline> tls;
    for (int s = 0; s < p.pipeline.n_stages; ++s)
      tls.push_back(cache.stage_plan(s, ls[s], PlanMode::Heu, time_limit_ms).timeline);
    SimOptions opts;
    opts.p2p_us = *rat_parse(p2p_us);
    SimReport r = simulate(p, ls, tls, opts);
    if (format == 1) return emit_trace(r, TraceFormat::Csv);
    if (format == 2) return emit_trace(r, TraceFormat::ChromeTrace);
    if (format == 3) return breakdown_table(r);
    return simreport_to_json(r);
  });
}

// simulate() on caller-provided timelines (JSON array, one per stage) plus the
// exact memory traces, which simreport_to_json does not carry.
char* lynx_ref_simulate_timelines(const char* profile_json, const int* layers, int n_layers,
                                  const char* timelines_json, const char* p2p_us) {
  return guard([&] {
    Profile p = load_profile_string(profile_json);
    std::vector<int> ls(layers, layers + n_layers);
    std::vector<StageRecomputeTimeline> tls;
    for (const auto& t : ordered_json::parse(timelines_json)) tls.push_back(timeline_from_json(t));
    SimOptions opts;
    opts.p2p_us = *rat_parse(p2p_us);
    SimReport r = simulate(p, ls, tls, opts);
    ordered_json j;
    j["report"] = ordered_json::parse(simreport_to_json(r));
    j["iteration_us_exact"] = rat_to_string(r.iteration_us);
    ordered_json traces = ordered_json::array();
    for (const auto& tr : r.memory_traces) {
      ordered_json a = ordered_json::array();
      for (const auto& [t, b] : tr) a.push_back({rat_to_string(t), rat_to_string(b)});
      traces.push_back(a);
    }
    j["memory_traces"] = traces;
    ordered_json peaks = ordered_json::array();
    for (const auto& pk : r.memory_peaks) peaks.push_back(rat_to_string(pk));
    j["memory_peaks"] = peaks;
    j["csv"] = emit_trace(r, TraceFormat::Csv);
    return j.dump();
  });
}

char* lynx_ref_stage_period(const char* profile_json, int stage, int stage_layers,
                            const char* timeline_json) {
  return guard([&] {
    Profile p = load_profile_string(profile_json);
    StageRecomputeTimeline tl = timeline_from_json(ordered_json::parse(timeline_json));
    return rat_to_string(stage_period_us(p, stage, stage_layers, tl));
  });
}

}  // extern "C"
