// extern "C" planner entry points (include/lynx_rt.h, "plan" section).
// Each mirrors one reference front-end command (proj/tools/lynx_main.cpp:72-226,
// proj/bindings/module.cpp:18-73) on in-memory JSON text, returns a malloc'd
// string (free with lynx_free) and reports the CLI's exit-code semantics in
// *status. Exceptions never cross the boundary.
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../../include/lynx_rt.h"
#include "host/report.hpp"
#include "lynx_ops_internal.h"

#include <nlohmann/json.hpp>

using namespace lynx::host;

namespace {

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

template <class F>
char* guarded(int* status, F&& f) {
  int st = 0;
  try {
    std::string out = f(st);
    if (status) *status = st;
    return dup(out);
  } catch (const PlanError& e) {
    if (status) *status = lynx::set_error(e.what(), e.status);
  } catch (const std::exception& e) {
    if (status) *status = lynx::set_error(e.what(), kStParse);  // the CLI's catch-all exit code
  }
  return nullptr;
}

std::vector<int> layers_for(const Profile& p, const int* layers, int n) {
  if (layers && n > 0) {
    if (n != p.pipeline.n_stages) throw ValidationError("partition stage count does not match the profile");
    int total = 0;
    for (int i = 0; i < n; ++i) total += layers[i];
    if (total != p.model.n_layers) throw ValidationError("partition layer count does not match the profile");
    return std::vector<int>(layers, layers + n);
  }
  return even_partition(p).layers;
}

PlanMode mode_of(const char* m) {
  const std::string s = m ? m : "heu";
  if (s == "heu") return PlanMode::Heu;
  if (s == "opt") return PlanMode::Opt;
  throw ParseError("--mode must be opt or heu");
}

}  // namespace

extern "C" {

void lynx_free(char* p) { std::free(p); }

char* lynx_plan_validate(const char* profile_json, int lenient, int* status) {
  return guarded(status, [&](int& st) {
    Profile p = parse_profile(profile_json, lenient != 0);
    const StageGraph g =
        expand_stage_graph(p.model, p.model.n_layers, !p.model.embed_ops.empty(), !p.model.head_ops.empty());
    std::string diag = graph_diagnostics(g);
    st = diag.empty() ? 0 : kStValidation;
    return diag;
  });
}

char* lynx_plan_serialize_profile(const char* profile_json, int lenient, int* status) {
  return guarded(status, [&](int&) { return profile_to_json(parse_profile(profile_json, lenient != 0)); });
}

char* lynx_plan_schedule(const char* profile_json, const char* mode, int stage, const int* layers, int n_layers,
                         long long time_limit_ms, int emit_lp, int* status) {
  return guarded(status, [&](int& st) -> std::string {
    Profile p = parse_profile(profile_json);
    if (stage < 0 || stage >= p.pipeline.n_stages) throw ValidationError("--stage out of range");
    const std::vector<int> ls = layers_for(p, layers, n_layers);
    const int L = ls[stage];
    if (mode_of(mode) == PlanMode::Opt) {
      const UnrolledStage u = stage_phase_graph(p, stage, L);
      const OptModel m = opt_model(u.graph, p.hardware, static_share_ceil(p, L));
      if (emit_lp) return to_lp_text(m.prog, "opt_stage_" + std::to_string(stage));
      const PhaseSchedule s = opt_solve(m, time_limit_ms);
      st = s.status == SolveStatus::Infeasible ? kStInfeasible : (s.status != SolveStatus::Optimal ? kStTimedOut : 0);
      return schedule_json(s, stage);
    }
    if (emit_lp) {
      const HeuModel hm = heu_model(p.model.layer, heu_context(p, stage, L));
      return to_lp_text(hm.prog, "heu_stage_" + std::to_string(stage));
    }
    StagePlanner sp(p);
    const StagePlan& plan = sp.plan(stage, L, PlanMode::Heu, time_limit_ms);
    st = plan.timeline.plan.status == SolveStatus::Optimal ? 0 : kStTimedOut;
    return plan_json(plan.timeline.plan, stage);
  });
}

char* lynx_plan_partition(const char* profile_json, const char* mode, long long time_limit_ms, int* status) {
  return guarded(status, [&](int&) {
    Profile p = parse_profile(profile_json);
    return partition_json(greedy_partition(p, mode_of(mode), time_limit_ms));
  });
}

char* lynx_plan_simulate(const char* profile_json, const char* mode, const int* layers, int n_layers,
                         const char* p2p_us, int format, int pybind_semantics, long long time_limit_ms,
                         int* status) {
  return guarded(status, [&](int&) -> std::string {
    Profile p = parse_profile(profile_json);
    const std::vector<int> ls = layers_for(p, layers, n_layers);
    const PlanMode md = mode_of(mode);
    std::vector<StageTimeline> tls;
    if (md == PlanMode::Heu || pybind_semantics) {
      StagePlanner sp(p);
      for (int s = 0; s < p.pipeline.n_stages; ++s) tls.push_back(sp.plan(s, ls[s], md, time_limit_ms).timeline);
    } else {
      for (int s = 0; s < p.pipeline.n_stages; ++s) {
        const UnrolledStage u = stage_phase_graph(p, s, ls[s]);
        const OptModel m = opt_model(u.graph, p.hardware, static_share_ceil(p, ls[s]));
        const PhaseSchedule sch = opt_solve(m, time_limit_ms);
        if (sch.status == SolveStatus::Infeasible) throw BudgetInfeasible("stage " + std::to_string(s));
        tls.push_back(timeline_from_schedule(p, s, ls[s], sch, u));
      }
    }
    auto p2p = parse_rat(p2p_us ? p2p_us : "0");
    if (!p2p || p2p->sign() < 0) throw ValidationError("--p2p-us must be a non-negative rational");
    const PipeResult r = run_pipeline(p, ls, tls, *p2p);
    if (format == 1) return trace_csv(r);
    if (format == 2) return trace_chrome(r);
    if (format == 3) return breakdown_text(r);
    return simreport_json(r);
  });
}

char* lynx_plan_stage(const char* profile_json, int stage, const int* layers, int n_layers, int baseline,
                      long long time_limit_ms, int* status) {
  return guarded(status, [&](int&) -> std::string {
    Profile p = parse_profile(profile_json);
    const std::vector<int> ls = layers_for(p, layers, n_layers);
    if (stage < 0 || stage >= p.pipeline.n_stages) throw ValidationError("stage out of range");
    StageTimeline tl;
    Rat period;
    std::string pj;
    if (baseline == 0) {
      StagePlanner sp(p);
      const StagePlan& plan = sp.plan(stage, ls[stage], PlanMode::Heu, time_limit_ms);
      tl = plan.timeline;
      period = plan.period_us;
      pj = plan_json(tl.plan, stage);
    } else {  // 1 = full recompute (Megatron full), 2 = retain all (no recompute), 3 = Megatron selective
      if (baseline < 1 || baseline > 3) throw ValidationError("baseline must be 0 (heu), 1, 2 or 3");
      const HeuCtx ctx = heu_context(p, stage, ls[stage]);
      const LayerPlan plan = baseline == 2   ? retain_all(p.model.layer, ctx)
                             : baseline == 3 ? selective_recompute(p.model.layer, ctx)
                                             : full_recompute(p.model.layer, ctx);
      tl = expand_to_stage(plan, ctx, p.pipeline, stage);
      period = steady_period(p, stage, ls[stage], tl);
      pj = plan_json(plan, stage);
    }
    nlohmann::ordered_json j;
    j["plan_json"] = pj;
    j["timeline"] = nlohmann::ordered_json::parse(timeline_json(tl));
    j["period_us"] = to_canonical(period);
    j["layers_per_stage"] = ls;
    return j.dump();
  });
}

char* lynx_plan_simulate_timelines(const char* profile_json, const int* layers, int n_layers,
                                   const char* timelines_json, const char* p2p_us, int* status) {
  return guarded(status, [&](int&) -> std::string {
    Profile p = parse_profile(profile_json);
    const std::vector<int> ls(layers, layers + n_layers);
    const std::vector<StageTimeline> tls = parse_timelines(timelines_json);
    auto p2p = parse_rat(p2p_us ? p2p_us : "0");
    if (!p2p) throw ValidationError("bad p2p_us");
    const PipeResult r = run_pipeline(p, ls, tls, *p2p);
    nlohmann::ordered_json j;
    j["report"] = nlohmann::ordered_json::parse(simreport_json(r));
    j["iteration_us_exact"] = to_canonical(r.iteration_us);
    nlohmann::ordered_json traces = nlohmann::ordered_json::array();
    for (const auto& tr : r.traces) {
      nlohmann::ordered_json a = nlohmann::ordered_json::array();
      for (const auto& [t, b] : tr) a.push_back({to_canonical(t), to_canonical(b)});
      traces.push_back(a);
    }
    j["memory_traces"] = traces;
    nlohmann::ordered_json peaks = nlohmann::ordered_json::array();
    for (const auto& pk : r.peaks) peaks.push_back(to_canonical(pk));
    j["memory_peaks"] = peaks;
    j["csv"] = trace_csv(r);
    return j.dump();
  });
}

char* lynx_plan_solve_heu(const char* profile_json, int stage, int stage_layers, int policy,
                          const char* delta_bytes, long long time_limit_ms, int* status) {
  return guarded(status, [&](int&) -> std::string {
    Profile p = parse_profile(profile_json);
    auto delta = parse_rat(delta_bytes ? delta_bytes : "0");
    if (!delta) throw ValidationError("bad delta_bytes");
    const HeuCtx ctx =
        heu_context(p, stage, stage_layers, policy ? Reserve::Unretained : Reserve::FixedBytes, *delta);
    const HeuModel hm = heu_model(p.model.layer, ctx);
    LayerPlan plan = heu_solve(hm, time_limit_ms);
    plan.peak_bytes = plan_peak(plan, ctx, p.model.layer);
    nlohmann::ordered_json j;
    j["plan_json"] = plan_json(plan, stage);
    j["n_vars"] = hm.prog.size();
    j["n_cons"] = static_cast<int>(hm.prog.rows().size());
    j["lp"] = to_lp_text(hm.prog, "heu_stage_" + std::to_string(stage));
    j["check"] = plan_violations(plan, ctx, p.model.layer);
    j["timeline"] = nlohmann::ordered_json::parse(timeline_json(expand_to_stage(plan, ctx, p.pipeline, stage)));
    return j.dump();
  });
}

}  // extern "C"
