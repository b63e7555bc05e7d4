// extern "C" planner entry points (include/lynx_rt.h, "plan" section).
// Each mirrors one reference front-end command (proj/tools/lynx_main.cpp:72-226,
// proj/bindings/module.cpp:18-73) on in-memory JSON text, returns a malloc'd
// string (free with lynx_free) and reports the CLI's exit-code semantics in
// *status. Exceptions never cross the boundary.
#include <cstdlib>
#include <map>
#include <set>
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

// OPT over a slice of `slice` consecutive layers of an L-layer stage: the
// unrolled phase grid of the full stage is Θ(n²) booleans (~10^6 at 7B), the slice's is small
// enough for an external MILP solver. The slice is solved for replication over the stage: one
// extra continuous variable Y bounds the slice's retained bytes at every phase entry
// (schedulable ops only: the embedding / head tensors are not replicated), and every ledger
// point carries the other L/k - 1 copies' Y on top: U_t_k + (L/k - 1) Y <= budget. The budget is
// the slice's static share plus the stage's activation budget minus `reserve` bytes (null: 0).
struct OptSlice {
  Profile p;
  int L = 0, k = 0;
  UnrolledStage u;
  OptModel m;
};

OptSlice opt_slice(const char* profile_json, int stage, const int* layers, int n_layers, int slice,
                   const char* reserve_bytes) {
  OptSlice o;
  o.p = parse_profile(profile_json);
  if (stage < 0 || stage >= o.p.pipeline.n_stages) throw ValidationError("stage out of range");
  o.L = layers_for(o.p, layers, n_layers)[stage];
  o.k = slice <= 0 ? o.L : slice;
  if (o.k > o.L || o.L % o.k != 0) throw ValidationError("slice_layers must divide the stage's layer count");
  const Rat st_L(static_share_ceil(o.p, o.L)), st_k(static_share_ceil(o.p, o.k));
  const Rat act = Rat(o.p.hardware.mem_budget_bytes) - st_L;
  Rat reserve(0);
  if (reserve_bytes && *reserve_bytes) {
    auto r = parse_rat(reserve_bytes);
    if (!r || r->sign() < 0) throw ValidationError("reserve_bytes must be a non-negative rational");
    reserve = *r;
  }
  if ((act - reserve).sign() <= 0) throw BudgetTooSmall("no activation budget left for the slice");
  HardwareProfile hw = o.p.hardware;
  const Rat b = st_k + act - reserve;
  hw.mem_budget_bytes = (b.num() / b.den()).to_i64();
  o.u = stage_phase_graph(o.p, stage, o.k);
  o.m = opt_model(o.u.graph, hw, static_share_ceil(o.p, o.k));
  const int copies = o.L / o.k - 1;
  if (copies > 0) {
    Program& P = o.m.prog;
    const StageGraph& g = o.u.graph;
    const int n_before = P.size();
    const int y = P.new_cont("Y_retained", Rat(0), Rat(hw.mem_budget_bytes));
    for (int t = 1; t < g.size(); ++t) {
      Linear e;
      e.add(1, y);
      for (int i = 0; i < t; ++i)
        if (g.schedulable[i] && g.ops[i].out_bytes > 0) e.add(Rat(-g.ops[i].out_bytes), o.m.S[t][i]);
      P.add_row(std::move(e), Sense::Ge, 0, "retained_" + std::to_string(t));
    }
    for (int v = 0; v < n_before; ++v)
      if (P.type(v) == VarType::Cont && P.name(v).rfind("U_", 0) == 0)
        P.add_row(Linear().add(1, v).add(copies, y), Sense::Le, Rat(hw.mem_budget_bytes), "copies_" + P.name(v));
  }
  return o;
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
    nlohmann::ordered_json starts = nlohmann::ordered_json::array();  // per stage, in pass order
    for (const auto& st : r.pass_starts) {
      nlohmann::ordered_json a = nlohmann::ordered_json::array();
      for (const Rat& t : st) a.push_back(to_canonical(t));
      starts.push_back(a);
    }
    j["pass_start_us"] = starts;
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

char* lynx_plan_opt_export(const char* profile_json, int stage, const int* layers, int n_layers, int slice_layers,
                           const char* reserve_bytes, int* status) {
  return guarded(status, [&](int&) -> std::string {
    const OptSlice o = opt_slice(profile_json, stage, layers, n_layers, slice_layers, reserve_bytes);
    const Program& P = o.m.prog;
    nlohmann::ordered_json j;
    j["stage"] = stage;
    j["stage_layers"] = o.L;
    j["slice_layers"] = o.k;
    j["n_ops"] = o.u.graph.size();
    j["budget_bytes"] = o.m.budget;
    j["static_bytes"] = o.m.static_bytes;
    j["stage_activation_bytes"] = to_canonical(Rat(o.p.hardware.mem_budget_bytes) - Rat(static_share_ceil(o.p, o.L)));
    nlohmann::ordered_json lo = nlohmann::ordered_json::array(), hi = lo, integ = lo;
    for (int v = 0; v < P.size(); ++v) {
      lo.push_back(P.lo(v).to_double());
      hi.push_back(P.hi(v).to_double());
      integ.push_back(P.type(v) == VarType::Bool ? 1 : 0);
    }
    j["n_vars"] = P.size();
    j["lo"] = lo;
    j["hi"] = hi;
    j["integer"] = integ;
    nlohmann::ordered_json c = nlohmann::ordered_json::array();
    for (const auto& [v, k] : P.objective().coef) c.push_back({v, k.to_double()});
    j["objective"] = c;
    // rows in coordinate form: row index, var, coefficient; sense -1 (<=), 0 (=), 1 (>=)
    nlohmann::ordered_json ri = nlohmann::ordered_json::array(), vi = ri, cv = ri, sense = ri, rhs = ri;
    int r = 0;
    for (const Row& row : P.rows()) {
      for (const auto& [v, k] : row.lhs.coef) {
        ri.push_back(r);
        vi.push_back(v);
        cv.push_back(k.to_double());
      }
      sense.push_back(row.sense == Sense::Le ? -1 : (row.sense == Sense::Eq ? 0 : 1));
      rhs.push_back((row.rhs - row.lhs.constant).to_double());
      ++r;
    }
    j["n_rows"] = r;
    j["row"] = ri;
    j["col"] = vi;
    j["val"] = cv;
    j["sense"] = sense;
    j["rhs"] = rhs;
    nlohmann::ordered_json R = nlohmann::ordered_json::array(), S = R;
    for (int t = 0; t < o.u.graph.size(); ++t) {
      R.push_back(o.m.R[t]);
      S.push_back(o.m.S[t]);
    }
    j["R"] = R;
    j["S"] = S;
    return j.dump();
  });
}

char* lynx_plan_opt_timeline(const char* profile_json, int stage, const int* layers, int n_layers, int slice_layers,
                             const char* reserve_bytes, const char* schedule, int* status) {
  return guarded(status, [&](int& st) -> std::string {
    const OptSlice o = opt_slice(profile_json, stage, layers, n_layers, slice_layers, reserve_bytes);
    const auto in = nlohmann::json::parse(schedule);
    PhaseSchedule s;
    s.status = SolveStatus::Optimal;
    if (in.contains("status") && in["status"].get<std::string>() != "optimal") s.status = SolveStatus::Feasible;
    for (const auto& pr : in["keep"]) s.keep.emplace_back(pr[0].get<int>(), pr[1].get<int>());
    for (const auto& pr : in["recompute"]) s.recompute.emplace_back(pr[0].get<int>(), pr[1].get<int>());
    const int n = o.u.graph.size();
    s.cost_us = Rat(0);
    for (int t = 0; t < n; ++t) s.cost_us += o.m.cost[t];
    for (auto [t, i] : s.recompute) {
      if (t < 0 || t >= n || i < 0 || i >= t) continue;  // reported by schedule_issues
      if (o.u.graph.is_comm(t)) s.overlapped.emplace_back(t, i);
      else s.cost_us += o.m.cost[i];
    }
    const std::string issues = schedule_issues(s, o.m);
    nlohmann::ordered_json j;
    j["issues"] = issues;
    j["cost_us"] = to_canonical(s.cost_us);
    j["n_recompute"] = static_cast<int>(s.recompute.size());
    j["n_overlapped"] = static_cast<int>(s.overlapped.size());
    if (!issues.empty()) {
      st = kStValidation;
      return j.dump();
    }
    std::vector<bool> in_layer;
    const StageTimeline slice_tl = timeline_from_schedule(o.p, stage, o.k, s, o.u, &in_layer);
    StageTimeline tl = slice_tl;
    tl.items.clear();
    const int copies = o.L / o.k;
    for (int r = 0; r < copies; ++r) {
      for (size_t x = 0; x < slice_tl.items.size(); ++x) {
        Recompute it = slice_tl.items[x];
        it.owner_layer += r * o.k;
        if (in_layer[x]) {
          it.host_layer += r * o.k;
        } else {
          // timeline_from_opt_schedule files hosts outside the layers (embedding / head phases) as
          // CriticalPath at layer 0, elem 0 — in the backward that is after every other layer's
          // consumer. The executor needs the copy before its consumer: regenerate on demand at
          // the start of the owner layer's backward instead.
          it.host = Recompute::Host::Critical;
          it.host_mb = it.owner_mb;
          it.host_bwd = true;
          it.host_layer = it.owner_layer;
          it.host_elem = 0;
        }
        tl.items.push_back(it);
      }
    }
    // timeline_from_opt_schedule marks an op discarded for every (microbatch, layer) once any of
    // its instances is recomputed (aggregate retention, report_io.cpp:249-261), while OPT may have
    // kept other instances; the reference simulator tolerates the gap (strict_deps = false), the
    // executor frees a discarded tensor and needs its copy. An owner (microbatch, layer) missing
    // a discarded op gets all its regenerations on demand at the start of its backward, in op
    // order (dependencies first).
    {
      const int nf = o.p.model.layer.n_fwd();
      std::vector<int> discarded;
      for (int i = 0; i < nf; ++i)
        if (!tl.plan.retained[i]) discarded.push_back(i);
      std::map<std::pair<int, int>, std::set<int>> have;
      for (const Recompute& it : tl.items) have[{it.owner_mb, it.owner_layer}].insert(it.op);
      std::set<std::pair<int, int>> rebuild;
      for (int mb = 0; mb < o.p.pipeline.n_microbatches; ++mb)
        for (int l = 0; l < o.L; ++l)
          for (int i : discarded)
            if (!have[{mb, l}].count(i)) rebuild.insert({mb, l});
      if (!rebuild.empty()) {
        std::vector<Recompute> kept;
        for (const Recompute& it : tl.items)
          if (!rebuild.count({it.owner_mb, it.owner_layer})) kept.push_back(it);
        for (auto [mb, l] : rebuild)
          for (int i : discarded) {
            Recompute it;
            it.owner_mb = mb;
            it.owner_layer = l;
            it.op = i;
            it.host = Recompute::Host::Critical;
            it.host_mb = mb;
            it.host_bwd = true;
            it.host_layer = l;
            it.host_elem = 0;
            kept.push_back(it);
          }
        tl.items = std::move(kept);
      }
      j["completed_owners"] = static_cast<int>(rebuild.size());
    }
    j["timeline"] = nlohmann::ordered_json::parse(timeline_json(tl));
    j["slice_items"] = static_cast<int>(slice_tl.items.size());
    return j.dump();
  });
}

}  // extern "C"
