#include "host/report.hpp"

#include <iomanip>
#include <sstream>

#include <nlohmann/json.hpp>

namespace lynx::host {

using Json = nlohmann::ordered_json;

namespace {
Json pairs(const std::vector<std::pair<int, int>>& v) {
  Json a = Json::array();
  for (auto [t, i] : v) a.push_back(Json::array({t, i}));
  return a;
}
const char* host_text(Recompute::Host h) {
  switch (h) {
    case Recompute::Host::Window: return "window";
    case Recompute::Host::Critical: return "critical";
    case Recompute::Host::Stall: return "stall";
  }
  return "?";
}
SolveStatus status_from(const std::string& s) {
  if (s == "optimal") return SolveStatus::Optimal;
  if (s == "feasible") return SolveStatus::Feasible;
  if (s == "timed_out") return SolveStatus::TimedOut;
  return SolveStatus::Infeasible;
}
Rat rat_field(const Json& j, const char* key) {
  if (!j.contains(key)) return Rat(0);
  auto r = parse_rat(j.at(key).get<std::string>());
  if (!r) throw ParseError(std::string("bad rational in timeline field ") + key);
  return *r;
}
Json timeline_obj(const StageTimeline& tl) {
  Json j;
  j["stage"] = tl.stage;
  j["role"] = tl.role == Role::Last ? "last" : "interior";
  j["strict_deps"] = tl.strict_deps;
  Json p;
  p["status"] = status_text(tl.plan.status);
  p["retained"] = Json::array();
  for (bool b : tl.plan.retained) p["retained"].push_back(b);
  p["phase"] = tl.plan.phase;
  p["critical_path_us"] = to_canonical(tl.plan.critical_us);
  p["peak_bytes"] = to_canonical(tl.plan.peak_bytes);
  p["delta_bytes"] = to_canonical(tl.plan.delta_bytes);
  p["role"] = tl.plan.role == Role::Last ? "last" : "interior";
  j["plan"] = p;
  Json items = Json::array();
  for (const Recompute& it : tl.items) {
    Json i;
    i["owner_mb"] = it.owner_mb;
    i["owner_layer"] = it.owner_layer;
    i["op"] = it.op;
    i["host"] = host_text(it.host);
    i["host_mb"] = it.host_mb;
    i["host_backward"] = it.host_bwd;
    i["host_layer"] = it.host_layer;
    i["host_window"] = it.host_window;
    i["host_elem"] = it.host_elem;
    items.push_back(i);
  }
  j["items"] = items;
  return j;
}
StageTimeline timeline_from(const Json& j) {
  StageTimeline tl;
  tl.stage = j.at("stage").get<int>();
  tl.role = j.at("role").get<std::string>() == "last" ? Role::Last : Role::Interior;
  tl.strict_deps = j.value("strict_deps", true);
  const Json& p = j.at("plan");
  tl.plan.status = status_from(p.value("status", std::string("optimal")));
  for (const auto& b : p.at("retained")) tl.plan.retained.push_back(b.get<bool>());
  tl.plan.phase = p.at("phase").get<std::vector<int>>();
  tl.plan.critical_us = rat_field(p, "critical_path_us");
  tl.plan.peak_bytes = rat_field(p, "peak_bytes");
  tl.plan.delta_bytes = rat_field(p, "delta_bytes");
  tl.plan.role = tl.role;
  for (const auto& i : j.at("items")) {
    Recompute it;
    it.owner_mb = i.at("owner_mb");
    it.owner_layer = i.at("owner_layer");
    it.op = i.at("op");
    const std::string h = i.at("host");
    it.host = h == "window" ? Recompute::Host::Window
                            : (h == "stall" ? Recompute::Host::Stall : Recompute::Host::Critical);
    it.host_mb = i.at("host_mb");
    it.host_bwd = i.at("host_backward");
    it.host_layer = i.at("host_layer");
    it.host_window = i.at("host_window");
    it.host_elem = i.at("host_elem");
    tl.items.push_back(it);
  }
  return tl;
}
}  // namespace

std::string plan_json(const LayerPlan& plan, int stage) {
  Json j;
  j["stage"] = stage;
  j["role"] = plan.role == Role::Last ? "last" : "interior";
  j["status"] = status_text(plan.status);
  Json s = Json::array();
  for (size_t i = 0; i < plan.retained.size(); ++i)
    if (plan.retained[i]) s.push_back(static_cast<int>(i));
  j["S"] = s;
  Json ph = Json::object();
  for (size_t i = 0; i < plan.retained.size(); ++i)
    if (!plan.retained[i]) ph[std::to_string(i)] = plan.phase[i];
  j["phase_assignment"] = ph;
  j["objective_us"] = to_canonical(plan.critical_us);
  j["peak_bytes"] = to_canonical(plan.peak_bytes);
  j["delta_bytes"] = to_canonical(plan.delta_bytes);
  return j.dump(2) + "\n";
}

std::string schedule_json(const PhaseSchedule& s, int stage) {
  Json j;
  j["stage"] = stage;
  j["status"] = status_text(s.status);
  j["objective_us"] = to_canonical(s.cost_us);
  if (s.status == SolveStatus::Feasible) j["bound_gap_us"] = to_canonical(s.gap);
  j["keep"] = pairs(s.keep);
  j["recompute"] = pairs(s.recompute);
  j["overlapped"] = pairs(s.overlapped);
  j["peak_bytes"] = Json::array();  // never filled by the reference either (optsched.hpp:50)
  return j.dump(2) + "\n";
}

std::string partition_json(const Partition& part) {
  Json j;
  j["layers_per_stage"] = part.layers;
  Json d = Json::array();
  for (const Rat& r : part.durations) d.push_back(to_fixed(r, 3));
  j["durations_us"] = d;
  j["mode"] = part.mode == PlanMode::Opt ? "opt" : "heu";
  j["iterations"] = part.iterations;
  Json mv = Json::array();
  for (const Move& m : part.moves) {
    Json o;
    o["from"] = m.from;
    o["to"] = m.to;
    o["accepted"] = m.accepted;
    mv.push_back(o);
  }
  j["moves"] = mv;
  return j.dump(2) + "\n";
}

std::string simreport_json(const PipeResult& r) {
  Json j;
  j["iteration_us"] = to_fixed(r.iteration_us, 3);
  Json st = Json::array();
  for (const auto& s : r.stages) {
    Json o;
    o["busy_us"] = to_fixed(s.busy, 3);
    o["comm_us"] = to_fixed(s.comm, 3);
    o["stall_us"] = to_fixed(s.stall, 3);
    o["recompute_on_demand_us"] = to_fixed(s.on_demand, 3);
    o["recompute_overlapped_us"] = to_fixed(s.overlapped, 3);
    st.push_back(o);
  }
  j["per_stage"] = st;
  Json bd = Json::array();
  for (const auto& b : r.breakdown) {
    Json o;
    o["no_recompute"] = to_fixed(b.no_recompute, 4);
    o["overlapped"] = to_fixed(b.overlapped, 4);
    o["on_demand"] = to_fixed(b.on_demand, 4);
    bd.push_back(o);
  }
  j["breakdown"] = bd;
  Json pk = Json::array();
  for (const Rat& p : r.peaks) pk.push_back(to_canonical(p));
  j["memory_peaks"] = pk;
  Json ev = Json::array();
  for (const Event& e : r.events) {
    Json o;
    o["stage"] = e.stage;
    o["microbatch"] = e.microbatch;
    o["kind"] = ev_kind_name(e.kind);
    if (e.op >= 0) o["op_id"] = e.op;
    o["start_us"] = to_fixed(e.start, 3);
    o["end_us"] = to_fixed(e.end, 3);
    o["overlapped"] = e.overlapped;
    ev.push_back(o);
  }
  j["timeline"] = ev;
  return j.dump(2) + "\n";
}

std::string breakdown_text(const PipeResult& r) {
  std::ostringstream os;
  os << "stage  no_recompute  overlapped  on_demand  iteration_us\n";
  for (size_t s = 0; s < r.breakdown.size(); ++s) {
    const auto& b = r.breakdown[s];
    os << std::left << std::setw(7) << s << std::setw(14) << to_fixed(b.no_recompute, 4) << std::setw(12)
       << to_fixed(b.overlapped, 4) << std::setw(11) << to_fixed(b.on_demand, 4);
    if (s == 0) os << to_fixed(r.iteration_us, 3);
    os << "\n";
  }
  return os.str();
}

PartitionDoc parse_partition(const std::string& text) {
  Json j;
  try {
    j = Json::parse(text);
  } catch (const nlohmann::json::exception& e) {
    throw ParseError(std::string("malformed partition document: ") + e.what());
  }
  PartitionDoc d;
  if (!j.contains("layers_per_stage")) throw ValidationError("partition document lacks layers_per_stage");
  d.layers = j["layers_per_stage"].get<std::vector<int>>();
  for (int l : d.layers)
    if (l < 1) throw ValidationError("layers_per_stage entries must be positive");
  if (j.contains("mode")) {
    d.has_mode = true;
    const std::string m = j["mode"].get<std::string>();
    if (m == "opt") {
      d.mode = PlanMode::Opt;
    } else if (m == "heu") {
      d.mode = PlanMode::Heu;
    } else {
      throw ValidationError("unknown partition mode '" + m + "'");
    }
  }
  return d;
}

std::string timeline_json(const StageTimeline& tl) { return timeline_obj(tl).dump(); }

StageTimeline parse_timeline(const std::string& text) {
  try {
    return timeline_from(Json::parse(text));
  } catch (const nlohmann::json::exception& e) {
    throw ParseError(std::string("malformed timeline document: ") + e.what());
  }
}

std::vector<StageTimeline> parse_timelines(const std::string& text) {
  try {
    std::vector<StageTimeline> v;
    for (const auto& o : Json::parse(text)) v.push_back(timeline_from(o));
    return v;
  } catch (const nlohmann::json::exception& e) {
    throw ParseError(std::string("malformed timeline document: ") + e.what());
  }
}

}  // namespace lynx::host
