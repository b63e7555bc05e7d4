#include "host/pipeline.hpp"

#include <algorithm>
#include <climits>
#include <map>
#include <set>
#include <sstream>
#include <stdexcept>
#include <tuple>

namespace lynx::host {

const char* ev_kind_name(EvKind k) {
  switch (k) {
    case EvKind::Fwd: return "fwd";
    case EvKind::Bwd: return "bwd";
    case EvKind::CommFwd: return "comm_fwd";
    case EvKind::CommBwd: return "comm_bwd";
    case EvKind::Recompute: return "recompute";
    case EvKind::StallRecompute: return "stall_recompute";
    case EvKind::P2P: return "p2p";
    case EvKind::Stall: return "stall";
  }
  return "?";
}

std::vector<Element> layer_elements(const LayerTemplate& layer, const HardwareProfile& hw, bool backward) {
  const int nf = layer.n_fwd();
  const int lo = backward ? nf : 0, hi = backward ? static_cast<int>(layer.ops.size()) : nf;
  const std::vector<int>& wins = backward ? layer.bwd_comm_ids : layer.fwd_comm_ids;
  std::vector<Element> out;
  for (int i = lo; i < hi; ++i) {
    const OpSpec& o = layer.ops[i];
    if (o.kind == OpKind::Comm) {
      Element e;
      e.comm = true;
      e.op = i;
      e.dur = op_time(o, hw);
      for (size_t w = 0; w < wins.size(); ++w)
        if (layer.index_of(wins[w]) == i) e.window = static_cast<int>(w);
      out.push_back(std::move(e));
    } else {
      if (out.empty() || out.back().comm) out.emplace_back();
      out.back().ops.push_back(i);
      out.back().dur += o.time_us;
    }
  }
  return out;
}

std::vector<std::pair<bool, int>> stage_passes(int S, int s, int M) {
  std::vector<std::pair<bool, int>> v;
  const int warm = std::min(S - s, M) - 1;
  for (int mb = 0; mb < std::min(warm, M); ++mb) v.emplace_back(false, mb);
  for (int mb = warm; mb < M; ++mb) {
    v.emplace_back(false, mb);
    v.emplace_back(true, mb - warm);
  }
  for (int mb = std::max(0, M - warm); mb < M; ++mb) v.emplace_back(true, mb);
  return v;
}

namespace {

struct Shape {  // per-template liveness tables
  std::vector<Element> fwd, bwd;
  int nf = 0, n = 0;
  std::vector<int> made_in;        // fwd op -> producing fwd element
  std::vector<int> last_fwd_use;   // fwd op -> last forward element consuming it (-1)
  std::vector<int> last_bwd_use;   // fwd op -> last backward element consuming it (-1)
  std::vector<int> bwd_elem;       // bwd op -> its element
  std::vector<int> bwd_last_use;   // bwd op -> last backward element consuming it (-1)
  std::vector<Rat> cost;
  std::vector<std::vector<int>> fdeps;
};

int element_of(const std::vector<Element>& els, int pos) {
  for (size_t e = 0; e < els.size(); ++e) {
    if (els[e].comm ? els[e].op == pos : std::count(els[e].ops.begin(), els[e].ops.end(), pos) > 0)
      return static_cast<int>(e);
  }
  return -1;
}

Shape make_shape(const LayerTemplate& L, const HardwareProfile& hw) {
  Shape sh;
  sh.nf = L.n_fwd();
  sh.n = static_cast<int>(L.ops.size());
  sh.fwd = layer_elements(L, hw, false);
  sh.bwd = layer_elements(L, hw, true);
  sh.made_in.assign(sh.nf, -1);
  sh.last_fwd_use.assign(sh.nf, -1);
  sh.last_bwd_use.assign(sh.nf, -1);
  sh.bwd_elem.assign(sh.n, -1);
  sh.bwd_last_use.assign(sh.n, -1);
  for (int i = 0; i < sh.n; ++i) sh.cost.push_back(op_time(L.ops[i], hw));
  for (int i = 0; i < sh.nf; ++i) {
    sh.made_in[i] = element_of(sh.fwd, i);
    std::vector<int> d;
    for (int id : L.ops[i].deps) d.push_back(L.index_of(id));
    sh.fdeps.push_back(std::move(d));
  }
  for (int i = sh.nf; i < sh.n; ++i) sh.bwd_elem[i] = element_of(sh.bwd, i);
  for (int i = 0; i < sh.n; ++i)
    for (int id : L.ops[i].deps) {
      const int d = L.index_of(id);
      if (i < sh.nf) {
        sh.last_fwd_use[d] = std::max(sh.last_fwd_use[d], sh.made_in[i]);
      } else if (d < sh.nf) {
        sh.last_bwd_use[d] = std::max(sh.last_bwd_use[d], sh.bwd_elem[i]);
      } else {
        sh.bwd_last_use[d] = std::max(sh.bwd_last_use[d], sh.bwd_elem[i]);
      }
    }
  return sh;
}

using Key4 = std::tuple<int, bool, int, int>;  // (mb, backward, layer, window|element)
using Key3 = std::tuple<int, int, int>;        // (mb, layer, op|element)

struct Lane {  // one pipeline stage
  int stage = 0, layers = 0;
  StageTimeline tl;
  std::vector<Element> pre, post;  // embed / head segments
  Rat pre_bytes, post_bytes;
  std::map<Key4, std::vector<Recompute>> in_window, on_demand;
  std::map<int, std::vector<Recompute>> in_stall;
  std::vector<std::pair<bool, int>> passes;
  size_t next = 0;
  Rat free_at;
  bool started = false;
  Rat resident, budget;
  bool track_memory = true;
  std::vector<std::pair<Rat, Rat>> deltas;
  std::map<Key3, Rat> regen_release;
  std::map<int, Rat> pass_release;
  std::set<Key3> regenerated;
  std::map<int, Rat> fwd_done, bwd_done;
  Rat exposed_comm, first, last;
  bool any = false;
  std::vector<Event>* sink = nullptr;
  std::vector<Rat> starts;  // pass start times (the executor's ledger clock for this stage)

  void event(EvKind k, int mb, int op, const Rat& s, const Rat& e, bool ov) {
    if (sink) sink->push_back(Event{stage, mb, k, op, s, e, ov});
    if (!any) {
      first = s;
      any = true;
    }
    last = rmax(last, e);
  }
  void take(const Rat& t, const Rat& b) {
    if (!track_memory || b.sign() == 0) return;
    resident += b;
    deltas.emplace_back(t, b);
  }
  void give(const Rat& t, const Rat& b) {
    if (!track_memory || b.sign() == 0) return;
    resident -= b;
    deltas.emplace_back(t, -b);
  }
};

class Model {
 public:
  Model(const Profile& p, const std::vector<int>& layers, const std::vector<StageTimeline>& tls, Rat p2p)
      : p_(p), layers_(layers), sh_(make_shape(p.model.layer, p.hardware)), p2p_(std::move(p2p)) {
    const int S = static_cast<int>(layers.size());
    if (static_cast<int>(tls.size()) != S) throw InconsistentPlan("one timeline per stage is required");
    lanes_.resize(S);
    for (int s = 0; s < S; ++s) setup(s, tls[s]);
  }

  PipeResult run() {
    PipeResult r;
    for (auto& ln : lanes_) ln.sink = &r.events;
    const int S = static_cast<int>(lanes_.size());
    for (;;) {
      int pick = -1;
      Rat when;
      for (int s = 0; s < S; ++s) {
        Lane& ln = lanes_[s];
        if (ln.next >= ln.passes.size()) continue;
        Rat in;
        if (!ready(s, ln.passes[ln.next].first, ln.passes[ln.next].second, in)) continue;
        const Rat start = rmax(ln.free_at, in);
        if (pick < 0 || start < when) {
          pick = s;
          when = start;
        }
      }
      if (pick < 0) {
        for (const auto& ln : lanes_)
          if (ln.next < ln.passes.size()) throw std::logic_error("pipeline deadlock: no runnable pass");
        break;
      }
      pass(pick);
    }
    finish(r);
    return r;
  }

  Rat period(int s) {
    Lane& ln = lanes_[s];
    ln.track_memory = false;
    ln.tl.strict_deps = false;
    ln.sink = nullptr;
    const int M = p_.pipeline.n_microbatches;
    const int nb = std::min(static_cast<int>(lanes_.size()) - s, M);
    const int steady = std::max(0, M - nb + 1);
    const int rep = steady >= 3 ? 1 : 0;
    const int fwd_mb = std::min(rep + nb - 1, M - 1);
    const Rat t = forward(ln, fwd_mb, Rat(0));
    return backward(ln, rep, t);
  }

 private:
  std::vector<Element> opaque(const std::vector<OpSpec>& ops) const {
    std::vector<Element> v;
    for (const OpSpec& o : ops) {
      if (o.kind == OpKind::Comm) {
        Element e;
        e.comm = true;
        e.dur = op_time(o, p_.hardware);
        v.push_back(std::move(e));
      } else {
        if (v.empty() || v.back().comm) v.emplace_back();
        v.back().dur += o.time_us;
      }
    }
    return v;
  }

  void setup(int s, const StageTimeline& tl) {
    Lane& ln = lanes_[s];
    const int S = static_cast<int>(lanes_.size());
    ln.stage = s;
    ln.layers = layers_[s];
    ln.tl = tl;
    if (ln.tl.plan.retained.empty()) {
      ln.tl.plan.retained.assign(sh_.nf, true);
    } else if (static_cast<int>(ln.tl.plan.retained.size()) != sh_.nf) {
      throw InconsistentPlan("plan retention vector does not match the layer template");
    }
    ln.budget = Rat(p_.hardware.mem_budget_bytes);
    const Rat share = Rat(p_.model.static_bytes) * Rat(ln.layers) / Rat(p_.model.n_layers);
    ln.resident = share;
    ln.deltas.emplace_back(Rat(0), share);
    if (s == 0) {
      ln.pre = opaque(p_.model.embed_ops);
      for (const auto& o : p_.model.embed_ops) ln.pre_bytes += Rat(o.out_bytes);
    }
    if (s == S - 1) {
      ln.post = opaque(p_.model.head_ops);
      for (const auto& o : p_.model.head_ops) ln.post_bytes += Rat(o.out_bytes);
    }
    for (const Recompute& it : ln.tl.items) {
      switch (it.host) {
        case Recompute::Host::Window:
          ln.in_window[{it.host_mb, it.host_bwd, it.host_layer, it.host_window}].push_back(it);
          break;
        case Recompute::Host::Critical:
          ln.on_demand[{it.host_mb, it.host_bwd, it.host_layer, it.host_elem}].push_back(it);
          break;
        case Recompute::Host::Stall:
          ln.in_stall[it.host_mb].push_back(it);
          break;
      }
    }
    ln.passes = stage_passes(S, s, p_.pipeline.n_microbatches);
  }

  bool ready(int s, bool bwd, int mb, Rat& out) const {
    const int S = static_cast<int>(lanes_.size());
    if (!bwd) {
      if (s == 0) {
        out = Rat(0);
        return true;
      }
      auto it = lanes_[s - 1].fwd_done.find(mb);
      if (it == lanes_[s - 1].fwd_done.end()) return false;
      out = it->second + p2p_;
      return true;
    }
    if (s == S - 1) {
      auto it = lanes_[s].fwd_done.find(mb);
      if (it == lanes_[s].fwd_done.end()) return false;
      out = it->second;
      return true;
    }
    auto it = lanes_[s + 1].bwd_done.find(mb);
    if (it == lanes_[s + 1].bwd_done.end()) return false;
    out = it->second + p2p_;
    return true;
  }

  void regenerate(Lane& ln, const Recompute& it, EvKind k, const Rat& s, const Rat& e, bool ov) {
    if (ln.tl.strict_deps) {
      for (int d : sh_.fdeps[it.op]) {
        if (ln.tl.plan.retained[d] || ln.regenerated.count({it.owner_mb, it.owner_layer, d})) continue;
        throw InconsistentPlan("recompute of op " + std::to_string(it.op) + " (mb " + std::to_string(it.owner_mb) +
                               ", layer " + std::to_string(it.owner_layer) + ") lacks dependency " +
                               std::to_string(d));
      }
    }
    ln.event(k, it.owner_mb, it.op, s, e, ov);
    ln.regenerated.insert({it.owner_mb, it.owner_layer, it.op});
    const Rat b(p_.model.layer.ops[it.op].out_bytes);
    if (ln.track_memory && b.sign() != 0) {
      ln.take(s, b);
      ln.regen_release[{it.owner_mb, it.owner_layer, sh_.last_bwd_use[it.op]}] += b;
    }
  }

  Rat window(Lane& ln, const Rat& t, const Rat& dur, const Key4& key) {
    Rat cur = t, hidden(0);
    const Rat end = t + dur;
    auto f = ln.in_window.find(key);
    if (f != ln.in_window.end()) {
      for (const Recompute& it : f->second) {
        const Rat c = sh_.cost[it.op];
        const Rat stop = cur + c;
        if (stop <= end) {
          regenerate(ln, it, EvKind::Recompute, cur, stop, true);
          hidden += c;
        } else if (cur < end) {  // preempted at the window end; the rest is on demand
          regenerate(ln, it, EvKind::Recompute, cur, end, true);
          ln.event(EvKind::Recompute, it.owner_mb, it.op, end, stop, false);
          hidden += end - cur;
        } else {
          regenerate(ln, it, EvKind::Recompute, cur, stop, false);
        }
        cur = stop;
      }
    }
    ln.exposed_comm += dur - rmin(hidden, dur);
    return cur;
  }

  void critical(Lane& ln, Rat& t, const Key4& key) {
    auto f = ln.on_demand.find(key);
    if (f == ln.on_demand.end()) return;
    std::stable_sort(f->second.begin(), f->second.end(), [](const Recompute& a, const Recompute& b) {
      return std::tie(a.owner_mb, a.owner_layer, a.op) < std::tie(b.owner_mb, b.owner_layer, b.op);
    });
    for (const Recompute& it : f->second) {
      const Rat c = sh_.cost[it.op];
      regenerate(ln, it, EvKind::Recompute, t, t + c, false);
      t += c;
    }
  }

  void fwd_memory(Lane& ln, int elem, const Rat& t, const Rat& tend) {
    if (!ln.track_memory) return;
    const LayerTemplate& L = p_.model.layer;
    const Element& e = sh_.fwd[elem];
    Rat made(0);
    if (e.comm) {
      made += Rat(L.ops[e.op].out_bytes);
    } else {
      for (int o : e.ops) made += Rat(L.ops[o].out_bytes);
    }
    ln.take(t, made);
    Rat dropped(0);
    for (int o = 0; o < sh_.nf; ++o) {
      if (ln.tl.plan.retained[o]) continue;
      if (std::max(sh_.made_in[o], sh_.last_fwd_use[o]) == elem) dropped += Rat(L.ops[o].out_bytes);
    }
    if (dropped.sign() != 0) ln.give(tend, dropped);
  }

  Rat forward(Lane& ln, int mb, const Rat& start) {
    Rat t = start;
    for (const Element& e : ln.pre) {
      ln.event(e.comm ? EvKind::CommFwd : EvKind::Fwd, mb, -1, t, t + e.dur, false);
      t += e.dur;
    }
    if (!ln.pre.empty() && ln.pre_bytes.sign() != 0) {
      ln.take(start, ln.pre_bytes);
      ln.pass_release[mb] += ln.pre_bytes;
    }
    for (int l = 0; l < ln.layers; ++l) {
      for (size_t ei = 0; ei < sh_.fwd.size(); ++ei) {
        const Element& e = sh_.fwd[ei];
        critical(ln, t, {mb, false, l, static_cast<int>(ei)});
        if (e.comm) {
          Rat busy = t;
          if (e.window >= 0) {
            busy = window(ln, t, e.dur, {mb, false, l, e.window});
          } else {
            ln.exposed_comm += e.dur;
          }
          ln.event(EvKind::CommFwd, mb, e.op, t, t + e.dur, false);
          fwd_memory(ln, static_cast<int>(ei), t, t + e.dur);
          t = rmax(t + e.dur, busy);
        } else {
          ln.event(EvKind::Fwd, mb, -1, t, t + e.dur, false);
          fwd_memory(ln, static_cast<int>(ei), t, t + e.dur);
          t += e.dur;
        }
      }
    }
    if (ln.stage + 1 == static_cast<int>(lanes_.size())) {
      for (const Element& e : ln.post) {
        ln.event(e.comm ? EvKind::CommFwd : EvKind::Fwd, mb, -1, t, t + e.dur, false);
        t += e.dur;
      }
      if (!ln.post.empty() && ln.post_bytes.sign() != 0) {
        ln.take(t, ln.post_bytes);
        ln.pass_release[mb] += ln.post_bytes;
      }
    }
    return t;
  }

  void bwd_release(Lane& ln, int mb, int l, int elem, const Rat& t) {
    if (!ln.track_memory) return;
    const LayerTemplate& L = p_.model.layer;
    Rat out(0);
    for (int o = 0; o < sh_.nf; ++o)
      if (sh_.last_bwd_use[o] == elem && ln.tl.plan.retained[o]) out += Rat(L.ops[o].out_bytes);
    auto rf = ln.regen_release.find({mb, l, elem});
    if (rf != ln.regen_release.end()) {
      out += rf->second;
      ln.regen_release.erase(rf);
    }
    for (int o = sh_.nf; o < sh_.n - 1; ++o) {  // the gradient sink (last op) crosses layers
      const int rel = sh_.bwd_last_use[o] >= 0 ? sh_.bwd_last_use[o] : sh_.bwd_elem[o];
      if (rel == elem) out += Rat(L.ops[o].out_bytes);
    }
    if (out.sign() != 0) ln.give(t, out);
  }

  Rat backward(Lane& ln, int mb, const Rat& start) {
    const LayerTemplate& L = p_.model.layer;
    Rat t = start, sink(0);
    for (int l = ln.layers - 1; l >= 0; --l) {
      bool first = true;
      for (size_t ei = 0; ei < sh_.bwd.size(); ++ei) {
        const Element& e = sh_.bwd[ei];
        critical(ln, t, {mb, true, l, static_cast<int>(ei)});
        const Rat tend = t + e.dur;
        if (e.comm) {
          Rat busy = t;
          if (e.window >= 0) {
            busy = window(ln, t, e.dur, {mb, true, l, e.window});
          } else {
            ln.exposed_comm += e.dur;
          }
          ln.event(EvKind::CommBwd, mb, e.op, t, tend, false);
          if (ln.track_memory) ln.take(t, Rat(L.ops[e.op].out_bytes));
          bwd_release(ln, mb, l, static_cast<int>(ei), tend);
          t = rmax(tend, busy);
        } else {
          ln.event(EvKind::Bwd, mb, -1, t, tend, false);
          if (ln.track_memory) {
            Rat made(0);
            for (int o : e.ops) made += Rat(L.ops[o].out_bytes);
            ln.take(t, made);
          }
          bwd_release(ln, mb, l, static_cast<int>(ei), tend);
          t = tend;
        }
        if (first) {  // the downstream layer's gradient has now been consumed
          first = false;
          if (ln.track_memory && sink.sign() != 0) ln.give(t, sink);
          sink = Rat(0);
        }
      }
      if (ln.track_memory) {
        Rat out(0);
        for (int o = 0; o < sh_.nf; ++o)
          if (sh_.last_bwd_use[o] == -1 && ln.tl.plan.retained[o]) out += Rat(L.ops[o].out_bytes);
        for (auto it = ln.regen_release.lower_bound({mb, l, INT_MIN});
             it != ln.regen_release.end() && std::get<0>(it->first) == mb && std::get<1>(it->first) == l;) {
          out += it->second;
          it = ln.regen_release.erase(it);
        }
        if (sh_.n > sh_.nf) sink = Rat(L.ops[sh_.n - 1].out_bytes);
        if (out.sign() != 0) ln.give(t, out);
        for (int o = 0; o < sh_.nf; ++o) ln.regenerated.erase({mb, l, o});
      }
    }
    if (ln.track_memory) {
      if (sink.sign() != 0) ln.give(t, sink);
      auto pe = ln.pass_release.find(mb);
      if (pe != ln.pass_release.end()) {
        ln.give(t, pe->second);
        ln.pass_release.erase(pe);
      }
    }
    return t;
  }

  void pass(int s) {
    Lane& ln = lanes_[s];
    const auto [bwd, mb] = ln.passes[ln.next];
    Rat in;
    ready(s, bwd, mb, in);
    const Rat start = rmax(ln.free_at, in);
    const int S = static_cast<int>(lanes_.size());
    if (p2p_.sign() >= 0 && ((!bwd && s > 0) || (bwd && s < S - 1)))
      ln.event(EvKind::P2P, mb, -1, in - p2p_, in, false);
    if (start > ln.free_at && ln.started) {  // idle gap: cool-down stall fill
      Rat t = ln.free_at;
      if (bwd) {
        auto si = ln.in_stall.find(mb);
        if (si != ln.in_stall.end()) {
          std::vector<Recompute> later;
          for (const Recompute& it : si->second) {
            const Rat c = sh_.cost[it.op];
            const Rat b(p_.model.layer.ops[it.op].out_bytes);
            if (t + c <= start && ln.resident + b <= ln.budget) {
              regenerate(ln, it, EvKind::StallRecompute, t, t + c, true);
              t += c;
            } else {
              later.push_back(it);
            }
          }
          for (const Recompute& it : later) ln.on_demand[{mb, true, it.owner_layer, 0}].push_back(it);
          ln.in_stall.erase(si);
        }
      }
      if (t < start) ln.event(EvKind::Stall, mb, -1, t, start, false);
    }
    ln.started = true;
    ln.starts.push_back(start);
    const Rat end = bwd ? backward(ln, mb, start) : forward(ln, mb, start);
    (bwd ? ln.bwd_done : ln.fwd_done)[mb] = end;
    ln.free_at = end;
    ++ln.next;
  }

  void finish(PipeResult& r) {
    const int S = static_cast<int>(lanes_.size());
    r.stages.assign(S, {});
    r.breakdown.assign(S, {});
    r.peaks.assign(S, Rat(0));
    r.traces.assign(S, {});
    r.pass_starts.assign(S, {});
    for (int s = 0; s < S; ++s) r.pass_starts[s] = lanes_[s].starts;
    r.iteration_us = Rat(0);
    for (const Event& e : r.events) r.iteration_us = rmax(r.iteration_us, e.end);
    for (const Event& e : r.events) {
      StageSummary& st = r.stages[e.stage];
      const Rat d = e.end - e.start;
      switch (e.kind) {
        case EvKind::Fwd:
        case EvKind::Bwd: st.busy += d; break;
        case EvKind::Recompute:
          st.busy += d;
          (e.overlapped ? st.overlapped : st.on_demand) += d;
          break;
        case EvKind::StallRecompute:
          st.busy += d;
          st.overlapped += d;
          break;
        case EvKind::CommFwd:
        case EvKind::CommBwd:
        case EvKind::P2P: st.comm += d; break;
        case EvKind::Stall: break;
      }
    }
    const int M = p_.pipeline.n_microbatches;
    for (int s = 0; s < S; ++s) {
      Lane& ln = lanes_[s];
      StageSummary& st = r.stages[s];
      const Rat span = ln.any ? ln.last - ln.first : Rat(0);
      const Rat idle = span - st.busy - ln.exposed_comm;
      st.stall = idle.sign() > 0 ? idle : Rat(0);
      Rat kept(0);
      for (int o = 0; o < sh_.nf; ++o)
        if (ln.tl.plan.retained[o]) kept += sh_.cost[o] * Rat(ln.layers) * Rat(M);
      const Rat total = kept + st.overlapped + st.on_demand;
      if (total.sign() == 0) {
        r.breakdown[s] = {Rat(1), Rat(0), Rat(0)};
      } else {
        r.breakdown[s] = {kept / total, st.overlapped / total, st.on_demand / total};
      }
      std::stable_sort(ln.deltas.begin(), ln.deltas.end(),
                       [](const auto& a, const auto& b) { return a.first < b.first; });
      Rat res(0), peak(0);
      auto& tr = r.traces[s];
      for (size_t i = 0; i < ln.deltas.size(); ++i) {
        res += ln.deltas[i].second;
        if (i + 1 < ln.deltas.size() && ln.deltas[i + 1].first == ln.deltas[i].first) continue;
        if (!tr.empty() && tr.back().first == ln.deltas[i].first) {
          tr.back().second = res;
        } else {
          tr.emplace_back(ln.deltas[i].first, res);
        }
        peak = rmax(peak, res);
      }
      r.peaks[s] = peak;
    }
    std::stable_sort(r.events.begin(), r.events.end(), [](const Event& a, const Event& b) {
      if (a.start != b.start) return a.start < b.start;
      if (a.stage != b.stage) return a.stage < b.stage;
      return static_cast<int>(a.kind) < static_cast<int>(b.kind);
    });
  }

  const Profile& p_;
  std::vector<int> layers_;
  Shape sh_;
  Rat p2p_;
  std::vector<Lane> lanes_;
};

}  // namespace

PipeResult run_pipeline(const Profile& p, const std::vector<int>& layers, const std::vector<StageTimeline>& tls,
                        const Rat& p2p_us) {
  Model m(p, layers, tls, p2p_us);
  return m.run();
}

Rat steady_period(const Profile& p, int stage, int stage_layers, const StageTimeline& tl) {
  const int S = p.pipeline.n_stages;
  std::vector<int> layers(S, 1);
  layers[stage] = stage_layers;
  std::vector<StageTimeline> tls(S);
  for (int s = 0; s < S; ++s) {
    tls[s].stage = s;
    tls[s].plan.retained.assign(p.model.layer.n_fwd(), true);
  }
  tls[stage] = tl;
  Model m(p, layers, tls, Rat(0));
  return m.period(stage);
}

std::string trace_csv(const PipeResult& r) {
  std::ostringstream os;
  os << "stage,microbatch,kind,op_id,start_us,end_us,overlapped\n";
  for (const Event& e : r.events)
    os << e.stage << "," << e.microbatch << "," << ev_kind_name(e.kind) << ","
       << (e.op < 0 ? "" : std::to_string(e.op)) << "," << to_fixed(e.start, 3) << "," << to_fixed(e.end, 3) << ","
       << (e.overlapped ? 1 : 0) << "\n";
  return os.str();
}

std::string trace_chrome(const PipeResult& r) {
  std::ostringstream os;
  os << "[";
  bool first = true;
  for (const Event& e : r.events) {
    if (!first) os << ",";
    first = false;
    const bool compute = e.kind != EvKind::CommFwd && e.kind != EvKind::CommBwd && e.kind != EvKind::P2P;
    os << "\n  {\"name\": \"" << ev_kind_name(e.kind);
    if (e.microbatch >= 0) os << " mb" << e.microbatch;
    if (e.op >= 0) os << " op" << e.op;
    os << "\", \"ph\": \"X\", \"pid\": " << e.stage << ", \"tid\": \"" << (compute ? "compute" : "comm")
       << "\", \"ts\": " << to_fixed(e.start, 3) << ", \"dur\": " << to_fixed(e.end - e.start, 3)
       << ", \"args\": {\"overlapped\": " << (e.overlapped ? "true" : "false") << "}}";
  }
  os << "\n]\n";
  return os.str();
}

}  // namespace lynx::host
