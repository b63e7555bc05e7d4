// The model-graph ("profile") contract the executor consumes.
//
// Same JSON document and validation rules as the reference loader
// (proj/include/lynx/profile.hpp:27-145, proj/src/profile.cpp:191-287):
// {model{name,n_layers,static_bytes,layer{ops,fwd_comm_ids,bwd_comm_ids,
// checkpoint_id},embed_ops,head_ops,embed_schedulable,head_schedulable},
// hardware{mem_budget_bytes,comm_scale},pipeline{n_stages,n_microbatches,
// schedule_kind}}. Times are exact rationals (µs), sizes integral bytes.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "host/errors.hpp"
#include "host/rational.hpp"

namespace lynx::host {

enum class OpKind { Compute, Comm };

struct OpSpec {
  int id = 0;
  std::string name;
  OpKind kind = OpKind::Compute;
  Rat time_us;
  int64_t out_bytes = 0;
  std::vector<int> deps;
};

struct LayerTemplate {
  std::vector<OpSpec> ops;
  std::vector<int> fwd_comm_ids, bwd_comm_ids;
  int checkpoint_id = 0;
  int index_of(int id) const;
  int ckpt_pos() const { return index_of(checkpoint_id); }
  int n_fwd() const { return ckpt_pos() + 1; }
};

struct ModelProfile {
  std::string name = "unnamed";
  int n_layers = 1;
  int64_t static_bytes = 0;
  LayerTemplate layer;
  std::vector<OpSpec> embed_ops, head_ops;
  bool embed_schedulable = false, head_schedulable = false;
};

struct HardwareProfile {
  int64_t mem_budget_bytes = 0;
  Rat comm_scale = 1;
};

struct PipelineConfig {
  int n_stages = 1;
  int n_microbatches = 1;
};

struct Profile {
  ModelProfile model;
  HardwareProfile hardware;
  PipelineConfig pipeline;
};

// Comm operators run `comm_scale` times their profiled time (NVLink vs PCIe).
inline Rat op_time(const OpSpec& op, const HardwareProfile& hw) {
  return op.kind == OpKind::Comm ? op.time_us * hw.comm_scale : op.time_us;
}

Profile parse_profile(const std::string& text, bool lenient = false);
std::string profile_to_json(const Profile& p);

// One stage's instantiated operator graph (reference expand_graph, profile.cpp:372-463).
struct StageGraph {
  std::vector<OpSpec> ops;                // ops[i].id == i
  std::vector<std::vector<int>> users;
  std::vector<bool> schedulable;
  int fwd_op_count = 0;
  std::vector<int> checkpoint_ops;
  int size() const { return static_cast<int>(ops.size()); }
  bool is_comm(int i) const { return ops[i].kind == OpKind::Comm; }
};
StageGraph expand_stage_graph(const ModelProfile& m, int stage_layers, bool with_embed, bool with_head);
// Diagnostics text exactly as the reference's ValidationReport::to_string().
std::string graph_diagnostics(const StageGraph& g);

}  // namespace lynx::host
