// Wire formats at the drop-in boundary: the reference's plan / schedule /
// partition / simreport JSON documents (proj/schemas/*.schema.json,
// emitters proj/src/report_io.cpp:47-185) plus the timeline document the
// executor consumes (one StageRecomputeTimeline per stage, heusched.hpp:115-135).
#pragma once

#include <string>
#include <vector>

#include "host/opt.hpp"
#include "host/partition.hpp"

namespace lynx::host {

std::string plan_json(const LayerPlan& plan, int stage);
std::string schedule_json(const PhaseSchedule& s, int stage);
std::string partition_json(const Partition& part);
std::string simreport_json(const PipeResult& r);
std::string breakdown_text(const PipeResult& r);

struct PartitionDoc {
  std::vector<int> layers;
  PlanMode mode = PlanMode::Heu;
  bool has_mode = false;
};
PartitionDoc parse_partition(const std::string& text);

std::string timeline_json(const StageTimeline& tl);              // one object
StageTimeline parse_timeline(const std::string& one_object_json);
std::vector<StageTimeline> parse_timelines(const std::string& array_json);

}  // namespace lynx::host
