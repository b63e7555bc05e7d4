// lynx_execute — the `lynx execute` sibling of the reference CLI's `simulate` subcommand
// (proj/tools/lynx_main.cpp:200-226), built against the drop-in C-ABI only (include/lynx_rt.h):
// it plans one stage of a profile exactly as the reference would (lynx_plan_stage: PlanCache::
// stage_plan + expand_plan_to_stage, partition.cpp:87-98 / heusched.cpp:343-427), hands the
// stage's StageRecomputeTimeline to the B200 executor, runs training iterations on synthetic
// tokens and prints the measured report in the reference's simreport.schema.json shape (or
// emit_trace's CSV / Chrome trace, or the executor counters).
//
//   lynx_execute <profile.json> <config.json> [--mode heu|full|retain_all|selective]
//                [--stage s] [--steps n] [--format json|csv|chrome|stats] [--out file]
//
// config.json is the executor configuration of lynx_rt_create (model shape, layers_per_stage,
// parallel, train, exec). Exit codes are the reference CLI's (lynx_main.cpp:30-35: 1 validation,
// 2 parse, 3 timed out, 4 infeasible, 5 no valid partition) plus 6 CUDA and 7 out of memory.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "lynx_rt.h"

namespace {

std::string read_file(const char* path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error(std::string("cannot read ") + path);
  std::ostringstream os;
  os << f.rdbuf();
  return os.str();
}

int fail(int st) {
  std::cerr << "lynx_execute: " << lynx_last_error() << "\n";
  return st ? st : 2;
}

// SplitMix64: synthetic token ids (uniform over the GPT-2 vocabulary), labels = next token.
uint64_t mix(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::cerr << "usage: lynx_execute <profile.json> <config.json> [--mode heu|full|retain_all|selective] "
                 "[--stage s] [--steps n] [--format json|csv|chrome|stats] [--out file]\n";
    return 1;
  }
  std::string mode = "heu", format = "json", out_path;
  int stage = 0, steps = 1;
  for (int i = 3; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--mode") mode = v;
    else if (k == "--stage") stage = std::stoi(v);
    else if (k == "--steps") steps = std::stoi(v);
    else if (k == "--format") format = v;
    else if (k == "--out") out_path = v;
    else {
      std::cerr << "unknown option " << k << "\n";
      return 1;
    }
  }
  std::string profile, config;
  try {
    profile = read_file(argv[1]);
    config = read_file(argv[2]);
  } catch (const std::exception& e) {
    std::cerr << e.what() << "\n";
    return 2;
  }
  const int baseline = mode == "heu" ? 0 : mode == "full" ? 1 : mode == "retain_all" ? 2 : mode == "selective" ? 3 : -1;
  if (baseline < 0) {
    std::cerr << "unknown mode " << mode << "\n";
    return 1;
  }
  nlohmann::json cfg = nlohmann::json::parse(config, nullptr, false);
  if (cfg.is_discarded()) {
    std::cerr << "config is not JSON\n";
    return 2;
  }
  std::vector<int> layers = cfg.value("layers_per_stage", std::vector<int>{});
  int st = 0;
  char* plan = lynx_plan_stage(profile.c_str(), stage, layers.empty() ? nullptr : layers.data(),
                               static_cast<int>(layers.size()), baseline, 10000, &st);
  if (!plan) return fail(st);
  const nlohmann::json pj = nlohmann::json::parse(plan);
  lynx_free(plan);
  cfg["layers_per_stage"] = pj.at("layers_per_stage");
  const std::string timeline = pj.at("timeline").dump();
  lynx_rt* rt = nullptr;
  if ((st = lynx_rt_create(profile.c_str(), timeline.c_str(), cfg.dump().c_str(), &rt))) return fail(st);

  const nlohmann::json prof = nlohmann::json::parse(profile);
  const auto& m = cfg.at("model");
  const long long n = static_cast<long long>(prof.at("pipeline").at("n_microbatches").get<int>()) *
                      m.at("micro_batch").get<int>() * m.at("seq").get<int>();
  std::vector<int> tokens(n), labels(n);
  uint64_t s = 1234;
  for (long long i = 0; i < n; ++i) tokens[i] = static_cast<int>(mix(s) % 50257);
  for (long long i = 0; i < n; ++i) labels[i] = i + 1 < n ? tokens[i + 1] : tokens[0];
  float loss = 0.f;
  for (int i = 0; i < steps; ++i)
    if ((st = lynx_rt_step(rt, tokens.data(), labels.data(), &loss))) {
      lynx_rt_destroy(rt);
      return fail(st);
    }
  char* out = format == "json"    ? lynx_rt_report_json(rt, &st)
              : format == "stats" ? lynx_rt_stats_json(rt, &st)
                                  : lynx_rt_trace(rt, format == "csv" ? 1 : 0, &st);
  if (!out) {
    lynx_rt_destroy(rt);
    return fail(st);
  }
  if (out_path.empty()) {
    std::fputs(out, stdout);
    if (format == "stats") std::fputs("\n", stdout);
  } else {
    std::ofstream f(out_path, std::ios::binary);
    f << out;
    if (!f) {
      std::cerr << "cannot write " << out_path << "\n";
      lynx_free(out);
      lynx_rt_destroy(rt);
      return 2;
    }
  }
  lynx_free(out);
  lynx_rt_destroy(rt);
  return 0;
}
