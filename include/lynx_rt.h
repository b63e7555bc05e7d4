/* lynx_rt.h — C-ABI of the host planner and the B200 executor.
 *
 * Drop-in boundary for the reference's hot path. The reference exposes a C++
 * value API, not a C-ABI:
 *
 *   simulate(const Profile&, const std::vector<int>& layers_per_stage,
 *            const std::vector<StageRecomputeTimeline>&, const SimOptions&) -> SimReport
 *                                              (proj/include/lynx/pipesim.hpp:86-88)
 *
 * fed by PlanCache::stage_plan (proj/include/lynx/partition.hpp:57-58) or
 * timeline_from_opt_schedule (proj/include/lynx/report_io.hpp:46-49), and the
 * front-ends `lynx validate|schedule|partition|simulate|report`
 * (proj/tools/lynx_main.cpp:72-226) and `_lynx.*` (proj/bindings/module.cpp:75-95).
 *
 * Section 1 (lynx_plan_*) restates those front-ends on in-memory JSON with
 * bit-identical output documents. Section 2 (lynx_rt_*) is the GPU executor
 * that replaces simulate(): it consumes the same profile and timelines and
 * returns a measured report in the simreport schema.
 *
 * Conventions: strings are NUL-terminated UTF-8 JSON; returned strings are
 * malloc'd by the library and released with lynx_free(). `status` receives
 * 0 on success or the reference CLI exit code (1 validation, 2 parse / other,
 * 3 timed out, 4 infeasible, 5 no valid partition) or 6 CUDA / 7 OOM; NULL is
 * returned on failure with the message in lynx_last_error(). No C++ exception
 * crosses this boundary. Single-threaded per handle.
 */
#ifndef LYNX_RT_H_
#define LYNX_RT_H_

#include "lynx_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

void lynx_free(char* p);

/* ---------------------------------------------------------------- 1. plan */

/* `lynx validate`: graph diagnostics text ("" when well-formed; status 1 otherwise).
 * Replaces cmd_validate (lynx_main.cpp:72-84) / _lynx.validate (module.cpp:66-72). */
char* lynx_plan_validate(const char* profile_json, int lenient, int* status);

/* Canonical profile serialization (profile.cpp:300-338, _lynx.serialize_profile). */
char* lynx_plan_serialize_profile(const char* profile_json, int lenient, int* status);

/* `lynx schedule --mode heu|opt --stage s [--emit-lp]`: plan JSON (plan.schema.json),
 * schedule JSON (schedule.schema.json) or CPLEX LP text. layers may be NULL
 * (initial_partition). Replaces cmd_schedule (lynx_main.cpp:117-157). */
char* lynx_plan_schedule(const char* profile_json, const char* mode, int stage, const int* layers, int n_layers,
                         long long time_limit_ms, int emit_lp, int* status);

/* `lynx partition --mode heu|opt`: partition JSON (Algorithm 1, partition.cpp:155-215). */
char* lynx_plan_partition(const char* profile_json, const char* mode, long long time_limit_ms, int* status);

/* `lynx simulate` / `lynx report`: format 0 simreport JSON, 1 CSV trace, 2 Chrome
 * trace, 3 breakdown table. pybind_semantics=1 reproduces _lynx.simulate's OPT
 * branch (plan_stage_opt timelines, module.cpp:43-64) instead of the CLI's. */
char* lynx_plan_simulate(const char* profile_json, const char* mode, const int* layers, int n_layers,
                         const char* p2p_us, int format, int pybind_semantics, long long time_limit_ms,
                         int* status);

/* One stage's plan + expanded RecomputeItem timeline + steady period:
 * baseline 0 = HEU (PlanCache::stage_plan), 1 = full recompute, 2 = retain all
 * (heusched.cpp:313-341). JSON {plan_json, timeline, period_us, layers_per_stage}. */
char* lynx_plan_stage(const char* profile_json, int stage, const int* layers, int n_layers, int baseline,
                      long long time_limit_ms, int* status);

/* simulate() on caller-provided timelines (JSON array of timeline objects):
 * {report, iteration_us_exact, memory_traces, memory_peaks, csv}. */
char* lynx_plan_simulate_timelines(const char* profile_json, const int* layers, int n_layers,
                                   const char* timelines_json, const char* p2p_us, int* status);

/* Solve one HEU context (policy 0 FixedBytes, 1 ReserveUnretained):
 * {plan_json, n_vars, n_cons, lp, check, timeline}. */
char* lynx_plan_solve_heu(const char* profile_json, int stage, int stage_layers, int policy,
                          const char* delta_bytes, long long time_limit_ms, int* status);

#ifdef __cplusplus
}
#endif

#endif /* LYNX_RT_H_ */
