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
 * baseline 0 = HEU (PlanCache::stage_plan), 1 = full recompute, 2 = retain all,
 * 3 = Megatron selective (only the core attention "attn" is recomputed; not a reference plan)
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

/* OPT at GPT scale through an external MILP solver (replaces the embedded
 * B&B of optsched.cpp:216-243, which cannot solve a 7B stage). The model is the reference's
 * OPT program (optsched.cpp:54-214) over `slice_layers` consecutive layers of the stage
 * (0 = all), extended for replication over the stage: a variable Y bounds the slice's retained
 * bytes at every phase entry and each ledger point carries (L/k - 1) Y for the other copies.
 * Slice budget = static(k) + (mem_budget - static(L)) - reserve_bytes (null: 0).
 * lynx_plan_opt_export: {n_vars, lo, hi, integer, objective [[var, c]], n_rows, row/col/val
 *   (coordinate form), sense (-1 <=, 0 =, 1 >=), rhs, R[t][i], S[t][i] (variable indices),
 *   budget_bytes, static_bytes, stage_activation_bytes, n_ops}; coefficients as doubles.
 * lynx_plan_opt_timeline: schedule_json = {"keep": [[t, i]...], "recompute": [[t, i]...]} from
 *   the solver. The schedule is checked exactly (check_schedule, optsched.cpp:245-338);
 *   violations return status 1 with {"issues"}. Otherwise timeline_from_opt_schedule
 *   (report_io.cpp:187-294) on the slice, replicated over the stage's layers:
 *   {issues: "", cost_us, n_recompute, n_overlapped, timeline, slice_items}. */
char* lynx_plan_opt_export(const char* profile_json, int stage, const int* layers, int n_layers, int slice_layers,
                           const char* reserve_bytes, int* status);
char* lynx_plan_opt_timeline(const char* profile_json, int stage, const int* layers, int n_layers, int slice_layers,
                             const char* reserve_bytes, const char* schedule_json, int* status);

/* ---------------------------------------------------------------- 2. execute */

/* One executor per (pipeline stage, TP rank) process; replaces simulate().
 * profile_json: the profile the plan was made for (GPT block template, see
 *   gpt_profile.py; the op names bind to kernels).
 * timeline_json: this stage's StageRecomputeTimeline as produced by
 *   lynx_plan_stage()["timeline"] (heusched.hpp:115-135 / report_io.hpp:46-49).
 * config_json: {"model": {hidden, heads, seq, micro_batch, vocab},
 *   "layers_per_stage": [...], "parallel": {tp, tp_rank, world_rank, world_size,
 *   nccl_id (hex, from lynx_rt_nccl_unique_id on rank 0)}, "train": {dropout,
 *   seed, lr, beta1, beta2, eps, weight_decay, init_std}, "exec": {trace,
 *   check_recompute, elide_recompute, dry_run, head_chunk, probe_fc1, probe_ops,
 *   reserve_pool, pool_internal_deps, standalone_stage, comm_standin_us, comm_standin_ctas, comm_standin_passes,
 *   standin_grad_wait_us, ledger_pass_start_us, window_join, elide_fill, op_timing,
 *   tp_fused, dw_concurrent}}; parallel.loopback = "<name>" instead of
 *   nccl_id runs every rank of the grid in this process on one GPU (one thread per rank).
 * Weights are initialised on the device from Philox streams keyed by seed. */
typedef struct lynx_rt lynx_rt;
int lynx_rt_create(const char* profile_json, const char* timeline_json, const char* config_json, lynx_rt** out);

/* One training iteration: H2D of this step's tokens / labels (int32
 * [n_microbatches * micro_batch * seq], host memory; NULL where the stage does
 * not need them), the stage's 1F1B passes with the plan's recomputation, AdamW.
 * Blocks until the iteration's final event; *loss = mean token loss (last stage). */
int lynx_rt_step(lynx_rt* h, const int* tokens, const int* labels, float* loss);

/* Measured report of the last step in the reference's simreport.schema.json shape
 * (SimReport, proj/include/lynx/pipesim.hpp:68-75, emitted like simreport_to_json,
 * report_io.cpp:103-143), for this executor's stage: iteration / busy / comm / stall
 * (pipeline-receive waits) / recompute on-demand (kernels + main-stream waits on the side
 * stream) / overlapped (window + stall fill) µs from CUDA events; breakdown weighted like
 * pipesim.cpp:705-720; memory_peaks = the LOGICAL ledger's peak (see lynx_rt_stats_json);
 * timeline = measured events of kinds fwd|bwd|comm_fwd|comm_bwd|recompute|stall_recompute|
 * stall (exec.trace, else empty). Arrays hold this stage only. */
char* lynx_rt_report_json(lynx_rt* h, int* status);
/* Executor counters of the last step (flat JSON): iteration / busy / comm / recompute
 * on-demand, overlapped, wait-on-recompute, exposed-recompute ms, launches, bit-identity check
 * counters, pool high-water bytes, host issue / allocation ms, and "ledger": the logical memory
 * ledger (pipesim.cpp:143-183, 483-605, 722-736) booked by this executor's own tensor
 * productions and drops on the plan clock — {memory_peak_bytes, memory_trace [[t_us, bytes]],
 * plan_clock}; with exec.ledger_pass_start_us = the simulator's pass starts it equals
 * simulate()'s memory_traces / memory_peaks entry for this stage exactly. */
char* lynx_rt_stats_json(lynx_rt* h, int* status);
/* Measured timeline of the last step (exec.trace) in emit_trace's formats
 * (pipesim.cpp:781-810): 0 Chrome trace JSON, 1 CSV. */
char* lynx_rt_trace(lynx_rt* h, int format, int* status);
/* Communication program of the last step (collectives / send / recv in issue order). */
char* lynx_rt_program_json(lynx_rt* h, int* status);
/* Parameter ("l0.w_qkv", "wte", ...) as bf16, or its fp32 gradient ("grad:l0.w_qkv"). */
int lynx_rt_get_tensor(lynx_rt* h, const char* name, void* host, size_t bytes);
/* Overwrite a parameter from fp32 host values (master and bf16 copy). */
int lynx_rt_set_tensor(lynx_rt* h, const char* name, const void* host, size_t bytes);
/* Hex-encoded ncclUniqueId for parallel.nccl_id (call on world rank 0). */
int lynx_rt_nccl_unique_id(char* hex_out, size_t len);
void lynx_rt_destroy(lynx_rt* h);

#ifdef __cplusplus
}
#endif

#endif /* LYNX_RT_H_ */
