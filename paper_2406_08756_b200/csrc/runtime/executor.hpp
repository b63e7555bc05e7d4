// The B200 executor: replays a Lynx recompute timeline for one pipeline stage
// on one TP rank — the GPU replacement for the reference's CPU executor
// simulate() (proj/src/pipesim.cpp:206-761).
//
// Same inputs (profile, layers per stage, the stage's StageRecomputeTimeline)
// and the same execution semantics:
//   * pass order: warm-up forwards, 1F1B pairs, cool-down backwards (pipesim.cpp:315-323);
//   * per layer, the template's elements: maximal compute runs and single comm
//     ops (pipesim.cpp:50-71);
//   * CriticalPath items run on the main stream before their element, sorted
//     by (owner_mb, owner_layer, op) (pipesim.cpp:426-440);
//   * Window items run on the recompute side stream, released when their
//     host all-reduce is issued, so they overlap the NCCL transfer
//     (pipesim.cpp:398-424); consumers wait on per-tensor events;
//   * StallFill items run on the side stream at the start of their backward
//     pass, filling the pipeline bubble while the gradient recv is pending
//     (pipesim.cpp:620-646);
//   * tensor liveness follows the ledger rules (discarded tensors dropped after
//     their last forward consumer, retained / regenerated ones after their last
//     backward consumer) on a stream-ordered device memory pool.
// TP all-reduces and PP send/recv go through NCCL on dedicated streams
// (tensor-parallel on one communicator; activations and gradients on two
// pipeline communicators so 1F1B cannot deadlock).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <map>
#include <memory>
#include <unordered_set>
#include <string>
#include <tuple>
#include <vector>

#include "host/pipeline.hpp"
#include "runtime/comm.hpp"
#include "runtime/gpt_stage.hpp"

namespace lynx::rt {

struct ExecOptions {
  bool trace = false;           // per-element CUDA-event timeline
  bool check_recompute = false; // keep forward copies, compare regenerated tensors bit-for-bit
  bool elide_recompute = false; // timing-only: skip recompute launches (exposed-recompute cross-check)
  bool window_join = true;      // main waits for a window's recomputes before the element after its all-reduce,
                                // and for a backward pass's stall-fill recomputes before the pass (reference
                                // semantics); false: they may keep running beside the main stream
  bool tp_fused = false;        // TP all-reduces fused into their consumers over peer memory (ops_tp.cu): the
                                // row-parallel partials go to symmetric staging slots, one kernel per site reads
                                // every rank's slot, sums and applies the epilogue
  bool elide_fill = false;      // elided mode: fill each stand-in buffer with uniform bf16 noise (timed apart,
                                // report elide_fill_ms) so consumers read realistic operands, not stale memory
  bool dry_run = false;         // build the launch program only (no device)
  bool probe_fc1 = false;       // CUDA events around every FC1 forward GEMM launch (roofline line)
  bool reserve_pool = true;     // map all free HBM (but 2 GiB) into the activation pool at construction
  bool pool_internal_deps = false;  // cudaMemPoolReuseAllowInternalDependencies on the activation pool: lets
                                    // an allocation on one stream reuse memory freed on another by making it
                                    // wait on the freeing stream (serialises the side stream behind main)
  bool op_timing = false;       // CUDA events around every template operator on the main stream (forward /
                                // backward ops, all-reduce epilogues, embedding, head): per-op device time
                                // of exactly the executor's kernel sequence (the profiler's source)
  bool probe_ops = false;       // one CUDA event after every operator launch on its stream: in-step
                                // time per operator name, gaps included (report "probe_ops")
  bool standalone = false;      // time one pipeline stage alone on one GPU: receives read synthetic
                                // activations / gradients, sends are skipped (measured partitioning)
  double comm_standin_us = 0;   // > 0 (standalone only): each TP all-reduce is replaced by a stand-in
  int comm_standin_ctas = 16;   // kernel holding the TP stream this long, so one GPU runs one TP rank
  bool dw_concurrent = true;    // attention backward: dW_proj on the aux stream beside dW_qkv (wave fill)
  int comm_standin_passes = 0;  // > 0: the stand-in also streams the all-reduce buffer through HBM this many
                                // times (in-place read + write): the local traffic of a real collective
                                // of a TP > 1 stage with the plan's comm windows (window overlap)
  std::vector<double> standin_grad_wait_us;  // standalone: per microbatch m, the pipeline stall before
                                             // B(m)'s gradient receive (from the simulator's trace),
                                             // held by a stand-in kernel so stall-fill recomputes
                                             // meet the bubble they are planned into
  std::vector<std::string> ledger_pass_start_us;  // plan-clock start of each pass of this stage (exact
                                                  // rationals, e.g. from lynx_plan_simulate_timelines'
                                                  // pass_start_us): the logical ledger is then timed on
                                                  // exactly the simulator's clock; default: passes back
                                                  // to back from 0
};

struct Slot {
  void* p = nullptr;
  size_t bytes = 0;
  cudaEvent_t ready = nullptr;  // set when produced off the main stream
  cudaStream_t stream = nullptr;
  bool regenerated = false;
  bool fused = false;      // produced early by the FC1 + GeLU epilogue; its own op call is a no-op
  bool booked = false;     // its profile bytes are in the logical ledger
  bool external = false;   // a communicator staging slot (exec.tp_fused), not a pool allocation
  void* shadow = nullptr;  // check_recompute: forward-produced copy
};

struct StepReport {
  double step_ms = 0, busy_ms = 0, comm_ms = 0, recompute_on_demand_ms = 0, recompute_overlapped_ms = 0,
         wait_on_recompute_ms = 0, recv_wait_ms = 0;
  double loss = 0;
  long long recompute_launches = 0, recompute_mismatch_words = 0, recompute_checked = 0;
  long long kernel_launches = 0;  // kernels of this library issued by the step
  size_t pool_high_water = 0;
  long long probe_launches = 0;  // exec.probe_fc1: FC1 forward GEMM launches timed in this step
  double probe_ms = 0;           // ... and their summed CUDA-event durations
  double alloc_host_ms = 0, alloc_host_max_ms = 0;  // host time inside pool allocations (stall diagnosis)
  double host_issue_ms = 0;                         // host time to issue the step (before the final sync)
  double elide_fill_ms = 0;                         // exec.elide_fill: device time of the stand-in fills
  size_t pool_reserved = 0;
};

struct CommOp {  // launch-program record (dry runs and tests)
  std::string kind;  // "allreduce" | "send" | "recv"
  std::string comm;  // "tp" | "pp_act" | "pp_grad"
  int peer = -1;
  size_t bytes = 0;
  std::string what;
};

class Executor {
 public:
  Executor(const std::string& profile_json, const std::string& timeline_json, const std::string& config_json);
  ~Executor();
  void step(const int* tokens_host, const int* labels_host, float* loss_out);
  std::string report_json() const;  // simreport.schema.json document of the last step (measured)
  std::string stats_json() const;   // executor counters, logical ledger trace, host timings
  host::PipeResult measured_result() const;
  std::string trace(int format) const;
  std::string program_json() const;
  void get_tensor(const std::string& name, void* host, size_t bytes);
  void set_tensor(const std::string& name, const void* host, size_t bytes);
  const StepReport& last() const { return rep_; }

 private:
  using Key4 = std::tuple<int, bool, int, int>;
  struct TimedSpan {
    cudaEvent_t a, b;
    int kind;  // 0 busy(pass), 1 comm, 2 on-demand recompute, 3 window recompute, 4 wait-on-recompute,
               // 5 recv wait, 6 stall-fill recompute
    int mb = -1, op = -1;
    bool on_side = false;
    bool bwd = false;
  };

  // setup
  void parse_config(const std::string& cfg);
  void bind_template();
  void validate_program();
  void* fused_partial();
  void init_device();
  void finish_production(Slot& out, size_t bytes, cudaStream_t s, bool recompute);
  void release_all();
  void alloc_persistent();

  // passes
  void forward_pass(int mb);
  void backward_pass(int mb);
  void run_items(const std::vector<host::Recompute>& items, cudaStream_t s, int span_kind, host::Rat* clock);
  void run_critical(const Key4& key, host::Rat& t);
  // TP all-reduce element starting at plan-clock time t; returns when its window recomputes end
  host::Rat comm_element(int mb, bool bwd, int l, const host::Element& e, const host::Rat& t);
  void fwd_op(int mb, int l, int pos, cudaStream_t s, bool recompute);
  void bwd_op(int mb, int l, int pos, cudaStream_t s);
  void head_forward(int mb);
  void head_backward(int mb);

  // tensors
  Slot& slot(int mb, int l, int pos) { return slots_[(static_cast<size_t>(mb) * cfg_.layers + l) * nf_ + pos]; }
  void* need(int mb, int l, int pos, cudaStream_t s);
  void* layer_input(int mb, int l, cudaStream_t s);
  void* alloc(size_t bytes, cudaStream_t s);
  void release(void* p, cudaStream_t s);
  void drop(Slot& sl, cudaStream_t s, bool keep_shadow);
  void mark_ready(Slot& sl, cudaStream_t s);
  uint64_t drop_stream(int l, int mb, Op op) const;

  // logical ledger (the simulator's memory ledger, pipesim.cpp:143-183 / 483-605 / 722-736), booked
  // by this executor's own tensor productions and drops on the plan clock
  void book(long long delta);
  host::Rat ledger_pass_start();
  void ledger_reset();
  std::pair<host::Rat, std::vector<std::pair<host::Rat, host::Rat>>> ledger_trace() const;

  // timing
  cudaEvent_t ev();
  void span_begin(cudaStream_t s, int kind, int mb = -1, int op = -1);
  void span_end(cudaStream_t s);
  void collect_spans();

  void ck(cudaError_t e, const char* what);
  void ck_op(int status, const char* what);
  void reserve_pool();

  host::Profile prof_;
  host::StageTimeline tl_;
  ModelCfg cfg_;
  ExecOptions opt_;
  std::string nccl_id_;
  int world_rank_ = 0, world_size_ = 1;
  bool needs_comms_ = false;
  bool tp_tmpl_ = false;
  int nf_ = 0, n_ = 0;
  std::vector<Op> op_of_;
  std::vector<host::Element> fel_, bel_;
  std::vector<int> made_in_, last_fwd_use_, last_bwd_user_, ckpt_pos_;
  std::vector<std::vector<int>> deps_;
  std::map<Key4, std::vector<host::Recompute>> win_, crit_;
  std::map<int, std::vector<host::Recompute>> stall_;

  cudaStream_t main_ = nullptr, side_ = nullptr, tp_s_ = nullptr, pa_s_ = nullptr, pg_s_ = nullptr;
  cudaStream_t aux_ = nullptr;  // intra-op concurrency of the main stream's work (attention backward dW GEMMs)
  std::unique_ptr<Comms> comms_;
  std::string loopback_;           // parallel.loopback: in-process grid name (all ranks on this GPU)
  cudaMemPool_t pool_ = nullptr;   // private stream-ordered pool of this executor (activations)
  std::unordered_set<void*> live_;  // every pool allocation not yet released (freed by release_all)
  ParamStore ps_;
  Scratch sc_main_, sc_side_;
  int *d_tokens_ = nullptr, *d_labels_ = nullptr;
  int *h_tokens_ = nullptr, *h_labels_ = nullptr;  // pinned staging
  float *d_loss_ = nullptr, *h_loss_ = nullptr;
  unsigned long long* d_mismatch_ = nullptr;
  std::vector<Slot> slots_;
  struct Grad {  // backward state of one microbatch (one layer in flight)
    void *dy = nullptr, *dln2 = nullptr, *dres = nullptr, *dln1 = nullptr;
  };
  std::vector<void*> stage_in_, head_dy_, ln_f_;  // per microbatch
  std::vector<Grad> grad_;
  std::vector<cudaEvent_t> act_sent_, grad_sent_;
  std::vector<cudaEvent_t> ev_pool_;
  size_t ev_next_ = 0;
  std::vector<TimedSpan> spans_;
  std::vector<std::pair<cudaStream_t, size_t>> open_;
  std::vector<CommOp> program_;
  StepReport rep_;
  int step_ = 0;
  int bwd_passes_ = 0;
  int dw_epi_ = 0;  // EPI_BF16 on the step's first backward pass, then EPI_ACC_BF16
  cudaEvent_t t0_ = nullptr, t1_ = nullptr;
  __nv_bfloat16 *syn_act_ = nullptr, *syn_grad_ = nullptr;  // standalone stage: stand-ins for PP receives
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> probes_;  // exec.probe_fc1 event pairs of this step
  size_t pool_reserved_init_ = 0;  // bytes mapped into the pool by reserve_pool()
  cudaStream_t probe_stream_ = nullptr;  // exec.probe_ops: the stream the current operator launches on
  std::vector<std::tuple<std::string, cudaStream_t, cudaEvent_t>> op_events_;  // exec.probe_ops, this step
  bool probe_recompute_ = false;
  std::vector<std::tuple<std::string, cudaEvent_t, cudaEvent_t>> op_tim_;  // exec.op_timing, this step
  std::map<std::string, std::vector<double>> op_tim_ms_;                  // ... resolved (ms per call)
  template <class F>
  void timed_op(const char* name, F&& f);  // exec.probe_ops: the current operator is a regeneration ("re: " prefix)
  std::vector<std::tuple<std::string, long long, double>> op_times_;           // name, launches, ms (last step)
  double op_stream_ms_[2] = {0, 0};                                            // main, side: sum of op times
  float* head_gw32_ = nullptr;  // last stage: LM-head weight gradient, fp32 across chunks / microbatches
  float *xent_max_ = nullptr, *xent_st_ = nullptr;  // vocab-parallel cross-entropy row statistics (one chunk)
  float* emb_gw32_ = nullptr;   // first stage: wte | wpe gradients, fp32 (sorted segment sums, no atomics)
  bool head_first_ = true;
  std::vector<std::tuple<int, int, int, int, double, double, bool>> trace_;  // stage, mb, kind, op, start, end, bwd
  bool cur_bwd_ = false;  // direction of the pass being issued (span tags)
  bool fused_ = false;          // exec.tp_fused in effect
  long long fused_seq_ = 0;     // fused reductions issued so far (identical on every TP rank): staging slot = seq % 2

  struct Ledger {
    bool override_starts = false;
    std::vector<host::Rat> starts;
    host::Rat t, free_at, resident, budget;
    bool started = false;
    size_t pass = 0;
    std::vector<std::pair<host::Rat, host::Rat>> deltas;  // (plan-clock time, +/- bytes), booking order
    std::map<int, long long> pass_release;
  } lg_;
  std::vector<host::Rat> cost_;        // plan-clock cost of each template op (op_time)
  std::vector<long long> out_bytes_;   // profile out_bytes of each template op
  std::vector<int> bwd_elem_, bwd_last_use_;
  host::Rat pre_dur_, post_dur_;
  long long pre_bytes_ = 0, post_bytes_ = 0;
  std::map<Key4, std::vector<host::Recompute>> deferred_;  // stall items the plan clock moves to the critical path
};

}  // namespace lynx::rt
