#include "runtime/executor.hpp"

#include <algorithm>
#include <chrono>
#include <map>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <stdexcept>

#include <nlohmann/json.hpp>

#include "host/report.hpp"
#include "lynx_ops_internal.h"

namespace lynx::rt {

using Json = nlohmann::ordered_json;
using host::Recompute;

namespace {
constexpr uint64_t kEmbedStream = 0xFFFFull << 32;
}  // namespace

// ============================================================ setup
// LYNX_TRACE_SLOTS=1: print every tensor production / drop (ledger debugging), read once.
static bool trace_slots() {
  static const bool on = std::getenv("LYNX_TRACE_SLOTS") != nullptr;
  return on;
}

void Executor::ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) cudaGetLastError();  // clear non-sticky errors so later launch checks do not see them
  if (e == cudaErrorMemoryAllocation) throw RtError(std::string(what) + ": out of device memory", kOutOfMemory);
  if (e != cudaSuccess) throw RtError(std::string(what) + ": " + cudaGetErrorString(e), kCudaError);
}
void Executor::ck_op(int status, const char* what) {
  if (status != kOk) throw RtError(std::string(what) + ": " + last_error(), status);
  if (opt_.probe_ops && probe_stream_) {
    cudaEvent_t e = ev();
    ck(cudaEventRecord(e, probe_stream_), "event");
    op_events_.emplace_back(std::string(probe_recompute_ ? "re: " : "") + what, probe_stream_, e);
  }
}

namespace {
// Sets the stream exec.probe_ops attributes operator launches to, for one scope.
struct ProbeStream {
  cudaStream_t& slot;
  cudaStream_t saved;
  ProbeStream(cudaStream_t& sl, cudaStream_t s) : slot(sl), saved(sl) { slot = s; }
  ~ProbeStream() { slot = saved; }
};
}  // namespace
Executor::Executor(const std::string& profile_json, const std::string& timeline_json, const std::string& config_json) {
  prof_ = host::parse_profile(profile_json);
  tl_ = host::parse_timeline(timeline_json);
  parse_config(config_json);
  bind_template();
  validate_program();
  if (opt_.dry_run) return;
  try {
    init_device();
  } catch (...) {
    release_all();  // a throwing constructor runs no destructor: free what was already allocated
    throw;
  }
}

// Replays the whole step's launch program on the host (dry run, no device work) before anything is
// allocated: a timeline whose regeneration comes after a consumer of the tensor — or a tensor produced
// twice — is rejected here, at lynx_rt_create, as the reference rejects it (InconsistentPlan, exit code 2,
// pipesim.cpp:364-376), instead of in the middle of a step.
void Executor::validate_program() {
  const bool dry = opt_.dry_run;
  const int step0 = step_;
  opt_.dry_run = true;
  try {
    step(nullptr, nullptr, nullptr);
  } catch (const RtError& e) {
    opt_.dry_run = dry;
    step_ = step0;
    throw RtError(std::string("InconsistentPlan: ") + e.what(), e.code == kValidation ? kValidation : kParse);
  }
  opt_.dry_run = dry;
  step_ = step0;
  for (auto& sl : slots_) sl = Slot{};
  std::fill(stage_in_.begin(), stage_in_.end(), nullptr);
  std::fill(head_dy_.begin(), head_dy_.end(), nullptr);
  std::fill(ln_f_.begin(), ln_f_.end(), nullptr);
  std::fill(grad_.begin(), grad_.end(), Grad{});
}

void Executor::init_device() {
  // Reserve the per-thread local-memory (stack) the library's kernels can need before the big
  // allocations: growing it lazily mid-step, with HBM nearly full, stalls the device (observed as
  // sporadic 1-4 s steps under high-memory plans).
  size_t stack = 0;
  ck(cudaDeviceGetLimit(&stack, cudaLimitStackSize), "stack limit");
  if (stack < 1024) ck(cudaDeviceSetLimit(cudaLimitStackSize, 1024), "stack limit");
  if (needs_comms_) {
    // A plan that regenerates an all-reduce output (phase 5 on ar1 / ar2, heusched.cpp:125) re-issues
    // the collective; its result must be bit-identical to the first one. Ring / Simple is deterministic
    // for a fixed communicator and size; the size-dependent choice among NVLS / tree / ring protocols is
    // pinned so the two calls cannot differ (unless the user set NCCL_ALGO / NCCL_PROTO).
    bool regen_ar = false;
    for (const host::Recompute& it : tl_.items)
      if (op_of_[it.op] == Op::AR1 || op_of_[it.op] == Op::AR2) regen_ar = true;
    if (regen_ar && loopback_.empty()) {
      setenv("NCCL_ALGO", "Ring", 0);
      setenv("NCCL_PROTO", "Simple", 0);
    }
    if (!loopback_.empty())
      comms_ = make_loopback_comms(loopback_, cfg_.tp, cfg_.pp, cfg_.pp_rank, cfg_.tp_rank);
    else
      comms_ = make_nccl_comms(nccl_id_, world_rank_, world_size_, cfg_.pp_rank, cfg_.tp_rank);
    if (fused_) comms_->fused_setup(static_cast<size_t>(cfg_.tokens()) * cfg_.hidden * 2);
  }
  for (cudaStream_t* s : {&main_, &side_, &tp_s_, &pa_s_, &pg_s_, &aux_})
    ck(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking), "stream");
  int dev = 0;
  ck(cudaGetDevice(&dev), "device");
  // A private pool: its high-water mark is this executor's alone, several executors can share a
  // process (the loopback grid), and destroying it returns every byte (the OOM error path).
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  ck(cudaMemPoolCreate(&pool_, &props), "mempool");
  uint64_t thr = UINT64_MAX;
  ck(cudaMemPoolSetAttribute(pool_, cudaMemPoolAttrReleaseThreshold, &thr), "mempool attr");
  int internal = opt_.pool_internal_deps ? 1 : 0;
  ck(cudaMemPoolSetAttribute(pool_, cudaMemPoolReuseAllowInternalDependencies, &internal), "mempool attr");
  ps_.allocate_and_init(cfg_, main_);
  alloc_persistent();
  if (opt_.reserve_pool) reserve_pool();
  ck(cudaEventCreate(&t0_), "event");
  ck(cudaEventCreate(&t1_), "event");
  for (int i = 0; i < cfg_.n_micro; ++i) {
    cudaEvent_t a, b;
    ck(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "event");
    act_sent_.push_back(a);
    grad_sent_.push_back(b);
  }
  ck(cudaStreamSynchronize(main_), "init");
}

// Map the activation pool's physical memory once, up front: all free HBM but a small reserve for
// the runtime, library workspaces and NCCL (2 GiB, 6 GiB with communicators), allocated from the pool and freed back into it (the release
// threshold keeps it mapped). Growing the pool lazily inside the steps, with HBM nearly full,
// made single cudaMallocFromPoolAsync calls block the host for up to 2.6 s while the driver
// mapped memory (seen as 3-10 s steps with `alloc_host_ms` in the report); afterwards the pool
// only splits and reuses what it holds.
void Executor::reserve_pool() {
  size_t free_b = 0, total_b = 0;
  ck(cudaMemGetInfo(&free_b, &total_b), "meminfo");
  // NCCL sets up P2P / NVLS buffers lazily at a communicator's first operation: leave it room
  const size_t keep = (needs_comms_ ? size_t{6} : size_t{2}) << 30, step = size_t{1} << 30;
  if (free_b <= keep + step) return;
  size_t want = (free_b - keep) / step * step;
  void* p = nullptr;
  while (want >= step) {
    if (cudaMallocFromPoolAsync(&p, want, pool_, main_) == cudaSuccess) break;
    cudaGetLastError();
    p = nullptr;
    want -= step;
  }
  if (!p) return;
  ck(cudaFreeAsync(p, main_), "pool reserve");
  ck(cudaStreamSynchronize(main_), "pool reserve");
  pool_reserved_init_ = want;
  uint64_t zero = 0;
  ck(cudaMemPoolSetAttribute(pool_, cudaMemPoolAttrUsedMemHigh, &zero), "mempool attr");
}

void Executor::parse_config(const std::string& text) {
  Json j = Json::parse(text);
  const Json& m = j.at("model");
  cfg_.n_layers_total = prof_.model.n_layers;
  cfg_.hidden = m.at("hidden");
  cfg_.heads = m.at("heads");
  cfg_.seq = m.at("seq");
  cfg_.micro_batch = m.at("micro_batch");
  cfg_.vocab = m.value("vocab", 50304);
  cfg_.head_dim = cfg_.hidden / cfg_.heads;
  const Json par = j.value("parallel", Json::object());
  cfg_.tp = par.value("tp", 1);
  cfg_.tp_rank = par.value("tp_rank", 0);
  cfg_.pp = prof_.pipeline.n_stages;
  cfg_.pp_rank = tl_.stage;
  cfg_.n_micro = prof_.pipeline.n_microbatches;
  const std::vector<int> lps = j.at("layers_per_stage").get<std::vector<int>>();
  if (static_cast<int>(lps.size()) != cfg_.pp) throw RtError("layers_per_stage does not match n_stages", kValidation);
  int total = 0;
  for (int x : lps) total += x;
  if (total != prof_.model.n_layers) throw RtError("layers_per_stage does not sum to n_layers", kValidation);
  cfg_.layers = lps[cfg_.pp_rank];
  cfg_.layer0 = 0;
  for (int s = 0; s < cfg_.pp_rank; ++s) cfg_.layer0 += lps[s];
  const Json tr = j.value("train", Json::object());
  cfg_.dropout = tr.value("dropout", 0.1f);
  cfg_.seed = tr.value("seed", 42ull);
  cfg_.lr = tr.value("lr", 1e-4f);
  cfg_.beta1 = tr.value("beta1", 0.9f);
  cfg_.beta2 = tr.value("beta2", 0.95f);
  cfg_.adam_eps = tr.value("eps", 1e-8f);
  cfg_.weight_decay = tr.value("weight_decay", 0.1f);
  cfg_.init_std = tr.value("init_std", 0.02f);
  cfg_.ln_eps = tr.value("ln_eps", 1e-5f);
  const Json ex = j.value("exec", Json::object());
  opt_.trace = ex.value("trace", false);
  opt_.check_recompute = ex.value("check_recompute", false);
  opt_.elide_recompute = ex.value("elide_recompute", false);
  opt_.elide_fill = ex.value("elide_fill", false);
  opt_.window_join = ex.value("window_join", true);
  opt_.tp_fused = ex.value("tp_fused", false);
  opt_.dry_run = ex.value("dry_run", false);
  opt_.standalone = ex.value("standalone_stage", false);
  opt_.probe_fc1 = ex.value("probe_fc1", false);
  opt_.probe_ops = ex.value("probe_ops", false);
  opt_.op_timing = ex.value("op_timing", false);
  opt_.reserve_pool = ex.value("reserve_pool", true);
  opt_.pool_internal_deps = ex.value("pool_internal_deps", false);
  opt_.comm_standin_us = ex.value("comm_standin_us", 0.0);
  opt_.comm_standin_ctas = ex.value("comm_standin_ctas", 16);
  opt_.comm_standin_passes = ex.value("comm_standin_passes", 0);
  opt_.dw_concurrent = ex.value("dw_concurrent", true);
  opt_.standin_grad_wait_us = ex.value("standin_grad_wait_us", std::vector<double>());
  opt_.ledger_pass_start_us = ex.value("ledger_pass_start_us", std::vector<std::string>());
  cfg_.head_chunk = static_cast<int>(std::min<long long>(ex.value("head_chunk", 4096), cfg_.tokens()));
  if (cfg_.hidden % cfg_.heads || cfg_.heads % cfg_.tp || (cfg_.hidden / cfg_.tp) % 128)
    throw RtError("hidden must split into heads and TP ranks in 128-column tiles", kValidation);
  if (cfg_.tokens() % 128 || cfg_.seq % 64 || cfg_.tokens() % cfg_.head_chunk || cfg_.head_chunk % 128)
    throw RtError("tokens per microbatch must be a multiple of 128 and of the head chunk", kValidation);
  if (cfg_.vocab % 128) throw RtError("vocab must be padded to a multiple of 128", kValidation);
  ps_.layout(cfg_);
  nccl_id_ = par.value("nccl_id", std::string());
  loopback_ = par.value("loopback", std::string());
  world_rank_ = par.value("world_rank", 0);
  world_size_ = par.value("world_size", 1);
  if (!loopback_.empty() && (opt_.standalone || !nccl_id_.empty()))
    throw RtError("parallel.loopback runs every rank in this process: no nccl_id, no standalone_stage", kValidation);
  if (opt_.standalone && world_size_ != 1)
    throw RtError("standalone_stage runs one stage in a single process", kValidation);
  if (opt_.standalone && cfg_.tp != 1 && opt_.comm_standin_us <= 0)
    throw RtError("standalone_stage at TP > 1 needs exec.comm_standin_us (one TP rank, stand-in all-reduces)",
                  kValidation);
  if (opt_.comm_standin_us > 0 && !opt_.standalone)
    throw RtError("exec.comm_standin_us is a standalone_stage option", kValidation);
  if (!opt_.standin_grad_wait_us.empty() && !opt_.standalone)
    throw RtError("exec.standin_grad_wait_us is a standalone_stage option", kValidation);
  if (opt_.comm_standin_ctas < 1 || opt_.comm_standin_ctas > 148)
    throw RtError("exec.comm_standin_ctas must be in [1, 148]", kValidation);
}

void Executor::bind_template() {
  const host::LayerTemplate& L = prof_.model.layer;
  nf_ = L.n_fwd();
  n_ = static_cast<int>(L.ops.size());
  for (const auto& o : L.ops) {
    const Op op = op_from_name(o.name);
    if (op == Op::UNKNOWN)
      throw RtError("profile op '" + o.name + "' has no B200 operator (see gpt_profile.py templates)", kValidation);
    op_of_.push_back(op);
    std::vector<int> d;
    for (int id : o.deps) d.push_back(L.index_of(id));
    deps_.push_back(d);
  }
  const bool tp_tmpl = !L.fwd_comm_ids.empty();
  if (cfg_.tp > 1 && !tp_tmpl) throw RtError("tp > 1 needs the tensor-parallel layer template", kValidation);
  const bool standin = opt_.comm_standin_us > 0;
  needs_comms_ = (!standin && (tp_tmpl || cfg_.tp > 1)) || (cfg_.pp > 1 && !opt_.standalone);
  tp_tmpl_ = tp_tmpl;
  static const std::vector<Op> t1 = {Op::LN1, Op::QKV, Op::ATTN, Op::PROJ_RES, Op::LN2, Op::FC1,
                                     Op::GELU, Op::FC2_RES, Op::MLP_BWD, Op::ATTN_BWD, Op::LN1_BWD};
  static const std::vector<Op> t2 = {Op::LN1, Op::QKV, Op::ATTN, Op::PROJ, Op::AR1, Op::LN2, Op::FC1, Op::GELU,
                                     Op::FC2, Op::AR2, Op::MLP_BWD, Op::AR_B1, Op::ATTN_BWD, Op::AR_B2, Op::LN1_BWD};
  if (op_of_ != (tp_tmpl ? t2 : t1)) throw RtError("profile layer template is not the GPT block template", kValidation);
  fel_ = host::layer_elements(L, prof_.hardware, false);
  bel_ = host::layer_elements(L, prof_.hardware, true);
  auto elem_of = [](const std::vector<host::Element>& els, int pos) {
    for (size_t e = 0; e < els.size(); ++e)
      if (els[e].comm ? els[e].op == pos : std::count(els[e].ops.begin(), els[e].ops.end(), pos) > 0)
        return static_cast<int>(e);
    return -1;
  };
  made_in_.assign(nf_, -1);
  last_fwd_use_.assign(nf_, -1);
  last_bwd_user_.assign(nf_, -1);
  for (int i = 0; i < nf_; ++i) made_in_[i] = elem_of(fel_, i);
  for (int i = 0; i < n_; ++i)
    for (int d : deps_[i]) {
      if (i < nf_) {
        last_fwd_use_[d] = std::max(last_fwd_use_[d], made_in_[i]);
      } else if (d < nf_) {
        last_bwd_user_[d] = std::max(last_bwd_user_[d], elem_of(bel_, i));
      }
    }
  if (static_cast<int>(tl_.plan.retained.size()) != nf_) {
    if (!tl_.plan.retained.empty()) throw RtError("plan retention vector does not match the layer template", kValidation);
    tl_.plan.retained.assign(nf_, true);
  }
  for (const Recompute& it : tl_.items) {
    if (it.owner_mb < 0 || it.owner_mb >= cfg_.n_micro || it.owner_layer < 0 || it.owner_layer >= cfg_.layers ||
        it.op < 0 || it.op >= nf_)
      throw RtError("recompute item out of range for this stage", kValidation);
    switch (it.host) {
      case Recompute::Host::Window: win_[{it.host_mb, it.host_bwd, it.host_layer, it.host_window}].push_back(it); break;
      case Recompute::Host::Critical: crit_[{it.host_mb, it.host_bwd, it.host_layer, it.host_elem}].push_back(it); break;
      case Recompute::Host::Stall: stall_[it.host_mb].push_back(it); break;
    }
  }
  for (auto& kv : crit_)
    std::stable_sort(kv.second.begin(), kv.second.end(), [](const Recompute& a, const Recompute& b) {
      return std::tie(a.owner_mb, a.owner_layer, a.op) < std::tie(b.owner_mb, b.owner_layer, b.op);
    });
  fused_ = opt_.tp_fused && tp_tmpl_ && cfg_.tp > 1;
  if (fused_) {
    if (opt_.standalone) throw RtError("exec.tp_fused needs every TP rank (not standalone_stage)", kValidation);
    for (const Recompute& it : tl_.items)
      if (op_of_[it.op] == Op::AR1 || op_of_[it.op] == Op::AR2)
        throw RtError("exec.tp_fused: the plan regenerates an all-reduce output (phase 5 on ar1 / ar2); run it "
                      "without tp_fused",
                      kValidation);
  }
  // plan clock and logical-ledger tables (pipesim.cpp:83-121 build_layout)
  bwd_elem_.assign(n_, -1);
  bwd_last_use_.assign(n_, -1);
  for (int i = 0; i < n_; ++i) {
    cost_.push_back(host::op_time(L.ops[i], prof_.hardware));
    out_bytes_.push_back(L.ops[i].out_bytes);
  }
  for (int i = nf_; i < n_; ++i) bwd_elem_[i] = elem_of(bel_, i);
  for (int i = nf_; i < n_; ++i)
    for (int d : deps_[i])
      if (d >= nf_) bwd_last_use_[d] = std::max(bwd_last_use_[d], bwd_elem_[i]);
  for (const auto& o : prof_.model.embed_ops) {
    pre_dur_ += o.kind == host::OpKind::Comm ? host::op_time(o, prof_.hardware) : o.time_us;
    pre_bytes_ += o.out_bytes;
  }
  for (const auto& o : prof_.model.head_ops) {
    post_dur_ += o.kind == host::OpKind::Comm ? host::op_time(o, prof_.hardware) : o.time_us;
    post_bytes_ += o.out_bytes;
  }
  for (const std::string& x : opt_.ledger_pass_start_us) {
    const auto r = host::parse_rat(x);
    if (!r) throw RtError("exec.ledger_pass_start_us: '" + x + "' is not a rational", kValidation);
    lg_.starts.push_back(*r);
  }
  lg_.override_starts = !lg_.starts.empty();
  if (lg_.override_starts && lg_.starts.size() != host::stage_passes(cfg_.pp, cfg_.pp_rank, cfg_.n_micro).size())
    throw RtError("exec.ledger_pass_start_us needs one start per pass of this stage", kValidation);
  slots_.assign(static_cast<size_t>(cfg_.n_micro) * cfg_.layers * nf_, Slot{});
  stage_in_.assign(cfg_.n_micro, nullptr);
  head_dy_.assign(cfg_.n_micro, nullptr);
  ln_f_.assign(cfg_.n_micro, nullptr);
  grad_.assign(cfg_.n_micro, Grad{});
}

void Executor::alloc_persistent() {
  const long long T = cfg_.tokens(), h = cfg_.hidden, hp = cfg_.hp();
  auto m = [&](size_t b) {
    void* p = nullptr;
    ck(cudaMalloc(&p, b), "scratch");
    return p;
  };
  const long long wide = 4 * hp;
  sc_main_.t_h = static_cast<__nv_bfloat16*>(m(T * h * 2));
  sc_main_.t_h2 = static_cast<__nv_bfloat16*>(m(T * h * 2));
  sc_main_.t_wide = static_cast<__nv_bfloat16*>(m(T * wide * 2));
  const size_t ws = std::max({layernorm_bwd_workspace(static_cast<int>(T), static_cast<int>(h)),
                              column_sum_workspace(T, static_cast<int>(wide)),
                              attention_bwd_workspace(cfg_.micro_batch, cfg_.seq, cfg_.heads_rank())});
  sc_main_.ws = static_cast<float*>(m(ws));
  sc_main_.ws_bytes = ws;
  if (cfg_.last()) {
    sc_main_.logits = static_cast<__nv_bfloat16*>(m(static_cast<size_t>(cfg_.head_chunk) * cfg_.vocab_rank() * 2));
    head_gw32_ = static_cast<float*>(m(static_cast<size_t>(cfg_.vocab_rank()) * h * 4));
    if (cfg_.vocab_parallel()) {
      xent_max_ = static_cast<float*>(m(static_cast<size_t>(cfg_.head_chunk) * 4));
      xent_st_ = static_cast<float*>(m(static_cast<size_t>(cfg_.head_chunk) * 8));
    }
  }
  if (cfg_.first()) emb_gw32_ = static_cast<float*>(m(static_cast<size_t>(cfg_.vocab + cfg_.seq) * h * 4));
  if (opt_.standalone) {  // activations ~ N(0, 1), gradients ~ N(0, 1e-2): realistic operands for timing
    syn_act_ = static_cast<__nv_bfloat16*>(m(static_cast<size_t>(T) * h * 2));
    syn_grad_ = static_cast<__nv_bfloat16*>(m(static_cast<size_t>(T) * h * 2));
    ck_op(init_normal_bf16(syn_act_, nullptr, T * h, 1.0f, cfg_.seed, 0xAC7ull, main_), "synthetic activations");
    ck_op(init_normal_bf16(syn_grad_, nullptr, T * h, 0.01f, cfg_.seed, 0x6AADull, main_), "synthetic gradients");
  }
  sc_side_.t_h = static_cast<__nv_bfloat16*>(m(T * h * 2));
  const size_t ntok = static_cast<size_t>(cfg_.n_micro) * T;
  d_tokens_ = static_cast<int*>(m(ntok * 4));
  d_labels_ = static_cast<int*>(m(ntok * 4));
  d_loss_ = static_cast<float*>(m(ntok * 4));
  d_mismatch_ = static_cast<unsigned long long*>(m(8));
  ck(cudaMallocHost(&h_tokens_, ntok * 4), "pinned");
  ck(cudaMallocHost(&h_labels_, ntok * 4), "pinned");
  ck(cudaMallocHost(&h_loss_, ntok * 4), "pinned");
}

Executor::~Executor() {
  if (opt_.dry_run) return;
  release_all();
}

void Executor::release_all() {
  // Own streams only: other executors of this process (loopback grid) keep running.
  for (cudaStream_t s : {main_, side_, tp_s_, pa_s_, pg_s_, aux_})
    if (s) cudaStreamSynchronize(s);
  // Every pool allocation still live — tensors of a step that threw (LYNX_E_OOM), per-microbatch
  // gradients and staging, forward copies kept for check_recompute — is freed before the pool.
  for (void* p : live_) cudaFree(p);
  live_.clear();
  for (auto& s : slots_) s = Slot{};
  std::fill(stage_in_.begin(), stage_in_.end(), nullptr);
  std::fill(head_dy_.begin(), head_dy_.end(), nullptr);
  std::fill(ln_f_.begin(), ln_f_.end(), nullptr);
  std::fill(grad_.begin(), grad_.end(), Grad{});
  ps_.release();
  for (void* p : {static_cast<void*>(sc_main_.t_h), static_cast<void*>(sc_main_.t_h2),
                  static_cast<void*>(sc_main_.t_wide), static_cast<void*>(sc_main_.ws),
                  static_cast<void*>(sc_main_.logits), static_cast<void*>(sc_side_.t_h), static_cast<void*>(d_tokens_),
                  static_cast<void*>(head_gw32_), static_cast<void*>(emb_gw32_), static_cast<void*>(syn_act_),
                  static_cast<void*>(syn_grad_), static_cast<void*>(xent_max_), static_cast<void*>(xent_st_),
                  static_cast<void*>(d_labels_), static_cast<void*>(d_loss_), static_cast<void*>(d_mismatch_)})
    if (p) cudaFree(p);
  xent_max_ = xent_st_ = nullptr;
  sc_main_ = Scratch{};
  sc_side_ = Scratch{};
  d_tokens_ = d_labels_ = nullptr;
  d_loss_ = nullptr;
  head_gw32_ = emb_gw32_ = nullptr;
  syn_act_ = syn_grad_ = nullptr;
  d_mismatch_ = nullptr;
  cudaFreeHost(h_tokens_);
  cudaFreeHost(h_labels_);
  cudaFreeHost(h_loss_);
  h_tokens_ = h_labels_ = nullptr;
  h_loss_ = nullptr;
  for (auto e : ev_pool_) cudaEventDestroy(e);
  for (auto e : act_sent_) cudaEventDestroy(e);
  for (auto e : grad_sent_) cudaEventDestroy(e);
  ev_pool_.clear();
  act_sent_.clear();
  grad_sent_.clear();
  ev_next_ = 0;
  if (t0_) cudaEventDestroy(t0_);
  if (t1_) cudaEventDestroy(t1_);
  t0_ = t1_ = nullptr;
  comms_.reset();
  for (cudaStream_t* s : {&main_, &side_, &tp_s_, &pa_s_, &pg_s_, &aux_})
    if (*s) {
      cudaStreamDestroy(*s);
      *s = nullptr;
    }
  if (pool_) cudaMemPoolDestroy(pool_);
  pool_ = nullptr;
  cudaGetLastError();
}

// ============================================================ tensors
void* Executor::alloc(size_t bytes, cudaStream_t s) {
  if (opt_.dry_run) return reinterpret_cast<void*>(0x1000);
  void* p = nullptr;
  const auto h0 = std::chrono::steady_clock::now();
  const cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool_, s);
  const double hms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
  rep_.alloc_host_ms += hms;
  rep_.alloc_host_max_ms = std::max(rep_.alloc_host_max_ms, hms);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    uint64_t used = 0, reserved = 0;
    size_t free_b = 0, total_b = 0;
    cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrUsedMemCurrent, &used);
    cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemGetInfo(&free_b, &total_b);
    throw RtError("activation allocation: out of device memory (request " + std::to_string(bytes) + " B, pool used " +
                      std::to_string(used) + " / reserved " + std::to_string(reserved) + " B, device free " +
                      std::to_string(free_b) + " of " + std::to_string(total_b) + " B)",
                  kOutOfMemory);
  }
  ck(e, "activation allocation");
  live_.insert(p);
  return p;
}

void Executor::release(void* p, cudaStream_t s) {
  if (!p || opt_.dry_run) return;
  live_.erase(p);
  ck(cudaFreeAsync(p, s), "activation free");
}

void Executor::mark_ready(Slot& sl, cudaStream_t s) {
  sl.stream = s;
  sl.ready = nullptr;
  if (s == main_ || opt_.dry_run) return;
  sl.ready = ev();
  ck(cudaEventRecord(sl.ready, s), "event");
}

void Executor::drop(Slot& sl, cudaStream_t s, bool keep_shadow) {
  if (!sl.p) return;
  if (sl.booked) book(-out_bytes_[static_cast<size_t>(&sl - slots_.data()) % nf_]);
  sl.booked = false;
  if (trace_slots()) {
    const size_t idx = static_cast<size_t>(&sl - slots_.data());
    std::fprintf(stderr, "drop mb%zu l%zu op%zu\n", idx / (cfg_.layers * nf_), (idx / nf_) % cfg_.layers, idx % nf_);
  }
  if (sl.external) {
    // a staging slot (exec.tp_fused): owned by the communicator
  } else if (keep_shadow && opt_.check_recompute && !sl.shadow) {
    sl.shadow = sl.p;  // forward-produced copy, compared against the regeneration
  } else {
    release(sl.p, s);
  }
  sl.external = false;
  sl.p = nullptr;
  sl.ready = nullptr;
  sl.regenerated = false;
  sl.fused = false;
}

void* Executor::need(int mb, int l, int pos, cudaStream_t s) {
  Slot& sl = slot(mb, l, pos);
  if (!sl.p && opt_.elide_recompute && sl.bytes) {
    // Timing-only mode: the plan's regeneration was skipped; the consumer gets a buffer of
    // the same size from the pool (stale activations of earlier ops: realistic bit patterns,
    // no extra memory), freed like a regenerated copy. Gradients of such a step are
    // meaningless and are discarded before the optimizer (see step()).
    sl.p = alloc(sl.bytes, s);
    sl.regenerated = true;
    sl.ready = nullptr;
    sl.stream = s;
    if (opt_.elide_fill && !opt_.dry_run) {
      span_begin(s, 7, mb, pos);
      ck_op(fill_noise_bf16(sl.p, sl.bytes, static_cast<uint64_t>(step_) * 7919 + pos, s), "elide fill");
      span_end(s);
    }
    return sl.p;
  }
  if (!sl.p)
    throw RtError("tensor " + std::string(op_name(op_of_[pos])) + " (mb " + std::to_string(mb) + ", layer " +
                      std::to_string(l) + ") is not resident: the timeline does not regenerate it before its consumer",
                  kParse);
  if (sl.ready && sl.stream != s) {
    if (s == main_) span_begin(main_, 4, mb, pos);
    ck(cudaStreamWaitEvent(s, sl.ready, 0), "wait");
    if (s == main_) span_end(main_);
  }
  return sl.p;
}

void* Executor::layer_input(int mb, int l, cudaStream_t s) {
  if (l == 0) return stage_in_[mb];
  const int ck_pos = nf_ - 1;  // the checkpoint is the forward sink
  return need(mb, l - 1, ck_pos, s);
}

// Philox stream of a dropout site: (global layer, microbatch, site). The TP template's all-reduce
// epilogues (AR1 / AR2) draw the same masks as the TP = 1 fused ops (PROJ_RES / FC2_RES), and no
// TP rank enters the key, so every TP rank — and a TP = 1 run of the same model — drops the same
// elements of the replicated residual stream.
uint64_t Executor::drop_stream(int l, int mb, Op op) const {
  const Op site = op == Op::AR1 ? Op::PROJ_RES : (op == Op::AR2 ? Op::FC2_RES : op);
  return (static_cast<uint64_t>(cfg_.layer0 + l + 1) << 32) | (static_cast<uint64_t>(mb) << 8) |
         static_cast<uint64_t>(site);
}

void* Executor::fused_partial() {
  return opt_.dry_run ? reinterpret_cast<void*>(0x2000) : comms_->fused_slot(static_cast<int>(fused_seq_ % 2));
}

// ============================================================ logical ledger
// The reference simulator's memory ledger (pipesim.cpp:143-183, 483-605, 722-736): every
// forward-template tensor this executor produces or drops books its profile out_bytes at the
// plan-clock time of the element (or recompute item) doing it; backward-op outputs, the embedding
// and the head are booked by the same rules (they are executor transients of other sizes). The
// trace and peak are then formed exactly like the simulator's (stable sort by time, equal
// timestamps netted), so with the simulator's pass start times (exec.ledger_pass_start_us) the
// executor's liveness decisions reproduce simulate()'s memory_traces / memory_peaks bit for bit.
void Executor::book(long long delta) {
  if (!delta) return;
  lg_.resident += host::Rat(delta);
  lg_.deltas.emplace_back(lg_.t, host::Rat(delta));
}

void Executor::ledger_reset() {
  lg_.t = lg_.free_at = host::Rat(0);
  lg_.started = false;
  lg_.pass = 0;
  lg_.deltas.clear();
  lg_.pass_release.clear();
  lg_.budget = host::Rat(prof_.hardware.mem_budget_bytes);
  const host::Rat share = host::Rat(prof_.model.static_bytes) * host::Rat(cfg_.layers) / host::Rat(prof_.model.n_layers);
  lg_.resident = share;
  lg_.deltas.emplace_back(host::Rat(0), share);
  deferred_.clear();
}

host::Rat Executor::ledger_pass_start() {
  host::Rat s = lg_.free_at;
  if (lg_.override_starts) s = lg_.starts.at(lg_.pass);
  ++lg_.pass;
  return s;
}

std::pair<host::Rat, std::vector<std::pair<host::Rat, host::Rat>>> Executor::ledger_trace() const {
  auto d = lg_.deltas;
  std::stable_sort(d.begin(), d.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  host::Rat res(0), peak(0);
  std::vector<std::pair<host::Rat, host::Rat>> tr;
  for (size_t i = 0; i < d.size(); ++i) {
    res += d[i].second;
    if (i + 1 < d.size() && d[i + 1].first == d[i].first) continue;
    if (!tr.empty() && tr.back().first == d[i].first) {
      tr.back().second = res;
    } else {
      tr.emplace_back(d[i].first, res);
    }
    peak = host::rmax(peak, res);
  }
  return {peak, tr};
}

// ============================================================ timing
cudaEvent_t Executor::ev() {
  if (ev_next_ == ev_pool_.size()) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "event");
    ev_pool_.push_back(e);
  }
  return ev_pool_[ev_next_++];
}

void Executor::span_begin(cudaStream_t s, int kind, int mb, int op) {
  if (opt_.dry_run) return;
  TimedSpan sp{ev(), ev(), kind, mb, op, s == side_, cur_bwd_};
  ck(cudaEventRecord(sp.a, s), "event");
  spans_.push_back(sp);
  open_.emplace_back(s, spans_.size() - 1);
}

void Executor::span_end(cudaStream_t s) {
  if (opt_.dry_run) return;
  for (size_t i = open_.size(); i-- > 0;)
    if (open_[i].first == s) {
      ck(cudaEventRecord(spans_[open_[i].second].b, s), "event");
      open_.erase(open_.begin() + static_cast<long>(i));
      return;
    }
}

template <class F>
void Executor::timed_op(const char* name, F&& f) {
  if (!opt_.op_timing || opt_.dry_run) {
    f();
    return;
  }
  cudaEvent_t a = ev(), b = ev();
  ck(cudaEventRecord(a, main_), "event");
  f();
  ck(cudaEventRecord(b, main_), "event");
  op_tim_.emplace_back(name, a, b);
}

void Executor::collect_spans() {
  rep_.busy_ms = rep_.comm_ms = rep_.recompute_on_demand_ms = rep_.recompute_overlapped_ms = 0;
  rep_.wait_on_recompute_ms = rep_.recv_wait_ms = rep_.elide_fill_ms = 0;
  trace_.clear();
  for (const TimedSpan& sp : spans_) {
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, sp.a, sp.b), "elapsed");
    switch (sp.kind) {
      case 0: rep_.busy_ms += ms; break;
      case 1: rep_.comm_ms += ms; break;
      case 2: rep_.recompute_on_demand_ms += ms; break;
      case 3:
      case 6: rep_.recompute_overlapped_ms += ms; break;
      case 7: rep_.elide_fill_ms += ms; break;
      case 4: rep_.wait_on_recompute_ms += ms; break;
      case 5: rep_.recv_wait_ms += ms; break;
      default: break;
    }
    if (opt_.trace) {
      float s0 = 0.f, s1 = 0.f;
      cudaEventElapsedTime(&s0, t0_, sp.a);
      cudaEventElapsedTime(&s1, t0_, sp.b);
      trace_.emplace_back(cfg_.pp_rank, sp.mb, sp.kind, sp.op, 1e3 * s0, 1e3 * s1, sp.bwd);
    }
  }
}

// ============================================================ forward operators
void Executor::fwd_op(int mb, int l, int pos, cudaStream_t s, bool recompute) {
  const ProbeStream probe(probe_stream_, s);
  struct Flag {
    bool& f;
    bool saved;
    Flag(bool& x, bool v) : f(x), saved(x) { f = v; }
    ~Flag() { f = saved; }
  } re(probe_recompute_, recompute);
  const Op op = op_of_[pos];
  Slot& out = slot(mb, l, pos);
  if (trace_slots())
    std::fprintf(stderr, "fwd mb%d l%d op%d %s%s\n", mb, l, pos, op_name(op), recompute ? " (recompute)" : "");
  if (out.p) {
    if (out.fused) {  // GeLU already written by the FC1 epilogue of this pass
      out.fused = false;
      if (!out.booked) {  // a regenerated GeLU is booked at its own item's plan time, like the simulator
        book(out_bytes_[pos]);
        out.booked = true;
      }
      return;
    }
    if (recompute) return;  // already resident (duplicate placement)
    throw RtError("forward tensor produced twice", kParse);
  }
  const long long T = cfg_.tokens();
  const int h = cfg_.hidden, hp = cfg_.hp();
  const LayerParams P = opt_.dry_run ? LayerParams{} : ps_.layer(l);
  Scratch& sc = s == side_ ? sc_side_ : sc_main_;
  const float p = cfg_.dropout;
  const uint64_t seed = cfg_.seed + static_cast<uint64_t>(step_) * 1000003ull;
  auto gemm = [&](const void* a, long long lda, const void* b, long long ldb, void* c, long long ldc, long long M,
                  long long N, long long K, const __nv_bfloat16* bias) {
    if (opt_.dry_run) return;
    GemmDesc g{a, lda, false, b, ldb, false, c, ldc, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K),
               bias, EPI_BF16};
    ck_op(gemm_run(g, s), op_name(op));
  };
  auto pos_of = [&](Op o) {
    for (int i = 0; i < nf_; ++i)
      if (op_of_[i] == o) return i;
    return -1;
  };
  size_t bytes = 2 * T * h;
  void *in = nullptr, *x = nullptr;
  switch (op) {
    case Op::LN1:
      bytes = 2 * T * h + 8 * T;
      x = layer_input(mb, l, s);
      break;
    case Op::QKV:
      bytes = 2 * T * 3 * hp;
      in = need(mb, l, pos_of(Op::LN1), s);
      break;
    case Op::ATTN:
      bytes = 2 * T * hp + 4LL * cfg_.micro_batch * cfg_.heads_rank() * cfg_.seq;
      in = need(mb, l, pos_of(Op::QKV), s);
      break;
    case Op::PROJ: in = need(mb, l, pos_of(Op::ATTN), s); break;
    case Op::PROJ_RES:
      in = need(mb, l, pos_of(Op::ATTN), s);
      x = layer_input(mb, l, s);
      break;
    case Op::LN2:
      bytes = 2 * T * h + 8 * T;
      in = need(mb, l, pos_of(tp_tmpl_ ? Op::AR1 : Op::PROJ_RES), s);
      break;
    case Op::FC1:
      bytes = 2 * T * 4 * hp;
      in = need(mb, l, pos_of(Op::LN2), s);
      break;
    case Op::GELU:
      bytes = 2 * T * 4 * hp;
      in = need(mb, l, pos_of(Op::FC1), s);
      break;
    case Op::FC2: in = need(mb, l, pos_of(Op::GELU), s); break;
    case Op::FC2_RES:
      in = need(mb, l, pos_of(Op::GELU), s);
      x = need(mb, l, pos_of(Op::PROJ_RES), s);
      break;
    default: throw RtError(std::string("operator ") + op_name(op) + " is not a compute forward op", kParse);
  }
  if (fused_ && (op == Op::PROJ || op == Op::FC2)) {  // row-parallel partial: into this rank's staging slot
    out.p = opt_.dry_run ? reinterpret_cast<void*>(0x2000) : comms_->fused_slot(static_cast<int>(fused_seq_ % 2));
    out.external = true;
  } else {
    out.p = alloc(bytes, s);
  }
  out.bytes = bytes;
  out.booked = true;
  book(out_bytes_[pos]);
  if (recompute) ++rep_.recompute_launches;
  // FC1 with its GeLU fused into the GEMM epilogue when the GeLU tensor is not resident (forward
  // pass, or both discarded and regenerated): the GeLU slot is produced here, its own op call
  // becomes a no-op. Same element, so the ledger's liveness is unchanged.
  Slot* gelu_slot = nullptr;
  if (op == Op::FC1) {
    const int gpos = pos_of(Op::GELU);
    if (gpos >= 0 && !slot(mb, l, gpos).p) {
      gelu_slot = &slot(mb, l, gpos);
      gelu_slot->p = alloc(2 * T * 4 * hp, s);
      gelu_slot->bytes = 2 * T * 4 * hp;
      gelu_slot->booked = !recompute;  // forward: same element as FC1; recompute: booked by GeLU's item
      if (!recompute) book(out_bytes_[gpos]);
      if (recompute) ++rep_.recompute_launches;
    }
  }
  if (!opt_.dry_run) {
    auto* o = static_cast<__nv_bfloat16*>(out.p);
    switch (op) {
      case Op::LN1:
      case Op::LN2: {
        auto* mean = reinterpret_cast<float*>(static_cast<char*>(out.p) + 2 * T * h);
        const auto* src = static_cast<const __nv_bfloat16*>(op == Op::LN1 ? x : in);
        ck_op(layernorm_fwd(src, op == Op::LN1 ? P.ln1_g : P.ln2_g, op == Op::LN1 ? P.ln1_b : P.ln2_b, o, mean,
                            mean + T, static_cast<int>(T), h, cfg_.ln_eps, s),
              "layernorm");
        break;
      }
      case Op::QKV: gemm(in, h, P.w_qkv, h, o, 3 * hp, T, 3 * hp, h, P.b_qkv); break;
      case Op::ATTN: {
        auto* lse = reinterpret_cast<float*>(static_cast<char*>(out.p) + 2 * T * hp);
        ck_op(attention_fwd(static_cast<const __nv_bfloat16*>(in), o, lse, cfg_.micro_batch, cfg_.seq,
                            cfg_.heads_rank(), cfg_.head_dim, s),
              "attention");
        break;
      }
      case Op::PROJ: gemm(in, hp, P.w_proj, hp, o, h, T, h, hp, nullptr); break;
      case Op::PROJ_RES: {  // out = x + dropout(attn W_proj^T + b), one GEMM with the residual epilogue
        GemmDesc g{in, hp, false, P.w_proj, hp, false, o, h, static_cast<int>(T), h, hp, P.b_proj, EPI_BF16_RESID};
        g.res = static_cast<const __nv_bfloat16*>(x);
        g.drop_p = p;
        g.drop_seed = seed;
        g.drop_stream = drop_stream(l, mb, Op::PROJ_RES);
        ck_op(gemm_run(g, s), "proj + residual");
        break;
      }
      case Op::FC1: {
        cudaEvent_t pa = nullptr, pb = nullptr;
        if (opt_.probe_fc1) {  // the bench's roofline kernel, timed on its own stream inside the step
          pa = ev();
          pb = ev();
          ck(cudaEventRecord(pa, s), "event");
        }
        if (gelu_slot) {
          GemmDesc g{in, h, false, P.w_fc1, h, false, o, 4 * hp, static_cast<int>(T), 4 * hp, h, P.b_fc1,
                     EPI_BF16_GELU, gelu_slot->p};
          ck_op(gemm_run(g, s), "fc1 + gelu");
        } else {
          gemm(in, h, P.w_fc1, h, o, 4 * hp, T, 4 * hp, h, P.b_fc1);
        }
        if (opt_.probe_fc1) {
          ck(cudaEventRecord(pb, s), "event");
          probes_.emplace_back(pa, pb);
        }
        break;
      }
      case Op::GELU: ck_op(gelu_fwd(static_cast<const __nv_bfloat16*>(in), o, T * 4 * hp, s), "gelu"); break;
      case Op::FC2: gemm(in, 4 * hp, P.w_fc2, 4 * hp, o, h, T, h, 4 * hp, nullptr); break;
      case Op::FC2_RES: {
        GemmDesc g{in, 4 * hp, false, P.w_fc2, 4 * hp, false, o, h, static_cast<int>(T), h, 4 * hp, P.b_fc2,
                   EPI_BF16_RESID};
        g.res = static_cast<const __nv_bfloat16*>(x);
        g.drop_p = p;
        g.drop_seed = seed;
        g.drop_stream = drop_stream(l, mb, Op::FC2_RES);
        ck_op(gemm_run(g, s), "fc2 + residual");
        break;
      }
      default: break;
    }
  }
  finish_production(out, bytes, s, recompute);
  if (gelu_slot) {
    finish_production(*gelu_slot, gelu_slot->bytes, s, recompute);
    gelu_slot->fused = true;
  }
}

void Executor::finish_production(Slot& out, size_t bytes, cudaStream_t s, bool recompute) {
  mark_ready(out, s);
  if (recompute) {
    out.regenerated = true;
    if (opt_.check_recompute && out.shadow && !opt_.dry_run) {
      ck(cudaMemsetAsync(d_mismatch_, 0, 8, s), "memset");
      ck_op(count_mismatch(out.p, out.shadow, bytes, d_mismatch_, s), "compare");
      unsigned long long mism = 0;
      ck(cudaMemcpyAsync(&mism, d_mismatch_, 8, cudaMemcpyDeviceToHost, s), "copy");
      ck(cudaStreamSynchronize(s), "sync");
      rep_.recompute_mismatch_words += static_cast<long long>(mism);
      ++rep_.recompute_checked;
      release(out.shadow, s);
      out.shadow = nullptr;
    }
  }
}

// Runs recompute items in order on stream s. With a plan clock, each item books its tensor at
// the clock and advances it by the op's cost (the simulator's item placement).
void Executor::run_items(const std::vector<Recompute>& items, cudaStream_t s, int span_kind, host::Rat* clock) {
  if (items.empty() || opt_.elide_recompute) return;
  span_begin(s, span_kind, items.front().owner_mb, items.front().op);
  for (const Recompute& it : items) {
    if (clock) lg_.t = *clock;
    const Op op = op_of_[it.op];
    if (op == Op::AR1 || op == Op::AR2) {
      // A discarded all-reduce output is only ever regenerated on the critical
      // path (heusched.cpp:125): re-issue its producer, then the collective.
      if (!slot(it.owner_mb, it.owner_layer, it.op).p) {
        const int prod = it.op - 1;  // PROJ / FC2 precede their all-reduce
        fwd_op(it.owner_mb, it.owner_layer, prod, main_, true);
        host::Element e;
        e.comm = true;
        e.op = it.op;
        comm_element(it.owner_mb, false, it.owner_layer, e, lg_.t);
        slot(it.owner_mb, it.owner_layer, it.op).regenerated = true;
      }
    } else {
      fwd_op(it.owner_mb, it.owner_layer, it.op, s, true);
    }
    if (clock) *clock += cost_[it.op];
  }
  span_end(s);
}

// Critical-path items of an element (plus stall-fill items the plan clock deferred to it), sorted
// by (owner_mb, owner_layer, op) as the simulator sorts them (pipesim.cpp:426-440).
void Executor::run_critical(const Key4& key, host::Rat& t) {
  auto f = crit_.find(key);
  auto d = deferred_.find(key);
  if (d == deferred_.end()) {
    if (f != crit_.end()) run_items(f->second, main_, 2, &t);
    return;
  }
  std::vector<Recompute> all = f != crit_.end() ? f->second : std::vector<Recompute>{};
  all.insert(all.end(), d->second.begin(), d->second.end());
  std::stable_sort(all.begin(), all.end(), [](const Recompute& a, const Recompute& b) {
    return std::tie(a.owner_mb, a.owner_layer, a.op) < std::tie(b.owner_mb, b.owner_layer, b.op);
  });
  deferred_.erase(d);
  run_items(all, main_, 2, &t);
}

// TP all-reduce element. Window items of (mb, bwd, l, window) are released on
// the side stream at the same instant, so their kernels overlap the NCCL transfer.
host::Rat Executor::comm_element(int mb, bool bwd, int l, const host::Element& e, const host::Rat& t) {
  const Op op = op_of_[e.op];
  host::Rat busy = t;  // plan clock: window items are packed from the comm start (pipesim.cpp:398-424)
  const long long T = cfg_.tokens();
  const int h = cfg_.hidden;
  void* buf = nullptr;
  auto pos_of = [&](Op o) {
    for (int i = 0; i < n_; ++i)
      if (op_of_[i] == o) return i;
    return -1;
  };
  if (!fused_) {
    if (op == Op::AR1) buf = need(mb, l, pos_of(Op::PROJ), main_);
    if (op == Op::AR2) buf = need(mb, l, pos_of(Op::FC2), main_);
    if (op == Op::AR_B1) buf = grad_[mb].dln2;
    if (op == Op::AR_B2) buf = grad_[mb].dln1;
  } else if (!bwd) {
    need(mb, l, pos_of(op == Op::AR1 ? Op::PROJ : Op::FC2), main_);  // the partial, in this rank's staging slot
  }
  program_.push_back({"allreduce", "tp", -1, static_cast<size_t>(T * h * 2),
                      std::string(op_name(op)) + " mb" + std::to_string(mb) + " l" + std::to_string(l)});
  cudaEvent_t go = nullptr;
  if (!opt_.dry_run) {
    go = ev();
    ck(cudaEventRecord(go, main_), "event");
    if (!fused_) ck(cudaStreamWaitEvent(tp_s_, go, 0), "wait");
  }
  // window items (the reference packs them from the comm start, pipesim.cpp:398-424)
  cudaEvent_t win_done = nullptr;
  int win_op = -1;
  if (e.window >= 0) {
    auto w = win_.find({mb, bwd, l, e.window});
    if (w != win_.end() && !opt_.elide_recompute) {
      if (!opt_.dry_run) ck(cudaStreamWaitEvent(side_, go, 0), "wait");
      run_items(w->second, side_, 3, &busy);
      if (opt_.window_join && !opt_.dry_run) {
        win_done = ev();
        ck(cudaEventRecord(win_done, side_), "event");
        win_op = w->second.front().op;
      }
    }
  }
  lg_.t = t;
  // The element after the all-reduce starts at max(comm end, window recompute end), as the reference
  // schedules it (pipesim.cpp:462, 527): a recompute that spills past the window is waited for (and
  // measured as exposed) instead of contending with the main stream for SMs.
  auto join_window = [&] {
    if (!win_done) return;
    span_begin(main_, 4, mb, win_op);
    ck(cudaStreamWaitEvent(main_, win_done, 0), "wait");
    span_end(main_);
  };
  TpPartials parts{};
  if (fused_ && !opt_.dry_run) {
    // exec.tp_fused: every rank's partial is read in place from its staging slot by one kernel on the main
    // stream that also does the consumer's elementwise work (ops_tp.cu) — no separate collective
    const long long k = fused_seq_++;
    span_begin(main_, 1, mb, e.op);
    comms_->fused_barrier(k, main_);
    const auto peers = comms_->fused_peers(static_cast<int>(k % 2));
    parts.n = static_cast<int>(peers.size());
    for (int r = 0; r < parts.n; ++r) parts.p[r] = static_cast<const __nv_bfloat16*>(peers[r]);
    if (bwd) {
      void* dst = alloc(T * h * 2, main_);
      ck_op(tp_reduce(parts, static_cast<__nv_bfloat16*>(dst), T * h, main_), "tp reduce");
      (op == Op::AR_B1 ? grad_[mb].dln2 : grad_[mb].dln1) = dst;
      span_end(main_);
      join_window();
      return busy;
    }
  } else if (fused_) {  // dry run: the reduced gradient buffer of a backward element
    if (bwd) (op == Op::AR_B1 ? grad_[mb].dln2 : grad_[mb].dln1) = alloc(T * h * 2, main_);
    if (bwd) return busy;
  } else if (!opt_.dry_run) {
    span_begin(tp_s_, 1, mb, e.op);
    if (opt_.comm_standin_us > 0)
      ck_op(comm_standin(static_cast<unsigned long long>(opt_.comm_standin_us * 1e3), opt_.comm_standin_ctas, tp_s_,
                         buf, T * h * 2, opt_.comm_standin_passes),
            "comm stand-in");
    else
      comms_->allreduce_sum_bf16(buf, static_cast<size_t>(T * h), tp_s_);
    span_end(tp_s_);
    cudaEvent_t done = ev();
    ck(cudaEventRecord(done, tp_s_), "event");
    ck(cudaStreamWaitEvent(main_, done, 0), "wait");
    join_window();
  }
  if (bwd) return busy;  // backward partials are reduced in place
  // forward: bias + dropout + residual epilogue produces the op's tensor
  Slot& out = slot(mb, l, e.op);
  out.p = alloc(2 * T * h, main_);
  out.bytes = 2 * T * h;
  out.booked = true;
  book(out_bytes_[e.op]);
  const void* resid = op == Op::AR1 ? layer_input(mb, l, main_) : need(mb, l, pos_of(Op::AR1), main_);
  if (!opt_.dry_run) {
    const LayerParams P = ps_.layer(l);
    const uint64_t seed = cfg_.seed + static_cast<uint64_t>(step_) * 1000003ull;
    if (fused_) {
      ck_op(tp_reduce_residual(parts, op == Op::AR1 ? P.b_proj : P.b_fc2, static_cast<const __nv_bfloat16*>(resid),
                               static_cast<__nv_bfloat16*>(out.p), T, h, cfg_.dropout, seed, drop_stream(l, mb, op),
                               main_),
            "tp reduce + residual");
      span_end(main_);
      join_window();
    } else {
      timed_op(op == Op::AR1 ? "ar1_epilogue" : "ar2_epilogue", [&] {
        ck_op(bias_dropout_residual_fwd(static_cast<const __nv_bfloat16*>(buf), op == Op::AR1 ? P.b_proj : P.b_fc2,
                                        static_cast<const __nv_bfloat16*>(resid), static_cast<__nv_bfloat16*>(out.p),
                                        T, h, cfg_.dropout, seed, drop_stream(l, mb, op), main_),
              "residual");
      });
    }
  }
  mark_ready(out, main_);
  // the partial (PROJ / FC2, 0 bytes in the profile) is consumed
  Slot& part = slot(mb, l, pos_of(op == Op::AR1 ? Op::PROJ : Op::FC2));
  if (!part.external) release(part.p, main_);
  part.p = nullptr;
  part.booked = false;
  part.external = false;
  return busy;
}

// ============================================================ backward operators
void Executor::bwd_op(int mb, int l, int pos, cudaStream_t s) {
  const ProbeStream probe(probe_stream_, s);
  const Op op = op_of_[pos];
  const long long T = cfg_.tokens();
  const int h = cfg_.hidden, hp = cfg_.hp();
  const LayerParams P = opt_.dry_run ? LayerParams{} : ps_.layer(l);
  Scratch& sc = sc_main_;
  const float p = cfg_.dropout;
  const uint64_t seed = cfg_.seed + static_cast<uint64_t>(step_) * 1000003ull;
  Grad& G = grad_[mb];
  auto gemm_on = [&](cudaStream_t st, const void* a, long long lda, bool amn, const void* b, long long ldb, bool bmn,
                     void* c, long long ldc, long long M, long long N, long long K, int epi) {
    if (opt_.dry_run) return;
    GemmDesc g{a, lda, amn, b, ldb, bmn, c, ldc, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), nullptr,
               epi};
    ck_op(gemm_run(g, st), amn && bmn ? "bwd dW gemm" : "bwd dX gemm");  // dW: both operands MN-major
  };
  auto gemm = [&](const void* a, long long lda, bool amn, const void* b, long long ldb, bool bmn, void* c, long long ldc,
                  long long M, long long N, long long K, int epi) { gemm_on(s, a, lda, amn, b, ldb, bmn, c, ldc, M, N, K, epi); };
  auto pos_of = [&](Op o) {
    for (int i = 0; i < nf_; ++i)
      if (op_of_[i] == o) return i;
    return -1;
  };
  auto colsum = [&](const void* x, __nv_bfloat16* acc, long long width) {
    if (!opt_.dry_run)
      ck_op(column_sum_acc(static_cast<const __nv_bfloat16*>(x), acc, 1, sc.ws, T, static_cast<int>(width), s),
            "colsum");
  };
  const bool tp = tp_tmpl_;  // template with all-reduce ops (ar1/ar2 carry the residual epilogues)
  switch (op) {
    case Op::MLP_BWD: {
      void* gelu = need(mb, l, pos_of(Op::GELU), s);
      void* fc1 = need(mb, l, pos_of(Op::FC1), s);
      void* y2 = need(mb, l, pos_of(Op::LN2), s);
      if (!opt_.dry_run)  // the FC2 branch gradient and its bias gradient in one pass
        ck_op(dropout_bwd_colsum(static_cast<const __nv_bfloat16*>(G.dy), sc.t_h, P.g_b_fc2, 1, sc.ws, T, h, p, seed,
                                 drop_stream(l, mb, tp ? Op::AR2 : Op::FC2_RES), s),
              "dropout_bwd + bias grad");
      gemm(sc.t_h, h, true, gelu, 4 * hp, true, P.g_w_fc2, 4 * hp, h, 4 * hp, T, dw_epi_);      // dW_fc2 += d^T gelu
      if (!opt_.dry_run) {  // dfc1 = (d W_fc2) * gelu'(fc1): the GeLU backward rides in the dX GEMM epilogue
        GemmDesc g{sc.t_h, h, false, P.w_fc2, 4 * hp, true, sc.t_wide, 4 * hp, static_cast<int>(T), 4 * hp, h,
                   nullptr, EPI_BF16_GELU_BWD};
        g.res = static_cast<const __nv_bfloat16*>(fc1);
        ck_op(gemm_run(g, s), "dgelu");
      }
      colsum(sc.t_wide, P.g_b_fc1, 4 * hp);
      gemm(sc.t_wide, 4 * hp, true, y2, h, true, P.g_w_fc1, h, 4 * hp, h, T, dw_epi_);       // dW_fc1 += dfc1^T y2
      // dln2 = dfc1 W_fc1: a partial over the TP ranks, all-reduced by AR_B1 (exec.tp_fused: written into
      // this rank's staging slot and reduced into a fresh buffer by the fused reduction)
      void* d2 = fused_ ? fused_partial() : (G.dln2 = alloc(T * h * 2, s));
      gemm(sc.t_wide, 4 * hp, false, P.w_fc1, h, true, d2, h, T, h, 4 * hp, EPI_BF16);
      break;
    }
    case Op::ATTN_BWD: {
      void* res1 = need(mb, l, pos_of(tp ? Op::AR1 : Op::PROJ_RES), s);
      void* ln2 = need(mb, l, pos_of(Op::LN2), s);
      void* attn = need(mb, l, pos_of(Op::ATTN), s);
      void* qkv = need(mb, l, pos_of(Op::QKV), s);
      void* ln1 = need(mb, l, pos_of(Op::LN1), s);
      const auto* mean2 = reinterpret_cast<const float*>(static_cast<char*>(ln2) + 2 * T * h);
      const auto* lse = reinterpret_cast<const float*>(static_cast<char*>(attn) + 2 * T * hp);
      G.dres = alloc(T * h * 2, s);
      if (!opt_.dry_run) {
        ck_op(layernorm_bwd(static_cast<const __nv_bfloat16*>(G.dln2), static_cast<const __nv_bfloat16*>(res1),
                            P.ln2_g, mean2, mean2 + T, static_cast<const __nv_bfloat16*>(G.dy),
                            static_cast<__nv_bfloat16*>(G.dres), P.g_ln2_g, P.g_ln2_b, 1, sc.ws, static_cast<int>(T), h, s),
              "ln2_bwd");
        ck_op(dropout_bwd_colsum(static_cast<const __nv_bfloat16*>(G.dres), sc.t_h, P.g_b_proj, 1, sc.ws, T, h, p,
                                 seed, drop_stream(l, mb, tp ? Op::AR1 : Op::PROJ_RES), s),
              "dropout_bwd + bias grad");
      }
      release(G.dln2, s);
      G.dln2 = nullptr;
      gemm(sc.t_h, h, false, P.w_proj, hp, true, sc.t_h2, hp, T, hp, h, EPI_BF16);         // dO = d W_proj
      if (!opt_.dry_run)
        ck_op(attention_bwd(static_cast<const __nv_bfloat16*>(qkv), static_cast<const __nv_bfloat16*>(attn), sc.t_h2,
                            lse, sc.t_wide, sc.ws, cfg_.micro_batch, cfg_.seq, cfg_.heads_rank(), cfg_.head_dim, s),
              "attention_bwd");
      colsum(sc.t_wide, P.g_b_qkv, 3 * hp);
      // The two weight-gradient GEMMs run concurrently (dW_proj on the aux stream, forked here and joined
      // before the op ends): at the 7B shapes dW_qkv has 384 wide tiles and dW_proj 128 for 74 CTA
      // pairs — 86.5 % of their last waves idle when run one after the other; together the proj tiles
      // fill dW_qkv's last wave. Both write only their own outputs: results are unchanged.
      const bool conc = opt_.dw_concurrent && !opt_.dry_run;
      if (conc) {
        cudaEvent_t fork = ev();
        ck(cudaEventRecord(fork, s), "event");
        ck(cudaStreamWaitEvent(aux_, fork, 0), "wait");
      }
      gemm(sc.t_wide, 3 * hp, true, ln1, h, true, P.g_w_qkv, h, 3 * hp, h, T, dw_epi_);    // dW_qkv += dqkv^T y1
      gemm_on(conc ? aux_ : s, sc.t_h, h, true, attn, hp, true, P.g_w_proj, hp, h, hp, T, dw_epi_);  // dW_proj += d^T O
      void* d1 = fused_ ? fused_partial() : (G.dln1 = alloc(T * h * 2, s));
      gemm(sc.t_wide, 3 * hp, false, P.w_qkv, h, true, d1, h, T, h, 3 * hp, EPI_BF16);  // dln1 = dqkv W_qkv
      if (conc) {
        cudaEvent_t joined = ev();
        ck(cudaEventRecord(joined, aux_), "event");
        ck(cudaStreamWaitEvent(s, joined, 0), "wait");
      }
      break;
    }
    case Op::LN1_BWD: {
      void* ln1 = need(mb, l, pos_of(Op::LN1), s);
      const auto* mean1 = reinterpret_cast<const float*>(static_cast<char*>(ln1) + 2 * T * h);
      void* x = layer_input(mb, l, s);
      void* dx = alloc(T * h * 2, s);
      if (!opt_.dry_run)
        ck_op(layernorm_bwd(static_cast<const __nv_bfloat16*>(G.dln1), static_cast<const __nv_bfloat16*>(x), P.ln1_g,
                            mean1, mean1 + T, static_cast<const __nv_bfloat16*>(G.dres), static_cast<__nv_bfloat16*>(dx),
                            P.g_ln1_g, P.g_ln1_b, 1, sc.ws, static_cast<int>(T), h, s),
              "ln1_bwd");
      release(G.dln1, s);
      release(G.dres, s);
      release(G.dy, s);  // the layer-output gradient is fully consumed
      G.dln1 = G.dres = nullptr;
      G.dy = dx;  // gradient sink -> the next (lower) layer's output gradient
      break;
    }
    default: throw RtError(std::string("operator ") + op_name(op) + " is not a compute backward op", kParse);
  }
}

// ============================================================ head / embedding
void Executor::head_forward(int mb) {
  const long long T = cfg_.tokens();
  const int h = cfg_.hidden, C = cfg_.head_chunk;
  const int V = cfg_.vocab_rank();  // this rank's vocabulary rows (all of them unless vocab-parallel)
  const bool vp = cfg_.vocab_parallel();
  void* x = need(mb, cfg_.layers - 1, nf_ - 1, main_);
  ln_f_[mb] = alloc(2 * T * h + 8 * T, main_);
  head_dy_[mb] = alloc(2 * T * h, main_);
  if (vp) {  // the launch program's collectives (dry runs record them too)
    for (long long c0 = 0; c0 < T; c0 += C) {
      program_.push_back({"allreduce", "tp", -1, static_cast<size_t>(C) * 4, "xent max mb" + std::to_string(mb)});
      program_.push_back({"allreduce", "tp", -1, static_cast<size_t>(C) * 8, "xent sum mb" + std::to_string(mb)});
    }
    program_.push_back({"allreduce", "tp", -1, static_cast<size_t>(T * h * 2), "head dX mb" + std::to_string(mb)});
  }
  if (opt_.dry_run) return;
  auto* y = static_cast<__nv_bfloat16*>(ln_f_[mb]);
  auto* mean = reinterpret_cast<float*>(static_cast<char*>(ln_f_[mb]) + 2 * T * h);
  ck_op(layernorm_fwd(static_cast<const __nv_bfloat16*>(x), ps_.p("lnf_g"), ps_.p("lnf_b"), y, mean, mean + T,
                      static_cast<int>(T), h, cfg_.ln_eps, main_),
        "final_ln");
  const __nv_bfloat16* w = ps_.p("w_head");
  float* gw = head_gw32_;  // fp32 across chunks and microbatches, added to the bf16 gradient at step end
  const float scale = 1.0f / static_cast<float>(T * cfg_.n_micro);
  const long long v0 = vp ? static_cast<long long>(cfg_.tp_rank) * V : 0;
  for (long long c0 = 0; c0 < T; c0 += C) {
    const __nv_bfloat16* yc = y + c0 * h;
    const int* lab = d_labels_ + mb * T + c0;
    GemmDesc lg{yc, h, false, w, h, false, sc_main_.logits, V, C, V, h, nullptr, EPI_BF16};
    ck_op(gemm_run(lg, main_), "lm_head");
    if (!vp) {
      ck_op(xent_fwd_bwd(sc_main_.logits, lab, d_loss_ + mb * T + c0, C, V, scale, main_), "xent");
    } else {
      // Megatron vocab-parallel cross-entropy: row max and (sum of exp, target logit) all-reduced over the
      // TP group between the three kernels. Standalone (one TP rank alone) skips them: timing only.
      ck_op(xent_vp_max(sc_main_.logits, xent_max_, C, V, main_), "xent max");
      if (comms_) comms_->allreduce_f32(xent_max_, static_cast<size_t>(C), true, main_);
      ck_op(xent_vp_sum(sc_main_.logits, lab, v0, xent_max_, xent_st_, C, V, main_), "xent sum");
      if (comms_) comms_->allreduce_f32(xent_st_, static_cast<size_t>(2 * C), false, main_);
      ck_op(xent_vp_finish(sc_main_.logits, lab, v0, xent_max_, xent_st_, d_loss_ + mb * T + c0, C, V, scale, main_),
            "xent finish");
    }
    GemmDesc dw{sc_main_.logits, V, true, yc, h, true, gw, h, V, h, C, nullptr,
                head_first_ ? EPI_STORE_F32 : EPI_ACC_F32};
    head_first_ = false;
    GemmDesc dx{sc_main_.logits, V, false, w, h, true, static_cast<__nv_bfloat16*>(head_dy_[mb]) + c0 * h, h, C, h, V,
                nullptr, EPI_BF16};
    // exec.dw_concurrent: dX (128 wide tiles at the 7B shape, 1.73 waves of CTA pairs) on the aux stream
    // beside dW (3152 tiles), joined before the next chunk's logits overwrite the buffer both read
    if (opt_.dw_concurrent) {
      cudaEvent_t fork = ev();
      ck(cudaEventRecord(fork, main_), "event");
      ck(cudaStreamWaitEvent(aux_, fork, 0), "wait");
      ck_op(gemm_run(dx, aux_), "lm_head dX");
      ck_op(gemm_run(dw, main_), "lm_head dW");
      cudaEvent_t joined = ev();
      ck(cudaEventRecord(joined, aux_), "event");
      ck(cudaStreamWaitEvent(main_, joined, 0), "wait");
    } else {
      ck_op(gemm_run(dw, main_), "lm_head dW");
      ck_op(gemm_run(dx, main_), "lm_head dX");
    }
  }
  if (vp) {  // the rows' gradient w.r.t. the final LayerNorm output: partial per vocabulary slice
    if (comms_)
      comms_->allreduce_sum_bf16(head_dy_[mb], static_cast<size_t>(T * h), main_);
    else if (opt_.comm_standin_us > 0)
      ck_op(comm_standin(static_cast<unsigned long long>(opt_.comm_standin_us * 1e3), opt_.comm_standin_ctas, main_,
                         head_dy_[mb], T * h * 2, opt_.comm_standin_passes),
            "head dX stand-in");
  }
}

void Executor::head_backward(int mb) {
  const long long T = cfg_.tokens();
  const int h = cfg_.hidden;
  void* x = need(mb, cfg_.layers - 1, nf_ - 1, main_);
  grad_[mb].dy = alloc(2 * T * h, main_);
  if (!opt_.dry_run) {
    const auto* mean = reinterpret_cast<const float*>(static_cast<char*>(ln_f_[mb]) + 2 * T * h);
    ck_op(layernorm_bwd(static_cast<const __nv_bfloat16*>(head_dy_[mb]), static_cast<const __nv_bfloat16*>(x),
                        ps_.p("lnf_g"), mean, mean + T, nullptr, static_cast<__nv_bfloat16*>(grad_[mb].dy),
                        ps_.g("lnf_g"), ps_.g("lnf_b"), 1, sc_main_.ws, static_cast<int>(T), h, main_),
          "final_ln_bwd");
  }
  release(head_dy_[mb], main_);
  release(ln_f_[mb], main_);
  head_dy_[mb] = ln_f_[mb] = nullptr;
}

// ============================================================ passes
void Executor::forward_pass(int mb) {
  cur_bwd_ = false;
  const long long T = cfg_.tokens();
  const int h = cfg_.hidden;
  const uint64_t seed = cfg_.seed + static_cast<uint64_t>(step_) * 1000003ull;
  stage_in_[mb] = alloc(2 * T * h, main_);
  if (cfg_.first()) {
    if (!opt_.dry_run)
      timed_op("embed", [&] {
        ck_op(embedding_fwd(d_tokens_ + mb * T, ps_.p("wte"), ps_.p("wpe"), static_cast<__nv_bfloat16*>(stage_in_[mb]),
                          cfg_.micro_batch, cfg_.seq, h, cfg_.dropout, seed, kEmbedStream | mb, main_),
            "embedding");
      });
  } else {
    program_.push_back({"recv", "pp_act", cfg_.pp_rank - 1, static_cast<size_t>(2 * T * h), "F mb" + std::to_string(mb)});
    if (opt_.standalone && !opt_.dry_run) {
      ck(cudaMemcpyAsync(stage_in_[mb], syn_act_, static_cast<size_t>(2 * T * h), cudaMemcpyDeviceToDevice, main_),
         "synthetic activation");
    } else if (!opt_.dry_run) {
      cudaEvent_t a = ev();
      ck(cudaEventRecord(a, main_), "event");  // buffer allocated on main
      ck(cudaStreamWaitEvent(pa_s_, a, 0), "wait");
      comms_->recv_bf16(stage_in_[mb], static_cast<size_t>(T * h), cfg_.pp_rank - 1, Channel::PP_ACT, pa_s_);
      cudaEvent_t b = ev();
      ck(cudaEventRecord(b, pa_s_), "event");
      span_begin(main_, 5, mb);
      ck(cudaStreamWaitEvent(main_, b, 0), "wait");
      span_end(main_);
    }
  }
  span_begin(main_, 0, mb);
  // plan clock (pipesim.cpp:442-481 expand_fwd): the ledger books at these times
  const host::Rat start = ledger_pass_start();
  lg_.started = true;
  host::Rat t = start;
  if (cfg_.first()) {
    t += pre_dur_;
    lg_.t = start;
    book(pre_bytes_);
    lg_.pass_release[mb] += pre_bytes_;
  }
  for (int l = 0; l < cfg_.layers; ++l) {
    for (size_t ei = 0; ei < fel_.size(); ++ei) {
      const host::Element& e = fel_[ei];
      run_critical({mb, false, l, static_cast<int>(ei)}, t);
      host::Rat next = t + e.dur;
      if (e.comm) {
        next = host::rmax(next, comm_element(mb, false, l, e, t));
      } else {
        lg_.t = t;
        for (int pos : e.ops) timed_op(op_name(op_of_[pos]), [&] { fwd_op(mb, l, pos, main_, false); });
      }
      // discarded tensors drop after their last forward consumer (pipesim.cpp:496-504)
      lg_.t = t + e.dur;
      for (int i = 0; i < nf_; ++i)
        if (!tl_.plan.retained[i] && std::max(made_in_[i], last_fwd_use_[i]) == static_cast<int>(ei))
          drop(slot(mb, l, i), main_, true);
      t = next;
    }
  }
  if (cfg_.last()) {
    t += post_dur_;
    lg_.t = t;
    book(post_bytes_);
    lg_.pass_release[mb] += post_bytes_;
  }
  lg_.free_at = t;
  if (cfg_.last()) {
    timed_op("head_fwd", [&] { head_forward(mb); });
  } else {
    void* out = need(mb, cfg_.layers - 1, nf_ - 1, main_);
    program_.push_back({"send", "pp_act", cfg_.pp_rank + 1, static_cast<size_t>(2 * T * h), "F mb" + std::to_string(mb)});
    if (opt_.standalone && !opt_.dry_run) {
      (void)out;
      ck(cudaEventRecord(act_sent_[mb], main_), "event");
    } else if (!opt_.dry_run) {
      cudaEvent_t a = ev();
      ck(cudaEventRecord(a, main_), "event");
      ck(cudaStreamWaitEvent(pa_s_, a, 0), "wait");
      comms_->send_bf16(out, static_cast<size_t>(T * h), cfg_.pp_rank + 1, Channel::PP_ACT, pa_s_);
      ck(cudaEventRecord(act_sent_[mb], pa_s_), "event");
    }
  }
  span_end(main_);
}

void Executor::backward_pass(int mb) {
  // The first backward pass of the step writes the layer weight gradients (bf16 store
  // epilogue); later microbatches accumulate into them in bf16 (fp32 sum in the epilogue,
  // one rounding per microbatch): the 2 B/parameter gradient of the paper's accounting.
  dw_epi_ = bwd_passes_ == 0 ? EPI_BF16 : EPI_ACC_BF16;  // bf16 gradients: store on the first pass
  ++bwd_passes_;
  cur_bwd_ = true;
  const long long T = cfg_.tokens();
  const int h = cfg_.hidden;
  const host::Rat start = ledger_pass_start();
  // cool-down stall fill: released on the side stream before the gradient arrives, so it fills the
  // bubble the receive leaves (pipesim.cpp:620-646). On the simulator's clock (ledger_pass_start_us)
  // an item that does not fit the gap or the budget moves to the critical path at element 0 of its
  // layer, as there; without it every item goes to the bubble (the gap is physical, not modelled).
  auto st = stall_.find(mb);
  cudaEvent_t stall_done = nullptr;
  int stall_op = -1;
  if (st != stall_.end() && !opt_.elide_recompute) {
    std::vector<Recompute> fit;
    host::Rat t = lg_.free_at;
    if (!lg_.override_starts) {
      fit = st->second;
    } else if (start > lg_.free_at && lg_.started) {
      host::Rat resident = lg_.resident;
      for (const Recompute& it : st->second) {
        const host::Rat b(out_bytes_[it.op]);
        if (t + cost_[it.op] <= start && resident + b <= lg_.budget) {
          fit.push_back(it);
          t += cost_[it.op];
          resident += b;
        } else {
          deferred_[{mb, true, it.owner_layer, 0}].push_back(it);
        }
      }
    } else {  // no gap on the simulator's clock: the reference never runs them (pipesim.cpp:620); the
              // executor still must regenerate them, on the critical path
      for (const Recompute& it : st->second) deferred_[{mb, true, it.owner_layer, 0}].push_back(it);
    }
    if (!fit.empty()) {
      if (!opt_.dry_run) {
        cudaEvent_t a = ev();
        ck(cudaEventRecord(a, main_), "event");
        ck(cudaStreamWaitEvent(side_, a, 0), "wait");
      }
      host::Rat clock = lg_.free_at;
      run_items(fit, side_, 6, &clock);
      if (opt_.window_join && !opt_.dry_run) {
        stall_done = ev();
        ck(cudaEventRecord(stall_done, side_), "event");
        stall_op = fit.front().op;
      }
    }
  }
  lg_.started = true;
  if (cfg_.last()) {
    timed_op("head_bwd", [&] { head_backward(mb); });
  } else {
    grad_[mb].dy = alloc(2 * T * h, main_);
    program_.push_back({"recv", "pp_grad", cfg_.pp_rank + 1, static_cast<size_t>(2 * T * h), "B mb" + std::to_string(mb)});
    if (opt_.standalone && !opt_.dry_run) {
      const double wait_us = mb < static_cast<int>(opt_.standin_grad_wait_us.size()) ? opt_.standin_grad_wait_us[mb] : 0;
      if (wait_us > 0) {  // the modelled pipeline stall before this gradient arrives
        cudaEvent_t a = ev();
        ck(cudaEventRecord(a, main_), "event");
        ck(cudaStreamWaitEvent(pg_s_, a, 0), "wait");
        ck_op(comm_standin(static_cast<unsigned long long>(wait_us * 1e3), 1, pg_s_), "recv stand-in");
        cudaEvent_t b = ev();
        ck(cudaEventRecord(b, pg_s_), "event");
        span_begin(main_, 5, mb);
        ck(cudaStreamWaitEvent(main_, b, 0), "wait");
        span_end(main_);
      }
      ck(cudaMemcpyAsync(grad_[mb].dy, syn_grad_, static_cast<size_t>(2 * T * h), cudaMemcpyDeviceToDevice, main_),
         "synthetic gradient");
    } else if (!opt_.dry_run) {
      cudaEvent_t a = ev();
      ck(cudaEventRecord(a, main_), "event");
      ck(cudaStreamWaitEvent(pg_s_, a, 0), "wait");
      comms_->recv_bf16(grad_[mb].dy, static_cast<size_t>(T * h), cfg_.pp_rank + 1, Channel::PP_GRAD, pg_s_);
      cudaEvent_t b = ev();
      ck(cudaEventRecord(b, pg_s_), "event");
      span_begin(main_, 5, mb);
      ck(cudaStreamWaitEvent(main_, b, 0), "wait");
      span_end(main_);
    }
  }
  if (stall_done) {
    // The pass starts once the stall-fill regenerations are done (they were planned into the bubble
    // before it, pipesim.cpp:620-646): an overrun is waited for and measured as exposed recompute,
    // not left to contend with the backward kernels for SMs.
    span_begin(main_, 4, mb, stall_op);
    ck(cudaStreamWaitEvent(main_, stall_done, 0), "wait");
    span_end(main_);
  }
  span_begin(main_, 0, mb);
  // plan clock (pipesim.cpp:509-605 expand_bwd / release_bwd)
  host::Rat t = start;
  long long sink = 0;
  for (int l = cfg_.layers - 1; l >= 0; --l) {
    bool first_elem = true;
    for (size_t ei = 0; ei < bel_.size(); ++ei) {
      const host::Element& e = bel_[ei];
      run_critical({mb, true, l, static_cast<int>(ei)}, t);
      const host::Rat tend = t + e.dur;
      host::Rat next = tend;
      lg_.t = t;
      if (e.comm) {
        book(out_bytes_[e.op]);  // logical: the all-reduced gradient (reduced in place here)
        next = host::rmax(next, comm_element(mb, true, l, e, t));
      } else {
        long long made = 0;  // logical: backward op outputs (executor transients of other sizes)
        for (int pos : e.ops) made += out_bytes_[pos];
        book(made);
        for (int pos : e.ops) timed_op(op_name(op_of_[pos]), [&] { bwd_op(mb, l, pos, main_); });
      }
      // retained / regenerated tensors drop after their last backward consumer
      lg_.t = tend;
      for (int i = 0; i < nf_; ++i)
        if (last_bwd_user_[i] == static_cast<int>(ei)) drop(slot(mb, l, i), main_, false);
      long long out = 0;  // backward transients whose last consumer this element is (the sink crosses layers)
      for (int o = nf_; o < n_ - 1; ++o)
        if ((bwd_last_use_[o] >= 0 ? bwd_last_use_[o] : bwd_elem_[o]) == static_cast<int>(ei)) out += out_bytes_[o];
      book(-out);
      t = next;
      if (first_elem) {  // the downstream layer's gradient has now been consumed
        first_elem = false;
        lg_.t = t;
        book(-sink);
        sink = 0;
      }
    }
    // end-of-layer sweep (pipesim.cpp:546-569): everything else of (mb, l)
    if (l == cfg_.layers - 1 && !cfg_.last() && !opt_.dry_run)
      ck(cudaStreamWaitEvent(main_, act_sent_[mb], 0), "wait");  // the activation send read it
    lg_.t = t;
    for (int i = 0; i < nf_; ++i) {
      Slot& sl = slot(mb, l, i);
      drop(sl, main_, false);
      if (sl.shadow) {
        release(sl.shadow, main_);
        sl.shadow = nullptr;
      }
    }
    if (n_ > nf_) sink = out_bytes_[n_ - 1];
  }
  lg_.t = t;
  book(-sink);
  if (auto pe = lg_.pass_release.find(mb); pe != lg_.pass_release.end()) {
    book(-pe->second);
    lg_.pass_release.erase(pe);
  }
  lg_.free_at = t;
  void* dx = grad_[mb].dy;
  if (cfg_.first()) {
    if (!opt_.dry_run) {
      void* ws = alloc(embedding_bwd_workspace(cfg_.micro_batch, cfg_.seq, h), main_);
      const uint64_t seed = cfg_.seed + static_cast<uint64_t>(step_) * 1000003ull;
      ck_op(embedding_bwd(d_tokens_ + mb * T, static_cast<const __nv_bfloat16*>(dx), emb_gw32_,
                          emb_gw32_ + static_cast<size_t>(cfg_.vocab) * h,
                          static_cast<float*>(ws), cfg_.micro_batch, cfg_.seq, h, cfg_.vocab, cfg_.dropout, seed,
                          kEmbedStream | mb, main_),
            "embedding_bwd");
      release(ws, main_);
    }
    release(dx, main_);
  } else {
    program_.push_back({"send", "pp_grad", cfg_.pp_rank - 1, static_cast<size_t>(2 * T * h), "B mb" + std::to_string(mb)});
    if (opt_.standalone && !opt_.dry_run) {
      release(dx, main_);
    } else {
      if (!opt_.dry_run) {
        cudaEvent_t a = ev();
        ck(cudaEventRecord(a, main_), "event");
        ck(cudaStreamWaitEvent(pg_s_, a, 0), "wait");
        comms_->send_bf16(dx, static_cast<size_t>(T * h), cfg_.pp_rank - 1, Channel::PP_GRAD, pg_s_);
        ck(cudaEventRecord(grad_sent_[mb], pg_s_), "event");
      }
      release(dx, pg_s_);  // stream-ordered after the send; main never waits on the peer
    }
  }
  grad_[mb].dy = nullptr;
  release(stage_in_[mb], main_);
  stage_in_[mb] = nullptr;
  span_end(main_);
}

// ============================================================ step
void Executor::step(const int* tokens, const int* labels, float* loss_out) {
  ++step_;
  ev_next_ = 0;
  spans_.clear();
  open_.clear();
  program_.clear();
  rep_ = StepReport{};
  probes_.clear();
  op_events_.clear();
  bwd_passes_ = 0;
  ledger_reset();
  const long long T = cfg_.tokens();
  const size_t ntok = static_cast<size_t>(cfg_.n_micro) * T;
  const auto passes = host::stage_passes(cfg_.pp, cfg_.pp_rank, cfg_.n_micro);
  if (opt_.dry_run) {
    for (auto [bwd, mb] : passes) bwd ? backward_pass(mb) : forward_pass(mb);
    return;
  }
  const long long launches0 = launch_count();
  const auto host0 = std::chrono::steady_clock::now();
  ck(cudaEventRecord(t0_, main_), "event");
  const ProbeStream probe(probe_stream_, main_);
  if (opt_.probe_ops) {  // the side stream's first operator is timed from here too
    cudaEvent_t e = ev();
    ck(cudaEventRecord(e, side_), "event");
    op_events_.emplace_back("(start)", side_, e);
    op_events_.emplace_back("(start)", main_, t0_);
  }
  if (cfg_.first() && tokens) {
    std::memcpy(h_tokens_, tokens, ntok * 4);
    ck(cudaMemcpyAsync(d_tokens_, h_tokens_, ntok * 4, cudaMemcpyHostToDevice, main_), "h2d tokens");
  }
  if (cfg_.last() && labels) {
    std::memcpy(h_labels_, labels, ntok * 4);
    ck(cudaMemcpyAsync(d_labels_, h_labels_, ntok * 4, cudaMemcpyHostToDevice, main_), "h2d labels");
  }
  ck(cudaMemsetAsync(ps_.grad, 0, static_cast<size_t>(ps_.count()) * 2, main_), "zero grads");
  head_first_ = true;
  if (cfg_.first())  // fp32 embedding-gradient accumulator (deterministic), folded into the bf16 grads at step end
    ck(cudaMemsetAsync(emb_gw32_, 0, static_cast<size_t>(cfg_.vocab + cfg_.seq) * cfg_.hidden * 4, main_),
       "zero embedding grads");
  for (auto [bwd, mb] : passes) bwd ? backward_pass(mb) : forward_pass(mb);
  ck(cudaStreamWaitEvent(main_, [&] {
       cudaEvent_t e = ev();
       ck(cudaEventRecord(e, side_), "event");
       return e;
     }(), 0),
     "join side");
  // Timing-only elided mode: the gradients are computed from stale buffers and may be
  // non-finite; they are zeroed and the update runs with a zero learning rate (same bytes
  // moved) so the weights, and the next steps' forward activations, stay valid.
  const size_t hsz = static_cast<size_t>(cfg_.hidden);
  if (cfg_.last() && !head_first_)
    ck_op(add_f32_to_bf16(head_gw32_, ps_.g("w_head"), static_cast<long long>(cfg_.vocab_rank()) * hsz, main_),
          "head grad");
  if (cfg_.first()) {
    ck_op(add_f32_to_bf16(emb_gw32_, ps_.g("wte"), static_cast<long long>(cfg_.vocab) * hsz, main_), "wte grad");
    ck_op(add_f32_to_bf16(emb_gw32_ + cfg_.vocab * hsz, ps_.g("wpe"), static_cast<long long>(cfg_.seq) * hsz, main_),
          "wpe grad");
  }
  if (opt_.elide_recompute)
    ck(cudaMemsetAsync(ps_.grad, 0, static_cast<size_t>(ps_.count()) * 2, main_), "zero grads (elided)");
  ck_op(adam_step(ps_.master, ps_.param, ps_.grad, 1, ps_.m, ps_.v, ps_.count(), opt_.elide_recompute ? 0.f : cfg_.lr,
                  cfg_.beta1, cfg_.beta2, cfg_.adam_eps, opt_.elide_recompute ? 0.f : cfg_.weight_decay, step_, 1.0f,
                  main_),
        "adam");
  if (cfg_.last()) ck(cudaMemcpyAsync(h_loss_, d_loss_, ntok * 4, cudaMemcpyDeviceToHost, main_), "d2h loss");
  ck(cudaEventRecord(t1_, main_), "event");
  rep_.host_issue_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host0).count();
  rep_.kernel_launches = launch_count() - launches0;
  ck(cudaEventSynchronize(t1_), "step");
  float ms = 0.f;
  ck(cudaEventElapsedTime(&ms, t0_, t1_), "elapsed");
  rep_.step_ms = ms;
  collect_spans();
  op_tim_ms_.clear();
  for (const auto& [name, a, b] : op_tim_) {
    float d = 0.f;
    ck(cudaEventElapsedTime(&d, a, b), "op timing");
    op_tim_ms_[name].push_back(d);
  }
  op_tim_.clear();
  for (const auto& [a, b] : probes_) {
    float pm = 0.f;
    ck(cudaEventElapsedTime(&pm, a, b), "probe");
    rep_.probe_ms += pm;
    ++rep_.probe_launches;
  }
  probes_.clear();
  if (opt_.probe_ops) {
    std::map<std::string, std::pair<long long, double>> acc;
    std::map<cudaStream_t, cudaEvent_t> prev;
    op_stream_ms_[0] = op_stream_ms_[1] = 0;
    for (const auto& [name, st, e] : op_events_) {
      auto it = prev.find(st);
      if (it != prev.end()) {
        float d = 0.f;
        ck(cudaEventElapsedTime(&d, it->second, e), "probe");
        auto& a = acc[std::string(st == side_ ? "side: " : "") + name];
        ++a.first;
        a.second += d;
        op_stream_ms_[st == side_ ? 1 : 0] += d;
      }
      prev[st] = e;
    }
    op_times_.clear();
    for (const auto& [k, v] : acc) op_times_.emplace_back(k, v.first, v.second);
    op_events_.clear();
  }
  if (cfg_.last()) {
    double s = 0;
    for (size_t i = 0; i < ntok; ++i) s += h_loss_[i];
    rep_.loss = s / static_cast<double>(ntok);
  }
  if (loss_out) *loss_out = static_cast<float>(rep_.loss);
  size_t hw = 0;
  cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrUsedMemHigh, &hw);
  rep_.pool_high_water = hw;
  uint64_t rsv = 0;
  cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrReservedMemCurrent, &rsv);
  rep_.pool_reserved = rsv;
}

// ============================================================ reports
std::string Executor::stats_json() const {
  Json j;
  j["stage"] = cfg_.pp_rank;
  j["tp_rank"] = cfg_.tp_rank;
  j["step"] = step_;
  j["iteration_ms"] = rep_.step_ms;
  j["busy_ms"] = rep_.busy_ms;
  j["comm_ms"] = rep_.comm_ms;
  j["recv_wait_ms"] = rep_.recv_wait_ms;
  j["recompute_on_demand_ms"] = rep_.recompute_on_demand_ms;
  j["recompute_overlapped_ms"] = rep_.recompute_overlapped_ms;
  j["wait_on_recompute_ms"] = rep_.wait_on_recompute_ms;
  j["exposed_recompute_ms"] = rep_.recompute_on_demand_ms + rep_.wait_on_recompute_ms;
  j["recompute_launches"] = rep_.recompute_launches;
  j["kernel_launches"] = rep_.kernel_launches;
  j["recompute_checked"] = rep_.recompute_checked;
  j["recompute_mismatch_words"] = rep_.recompute_mismatch_words;
  j["loss"] = rep_.loss;
  j["pool_high_water_bytes"] = rep_.pool_high_water;
  j["probe_fc1_launches"] = rep_.probe_launches;
  j["probe_fc1_ms"] = rep_.probe_ms;
  j["alloc_host_ms"] = rep_.alloc_host_ms;
  j["alloc_host_max_ms"] = rep_.alloc_host_max_ms;
  j["host_issue_ms"] = rep_.host_issue_ms;
  j["elide_fill_ms"] = rep_.elide_fill_ms;
  if (opt_.op_timing) j["op_timing_ms"] = op_tim_ms_;
  j["pool_reserved_bytes"] = rep_.pool_reserved;
  j["pool_reserved_at_init_bytes"] = pool_reserved_init_;
  if (opt_.probe_ops) {
    Json po = Json::object();
    for (const auto& [k, n, ms] : op_times_) po[k] = {n, ms};
    j["probe_ops"] = po;
    j["probe_ops_main_ms"] = op_stream_ms_[0];
    j["probe_ops_side_ms"] = op_stream_ms_[1];
  }
  j["static_bytes_allocated"] = static_cast<long long>(ps_.count()) * 16;
  j["params"] = ps_.count();
  j["layers"] = cfg_.layers;
  j["microbatches"] = cfg_.n_micro;
  j["tokens_per_microbatch"] = cfg_.tokens();
  // logical ledger of the last step (plan clock): simulate()'s memory_peaks / memory_traces entry for
  // this stage when exec.ledger_pass_start_us carries the simulator's pass starts
  const auto [peak, tr] = ledger_trace();
  Json lt = Json::array();
  for (const auto& [t, b] : tr) lt.push_back({host::to_canonical(t), host::to_canonical(b)});
  j["ledger"] = {{"memory_peak_bytes", host::to_canonical(peak)}, {"memory_trace", lt},
                 {"deltas", lg_.deltas.size()}, {"plan_clock", lg_.override_starts ? "simulator" : "back-to-back"}};
  return j.dump();
}

// Measured counterpart of simulate()'s SimReport for this stage (pipesim.hpp:68-75): CUDA-event
// times on the executor's streams, the logical ledger's peak, and (exec.trace) the timeline.
host::PipeResult Executor::measured_result() const {
  auto us = [](double v) { return host::Rat::frac(std::llround(v * 1000.0), 1000); };  // ns resolution
  host::PipeResult r;
  r.iteration_us = us(rep_.step_ms * 1000.0);
  host::StageSummary st;
  st.busy = us(rep_.busy_ms * 1000.0);
  st.comm = us(rep_.comm_ms * 1000.0);
  st.stall = us(rep_.recv_wait_ms * 1000.0);
  st.on_demand = us((rep_.recompute_on_demand_ms + rep_.wait_on_recompute_ms) * 1000.0);
  st.overlapped = us(rep_.recompute_overlapped_ms * 1000.0);
  r.stages.push_back(st);
  host::Rat kept(0);  // tensor-path breakdown, weighted like pipesim.cpp:705-720
  for (int o = 0; o < nf_; ++o)
    if (tl_.plan.retained[o]) kept += cost_[o] * host::Rat(cfg_.layers) * host::Rat(cfg_.n_micro);
  const host::Rat total = kept + st.overlapped + st.on_demand;
  if (total.sign() == 0)
    r.breakdown.push_back({host::Rat(1), host::Rat(0), host::Rat(0)});
  else
    r.breakdown.push_back({kept / total, st.overlapped / total, st.on_demand / total});
  const auto lt = ledger_trace();
  r.peaks.push_back(lt.first);
  r.traces.push_back(lt.second);
  for (const auto& [stage, mb, k, op, a, b, bwd] : trace_) {
    host::Event e;
    e.stage = stage;
    e.microbatch = mb;
    e.op = k == 0 || k == 5 ? -1 : op;
    e.start = us(a);
    e.end = us(b);
    switch (k) {
      case 0: e.kind = bwd ? host::EvKind::Bwd : host::EvKind::Fwd; break;
      case 1: e.kind = bwd ? host::EvKind::CommBwd : host::EvKind::CommFwd; break;
      case 2:
      case 4: e.kind = host::EvKind::Recompute; break;  // on demand: kernels, or main waiting on the side stream
      case 3:
        e.kind = host::EvKind::Recompute;
        e.overlapped = true;
        break;
      case 5: e.kind = host::EvKind::Stall; break;  // waiting for a pipeline receive
      case 6:
        e.kind = host::EvKind::StallRecompute;
        e.overlapped = true;
        break;
      default: continue;
    }
    r.events.push_back(e);
  }
  std::stable_sort(r.events.begin(), r.events.end(), [](const host::Event& a, const host::Event& b) {
    if (a.start != b.start) return a.start < b.start;
    if (a.stage != b.stage) return a.stage < b.stage;
    return static_cast<int>(a.kind) < static_cast<int>(b.kind);
  });
  return r;
}

std::string Executor::report_json() const { return host::simreport_json(measured_result()); }

// emit_trace (pipesim.cpp:781-810) of the measured timeline: 0 Chrome trace, 1 CSV.
std::string Executor::trace(int format) const {
  const host::PipeResult r = measured_result();
  return format == 1 ? host::trace_csv(r) : host::trace_chrome(r);
}

std::string Executor::program_json() const {
  Json a = Json::array();
  for (const CommOp& c : program_) {
    Json o;
    o["kind"] = c.kind;
    o["comm"] = c.comm;
    o["peer"] = c.peer;
    o["bytes"] = c.bytes;
    o["what"] = c.what;
    a.push_back(o);
  }
  return a.dump();
}

void Executor::get_tensor(const std::string& name, void* host, size_t bytes) {
  if (opt_.dry_run) throw RtError("dry run has no tensors", kValidation);
  const bool grad = name.rfind("grad:", 0) == 0;
  const std::string base = grad ? name.substr(5) : name;
  for (const auto& r : ps_.refs())
    if (r.name == base) {
      const size_t want = static_cast<size_t>(r.n) * (grad ? 4 : 2);  // gradients are returned as fp32
      if (bytes != want) throw RtError("tensor " + name + " has " + std::to_string(want) + " bytes", kValidation);
      ck(cudaStreamSynchronize(main_), "sync");
      if (grad) {
        std::vector<__nv_bfloat16> tmp(static_cast<size_t>(r.n));
        ck(cudaMemcpy(tmp.data(), ps_.grad + r.off, tmp.size() * 2, cudaMemcpyDeviceToHost), "d2h");
        float* out = static_cast<float*>(host);
        for (size_t i = 0; i < tmp.size(); ++i) out[i] = __bfloat162float(tmp[i]);
      } else {
        ck(cudaMemcpy(host, ps_.param + r.off, bytes, cudaMemcpyDeviceToHost), "d2h");
      }
      return;
    }
  throw RtError("unknown tensor " + name, kValidation);
}

void Executor::set_tensor(const std::string& name, const void* host, size_t bytes) {
  // fp32 master values; the bf16 working copy is derived
  for (const auto& r : ps_.refs())
    if (r.name == name) {
      if (bytes != static_cast<size_t>(r.n) * 4) throw RtError("set_tensor expects fp32 values", kValidation);
      ck(cudaMemcpy(ps_.master + r.off, host, bytes, cudaMemcpyHostToDevice), "h2d");
      ck_op(f32_to_bf16(ps_.master + r.off, ps_.param + r.off, r.n, main_), "copy");  // Adam state untouched
      ck(cudaStreamSynchronize(main_), "sync");
      return;
    }
  throw RtError("unknown tensor " + name, kValidation);
}

}  // namespace lynx::rt

// ============================================================ C-ABI
#include "../../../include/lynx_rt.h"

namespace {
char* dupstr(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const lynx::rt::RtError& e) {
    return lynx::set_error(e.what(), e.code);
  } catch (const lynx::host::PlanError& e) {
    return lynx::set_error(e.what(), e.status);
  } catch (const std::exception& e) {
    return lynx::set_error(e.what(), lynx::kParse);
  }
}
}  // namespace

struct lynx_rt {
  std::unique_ptr<lynx::rt::Executor> ex;
};

extern "C" {

int lynx_rt_create(const char* profile_json, const char* timeline_json, const char* config_json, lynx_rt** out) {
  *out = nullptr;
  return guard([&] {
    auto h = std::make_unique<lynx_rt>();
    h->ex = std::make_unique<lynx::rt::Executor>(profile_json, timeline_json, config_json);
    *out = h.release();
  });
}

int lynx_rt_step(lynx_rt* h, const int* tokens, const int* labels, float* loss) {
  return guard([&] { h->ex->step(tokens, labels, loss); });
}

char* lynx_rt_report_json(lynx_rt* h, int* status) {
  std::string s;
  const int st = guard([&] { s = h->ex->report_json(); });
  if (status) *status = st;
  return st ? nullptr : dupstr(s);
}

char* lynx_rt_stats_json(lynx_rt* h, int* status) {
  std::string s;
  const int st = guard([&] { s = h->ex->stats_json(); });
  if (status) *status = st;
  return st ? nullptr : dupstr(s);
}

char* lynx_rt_trace(lynx_rt* h, int format, int* status) {
  std::string s;
  const int st = guard([&] { s = h->ex->trace(format); });
  if (status) *status = st;
  return st ? nullptr : dupstr(s);
}

char* lynx_rt_program_json(lynx_rt* h, int* status) {
  std::string s;
  const int st = guard([&] { s = h->ex->program_json(); });
  if (status) *status = st;
  return st ? nullptr : dupstr(s);
}

int lynx_rt_get_tensor(lynx_rt* h, const char* name, void* host, size_t bytes) {
  return guard([&] { h->ex->get_tensor(name, host, bytes); });
}

int lynx_rt_set_tensor(lynx_rt* h, const char* name, const void* host, size_t bytes) {
  return guard([&] { h->ex->set_tensor(name, host, bytes); });
}

int lynx_rt_nccl_unique_id(char* hex_out, size_t len) {
  return guard([&] {
    const std::string hex = lynx::rt::nccl_unique_id_hex();
    if (len < hex.size() + 1) throw lynx::rt::RtError("buffer too small", lynx::kValidation);
    std::memcpy(hex_out, hex.c_str(), hex.size() + 1);
  });
}

void lynx_rt_destroy(lynx_rt* h) { delete h; }

}  // extern "C"
