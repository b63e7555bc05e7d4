#include <cmath>
#include <stdexcept>

#include "lynx_ops_internal.h"
#include "runtime/gpt_stage.hpp"

namespace lynx::rt {

Op op_from_name(const std::string& n) {
  static const char* names[] = {"ln1",     "qkv", "attn",    "proj",     "ar1",   "proj_res", "ln2",    "fc1", "gelu",
                                "fc2",     "ar2", "fc2_res", "mlp_bwd",  "ar_b1", "attn_bwd", "ar_b2",  "ln1_bwd"};
  for (int i = 0; i < static_cast<int>(Op::UNKNOWN); ++i)
    if (n == names[i]) return static_cast<Op>(i);
  return Op::UNKNOWN;
}

const char* op_name(Op op) {
  static const char* names[] = {"ln1", "qkv", "attn", "proj", "ar1", "proj_res", "ln2", "fc1", "gelu", "fc2",
                                "ar2", "fc2_res", "mlp_bwd", "ar_b1", "attn_bwd", "ar_b2", "ln1_bwd", "?"};
  return names[static_cast<int>(op)];
}

namespace {
constexpr long long kAlign = 64;  // elements: 128-byte aligned bf16 tensors, 256-byte fp32
long long align_up(long long x) { return (x + kAlign - 1) / kAlign * kAlign; }
}  // namespace

long long ParamStore::add(const std::string& name, long long n) {
  refs_.push_back({name, total_, n});
  total_ = align_up(total_ + n);
  return refs_.back().off;
}

void ParamStore::layout(const ModelCfg& c) {
  refs_.clear();
  total_ = 0;
  const long long h = c.hidden, hp = c.hp();
  if (c.first()) {
    add("wte", static_cast<long long>(c.vocab) * h);
    add("wpe", static_cast<long long>(c.seq) * h);
  }
  for (int l = 0; l < c.layers; ++l) {
    const std::string p = "l" + std::to_string(l) + ".";
    add(p + "ln1_g", h);
    add(p + "ln1_b", h);
    add(p + "w_qkv", 3 * hp * h);
    add(p + "b_qkv", 3 * hp);
    add(p + "w_proj", h * hp);
    add(p + "b_proj", h);
    add(p + "ln2_g", h);
    add(p + "ln2_b", h);
    add(p + "w_fc1", 4 * hp * h);
    add(p + "b_fc1", 4 * hp);
    add(p + "w_fc2", h * 4 * hp);
    add(p + "b_fc2", h);
  }
  if (c.last()) {
    add("lnf_g", h);
    add("lnf_b", h);
    add("w_head", static_cast<long long>(c.vocab_rank()) * h);
  }
}

const ParamRef& ParamStore::find(const std::string& name) const {
  for (const auto& r : refs_)
    if (r.name == name) return r;
  throw std::runtime_error("unknown parameter " + name);
}

__nv_bfloat16* ParamStore::p(const std::string& name) const { return param + find(name).off; }
__nv_bfloat16* ParamStore::g(const std::string& name) const { return grad + find(name).off; }

LayerParams ParamStore::resolve(int l) const {
  const std::string p = "l" + std::to_string(l) + ".";
  LayerParams L{};
  L.ln1_g = this->p(p + "ln1_g");
  L.ln1_b = this->p(p + "ln1_b");
  L.w_qkv = this->p(p + "w_qkv");
  L.b_qkv = this->p(p + "b_qkv");
  L.w_proj = this->p(p + "w_proj");
  L.b_proj = this->p(p + "b_proj");
  L.ln2_g = this->p(p + "ln2_g");
  L.ln2_b = this->p(p + "ln2_b");
  L.w_fc1 = this->p(p + "w_fc1");
  L.b_fc1 = this->p(p + "b_fc1");
  L.w_fc2 = this->p(p + "w_fc2");
  L.b_fc2 = this->p(p + "b_fc2");
  L.g_ln1_g = g(p + "ln1_g");
  L.g_ln1_b = g(p + "ln1_b");
  L.g_w_qkv = g(p + "w_qkv");
  L.g_b_qkv = g(p + "b_qkv");
  L.g_w_proj = g(p + "w_proj");
  L.g_b_proj = g(p + "b_proj");
  L.g_ln2_g = g(p + "ln2_g");
  L.g_ln2_b = g(p + "ln2_b");
  L.g_w_fc1 = g(p + "w_fc1");
  L.g_b_fc1 = g(p + "b_fc1");
  L.g_w_fc2 = g(p + "w_fc2");
  L.g_b_fc2 = g(p + "b_fc2");
  return L;
}

void ParamStore::allocate_and_init(const ModelCfg& c, cudaStream_t s) {
  const size_t n = static_cast<size_t>(total_);
  auto ck = [](cudaError_t e) {
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw std::runtime_error(std::string("parameter allocation: ") + cudaGetErrorString(e));
    }
  };
  ck(cudaMalloc(&param, n * 2));
  ck(cudaMalloc(&master, n * 4));
  ck(cudaMalloc(&grad, n * 2));
  ck(cudaMalloc(&m, n * 4));
  ck(cudaMalloc(&v, n * 4));
  ck(cudaMemsetAsync(grad, 0, n * 2, s));
  ck(cudaMemsetAsync(m, 0, n * 4, s));
  ck(cudaMemsetAsync(v, 0, n * 4, s));
  ck(cudaMemsetAsync(param, 0, n * 2, s));  // alignment padding stays zero
  ck(cudaMemsetAsync(master, 0, n * 4, s));
  layers_.clear();
  for (int l = 0; l < c.layers; ++l) layers_.push_back(resolve(l));
  // Weights ~ N(0, std) defined on the UNSHARDED tensor: the Philox stream is keyed by
  // (global layer, tensor kind) only — no TP rank, no stage-local position — and each TP rank
  // materialises its Megatron slice of the full tensor (init_normal_sharded_bf16). Every TP / PP
  // layout of a model therefore holds exactly the weights of its TP = 1, PP = 1 run: replicated
  // tensors (embeddings, LM head, LayerNorms, row-parallel biases) are identical on all TP ranks,
  // and the unsharded CPU oracle sees the same values.
  const float out_std = c.init_std / std::sqrt(2.0f * c.n_layers_total);
  const long long h = c.hidden, hp = c.hp();
  for (const auto& r : refs_) {
    const std::string& nm = r.name;
    const size_t dot = nm.find('.');
    const bool layer = nm[0] == 'l' && dot != std::string::npos;
    const std::string base = layer ? nm.substr(dot + 1) : nm;
    const uint64_t layer_global = layer ? static_cast<uint64_t>(c.layer0 + std::stoi(nm.substr(1)) + 1) : 0;
    int st = 0;
    if (base == "ln1_g" || base == "ln2_g" || base == "lnf_g") {
      st = fill_param(param + r.off, master + r.off, 1.0f, r.n, s);
    } else if (base.rfind("b_", 0) == 0 || base == "ln1_b" || base == "ln2_b" || base == "lnf_b") {
      st = fill_param(param + r.off, master + r.off, 0.0f, r.n, s);
    } else {
      // kind id, local [rows, cols], column-split row block / row-split flag
      static const struct { const char* name; int kind; } kinds[] = {
          {"wte", 1}, {"wpe", 2}, {"w_qkv", 3}, {"w_proj", 4}, {"w_fc1", 5}, {"w_fc2", 6}, {"w_head", 7}};
      int kind = 0;
      for (const auto& k : kinds)
        if (base == k.name) kind = k.kind;
      if (!kind) throw std::runtime_error("parameter init: no rule for " + nm);
      long long rows = r.n / h, cols = h, row_blk = 0;
      int col_split = 0;
      if (base == "w_qkv") row_blk = hp;                      // [3 hp, h]: q | k | v blocks of hp rows
      if (base == "w_fc1") row_blk = 4 * hp;                  // [4 hp, h]
      if (base == "w_head" && c.vocab_parallel()) row_blk = c.vocab_rank();  // [V / tp, h]: vocab rows
      if (base == "w_proj" || base == "w_fc2") {              // [h, hp] / [h, 4 hp]: column slices
        rows = h;
        cols = r.n / h;
        col_split = 1;
      }
      const bool out_proj = base == "w_proj" || base == "w_fc2";
      const uint64_t sid = (layer_global << 24) ^ (static_cast<uint64_t>(kind) << 8);
      st = init_normal_sharded_bf16(param + r.off, master + r.off, rows, cols, row_blk, col_split, c.tp, c.tp_rank,
                                    out_proj ? out_std : c.init_std, c.seed, sid, s);
    }
    if (st) throw std::runtime_error(std::string("parameter init: ") + last_error());
  }
}

void ParamStore::release() {
  layers_.clear();
  cudaFree(param);
  cudaFree(master);
  cudaFree(grad);
  cudaFree(m);
  cudaFree(v);
  param = nullptr;
  grad = nullptr;
  master = m = v = nullptr;
}

}  // namespace lynx::rt
