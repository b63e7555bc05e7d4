// One pipeline stage of a Megatron-style GPT on one TP rank: parameter and
// optimizer state in flat device buffers, and the kernel sequence behind each
// operator of the profile's layer template (forward, backward, recompute).
//
// The reference has no numerics at all (operators are names in the profile
// JSON); this is the operator library the plan's op names are
// bound to. Forward ops write exactly the tensor the profile accounts for
// (out_bytes); a recomputation is the same launch sequence with the same
// Philox dropout streams, so regenerated tensors are bit-identical.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>
#include <vector>

namespace lynx::rt {

// Template operators of the two GPT layer templates (gpt_profile.py).
enum class Op {
  LN1, QKV, ATTN, PROJ, AR1, PROJ_RES, LN2, FC1, GELU, FC2, AR2, FC2_RES,
  MLP_BWD, AR_B1, ATTN_BWD, AR_B2, LN1_BWD, UNKNOWN
};
Op op_from_name(const std::string& name);
const char* op_name(Op op);

struct ModelCfg {
  int n_layers_total = 4;  // whole model
  int layers = 4;          // on this stage
  int layer0 = 0;          // global index of this stage's first layer
  int hidden = 512, heads = 8, head_dim = 64, seq = 256, micro_batch = 2, vocab = 50304;
  int tp = 1, tp_rank = 0, pp = 1, pp_rank = 0, n_micro = 1;
  float dropout = 0.1f, ln_eps = 1e-5f, init_std = 0.02f;
  uint64_t seed = 42;
  float lr = 1e-4f, beta1 = 0.9f, beta2 = 0.95f, adam_eps = 1e-8f, weight_decay = 0.1f;
  int head_chunk = 4096;  // LM-head rows per logits chunk
  bool first() const { return pp_rank == 0; }
  bool last() const { return pp_rank == pp - 1; }
  long long tokens() const { return static_cast<long long>(micro_batch) * seq; }
  int hp() const { return hidden / tp; }  // per-rank attention width
  // Megatron vocab-parallel LM head + cross-entropy (TP > 1, vocabulary padded to 128 * tp rows):
  // each TP rank holds vocab / tp rows of the head; otherwise the head is replicated.
  bool vocab_parallel() const { return tp > 1 && vocab % (128 * tp) == 0; }
  int vocab_rank() const { return vocab_parallel() ? vocab / tp : vocab; }
  int heads_rank() const { return heads / tp; }
};

struct ParamRef {
  std::string name;
  long long off = 0, n = 0;  // element offset / count in the flat buffers
};

struct LayerParams {
  __nv_bfloat16 *ln1_g, *ln1_b, *w_qkv, *b_qkv, *w_proj, *b_proj, *ln2_g, *ln2_b, *w_fc1, *b_fc1, *w_fc2, *b_fc2;
  __nv_bfloat16 *g_ln1_g, *g_ln1_b, *g_w_qkv, *g_b_qkv, *g_w_proj, *g_b_proj, *g_ln2_g, *g_ln2_b, *g_w_fc1, *g_b_fc1,
      *g_w_fc2, *g_b_fc2;
};

// Flat bf16 params + bf16 grads + fp32 master / Adam m / v: 16 B per parameter, the model-state
// accounting of the paper (FP16 params and gradients, FP32 optimizer data).
class ParamStore {
 public:
  void layout(const ModelCfg& c);
  void allocate_and_init(const ModelCfg& c, cudaStream_t s);
  void release();
  LayerParams layer(int l) const { return layers_.at(static_cast<size_t>(l)); }  // resolved once at allocation
  __nv_bfloat16* p(const std::string& name) const;
  __nv_bfloat16* g(const std::string& name) const;
  long long count() const { return total_; }
  const std::vector<ParamRef>& refs() const { return refs_; }
  __nv_bfloat16* param = nullptr;
  __nv_bfloat16* grad = nullptr;
  float *master = nullptr, *m = nullptr, *v = nullptr;

 private:
  const ParamRef& find(const std::string& name) const;
  long long add(const std::string& name, long long n);
  LayerParams resolve(int l) const;
  std::vector<ParamRef> refs_;
  std::vector<LayerParams> layers_;
  long long total_ = 0;
};

// Per-stream scratch for backward transients and GEMM staging.
struct Scratch {
  __nv_bfloat16 *t_h = nullptr;     // [T, h]
  __nv_bfloat16 *t_h2 = nullptr;    // [T, h]
  __nv_bfloat16 *t_wide = nullptr;  // [T, max(4hp, 3hp)]
  __nv_bfloat16 *logits = nullptr;  // [head_chunk, V]
  float* ws = nullptr;              // reduction workspaces
  size_t ws_bytes = 0;
};

}  // namespace lynx::rt
