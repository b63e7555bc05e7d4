// Internal (C++) interface of the operator library shared by the kernel
// translation units, the C-ABI wrappers (capi_ops.cu) and the runtime.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace lynx {

// Status codes shared with the C-ABI (include/lynx_b200.h).
enum Status {
  kOk = 0,
  kValidation = 1,
  kParse = 2,
  kTimedOut = 3,
  kInfeasible = 4,
  kNoValidPartition = 5,
  kCudaError = 6,
  kOutOfMemory = 7,
};

int set_error(const std::string& msg, int code = kCudaError);
// Checks the last launch and counts `kernels` launches of this library
// (the bench's gpu_launches claim).
int check_launch(const char* what, int kernels = 1);
long long launch_count();
const char* last_error();

// EPI_BF16_GELU: c = bf16(acc + bias) and c2 = bf16(gelu(c)) (FC1 with its GeLU fused).
// EPI_BF16_RESID: c = bf16(res + dropout(bf16(acc + bias))) with the Philox mask of
// bias_dropout_residual_fwd (element index row * ldc + col), i.e. PROJ_RES / FC2_RES in one kernel.
// EPI_BF16_GELU_BWD: c = bf16(acc * gelu'(res)) with res the FC1 output (GeLU backward fused into the
// dX GEMM of FC2).
enum EpiMode {
  EPI_BF16 = 0,
  EPI_ACC_F32 = 1,
  EPI_STORE_F32 = 2,
  EPI_ACC_BF16 = 3,
  EPI_BF16_GELU = 4,
  EPI_BF16_RESID = 5,
  EPI_BF16_GELU_BWD = 6
};

struct GemmDesc {
  const void* a;  // bf16
  long long lda;  // elements between consecutive rows of the stored matrix
  bool a_mn;      // A stored MN-major ([K][M]) instead of K-major ([M][K])
  const void* b;
  long long ldb;
  bool b_mn;  // B stored MN-major ([K][N]) instead of K-major ([N][K])
  void* c;
  long long ldc;
  int M, N, K;
  const __nv_bfloat16* bias;  // EPI_BF16 / EPI_BF16_GELU only, may be null
  int epi;
  void* c2 = nullptr;  // EPI_BF16_GELU: second bf16 output (same shape and ldc as c)
  const __nv_bfloat16* res = nullptr;  // EPI_BF16_RESID residual / EPI_BF16_GELU_BWD GeLU input (shape, ldc of c)
  float drop_p = 0.f;
  uint64_t drop_seed = 0, drop_stream = 0;
};

int gemm_run(const GemmDesc& g, cudaStream_t stream, int max_ctas = 0);
// -1: 2-CTA (cta_group::2) kernel wherever the shape allows (default); 0: 1-CTA kernel only.
void gemm_set_mode(int mode);

// ---- norm / elementwise / attention / loss (see the .cu files for contracts)
int layernorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* gamma, const __nv_bfloat16* beta, __nv_bfloat16* y,
                  float* mean, float* rstd, int rows, int width, float eps, cudaStream_t s);
// dgamma_acc / dbeta_acc are fp32 (acc_bf16 = 0) or bf16 (acc_bf16 = 1) accumulators.
int layernorm_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* x, const __nv_bfloat16* gamma, const float* mean,
                  const float* rstd, const __nv_bfloat16* dres, __nv_bfloat16* dx, void* dgamma_acc,
                  void* dbeta_acc, int acc_bf16, float* workspace, int rows, int width, cudaStream_t s);
size_t layernorm_bwd_workspace(int rows, int width);

int bias_dropout_residual_fwd(const __nv_bfloat16* y, const __nv_bfloat16* bias, const __nv_bfloat16* res,
                              __nv_bfloat16* out, long long rows, int width, float p, uint64_t seed,
                              uint64_t stream_id, cudaStream_t s);
int dropout_bwd(const __nv_bfloat16* dout, __nv_bfloat16* dy, long long rows, int width, float p, uint64_t seed,
                uint64_t stream_id, cudaStream_t s);
int column_sum_acc(const __nv_bfloat16* x, void* acc, int acc_bf16, float* workspace, long long rows, int width,
                   cudaStream_t s);
// dy = dropout_bwd(dout) and acc += column sums of dy (bias gradient) in one pass; dy and acc are
// bit-identical to dropout_bwd followed by column_sum_acc.
int dropout_bwd_colsum(const __nv_bfloat16* dout, __nv_bfloat16* dy, void* acc, int acc_bf16, float* workspace,
                       long long rows, int width, float p, uint64_t seed, uint64_t stream_id, cudaStream_t s);
// dst(bf16) += src(fp32), elementwise (n % 8 == 0 not required).
int add_f32_to_bf16(const float* src, __nv_bfloat16* dst, long long n, cudaStream_t s);
size_t column_sum_workspace(long long rows, int width);
int gelu_fwd(const __nv_bfloat16* x, __nv_bfloat16* y, long long n, cudaStream_t s);
int gelu_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* x, __nv_bfloat16* dx, long long n, cudaStream_t s);
int add_bf16(const __nv_bfloat16* a, const __nv_bfloat16* b, __nv_bfloat16* out, long long n, cudaStream_t s);

int embedding_fwd(const int32_t* tokens, const __nv_bfloat16* wte, const __nv_bfloat16* wpe, __nv_bfloat16* out,
                  int batch, int seq, int width, float p, uint64_t seed, uint64_t stream_id, cudaStream_t s);
int embedding_bwd(const int32_t* tokens, const __nv_bfloat16* dout, float* dwte, float* dwpe, float* workspace,
                  int batch, int seq, int width, int vocab, float p, uint64_t seed, uint64_t stream_id,
                  cudaStream_t s);
size_t embedding_bwd_workspace(int batch, int seq, int width);

int xent_fwd_bwd(__nv_bfloat16* logits, const int32_t* labels, float* loss_rows, long long rows, int vocab,
                 float grad_scale, cudaStream_t s);
// Vocab-parallel cross-entropy (TP > 1): the rank's logits cover vocabulary columns [v0, v0 + vl);
// row_max is all-reduced (MAX) after xent_vp_max, sum_target ([2 * rows]: sums, then target logits)
// (SUM) after xent_vp_sum; xent_vp_finish writes the loss rows and the logit gradients in place.
int xent_vp_max(const __nv_bfloat16* logits, float* row_max, long long rows, int vl, cudaStream_t s);
int xent_vp_sum(const __nv_bfloat16* logits, const int32_t* labels, long long v0, const float* row_max,
                float* sum_target, long long rows, int vl, cudaStream_t s);
int xent_vp_finish(__nv_bfloat16* logits, const int32_t* labels, long long v0, const float* row_max,
                   const float* sum_target, float* loss_rows, long long rows, int vl, float grad_scale,
                   cudaStream_t s);

int attention_fwd(const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, int batch, int seq, int heads,
                  int head_dim, cudaStream_t s);
int attention_bwd(const __nv_bfloat16* qkv, const __nv_bfloat16* out, const __nv_bfloat16* dout, const float* lse,
                  __nv_bfloat16* dqkv, float* workspace, int batch, int seq, int heads, int head_dim,
                  cudaStream_t s);
size_t attention_bwd_workspace(int batch, int seq, int heads);
// tcgen05 attention (ops_attention_tc.cu): head_dim 64/128, seq % 128 == 0.
// attention_set_mode: -1 (default) tcgen05 kernels where the shape allows, 0 mma.sync kernels only.
void attention_set_mode(int mode);
// tcgen05 backward kernels: 2 or 4 row warpgroups (0: default).
void attention_set_bwd_warpgroups(int n);
// tcgen05 forward: 1 or 2 query tiles per CTA (0: default, 2).
void attention_set_fwd_tiles(int n);
int attention_mode();
bool attention_tc_supported(int seq, int head_dim);
int attention_fwd_tc(const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, int batch, int seq, int heads,
                     int head_dim, cudaStream_t s);
int attention_bwd_tc(const __nv_bfloat16* qkv, const __nv_bfloat16* dout, const float* lse, const float* dvec,
                     __nv_bfloat16* dqkv, int batch, int seq, int heads, int head_dim, cudaStream_t s);

// ---- fused tensor-parallel reductions (ops_tp.cu): every rank's row-parallel partial read in place
constexpr int kMaxTpRanks = 8;
struct TpPartials {
  const __nv_bfloat16* p[kMaxTpRanks];  // rank order
  int n;
};
struct TpFlags {
  unsigned long long* f[kMaxTpRanks];  // every rank's flag array (peer mappings), rank order
};
// out = res + dropout(bias + bf16(sum of partials)) with bias_dropout_residual_fwd's mask and rounding.
int tp_reduce_residual(const TpPartials& parts, const __nv_bfloat16* bias, const __nv_bfloat16* res,
                       __nv_bfloat16* out, long long rows, int width, float p, uint64_t seed, uint64_t stream_id,
                       cudaStream_t s);
// out = bf16(sum of partials), n elements.
int tp_reduce(const TpPartials& parts, __nv_bfloat16* out, long long n, cudaStream_t s);
// Cross-process "partials of call k are written" barrier over device flags (k + 1 = value).
int tp_signal_wait(const TpFlags& peers, const unsigned long long* my_flags, int n, int me, unsigned long long value,
                   cudaStream_t s);

// grad is fp32 (grad_bf16 = 0) or bf16 (grad_bf16 = 1).
int adam_step(float* master, __nv_bfloat16* param, const void* grad, int grad_bf16, float* m, float* v, long long n,
              float lr, float beta1, float beta2, float eps, float weight_decay, int step, float grad_scale,
              cudaStream_t s);
int fill_f32(float* p, float v, long long n, cudaStream_t s);
int fill_param(__nv_bfloat16* p, float* master, float v, long long n, cudaStream_t s);
// Number of 32-bit words that differ between two device buffers (bit-identity checks).
int count_mismatch(const void* a, const void* b, size_t bytes, unsigned long long* d_count, cudaStream_t s);
int init_normal_bf16(__nv_bfloat16* p, float* master, long long n, float std, uint64_t seed, uint64_t stream_id,
                     cudaStream_t s);
// Shard of an unsharded N(0, std) tensor (values identical to init_normal_bf16 of the full tensor;
// see ops_elementwise.cu for the index map): Megatron column splits use row_blk (QKV: hp, FC1: 4hp),
// row splits col_split (projection, FC2).
int init_normal_sharded_bf16(__nv_bfloat16* p, float* master, long long rows, long long cols, long long row_blk,
                             int col_split, int tp, int tp_rank, float std, uint64_t seed, uint64_t stream_id,
                             cudaStream_t s);
int f32_to_bf16(const float* src, __nv_bfloat16* dst, long long n, cudaStream_t s);
// bytes / 4 words of uniform bf16 pairs in [-1, 1) (timing-only stand-in buffers).
int fill_noise_bf16(void* p, size_t bytes, uint64_t seed, cudaStream_t s);
// Single-GPU stand-in for a collective (exec.comm_standin_us): `ctas` CTAs of 512 threads hold
// the stream for `ns` nanoseconds of %globaltimer, sleeping between polls. Models the transfer
// time of an NCCL all-reduce the plan's window capacity assumes; not its SM / HBM traffic.
// With buf / passes > 0 the CTAs first stream `bytes` of buf in place (read + write, `passes` times): the
// local HBM traffic and SM occupancy of a real collective on that buffer.
int comm_standin(unsigned long long ns, int ctas, cudaStream_t s, void* buf = nullptr, long long bytes = 0,
                 int passes = 0);

}  // namespace lynx
