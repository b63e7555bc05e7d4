// extern "C" entry points of the operator library (include/lynx_b200.h).
// Plain device pointers, sizes and a cudaStream_t passed as void*; every
// function returns a Status code and leaves a message in lynx_last_error().
#include <atomic>
#include <cstdio>
#include <string>

#include "../../include/lynx_b200.h"
#include "lynx_ops_internal.h"

namespace lynx {

namespace {
thread_local std::string g_last_error;
}

int set_error(const std::string& msg, int code) {
  g_last_error = msg;
  return code;
}

namespace {
std::atomic<long long> g_launches{0};
}

long long launch_count() { return g_launches.load(); }

int check_launch(const char* what, int kernels) {
  g_launches += kernels;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(std::string(what) + ": " + cudaGetErrorString(e), kCudaError);
  return kOk;
}

const char* last_error() { return g_last_error.c_str(); }

}  // namespace lynx

using namespace lynx;

#define BF(p) reinterpret_cast<__nv_bfloat16*>(p)
#define CBF(p) reinterpret_cast<const __nv_bfloat16*>(p)
#define STREAM(s) reinterpret_cast<cudaStream_t>(s)

extern "C" {

const char* lynx_last_error(void) { return lynx::last_error(); }
int lynx_abi_version(void) { return LYNX_ABI_VERSION; }

int lynx_op_gemm(const void* a, long long lda, int a_mn_major, const void* b, long long ldb, int b_mn_major, void* c,
                 long long ldc, int m, int n, int k, const void* bias, int epilogue, void* stream) {
  GemmDesc g{a, lda, a_mn_major != 0, b, ldb, b_mn_major != 0, c, ldc, m, n, k, CBF(bias), epilogue};
  return gemm_run(g, STREAM(stream));
}

// exec.tp_fused building blocks (the executor's row-parallel reductions), for multi-process checks:
// `partials` / `peer_flags` hold n device pointers in rank order (this rank's own at index me).
int lynx_op_tp_signal_wait(void* const* peer_flags, const void* my_flags, int n, int me, unsigned long long value,
                           void* stream) {
  if (n < 1 || n > kMaxTpRanks || me < 0 || me >= n) return set_error("tp_signal_wait: ranks", kValidation);
  TpFlags f{};
  for (int r = 0; r < n; ++r) f.f[r] = static_cast<unsigned long long*>(peer_flags[r]);
  return tp_signal_wait(f, static_cast<const unsigned long long*>(my_flags), n, me, value, STREAM(stream));
}

int lynx_op_tp_reduce_residual(const void* const* partials, int n, const void* bias, const void* res, void* out,
                               long long rows, int width, float p, unsigned long long seed,
                               unsigned long long stream_id, void* stream) {
  if (n < 1 || n > kMaxTpRanks) return set_error("tp_reduce_residual: ranks", kValidation);
  TpPartials parts{};
  parts.n = n;
  for (int r = 0; r < n; ++r) parts.p[r] = CBF(partials[r]);
  return tp_reduce_residual(parts, CBF(bias), CBF(res), BF(out), rows, width, p, seed, stream_id, STREAM(stream));
}

int lynx_op_gemm_gelu(const void* a, long long lda, int a_mn_major, const void* b, long long ldb, int b_mn_major,
                      void* c, void* c_gelu, long long ldc, int m, int n, int k, const void* bias, void* stream) {
  GemmDesc g{a, lda, a_mn_major != 0, b, ldb, b_mn_major != 0, c, ldc, m, n, k, CBF(bias), EPI_BF16_GELU, c_gelu};
  return gemm_run(g, STREAM(stream));
}

int lynx_op_gemm_residual(const void* a, long long lda, const void* b, long long ldb, void* c, long long ldc, int m,
                          int n, int k, const void* bias, const void* res, float p, unsigned long long seed,
                          unsigned long long stream_id, void* stream) {
  GemmDesc g{a, lda, false, b, ldb, false, c, ldc, m, n, k, CBF(bias), EPI_BF16_RESID};
  g.res = CBF(res);
  g.drop_p = p;
  g.drop_seed = seed;
  g.drop_stream = stream_id;
  return gemm_run(g, STREAM(stream));
}

int lynx_op_gemm_gelu_bwd(const void* a, long long lda, const void* b, long long ldb, int b_mn_major, void* c,
                          long long ldc, int m, int n, int k, const void* x, void* stream) {
  GemmDesc g{a, lda, false, b, ldb, b_mn_major != 0, c, ldc, m, n, k, nullptr, EPI_BF16_GELU_BWD};
  g.res = CBF(x);
  return gemm_run(g, STREAM(stream));
}

void lynx_op_gemm_mode(int mode) { gemm_set_mode(mode); }
void lynx_op_attention_mode(int mode) { attention_set_mode(mode); }
void lynx_op_attention_bwd_warpgroups(int n) { attention_set_bwd_warpgroups(n); }
void lynx_op_attention_fwd_tiles(int n) { attention_set_fwd_tiles(n); }
int lynx_op_attention_tc_supported(int seq, int head_dim) { return attention_tc_supported(seq, head_dim) ? 1 : 0; }

int lynx_op_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd,
                          int rows, int width, float eps, void* stream) {
  return layernorm_fwd(CBF(x), CBF(gamma), CBF(beta), BF(y), mean, rstd, rows, width, eps, STREAM(stream));
}

size_t lynx_op_layernorm_bwd_workspace(int rows, int width) { return layernorm_bwd_workspace(rows, width); }

int lynx_op_layernorm_bwd(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
                          const void* dres, void* dx, float* dgamma_acc, float* dbeta_acc, float* workspace,
                          int rows, int width, void* stream) {
  return layernorm_bwd(CBF(dy), CBF(x), CBF(gamma), mean, rstd, CBF(dres), BF(dx), dgamma_acc, dbeta_acc, 0, workspace,
                       rows, width, STREAM(stream));
}

int lynx_op_bias_dropout_residual(const void* y, const void* bias, const void* res, void* out, long long rows,
                                  int width, float p, unsigned long long seed, unsigned long long stream_id,
                                  void* stream) {
  return bias_dropout_residual_fwd(CBF(y), CBF(bias), CBF(res), BF(out), rows, width, p, seed, stream_id,
                                   STREAM(stream));
}

int lynx_op_dropout_bwd(const void* dout, void* dy, long long rows, int width, float p, unsigned long long seed,
                        unsigned long long stream_id, void* stream) {
  return dropout_bwd(CBF(dout), BF(dy), rows, width, p, seed, stream_id, STREAM(stream));
}

size_t lynx_op_column_sum_workspace(long long rows, int width) { return column_sum_workspace(rows, width); }

int lynx_op_column_sum_acc(const void* x, float* acc, float* workspace, long long rows, int width, void* stream) {
  return column_sum_acc(CBF(x), acc, 0, workspace, rows, width, STREAM(stream));
}

int lynx_op_dropout_bwd_colsum(const void* dout, void* dy, float* acc, float* workspace, long long rows, int width,
                               float p, unsigned long long seed, unsigned long long stream_id, void* stream) {
  return dropout_bwd_colsum(CBF(dout), BF(dy), acc, 0, workspace, rows, width, p, seed, stream_id, STREAM(stream));
}

int lynx_op_gelu_fwd(const void* x, void* y, long long n, void* stream) {
  return gelu_fwd(CBF(x), BF(y), n, STREAM(stream));
}

int lynx_op_gelu_bwd(const void* dy, const void* x, void* dx, long long n, void* stream) {
  return gelu_bwd(CBF(dy), CBF(x), BF(dx), n, STREAM(stream));
}

int lynx_op_attention_fwd(const void* qkv, void* out, float* lse, int batch, int seq, int heads, int head_dim,
                          void* stream) {
  return attention_fwd(CBF(qkv), BF(out), lse, batch, seq, heads, head_dim, STREAM(stream));
}

size_t lynx_op_attention_bwd_workspace(int batch, int seq, int heads) {
  return attention_bwd_workspace(batch, seq, heads);
}

int lynx_op_attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv,
                          float* workspace, int batch, int seq, int heads, int head_dim, void* stream) {
  return attention_bwd(CBF(qkv), CBF(out), CBF(dout), lse, BF(dqkv), workspace, batch, seq, heads, head_dim,
                       STREAM(stream));
}

int lynx_op_embedding_fwd(const int* tokens, const void* wte, const void* wpe, void* out, int batch, int seq,
                          int width, float p, unsigned long long seed, unsigned long long stream_id, void* stream) {
  return embedding_fwd(tokens, CBF(wte), CBF(wpe), BF(out), batch, seq, width, p, seed, stream_id, STREAM(stream));
}

size_t lynx_op_embedding_bwd_workspace(int batch, int seq, int width) {
  return embedding_bwd_workspace(batch, seq, width);
}

int lynx_op_embedding_bwd(const int* tokens, const void* dout, float* dwte, float* dwpe, float* workspace, int batch,
                          int seq, int width, int vocab, float p, unsigned long long seed,
                          unsigned long long stream_id, void* stream) {
  return embedding_bwd(tokens, CBF(dout), dwte, dwpe, workspace, batch, seq, width, vocab, p, seed, stream_id,
                       STREAM(stream));
}

int lynx_op_xent_fwd_bwd(void* logits, const int* labels, float* loss_rows, long long rows, int vocab,
                         float grad_scale, void* stream) {
  return xent_fwd_bwd(BF(logits), labels, loss_rows, rows, vocab, grad_scale, STREAM(stream));
}

int lynx_op_adam(float* master, void* param, const float* grad, float* m, float* v, long long n, float lr,
                 float beta1, float beta2, float eps, float weight_decay, int step, float grad_scale, void* stream) {
  return adam_step(master, BF(param), grad, 0, m, v, n, lr, beta1, beta2, eps, weight_decay, step, grad_scale,
                   STREAM(stream));
}

int lynx_op_init_normal(void* param, float* master, long long n, float std, unsigned long long seed,
                        unsigned long long stream_id, void* stream) {
  return init_normal_bf16(BF(param), master, n, std, seed, stream_id, STREAM(stream));
}

}  // extern "C"
