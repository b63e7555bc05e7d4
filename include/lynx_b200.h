/* lynx_b200.h — C-ABI of the B200 operator library (sm_100a kernels).
 *
 * These are the GPT-block operators the executor (include/lynx_rt.h) launches
 * for every forward op, backward op and recomputation of a Lynx plan. The
 * reference has no operator library at all: its operators are names, times and
 * byte counts in the profile JSON (reference proj/tests/fixtures/gpt-tiny.json:8-15,
 * schema proj/include/lynx/profile.hpp:27-34). These entry points are what a
 * GPU "model deployer" (Fig. 5, out of the reference's scope per
 * SPEC.md:9,14) binds to.
 *
 * Conventions: device pointers; bf16 tensors are row-major; `stream` is a
 * cudaStream_t (NULL = legacy default stream). Every function returns
 * LYNX_OK (0) or an error code, with the message in lynx_last_error()
 * (thread-local). No function allocates device memory; callers pass the
 * workspace sizes reported by the *_workspace queries.
 */
#ifndef LYNX_B200_H_
#define LYNX_B200_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LYNX_ABI_VERSION 1

/* Status codes: 0-5 follow the reference CLI exit codes
 * (proj/tools/lynx_main.cpp:30-35); 6-7 are added for the device side. */
#define LYNX_OK 0
#define LYNX_E_VALIDATION 1
#define LYNX_E_PARSE 2
#define LYNX_E_TIMED_OUT 3
#define LYNX_E_INFEASIBLE 4
#define LYNX_E_NO_PARTITION 5
#define LYNX_E_CUDA 6
#define LYNX_E_OOM 7

/* GEMM epilogues */
#define LYNX_EPI_BF16 0    /* C(bf16) = A*B^T (+ bias[n]) */
#define LYNX_EPI_ACC_F32 1 /* C(f32) += A*B^T  (weight-gradient accumulation) */
#define LYNX_EPI_F32 2     /* C(f32)  = A*B^T */
#define LYNX_EPI_ACC_BF16 3 /* C(bf16) += A*B^T (bf16 gradient accumulation, 16 B/parameter model states) */

const char* lynx_last_error(void);
int lynx_abi_version(void);

/* exec.tp_fused building blocks (the executor's row-parallel reductions; ops_tp.cu). Replace the TP
 * all-reduce + bias_dropout_residual of Megatron's row-parallel layers (the reference's CTime windows,
 * heusched.cpp:62-70). peer_flags / partials: n device pointers in rank order, this rank's own at `me`.
 * signal_wait: every rank's flag array gets `value` in slot `me` (st.release.sys), then the stream waits
 * until all n slots of `my_flags` reached `value` (ld.acquire.sys; traps after 60 s).
 * reduce_residual: out = res + dropout(bias + bf16(sum of partials in rank order)). */
int lynx_op_tp_signal_wait(void* const* peer_flags, const void* my_flags, int n, int me, unsigned long long value,
                           void* stream);
int lynx_op_tp_reduce_residual(const void* const* partials, int n, const void* bias, const void* res, void* out,
                               long long rows, int width, float p, unsigned long long seed,
                               unsigned long long stream_id, void* stream);
/* C[M,N] = A[M,K] * B[N,K]^T on tcgen05 tensor cores (fp32 accumulation in TMEM).
 * a_mn_major=0: A stored [M][K] (row pitch lda); 1: A stored [K][M] (pitch lda).
 * b_mn_major=0: B stored [N][K] (row pitch ldb); 1: B stored [K][N] (pitch ldb).
 * Requires M % 128 == 0, N % 128 == 0, K % 64 == 0, 16-byte aligned rows. */
int lynx_op_gemm(const void* a, long long lda, int a_mn_major, const void* b, long long ldb, int b_mn_major, void* c,
                 long long ldc, int m, int n, int k, const void* bias, int epilogue, void* stream);
/* FC1 with its GeLU fused into the epilogue: c = bf16(A*B^T + bias[n]) and
 * c_gelu = bf16(gelu(c)) (GPT-2 tanh GeLU of the bf16-rounded c, bit-identical to lynx_op_gelu_fwd
 * on c). Same shape / layout rules as lynx_op_gemm; c and c_gelu share ldc. */
int lynx_op_gemm_gelu(const void* a, long long lda, int a_mn_major, const void* b, long long ldb, int b_mn_major,
                      void* c, void* c_gelu, long long ldc, int m, int n, int k, const void* bias, void* stream);
/* Projection + bias + dropout + residual in one kernel: c = bf16(res + dropout_p(bf16(A*B^T + bias)))
 * with the keep mask of lynx_op_bias_dropout_residual (Philox(seed, stream_id, row*ldc + col)); A [m,k]
 * and B [n,k] K-major, res and c [m,n] with pitch ldc. */
int lynx_op_gemm_residual(const void* a, long long lda, const void* b, long long ldb, void* c, long long ldc, int m,
                          int n, int k, const void* bias, const void* res, float p, unsigned long long seed,
                          unsigned long long stream_id, void* stream);
/* GeLU backward fused into a dX GEMM: c = bf16((A*B^T) * gelu'(x)), x the GeLU input [m,n] (pitch ldc).
 * A [m,k] K-major; B [n,k] (b_mn_major = 0) or [k,n] (1). */
int lynx_op_gemm_gelu_bwd(const void* a, long long lda, const void* b, long long ldb, int b_mn_major, void* c,
                          long long ldc, int m, int n, int k, const void* x, void* stream);
/* GEMM kernel selection: -1 (default) the 512x256 "wide" CTA-pair kernel (two cta_group::2 MMAs per
 * k-step sharing the B stage) for K >= 8192 when M % 512 == 0 and N % 256 == 0, else the 256x256
 * CTA-pair (tcgen05.mma.cta_group::2) kernel for K-major A when M % 256 == 0 and N % 256 == 0, else
 * the single-CTA 128xBN kernel; 0 single-CTA only; 1 256x256 CTA-pair wherever the shape allows;
 * 2 wide pair wherever the shape allows, then as 1. */
void lynx_op_gemm_mode(int mode);

/* y = (x - mean) * rstd * gamma + beta over rows of `width`; mean/rstd fp32 [rows]. */
int lynx_op_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd,
                          int rows, int width, float eps, void* stream);
size_t lynx_op_layernorm_bwd_workspace(int rows, int width);
/* dx = LN'(dy) (+ dres if non-NULL); dgamma_acc/dbeta_acc (fp32) += column sums. Deterministic. */
int lynx_op_layernorm_bwd(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
                          const void* dres, void* dx, float* dgamma_acc, float* dbeta_acc, float* workspace,
                          int rows, int width, void* stream);

/* out = res + dropout_p(y + bias[col]); mask = Philox(seed, stream_id, element). bias may be NULL. */
int lynx_op_bias_dropout_residual(const void* y, const void* bias, const void* res, void* out, long long rows,
                                  int width, float p, unsigned long long seed, unsigned long long stream_id,
                                  void* stream);
/* dy = dout * mask / (1 - p) with the same mask as the forward call. */
int lynx_op_dropout_bwd(const void* dout, void* dy, long long rows, int width, float p, unsigned long long seed,
                        unsigned long long stream_id, void* stream);
size_t lynx_op_column_sum_workspace(long long rows, int width);
/* acc[col] += sum_rows x[row][col] (bias gradients), deterministic. */
int lynx_op_column_sum_acc(const void* x, float* acc, float* workspace, long long rows, int width, void* stream);
/* dy = dropout_bwd(dout) and acc[col] += sum_rows dy[row][col] in one pass (the residual branch's
 * gradient and its bias gradient); bit-identical to lynx_op_dropout_bwd + lynx_op_column_sum_acc.
 * workspace: lynx_op_column_sum_workspace(rows, width) bytes. */
int lynx_op_dropout_bwd_colsum(const void* dout, void* dy, float* acc, float* workspace, long long rows, int width,
                               float p, unsigned long long seed, unsigned long long stream_id, void* stream);

/* GPT-2 tanh GeLU on n bf16 elements (n % 8 == 0). */
int lynx_op_gelu_fwd(const void* x, void* y, long long n, void* stream);
int lynx_op_gelu_bwd(const void* dy, const void* x, void* dx, long long n, void* stream);

/* Causal attention. qkv [batch*seq, 3*heads*head_dim] ([Q|K|V], head-major inside each),
 * out [batch*seq, heads*head_dim], lse [batch, heads, seq] (natural log). head_dim in {64,96,112,128},
 * seq % 64 == 0. Backward writes dQ|dK|dV into dqkv with the qkv layout; deterministic. */
int lynx_op_attention_fwd(const void* qkv, void* out, float* lse, int batch, int seq, int heads, int head_dim,
                          void* stream);
size_t lynx_op_attention_bwd_workspace(int batch, int seq, int heads);
int lynx_op_attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv,
                          float* workspace, int batch, int seq, int heads, int head_dim, void* stream);
/* Attention kernel selection: -1 (default) the tcgen05 kernels (TMEM accumulators, TMA tiles) when
 * head_dim is 64 or 128 and seq % 128 == 0, else the mma.sync kernels; 0 mma.sync kernels only. */
void lynx_op_attention_mode(int mode);
/* Row warpgroups of the tcgen05 attention backward kernels: 2 or 4 (0: the default, 2). */
void lynx_op_attention_bwd_warpgroups(int n);
/* tcgen05 attention forward variant (0: the default, 2): 1 = one query tile per CTA, 2 = two query tiles
 * per CTA (persistent), 3 = 64-key blocks with P apart from S, 4 = CTA pair (cta_group::2; head_dim 128
 * and an even tile count, else 2). Environment: LYNX_ATTN_FWD_TILES. */
void lynx_op_attention_fwd_tiles(int n);
/* 1 when attention of this shape runs on the tcgen05 kernels (head_dim 64/96/112/128, seq % 128 == 0). */
int lynx_op_attention_tc_supported(int seq, int head_dim);

/* out[b,s] = dropout(wte[tokens[b,s]] + wpe[s]); backward accumulates fp32 dwte/dwpe. */
int lynx_op_embedding_fwd(const int* tokens, const void* wte, const void* wpe, void* out, int batch, int seq,
                          int width, float p, unsigned long long seed, unsigned long long stream_id, void* stream);
size_t lynx_op_embedding_bwd_workspace(int batch, int seq, int width);
int lynx_op_embedding_bwd(const int* tokens, const void* dout, float* dwte, float* dwpe, float* workspace, int batch,
                          int seq, int width, int vocab, float p, unsigned long long seed,
                          unsigned long long stream_id, void* stream);

/* In place: logits[rows, vocab] -> (softmax - onehot(labels)) * grad_scale; loss_rows = lse - logit[label]. */
int lynx_op_xent_fwd_bwd(void* logits, const int* labels, float* loss_rows, long long rows, int vocab,
                         float grad_scale, void* stream);

/* AdamW over flat fp32 master / m / v, writes the bf16 working copy. grad is scaled by grad_scale. */
int lynx_op_adam(float* master, void* param, const float* grad, float* m, float* v, long long n, float lr,
                 float beta1, float beta2, float eps, float weight_decay, int step, float grad_scale, void* stream);
/* param (bf16) ~ N(0, std) from Philox(seed, stream_id, index); master (may be NULL) = float(param). */
int lynx_op_init_normal(void* param, float* master, long long n, float std, unsigned long long seed,
                        unsigned long long stream_id, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LYNX_B200_H_ */
