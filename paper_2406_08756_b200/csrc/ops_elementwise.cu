// Elementwise / memory-bound kernels of the GPT block: bias + dropout +
// residual, GeLU, embedding, vocab cross-entropy, AdamW, initialisation.
// All are 16-byte vectorised (8 x bf16 per thread-step), grid-stride over a
// grid sized in multiples of the SM count, and HBM-bound; DESIGN.md lists the
// algorithmic bytes per element used for their roofline.
//
// Dropout masks come from Philox-4x32-10 keyed by (seed, stream_id, element):
// stream_id encodes (global layer, microbatch, op) so a recomputed forward op
// reproduces the original mask bit-for-bit.
#include "common.cuh"
#include "lynx_ops_internal.h"

namespace lynx {
namespace {

constexpr int kBlock = 256;

int grid_for(long long nvec) {
  long long g = (nvec + kBlock - 1) / kBlock;
  const long long cap = 148 * 16;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

__global__ void bias_dropout_residual_kernel(const BF8* __restrict__ y, const BF8* __restrict__ bias,
                                             const BF8* __restrict__ res, BF8* __restrict__ out, long long nvec,
                                             int wvec, float p, uint64_t seed, uint64_t stream) {
  const uint32_t thr = drop_threshold(p);
  const float scale = p > 0.f ? 1.f / (1.f - p) : 1.f;
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < nvec;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    float a[8], r[8], b[8];
    bf8_to_f(y[v], a);
    bf8_to_f(res[v], r);
    if (bias) {
      bf8_to_f(bias[v % wvec], b);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = 0.f;
    }
    const uint32_t keep = p > 0.f ? keep_bits8(seed, stream, v, thr) : 0xFFu;
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = r[j] + (((keep >> j) & 1u) ? (a[j] + b[j]) * scale : 0.f);
    out[v] = f_to_bf8(o);
  }
}

__global__ void dropout_bwd_kernel(const BF8* __restrict__ dout, BF8* __restrict__ dy, long long nvec, float p,
                                   uint64_t seed, uint64_t stream) {
  const uint32_t thr = drop_threshold(p);
  const float scale = p > 0.f ? 1.f / (1.f - p) : 1.f;
#pragma unroll 4  // several 16-byte vectors in flight per thread (HBM-bound)
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < nvec;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    float d[8], o[8];
    bf8_to_f(dout[v], d);
    const uint32_t keep = p > 0.f ? keep_bits8(seed, stream, v, thr) : 0xFFu;
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = ((keep >> j) & 1u) ? d[j] * scale : 0.f;
    dy[v] = f_to_bf8(o);
  }
}

// GPT-2 tanh GeLU.
LYNX_DEV float gelu_f(float x) { return gelu_exact(x); }
LYNX_DEV float gelu_grad(float x) { return gelu_grad_f(x); }

__global__ void gelu_fwd_kernel(const BF8* __restrict__ x, BF8* __restrict__ y, long long nvec) {
#pragma unroll 4  // several 16-byte vectors in flight per thread (HBM-bound)
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < nvec;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    float a[8];
    bf8_to_f(x[v], a);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = gelu_f(a[j]);
    y[v] = f_to_bf8(a);
  }
}

__global__ void gelu_bwd_kernel(const BF8* __restrict__ dy, const BF8* __restrict__ x, BF8* __restrict__ dx,
                                long long nvec) {
#pragma unroll 4  // several 16-byte vectors in flight per thread (HBM-bound)
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < nvec;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    float a[8], d[8];
    bf8_to_f(x[v], a);
    bf8_to_f(dy[v], d);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = d[j] * gelu_grad(a[j]);
    dx[v] = f_to_bf8(a);
  }
}

__global__ void add_kernel(const BF8* __restrict__ a, const BF8* __restrict__ b, BF8* __restrict__ o, long long nvec) {
#pragma unroll 4  // several 16-byte vectors in flight per thread (HBM-bound)
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < nvec;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    float x[8], y[8];
    bf8_to_f(a[v], x);
    bf8_to_f(b[v], y);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] += y[j];
    o[v] = f_to_bf8(x);
  }
}

// out[b,s,:] = dropout(wte[tok[b,s],:] + wpe[s,:])
__global__ void embedding_fwd_kernel(const int32_t* __restrict__ tok, const BF8* __restrict__ wte,
                                     const BF8* __restrict__ wpe, BF8* __restrict__ out, long long nvec, int wvec,
                                     int seq, float p, uint64_t seed, uint64_t stream) {
  const uint32_t thr = drop_threshold(p);
  const float scale = p > 0.f ? 1.f / (1.f - p) : 1.f;
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < nvec;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long row = v / wvec;
    const int c = static_cast<int>(v % wvec);
    const int pos = static_cast<int>(row % seq);
    float a[8], b[8];
    bf8_to_f(wte[static_cast<long long>(tok[row]) * wvec + c], a);
    bf8_to_f(wpe[static_cast<long long>(pos) * wvec + c], b);
    const uint32_t keep = p > 0.f ? keep_bits8(seed, stream, v, thr) : 0xFFu;
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = ((keep >> j) & 1u) ? (a[j] + b[j]) * scale : 0.f;
    out[v] = f_to_bf8(a);
  }
}

// d(pre-dropout) for the embedding: masked gradient, then dwte (fp32 atomics,
// see DESIGN.md) and dwpe (deterministic: reduced over the batch in order).
__global__ void embedding_wte_bwd_kernel(const int32_t* __restrict__ tok, const BF8* __restrict__ dout,
                                         float* __restrict__ dwte, float* __restrict__ gmasked, long long nvec,
                                         int wvec, float p, uint64_t seed, uint64_t stream) {
  const uint32_t thr = drop_threshold(p);
  const float scale = p > 0.f ? 1.f / (1.f - p) : 1.f;
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < nvec;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long row = v / wvec;
    const int c = static_cast<int>(v % wvec);
    float d[8];
    bf8_to_f(dout[v], d);
    const uint32_t keep = p > 0.f ? keep_bits8(seed, stream, v, thr) : 0xFFu;
    float* dst = dwte + static_cast<long long>(tok[row]) * wvec * 8 + c * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float g = ((keep >> j) & 1u) ? d[j] * scale : 0.f;
      gmasked[v * 8 + j] = g;
      atomicAdd(dst + j, g);
    }
  }
}

__global__ void embedding_wpe_bwd_kernel(const float* __restrict__ gmasked, float* __restrict__ dwpe, int batch,
                                         int seq, int width) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(seq) * width) return;
  float s = 0.f;
  for (int b = 0; b < batch; ++b) s += gmasked[static_cast<long long>(b) * seq * width + idx];
  dwpe[idx] += s;
}

// Row-wise cross-entropy over the vocabulary, in place: logits -> dlogits.
// loss_rows[r] = logsumexp(row) - row[label]; d = (softmax - onehot) * grad_scale.
__global__ void __launch_bounds__(kBlock) xent_kernel(__nv_bfloat16* __restrict__ logits,
                                                      const int32_t* __restrict__ labels,
                                                      float* __restrict__ loss_rows, int vocab, float grad_scale) {
  __shared__ float red[kBlock / 32];
  __shared__ float bcast;
  const long long row = blockIdx.x;
  BF8* lr = reinterpret_cast<BF8*>(logits + row * vocab);
  const int nvec = vocab / 8;
  float mx = -INFINITY;
  for (int c = threadIdx.x; c < nvec; c += kBlock) {
    float a[8];
    bf8_to_f(lr[c], a);
#pragma unroll
    for (int j = 0; j < 8; ++j) mx = fmaxf(mx, a[j]);
  }
  mx = warp_max(mx);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = red[0];
    for (int i = 1; i < kBlock / 32; ++i) m = fmaxf(m, red[i]);
    bcast = m;
  }
  __syncthreads();
  mx = bcast;
  float s = 0.f;
  for (int c = threadIdx.x; c < nvec; c += kBlock) {
    float a[8];
    bf8_to_f(lr[c], a);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += __expf(a[j] - mx);
  }
  s = warp_sum(s);
  __syncthreads();
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < kBlock / 32; ++i) t += red[i];
    bcast = t;
  }
  __syncthreads();
  const float lse = mx + logf(bcast);
  const int label = labels[row];
  const float target = bf2f(logits[row * vocab + label]);
  __syncthreads();
  for (int c = threadIdx.x; c < nvec; c += kBlock) {
    float a[8];
    bf8_to_f(lr[c], a);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float pj = __expf(a[j] - lse);
      a[j] = (pj - ((c * 8 + j) == label ? 1.f : 0.f)) * grad_scale;
    }
    lr[c] = f_to_bf8(a);
  }
  if (threadIdx.x == 0) loss_rows[row] = lse - target;
}

LYNX_DEV float grad_at(const float* g, long long i) { return g[i]; }
LYNX_DEV float grad_at(const __nv_bfloat16* g, long long i) { return bf2f(g[i]); }

template <class G>
__global__ void adam_kernel(float* __restrict__ master, __nv_bfloat16* __restrict__ param, const G* __restrict__ grad,
                            float* __restrict__ m, float* __restrict__ v, long long n, float lr, float b1, float b2,
                            float eps, float wd, float bc1, float bc2, float gscale) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float g = grad_at(grad, i) * gscale;
    const float mi = b1 * m[i] + (1.f - b1) * g;
    const float vi = b2 * v[i] + (1.f - b2) * g * g;
    m[i] = mi;
    v[i] = vi;
    float w = master[i];
    w -= lr * ((mi / bc1) / (sqrtf(vi / bc2) + eps) + wd * w);
    master[i] = w;
    param[i] = f2bf(w);
  }
}

// Same arithmetic as adam_kernel, 4 parameters per thread with 16-byte loads/stores
// (HBM-bound: 30 B per parameter). n4 = n / 4; the tail is left to adam_kernel.
__device__ __forceinline__ float adam_one(float g, float& mi, float& vi, float w, float lr, float b1, float b2,
                                          float eps, float wd, float bc1, float bc2) {
  mi = b1 * mi + (1.f - b1) * g;
  vi = b2 * vi + (1.f - b2) * g * g;
  return w - lr * ((mi / bc1) / (sqrtf(vi / bc2) + eps) + wd * w);
}

LYNX_DEV float4 grad4_at(const float4* g, long long i) { return g[i]; }
LYNX_DEV float4 grad4_at(const uint2* g, long long i) {
  const uint2 w = g[i];
  const float2 a = unpack_bf16x2(w.x), b = unpack_bf16x2(w.y);
  return make_float4(a.x, a.y, b.x, b.y);
}

template <class G4>
__global__ void __launch_bounds__(256) adam_vec4_kernel(float4* __restrict__ master, uint2* __restrict__ param,
                                                        const G4* __restrict__ grad, float4* __restrict__ m,
                                                        float4* __restrict__ v, long long n4, float lr, float b1,
                                                        float b2, float eps, float wd, float bc1, float bc2,
                                                        float gscale) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float4 g = grad4_at(grad, i);
    float4 mi = m[i], vi = v[i], w = master[i];
    w.x = adam_one(g.x * gscale, mi.x, vi.x, w.x, lr, b1, b2, eps, wd, bc1, bc2);
    w.y = adam_one(g.y * gscale, mi.y, vi.y, w.y, lr, b1, b2, eps, wd, bc1, bc2);
    w.z = adam_one(g.z * gscale, mi.z, vi.z, w.z, lr, b1, b2, eps, wd, bc1, bc2);
    w.w = adam_one(g.w * gscale, mi.w, vi.w, w.w, lr, b1, b2, eps, wd, bc1, bc2);
    m[i] = mi;
    v[i] = vi;
    master[i] = w;
    param[i] = make_uint2(pack_bf16x2(w.x, w.y), pack_bf16x2(w.z, w.w));
  }
}

__global__ void fill_kernel(float* p, float v, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    p[i] = v;
}

__global__ void fill_param_kernel(__nv_bfloat16* p, float* m, float v, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    p[i] = f2bf(v);
    if (m) m[i] = v;
  }
}

__global__ void mismatch_kernel(const uint32_t* a, const uint32_t* b, long long n, unsigned long long* out) {
  unsigned long long c = 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    c += a[i] != b[i];
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Box-Muller on Philox draws: deterministic in (seed, stream, index).
__global__ void init_normal_kernel(__nv_bfloat16* __restrict__ p, float* __restrict__ master, long long n, float std,
                                   uint64_t seed, uint64_t stream) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; 2 * i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const uint4 r = philox_group(seed, stream, static_cast<uint64_t>(i));
    const float u1 = (r.x + 1.0f) * 2.3283064365386963e-10f;  // (0, 1]
    const float u2 = r.y * 2.3283064365386963e-10f;
    const float rad = sqrtf(-2.f * logf(u1));
    const float z0 = rad * cosf(6.283185307179586f * u2) * std;
    const float z1 = rad * sinf(6.283185307179586f * u2) * std;
    const __nv_bfloat16 b0 = f2bf(z0), b1 = f2bf(z1);
    p[2 * i] = b0;
    if (master) master[2 * i] = bf2f(b0);
    if (2 * i + 1 < n) {
      p[2 * i + 1] = b1;
      if (master) master[2 * i + 1] = bf2f(b1);
    }
  }
}

}  // namespace

int bias_dropout_residual_fwd(const __nv_bfloat16* y, const __nv_bfloat16* bias, const __nv_bfloat16* res,
                              __nv_bfloat16* out, long long rows, int width, float p, uint64_t seed,
                              uint64_t stream_id, cudaStream_t s) {
  if (width % 8) return set_error("bias_dropout_residual: width % 8", kValidation);
  const long long nvec = rows * width / 8;
  if (!nvec) return kOk;
  bias_dropout_residual_kernel<<<grid_for(nvec), kBlock, 0, s>>>(
      reinterpret_cast<const BF8*>(y), reinterpret_cast<const BF8*>(bias), reinterpret_cast<const BF8*>(res),
      reinterpret_cast<BF8*>(out), nvec, width / 8, p, seed, stream_id);
  return check_launch("bias_dropout_residual_fwd");
}

int dropout_bwd(const __nv_bfloat16* dout, __nv_bfloat16* dy, long long rows, int width, float p, uint64_t seed,
                uint64_t stream_id, cudaStream_t s) {
  if (width % 8) return set_error("dropout_bwd: width % 8", kValidation);
  const long long nvec = rows * width / 8;
  if (!nvec) return kOk;
  dropout_bwd_kernel<<<grid_for(nvec), kBlock, 0, s>>>(reinterpret_cast<const BF8*>(dout),
                                                       reinterpret_cast<BF8*>(dy), nvec, p, seed, stream_id);
  return check_launch("dropout_bwd");
}

int gelu_fwd(const __nv_bfloat16* x, __nv_bfloat16* y, long long n, cudaStream_t s) {
  if (n % 8) return set_error("gelu: n % 8", kValidation);
  if (!n) return kOk;
  gelu_fwd_kernel<<<grid_for(n / 8), kBlock, 0, s>>>(reinterpret_cast<const BF8*>(x), reinterpret_cast<BF8*>(y),
                                                     n / 8);
  return check_launch("gelu_fwd");
}

int gelu_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* x, __nv_bfloat16* dx, long long n, cudaStream_t s) {
  if (n % 8) return set_error("gelu: n % 8", kValidation);
  if (!n) return kOk;
  gelu_bwd_kernel<<<grid_for(n / 8), kBlock, 0, s>>>(reinterpret_cast<const BF8*>(dy),
                                                     reinterpret_cast<const BF8*>(x), reinterpret_cast<BF8*>(dx),
                                                     n / 8);
  return check_launch("gelu_bwd");
}

int add_bf16(const __nv_bfloat16* a, const __nv_bfloat16* b, __nv_bfloat16* out, long long n, cudaStream_t s) {
  if (n % 8) return set_error("add: n % 8", kValidation);
  if (!n) return kOk;
  add_kernel<<<grid_for(n / 8), kBlock, 0, s>>>(reinterpret_cast<const BF8*>(a), reinterpret_cast<const BF8*>(b),
                                                reinterpret_cast<BF8*>(out), n / 8);
  return check_launch("add_bf16");
}

int embedding_fwd(const int32_t* tokens, const __nv_bfloat16* wte, const __nv_bfloat16* wpe, __nv_bfloat16* out,
                  int batch, int seq, int width, float p, uint64_t seed, uint64_t stream_id, cudaStream_t s) {
  if (width % 8) return set_error("embedding: width % 8", kValidation);
  const long long nvec = static_cast<long long>(batch) * seq * width / 8;
  embedding_fwd_kernel<<<grid_for(nvec), kBlock, 0, s>>>(tokens, reinterpret_cast<const BF8*>(wte),
                                                         reinterpret_cast<const BF8*>(wpe),
                                                         reinterpret_cast<BF8*>(out), nvec, width / 8, seq, p, seed,
                                                         stream_id);
  return check_launch("embedding_fwd");
}

size_t embedding_bwd_workspace(int batch, int seq, int width) {
  return static_cast<size_t>(batch) * seq * width * sizeof(float);
}

int embedding_bwd(const int32_t* tokens, const __nv_bfloat16* dout, float* dwte, float* dwpe, float* workspace,
                  int batch, int seq, int width, int vocab, float p, uint64_t seed, uint64_t stream_id,
                  cudaStream_t s) {
  (void)vocab;
  if (width % 8) return set_error("embedding: width % 8", kValidation);
  const long long nvec = static_cast<long long>(batch) * seq * width / 8;
  embedding_wte_bwd_kernel<<<grid_for(nvec), kBlock, 0, s>>>(tokens, reinterpret_cast<const BF8*>(dout), dwte,
                                                             workspace, nvec, width / 8, p, seed, stream_id);
  const long long n = static_cast<long long>(seq) * width;
  embedding_wpe_bwd_kernel<<<static_cast<int>((n + kBlock - 1) / kBlock), kBlock, 0, s>>>(workspace, dwpe, batch,
                                                                                           seq, width);
  return check_launch("embedding_bwd", 2);
}

int xent_fwd_bwd(__nv_bfloat16* logits, const int32_t* labels, float* loss_rows, long long rows, int vocab,
                 float grad_scale, cudaStream_t s) {
  if (vocab % 8) return set_error("xent: vocab % 8", kValidation);
  if (!rows) return kOk;
  xent_kernel<<<static_cast<unsigned>(rows), kBlock, 0, s>>>(logits, labels, loss_rows, vocab, grad_scale);
  return check_launch("xent_fwd_bwd");
}

int adam_step(float* master, __nv_bfloat16* param, const void* grad, int grad_bf16, float* m, float* v, long long n,
              float lr, float beta1, float beta2, float eps, float weight_decay, int step, float grad_scale,
              cudaStream_t s) {
  const float bc1 = 1.f - powf(beta1, static_cast<float>(step));
  const float bc2 = 1.f - powf(beta2, static_cast<float>(step));
  const size_t gsz = grad_bf16 ? 2 : 4;
  const bool aligned = ((reinterpret_cast<uintptr_t>(master) | reinterpret_cast<uintptr_t>(m) |
                         reinterpret_cast<uintptr_t>(v)) % 16 == 0) &&
                       reinterpret_cast<uintptr_t>(grad) % (4 * gsz) == 0 && reinterpret_cast<uintptr_t>(param) % 8 == 0;
  const long long n4 = aligned ? n / 4 : 0;
  if (n4) {
    auto* m4 = reinterpret_cast<float4*>(master);
    auto* p4 = reinterpret_cast<uint2*>(param);
    if (grad_bf16)
      adam_vec4_kernel<uint2><<<grid_for(n4), 256, 0, s>>>(m4, p4, static_cast<const uint2*>(grad),
                                                           reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v),
                                                           n4, lr, beta1, beta2, eps, weight_decay, bc1, bc2,
                                                           grad_scale);
    else
      adam_vec4_kernel<float4><<<grid_for(n4), 256, 0, s>>>(m4, p4, static_cast<const float4*>(grad),
                                                            reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v),
                                                            n4, lr, beta1, beta2, eps, weight_decay, bc1, bc2,
                                                            grad_scale);
  }
  const long long done = 4 * n4;
  if (n > done) {
    if (grad_bf16)
      adam_kernel<__nv_bfloat16><<<grid_for(n - done), kBlock, 0, s>>>(
          master + done, param + done, static_cast<const __nv_bfloat16*>(grad) + done, m + done, v + done, n - done,
          lr, beta1, beta2, eps, weight_decay, bc1, bc2, grad_scale);
    else
      adam_kernel<float><<<grid_for(n - done), kBlock, 0, s>>>(master + done, param + done,
                                                               static_cast<const float*>(grad) + done, m + done,
                                                               v + done, n - done, lr, beta1, beta2, eps,
                                                               weight_decay, bc1, bc2, grad_scale);
  }
  return check_launch("adam_step");
}

__global__ void add_f32_to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = f2bf(bf2f(dst[i]) + src[i]);
}

int add_f32_to_bf16(const float* src, __nv_bfloat16* dst, long long n, cudaStream_t s) {
  if (!n) return kOk;
  add_f32_to_bf16_kernel<<<grid_for(n), kBlock, 0, s>>>(src, dst, n);
  return check_launch("add_f32_to_bf16");
}

int fill_f32(float* p, float v, long long n, cudaStream_t s) {
  if (!n) return kOk;
  fill_kernel<<<grid_for(n), kBlock, 0, s>>>(p, v, n);
  return check_launch("fill_f32");
}

int fill_param(__nv_bfloat16* p, float* master, float v, long long n, cudaStream_t s) {
  if (!n) return kOk;
  fill_param_kernel<<<grid_for(n), kBlock, 0, s>>>(p, master, v, n);
  return check_launch("fill_param");
}

int count_mismatch(const void* a, const void* b, size_t bytes, unsigned long long* d_count, cudaStream_t s) {
  const long long n = static_cast<long long>(bytes / 4);
  if (!n) return kOk;
  mismatch_kernel<<<grid_for(n), kBlock, 0, s>>>(static_cast<const uint32_t*>(a), static_cast<const uint32_t*>(b), n,
                                                 d_count);
  return check_launch("count_mismatch");
}

int init_normal_bf16(__nv_bfloat16* p, float* master, long long n, float std, uint64_t seed, uint64_t stream_id,
                     cudaStream_t s) {
  if (!n) return kOk;
  init_normal_kernel<<<grid_for((n + 1) / 2), kBlock, 0, s>>>(p, master, n, std, seed, stream_id);
  return check_launch("init_normal_bf16");
}

// ---------------------------------------------------------------- collective stand-in
__global__ void __launch_bounds__(512) comm_standin_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(500);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

int comm_standin(unsigned long long ns, int ctas, cudaStream_t s) {
  comm_standin_kernel<<<ctas, 512, 0, s>>>(ns);
  return check_launch("comm_standin");
}

}  // namespace lynx
