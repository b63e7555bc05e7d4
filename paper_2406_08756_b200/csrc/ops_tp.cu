// Tensor-parallel reductions fused into their consumer (exec.tp_fused): each TP rank
// reads every rank's row-parallel partial straight from that rank's memory — the same device in the
// in-process loopback grid, NVLink peer mappings across processes — sums them in rank order in fp32 and
// rounds once to bf16 (the value a two-rank ring all-reduce produces), and applies the consumer's
// elementwise work in the same pass: the attention projection's / FC2's bias + dropout + residual
// epilogue (forward), or nothing (the backward dX partials of FC1 / QKV, consumed by LayerNorm
// backward). One kernel replaces the collective and the epilogue that followed it.
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

__device__ __forceinline__ void sum_ranks(const TpPartials& parts, long long v, float* acc) {
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  for (int r = 0; r < parts.n; ++r) {
    // .cg: not through L1 — a peer's staging slot is rewritten every second call
    const uint4 raw = __ldcg(reinterpret_cast<const uint4*>(parts.p[r]) + v);
    BF8 x;
    x.w[0] = raw.x, x.w[1] = raw.y, x.w[2] = raw.z, x.w[3] = raw.w;
    float f[8];
    bf8_to_f(x, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += f[j];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = bf2f(f2bf(acc[j]));  // the all-reduced bf16 value
}

__global__ void tp_reduce_residual_kernel(TpPartials parts, const BF8* __restrict__ bias, const BF8* __restrict__ res,
                                          BF8* __restrict__ out, long long nvec, int wvec, float p, uint64_t seed,
                                          uint64_t stream) {
  const uint32_t thr = drop_threshold(p);
  const float scale = p > 0.f ? 1.f / (1.f - p) : 1.f;
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < nvec;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    float a[8], r[8], b[8];
    sum_ranks(parts, v, a);
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

__global__ void tp_reduce_kernel(TpPartials parts, BF8* __restrict__ out, long long nvec) {
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < nvec;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    float a[8];
    sum_ranks(parts, v, a);
    out[v] = f_to_bf8(a);
  }
}

// Cross-process readiness of call k's partials: every rank stores k + 1 into its slot of every rank's
// flag array (system-scope release after a system fence: the partial's producer kernel completed
// earlier on this stream), then waits until all ranks' slots of its own array reached k + 1.
__global__ void tp_signal_kernel(TpFlags peers, int n, int me, unsigned long long value) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int r = 0; r < n; ++r)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peers.f[r] + me), "l"(value) : "memory");
}

// A peer that never signals (a rank died, or took a different path) must not hang the GPU: after
// kWaitTimeoutNs the kernel traps, the launch fails and the executor reports a CUDA error.
constexpr unsigned long long kWaitTimeoutNs = 60ull * 1000 * 1000 * 1000;

__global__ void tp_wait_kernel(const unsigned long long* flags, int n, unsigned long long value) {
  const int r = threadIdx.x;
  if (r >= n) return;
  unsigned long long v = 0, t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + r) : "memory");
    if (v < value) {
      __nanosleep(200);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > kWaitTimeoutNs) __trap();
    }
  } while (v < value);
}

}  // namespace

int tp_reduce_residual(const TpPartials& parts, const __nv_bfloat16* bias, const __nv_bfloat16* res,
                       __nv_bfloat16* out, long long rows, int width, float p, uint64_t seed, uint64_t stream_id,
                       cudaStream_t s) {
  if (width % 8 || parts.n < 1 || parts.n > kMaxTpRanks) return set_error("tp_reduce_residual: shape", kValidation);
  const long long nvec = rows * width / 8;
  if (!nvec) return kOk;
  tp_reduce_residual_kernel<<<grid_for(nvec), kBlock, 0, s>>>(parts, reinterpret_cast<const BF8*>(bias),
                                                               reinterpret_cast<const BF8*>(res),
                                                               reinterpret_cast<BF8*>(out), nvec, width / 8, p, seed,
                                                               stream_id);
  return check_launch("tp_reduce_residual");
}

int tp_reduce(const TpPartials& parts, __nv_bfloat16* out, long long n, cudaStream_t s) {
  if (n % 8 || parts.n < 1 || parts.n > kMaxTpRanks) return set_error("tp_reduce: shape", kValidation);
  if (!n) return kOk;
  tp_reduce_kernel<<<grid_for(n / 8), kBlock, 0, s>>>(parts, reinterpret_cast<BF8*>(out), n / 8);
  return check_launch("tp_reduce");
}

int tp_signal_wait(const TpFlags& peers, const unsigned long long* my_flags, int n, int me, unsigned long long value,
                   cudaStream_t s) {
  tp_signal_kernel<<<1, 32, 0, s>>>(peers, n, me, value);
  tp_wait_kernel<<<1, 32, 0, s>>>(my_flags, n, value);
  return check_launch("tp_signal_wait", 2);
}

}  // namespace lynx
