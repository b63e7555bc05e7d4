// LayerNorm forward / backward and deterministic column reductions.
//
// Forward: one CTA per row, 16-byte vectorised loads (8 x bf16 per chunk), the
// row held in registers, two-pass mean/variance with a fixed warp-shuffle +
// shared-memory reduction tree, fp32 statistics. HBM-bound: algorithmic bytes
// per row = 2*width (x) + 2*width (y) + 8 (mean, rstd).
//
// Backward: per-row dx (+ optional residual gradient) and dgamma/dbeta partial
// sums accumulated per CTA over a fixed contiguous row range, then reduced in
// a fixed order by a second kernel — no atomics, so gradients are
// bit-reproducible run to run.
#include "common.cuh"
#include "lynx_ops_internal.h"

namespace lynx {
namespace {

constexpr int kNT = 256;    // threads per row-CTA
constexpr int kMaxC = 4;    // chunks of 8 per thread -> width <= 8192
constexpr int kPartBlocks = 512;

template <int NT>
LYNX_DEV float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) t += red[i];
  return t;
}

__global__ void __launch_bounds__(kNT) ln_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                     const __nv_bfloat16* __restrict__ gamma,
                                                     const __nv_bfloat16* __restrict__ beta,
                                                     __nv_bfloat16* __restrict__ y, float* __restrict__ mean,
                                                     float* __restrict__ rstd, int width, float eps) {
  __shared__ float red[kNT / 32];
  const long long row = blockIdx.x;
  const int nchunk = width / 8;
  const BF8* xr = reinterpret_cast<const BF8*>(x + row * width);
  float v[kMaxC][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxC; ++i) {
    const int c = threadIdx.x + i * kNT;
    if (c < nchunk) {
      bf8_to_f(xr[c], v[i]);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[i][j];
    }
  }
  const float mu = block_sum<kNT>(s, red) / width;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxC; ++i) {
    const int c = threadIdx.x + i * kNT;
    if (c < nchunk) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float d = v[i][j] - mu;
        q += d * d;
      }
    }
  }
  const float var = block_sum<kNT>(q, red) / width;
  const float rs = rsqrtf(var + eps);
  const BF8* gr = reinterpret_cast<const BF8*>(gamma);
  const BF8* br = reinterpret_cast<const BF8*>(beta);
  BF8* yr = reinterpret_cast<BF8*>(y + row * width);
#pragma unroll
  for (int i = 0; i < kMaxC; ++i) {
    const int c = threadIdx.x + i * kNT;
    if (c < nchunk) {
      float g[8], b[8], o[8];
      bf8_to_f(gr[c], g);
      bf8_to_f(br[c], b);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = (v[i][j] - mu) * rs * g[j] + b[j];
      yr[c] = f_to_bf8(o);
    }
  }
  if (threadIdx.x == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

// dx for rows [r0, r1) of this CTA's range; partial dgamma/dbeta to ws.
__global__ void __launch_bounds__(kNT) ln_bwd_kernel(const __nv_bfloat16* __restrict__ dy,
                                                     const __nv_bfloat16* __restrict__ x,
                                                     const __nv_bfloat16* __restrict__ gamma,
                                                     const float* __restrict__ mean, const float* __restrict__ rstd,
                                                     const __nv_bfloat16* __restrict__ dres,
                                                     __nv_bfloat16* __restrict__ dx, float* __restrict__ ws,
                                                     int rows, int width) {
  __shared__ float red[kNT / 32];
  const int nchunk = width / 8;
  const int per = (rows + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per;
  const int r1 = min(rows, r0 + per);
  float gsum[kMaxC][8], bsum[kMaxC][8], g[kMaxC][8];
  const BF8* gp = reinterpret_cast<const BF8*>(gamma);
#pragma unroll
  for (int i = 0; i < kMaxC; ++i) {
    const int c = threadIdx.x + i * kNT;
#pragma unroll
    for (int j = 0; j < 8; ++j) gsum[i][j] = bsum[i][j] = 0.f;
    if (c < nchunk) bf8_to_f(gp[c], g[i]);
  }
  for (int row = r0; row < r1; ++row) {
    const BF8* dyr = reinterpret_cast<const BF8*>(dy + static_cast<long long>(row) * width);
    const BF8* xr = reinterpret_cast<const BF8*>(x + static_cast<long long>(row) * width);
    const float mu = mean[row], rs = rstd[row];
    float xh[kMaxC][8], gy[kMaxC][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxC; ++i) {
      const int c = threadIdx.x + i * kNT;
      if (c < nchunk) {
        float d[8], xv[8];
        bf8_to_f(dyr[c], d);
        bf8_to_f(xr[c], xv);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          xh[i][j] = (xv[j] - mu) * rs;
          gy[i][j] = d[j] * g[i][j];
          s1 += gy[i][j];
          s2 += gy[i][j] * xh[i][j];
          gsum[i][j] += d[j] * xh[i][j];
          bsum[i][j] += d[j];
        }
      }
    }
    const float m1 = block_sum<kNT>(s1, red) / width;
    const float m2 = block_sum<kNT>(s2, red) / width;
    BF8* dxr = reinterpret_cast<BF8*>(dx + static_cast<long long>(row) * width);
    const BF8* drr = dres ? reinterpret_cast<const BF8*>(dres + static_cast<long long>(row) * width) : nullptr;
#pragma unroll
    for (int i = 0; i < kMaxC; ++i) {
      const int c = threadIdx.x + i * kNT;
      if (c < nchunk) {
        float o[8], r[8];
        if (drr) bf8_to_f(drr[c], r);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          o[j] = rs * (gy[i][j] - m1 - xh[i][j] * m2);
          if (drr) o[j] += r[j];
        }
        dxr[c] = f_to_bf8(o);
      }
    }
  }
  float* wg = ws + static_cast<long long>(blockIdx.x) * 2 * width;
  float* wb = wg + width;
#pragma unroll
  for (int i = 0; i < kMaxC; ++i) {
    const int c = threadIdx.x + i * kNT;
    if (c < nchunk) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        wg[c * 8 + j] = gsum[i][j];
        wb[c * 8 + j] = bsum[i][j];
      }
    }
  }
}

// acc[k][col] += sum_b ws[b][k][col] in block order (k = 0..nvec-1).
__global__ void reduce_partials_kernel(const float* __restrict__ ws, float* __restrict__ acc0,
                                       float* __restrict__ acc1, int nblocks, int width, int nvec) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= width) return;
  float s0 = 0.f, s1 = 0.f;
  for (int b = 0; b < nblocks; ++b) {
    s0 += ws[(static_cast<long long>(b) * nvec) * width + col];
    if (nvec > 1) s1 += ws[(static_cast<long long>(b) * nvec + 1) * width + col];
  }
  acc0[col] += s0;
  if (nvec > 1) acc1[col] += s1;
}

// Per-CTA partial column sums of a [rows, width] bf16 matrix.
__global__ void __launch_bounds__(kNT) column_partial_kernel(const __nv_bfloat16* __restrict__ x,
                                                             float* __restrict__ ws, long long rows, int width) {
  const int nchunk = width / 8;
  const long long per = (rows + gridDim.x - 1) / gridDim.x;
  const long long r0 = blockIdx.x * per;
  const long long r1 = min(rows, r0 + per);
  for (int c = threadIdx.x; c < nchunk; c += kNT) {
    float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (long long row = r0; row < r1; ++row) {
      float v[8];
      bf8_to_f(reinterpret_cast<const BF8*>(x + row * width)[c], v);
#pragma unroll
      for (int j = 0; j < 8; ++j) s[j] += v[j];
    }
    float* w = ws + static_cast<long long>(blockIdx.x) * width + c * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) w[j] = s[j];
  }
}

int part_blocks(long long rows) { return static_cast<int>(rows < kPartBlocks ? rows : kPartBlocks); }

}  // namespace

int layernorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* gamma, const __nv_bfloat16* beta, __nv_bfloat16* y,
                  float* mean, float* rstd, int rows, int width, float eps, cudaStream_t s) {
  if (width % 8 || width > kNT * kMaxC * 8) return set_error("layernorm: width must be a multiple of 8, <= 8192", kValidation);
  if (rows == 0) return kOk;
  ln_fwd_kernel<<<rows, kNT, 0, s>>>(x, gamma, beta, y, mean, rstd, width, eps);
  return check_launch("layernorm_fwd");
}

size_t layernorm_bwd_workspace(int rows, int width) {
  return static_cast<size_t>(part_blocks(rows)) * 2 * width * sizeof(float);
}

int layernorm_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* x, const __nv_bfloat16* gamma, const float* mean,
                  const float* rstd, const __nv_bfloat16* dres, __nv_bfloat16* dx, float* dgamma_acc,
                  float* dbeta_acc, float* workspace, int rows, int width, cudaStream_t s) {
  if (width % 8 || width > kNT * kMaxC * 8) return set_error("layernorm: width must be a multiple of 8, <= 8192", kValidation);
  if (rows == 0) return kOk;
  const int nb = part_blocks(rows);
  ln_bwd_kernel<<<nb, kNT, 0, s>>>(dy, x, gamma, mean, rstd, dres, dx, workspace, rows, width);
  reduce_partials_kernel<<<(width + 255) / 256, 256, 0, s>>>(workspace, dgamma_acc, dbeta_acc, nb, width, 2);
  return check_launch("layernorm_bwd", 2);
}

size_t column_sum_workspace(long long rows, int width) {
  return static_cast<size_t>(part_blocks(rows)) * width * sizeof(float);
}

int column_sum_acc(const __nv_bfloat16* x, float* acc, float* workspace, long long rows, int width, cudaStream_t s) {
  if (width % 8) return set_error("column_sum: width must be a multiple of 8", kValidation);
  if (rows == 0) return kOk;
  const int nb = part_blocks(rows);
  column_partial_kernel<<<nb, kNT, 0, s>>>(x, workspace, rows, width);
  reduce_partials_kernel<<<(width + 255) / 256, 256, 0, s>>>(workspace, acc, nullptr, nb, width, 1);
  return check_launch("column_sum_acc", 2);
}

}  // namespace lynx
