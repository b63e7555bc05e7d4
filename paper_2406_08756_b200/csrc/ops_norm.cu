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
#include <cstdlib>

#include "common.cuh"
#include "lynx_ops_internal.h"

namespace lynx {
namespace {

constexpr int kNT = 256;    // threads per row-CTA
constexpr int kMaxC = 4;    // chunks of 8 per thread -> width <= 8192
constexpr int kPartBlocks = 1184;  // 8 x 148 SMs: row-partitioned partial sums (bias gradients)

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

// Warp-group-per-row forward for width = 256*C*W: W warps (1 or 2) share a row, each lane
// streams C 16-byte chunks (all loads in flight at once), statistics by warp shuffles plus,
// for W = 2, one shared-memory exchange; the row stays raw bf16 in registers. 8/W rows per
// 256-thread CTA. W = 2 for wide rows keeps registers low enough for 2+ CTAs per SM (a
// 16-chunk-per-lane warp needed 254 registers and ran latency-bound at one CTA per SM).
template <int C, int W>
__global__ void __launch_bounds__(256) ln_fwd_warp_kernel(const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ gamma,
                                                          const __nv_bfloat16* __restrict__ beta,
                                                          __nv_bfloat16* __restrict__ y, float* __restrict__ mean,
                                                          float* __restrict__ rstd, int rows, int width, float eps) {
  __shared__ float xch[8][2];
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, part = warp % W;
  const long long row = blockIdx.x * (8LL / W) + warp / W;
  const bool live = row < rows;
  const BF8* xr = reinterpret_cast<const BF8*>(x + (live ? row : 0) * width);
  const int c0 = part * 32 * C + lane;  // this lane's chunks: c0 + 32 i
  BF8 raw[C];
#pragma unroll
  for (int i = 0; i < C; ++i) raw[i] = xr[c0 + 32 * i];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < C; ++i) {
    float v[8];
    bf8_to_f(raw[i], v);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  s = warp_sum(s);
  if (W > 1) {
    if (lane == 0) xch[warp][0] = s;
    __syncthreads();
    s = 0.f;
#pragma unroll
    for (int k = 0; k < W; ++k) s += xch[warp - part + k][0];  // fixed order: every part gets the same sum
  }
  const float mu = s / width;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < C; ++i) {
    float v[8];
    bf8_to_f(raw[i], v);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float d = v[j] - mu;
      q += d * d;
    }
  }
  q = warp_sum(q);
  if (W > 1) {
    if (lane == 0) xch[warp][1] = q;
    __syncthreads();
    q = 0.f;
#pragma unroll
    for (int k = 0; k < W; ++k) q += xch[warp - part + k][1];
  }
  const float rs = rsqrtf(q / width + eps);
  if (!live) return;
  const BF8* gr = reinterpret_cast<const BF8*>(gamma);
  const BF8* br = reinterpret_cast<const BF8*>(beta);
  BF8* yr = reinterpret_cast<BF8*>(y + row * width);
#pragma unroll
  for (int i = 0; i < C; ++i) {
    float v[8], g[8], b[8], o[8];
    bf8_to_f(raw[i], v);
    bf8_to_f(gr[c0 + 32 * i], g);
    bf8_to_f(br[c0 + 32 * i], b);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (v[j] - mu) * rs * g[j] + b[j];
    yr[c0 + 32 * i] = f_to_bf8(o);
  }
  if (lane == 0 && part == 0) {
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

// Row-batched backward: each CTA owns a contiguous row range and walks it R rows at a
// time, so every thread has R*C*(2 or 3) 16-byte loads in flight per barrier round
// (the one-row-at-a-time kernel above is latency-bound at ~20% of HBM bandwidth).
// The thread owns the same C chunks of every row, so the dgamma/dbeta partials stay
// in registers. The per-row sums s1 = sum(g*dy), s2 = sum(g*dy*xhat) of all R rows
// are reduced in one shared-memory round (double-buffered, one barrier per batch).
constexpr int kLnBlocks = 296;  // 2 CTAs per SM on 148 SMs

// R = 4 / C rows per batch keeps the in-flight loads (3*R*C 16-B vectors) and the
// register-resident dgamma/dbeta partials (16*C floats) within 128 registers.
template <int C>
__global__ void __launch_bounds__(256, C <= 2 ? 2 : 1) ln_bwd_rows_kernel(const __nv_bfloat16* __restrict__ dy,
                                                             const __nv_bfloat16* __restrict__ x,
                                                             const __nv_bfloat16* __restrict__ gamma,
                                                             const float* __restrict__ mean,
                                                             const float* __restrict__ rstd,
                                                             const __nv_bfloat16* __restrict__ dres,
                                                             __nv_bfloat16* __restrict__ dx, float* __restrict__ ws,
                                                             int rows, int width) {
  constexpr int R = C >= 4 ? 1 : 4 / C;
  __shared__ float red[2][2 * R][8];
  const int nt = blockDim.x, nw = nt / 32, warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int per = (rows + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per;
  const int r1 = min(rows, r0 + per);
  const float inv_w = 1.f / width;
  float g[C][8], gsum[C][8], bsum[C][8];
#pragma unroll
  for (int i = 0; i < C; ++i) {
    bf8_to_f(reinterpret_cast<const BF8*>(gamma)[threadIdx.x + i * nt], g[i]);
#pragma unroll
    for (int j = 0; j < 8; ++j) gsum[i][j] = bsum[i][j] = 0.f;
  }
  int it = 0;
  for (int row = r0; row < r1; row += R, it ^= 1) {
    BF8 dv[R][C], xv[R][C], rv[R][C];
    float mu[R], rs[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const bool ok = row + rr < r1;
      const long long base = static_cast<long long>(ok ? row + rr : row) * width;
      mu[rr] = mean[ok ? row + rr : row];
      rs[rr] = ok ? rstd[row + rr] : 0.f;  // rs = 0 zeroes an out-of-range row's contributions
#pragma unroll
      for (int i = 0; i < C; ++i) {
        const int c = threadIdx.x + i * nt;
        dv[rr][i] = reinterpret_cast<const BF8*>(dy + base)[c];
        xv[rr][i] = reinterpret_cast<const BF8*>(x + base)[c];
        if (dres) rv[rr][i] = reinterpret_cast<const BF8*>(dres + base)[c];
      }
    }
    float s[2 * R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      float s1 = 0.f, s2 = 0.f;
      const float keep = rs[rr] != 0.f ? 1.f : 0.f;
#pragma unroll
      for (int i = 0; i < C; ++i) {
        float d[8], xx[8];
        bf8_to_f(dv[rr][i], d);
        bf8_to_f(xv[rr][i], xx);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (xx[j] - mu[rr]) * rs[rr], gy = d[j] * g[i][j];
          s1 += gy;
          s2 += gy * xh;
          gsum[i][j] += d[j] * xh;
          bsum[i][j] += d[j] * keep;
        }
      }
      s[2 * rr] = warp_sum(s1);
      s[2 * rr + 1] = warp_sum(s2);
    }
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 2 * R; ++k) red[it][k][warp] = s[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 2 * R; ++k) {
      float t = 0.f;
      for (int w = 0; w < nw; ++w) t += red[it][k][w];
      s[k] = t * inv_w;
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (row + rr >= r1) break;
      BF8* dxr = reinterpret_cast<BF8*>(dx + static_cast<long long>(row + rr) * width);
#pragma unroll
      for (int i = 0; i < C; ++i) {
        float d[8], xx[8], o[8], r[8];
        bf8_to_f(dv[rr][i], d);
        bf8_to_f(xv[rr][i], xx);
        if (dres) bf8_to_f(rv[rr][i], r);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (xx[j] - mu[rr]) * rs[rr], gy = d[j] * g[i][j];
          o[j] = rs[rr] * (gy - s[2 * rr] - xh * s[2 * rr + 1]);
          if (dres) o[j] += r[j];
        }
        dxr[threadIdx.x + i * nt] = f_to_bf8(o);
      }
    }
  }
  float* wg = ws + static_cast<long long>(blockIdx.x) * 2 * width;
  float* wb = wg + width;
#pragma unroll
  for (int i = 0; i < C; ++i) {
    const int c = threadIdx.x + i * nt;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      wg[c * 8 + j] = gsum[i][j];
      wb[c * 8 + j] = bsum[i][j];
    }
  }
}

// Chunks-per-thread for the row-batched kernel (0: unsupported width -> one-row kernel).
int ln_rows_chunks(int width) {
  const int nchunk = width / 8;
  for (int c : {1, 2, 4})
    if (nchunk % c == 0 && nchunk / c <= 256 && (nchunk / c) % 32 == 0) return c;
  return 0;
}

// acc[k][col] += sum_b ws[b][k][col] in block order (k = 0..nvec-1).
// 32 columns per CTA; warp w sums the contiguous block range [w*per, (w+1)*per) with
// 4-way unrolled loads, then warp 0 adds the 8 warp sums in order: a fixed tree, so
// the result is bit-reproducible, with 8x the loads in flight of a one-thread-per-column loop.
__global__ void __launch_bounds__(256) reduce_partials_kernel(const float* __restrict__ ws, void* __restrict__ acc0,
                                                              void* __restrict__ acc1, int nblocks, int width,
                                                              int nvec, int acc_bf16) {
  __shared__ float part[8][2][32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int col = blockIdx.x * 32 + lane;
  const int per = (nblocks + 7) / 8;
  const int b0 = warp * per, b1 = min(nblocks, b0 + per);
  float s0 = 0.f, s1 = 0.f;
  if (col < width) {
#pragma unroll 4
    for (int b = b0; b < b1; ++b) {
      s0 += ws[(static_cast<long long>(b) * nvec) * width + col];
      if (nvec > 1) s1 += ws[(static_cast<long long>(b) * nvec + 1) * width + col];
    }
  }
  part[warp][0][lane] = s0;
  part[warp][1][lane] = s1;
  __syncthreads();
  if (warp == 0 && col < width) {
    float t0 = 0.f, t1 = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      t0 += part[w][0][lane];
      t1 += part[w][1][lane];
    }
    if (acc_bf16) {  // bf16 gradient accumulators (16 B / parameter model states)
      auto* a0 = static_cast<__nv_bfloat16*>(acc0);
      a0[col] = f2bf(bf2f(a0[col]) + t0);
      if (nvec > 1) {
        auto* a1 = static_cast<__nv_bfloat16*>(acc1);
        a1[col] = f2bf(bf2f(a1[col]) + t1);
      }
    } else {
      static_cast<float*>(acc0)[col] += t0;
      if (nvec > 1) static_cast<float*>(acc1)[col] += t1;
    }
  }
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
#pragma unroll 4  // independent row loads in flight (the sums stay in row order)
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

// dy = dropout_bwd(dout) (the Philox mask of dropout_bwd_kernel, element vector index
// row * width / 8 + c) and the column partial sums of the bf16 dy in one pass: the bias gradient
// of the projection / FC2 branch. Same row partition and summation order as column_partial_kernel,
// so the bias gradient is bit-identical to the two-kernel path.
__global__ void __launch_bounds__(kNT) dropout_bwd_colsum_kernel(const __nv_bfloat16* __restrict__ dout,
                                                                 __nv_bfloat16* __restrict__ dy, float* __restrict__ ws,
                                                                 long long rows, int width, float p, uint64_t seed,
                                                                 uint64_t stream) {
  const uint32_t thr = drop_threshold(p);
  const float scale = p > 0.f ? 1.f / (1.f - p) : 1.f;
  const int nchunk = width / 8;
  const long long per = (rows + gridDim.x - 1) / gridDim.x;
  const long long r0 = blockIdx.x * per;
  const long long r1 = min(rows, r0 + per);
  for (int c = threadIdx.x; c < nchunk; c += kNT) {
    float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
    for (long long row = r0; row < r1; ++row) {
      float d[8], o[8];
      const long long vec = row * nchunk + c;
      bf8_to_f(reinterpret_cast<const BF8*>(dout)[vec], d);
      const uint32_t keep = p > 0.f ? keep_bits8(seed, stream, vec, thr) : 0xFFu;
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = ((keep >> j) & 1u) ? d[j] * scale : 0.f;
      const BF8 ob = f_to_bf8(o);
      reinterpret_cast<BF8*>(dy)[vec] = ob;
      bf8_to_f(ob, o);
#pragma unroll
      for (int j = 0; j < 8; ++j) s[j] += o[j];
    }
    float* w = ws + static_cast<long long>(blockIdx.x) * width + c * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) w[j] = s[j];
  }
}

int part_blocks(long long rows) { return static_cast<int>(rows < kPartBlocks ? rows : kPartBlocks); }

}  // namespace

// Warps per row for the wide (16-24 chunk) LayerNorm forward: 4 by default (2 rows per 256-thread
// CTA: 0.219 ms at [65536, 4096] = 75 % of HBM, vs 0.259 ms with 2 warps per row); LYNX_LN_PARTS=2|8.
int ln_fwd_parts() {
  static const int w = [] {
    const char* e = std::getenv("LYNX_LN_PARTS");
    return e && e[0] == '2' ? 2 : (e && e[0] == '8' ? 8 : 4);
  }();
  return w;
}

int layernorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* gamma, const __nv_bfloat16* beta, __nv_bfloat16* y,
                  float* mean, float* rstd, int rows, int width, float eps, cudaStream_t s) {
  if (width % 8 || width > kNT * kMaxC * 8) return set_error("layernorm: width must be a multiple of 8, <= 8192", kValidation);
  if (rows == 0) return kOk;
  const unsigned grid1 = static_cast<unsigned>((rows + 7) / 8), grid2 = static_cast<unsigned>((rows + 3) / 4),
                 grid4 = static_cast<unsigned>((rows + 1) / 2), grid8 = static_cast<unsigned>(rows);
  switch (width % 256 ? 0 : width / 256) {
#define LN_FWD_W1(C) \
  case C: ln_fwd_warp_kernel<C, 1><<<grid1, 256, 0, s>>>(x, gamma, beta, y, mean, rstd, rows, width, eps); break;
#define LN_FWD_W2(C)                                                                                          \
  case C:                                                                                                    \
    if (ln_fwd_parts() == 8 && C % 8 == 0)                                                                   \
      ln_fwd_warp_kernel<C / 8, 8><<<grid8, 256, 0, s>>>(x, gamma, beta, y, mean, rstd, rows, width, eps);   \
    else if (ln_fwd_parts() == 2)                                                                            \
      ln_fwd_warp_kernel<C / 2, 2><<<grid2, 256, 0, s>>>(x, gamma, beta, y, mean, rstd, rows, width, eps);   \
    else                                                                                                     \
      ln_fwd_warp_kernel<C / 4, 4><<<grid4, 256, 0, s>>>(x, gamma, beta, y, mean, rstd, rows, width, eps);   \
    break;
    LN_FWD_W1(1)
    LN_FWD_W1(2)
    LN_FWD_W1(4)
    LN_FWD_W1(7)
    LN_FWD_W1(8)
    LN_FWD_W2(16)
    LN_FWD_W2(20)
    LN_FWD_W2(24)
#undef LN_FWD_W1
#undef LN_FWD_W2
    default: ln_fwd_kernel<<<rows, kNT, 0, s>>>(x, gamma, beta, y, mean, rstd, width, eps);
  }
  return check_launch("layernorm_fwd");
}

size_t layernorm_bwd_workspace(int rows, int width) {
  return static_cast<size_t>(part_blocks(rows)) * 2 * width * sizeof(float);
}

int layernorm_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* x, const __nv_bfloat16* gamma, const float* mean,
                  const float* rstd, const __nv_bfloat16* dres, __nv_bfloat16* dx, void* dgamma_acc,
                  void* dbeta_acc, int acc_bf16, float* workspace, int rows, int width, cudaStream_t s) {
  if (width % 8 || width > kNT * kMaxC * 8) return set_error("layernorm: width must be a multiple of 8, <= 8192", kValidation);
  if (rows == 0) return kOk;
  const int cpt = ln_rows_chunks(width);
  const int nb = cpt ? (rows < kLnBlocks ? rows : kLnBlocks) : part_blocks(rows);
  const int nt = cpt ? width / 8 / cpt : kNT;
  switch (cpt) {
    case 1: ln_bwd_rows_kernel<1><<<nb, nt, 0, s>>>(dy, x, gamma, mean, rstd, dres, dx, workspace, rows, width); break;
    case 2: ln_bwd_rows_kernel<2><<<nb, nt, 0, s>>>(dy, x, gamma, mean, rstd, dres, dx, workspace, rows, width); break;
    case 4: ln_bwd_rows_kernel<4><<<nb, nt, 0, s>>>(dy, x, gamma, mean, rstd, dres, dx, workspace, rows, width); break;
    default: ln_bwd_kernel<<<nb, kNT, 0, s>>>(dy, x, gamma, mean, rstd, dres, dx, workspace, rows, width);
  }
  reduce_partials_kernel<<<(width + 31) / 32, 256, 0, s>>>(workspace, dgamma_acc, dbeta_acc, nb, width, 2,
                                                           acc_bf16);
  return check_launch("layernorm_bwd", 2);
}

size_t column_sum_workspace(long long rows, int width) {
  return static_cast<size_t>(part_blocks(rows)) * width * sizeof(float);
}

int column_sum_acc(const __nv_bfloat16* x, void* acc, int acc_bf16, float* workspace, long long rows, int width,
                   cudaStream_t s) {
  if (width % 8) return set_error("column_sum: width must be a multiple of 8", kValidation);
  if (rows == 0) return kOk;
  const int nb = part_blocks(rows);
  column_partial_kernel<<<nb, kNT, 0, s>>>(x, workspace, rows, width);
  reduce_partials_kernel<<<(width + 31) / 32, 256, 0, s>>>(workspace, acc, nullptr, nb, width, 1, acc_bf16);
  return check_launch("column_sum_acc", 2);
}

int dropout_bwd_colsum(const __nv_bfloat16* dout, __nv_bfloat16* dy, void* acc, int acc_bf16, float* workspace,
                       long long rows, int width, float p, uint64_t seed, uint64_t stream_id, cudaStream_t s) {
  if (width % 8) return set_error("dropout_bwd_colsum: width must be a multiple of 8", kValidation);
  if (p < 0.f || p >= 1.f) return set_error("dropout: p must be in [0, 1)", kValidation);
  if (rows == 0) return kOk;
  const int nb = part_blocks(rows);
  dropout_bwd_colsum_kernel<<<nb, kNT, 0, s>>>(dout, dy, workspace, rows, width, p, seed, stream_id);
  reduce_partials_kernel<<<(width + 31) / 32, 256, 0, s>>>(workspace, acc, nullptr, nb, width, 1, acc_bf16);
  return check_launch("dropout_bwd_colsum", 2);
}

}  // namespace lynx
