// Causal multi-head attention (flash style), forward and backward.
//
// Layout (per TP rank): qkv [T, 3*H*D] bf16 with row t = b*S + s and columns
// [Q heads | K heads | V heads], head h at h*D; out [T, H*D]; lse [B, H, S] fp32.
//
// Forward: one CTA per (64-query block, head, batch), 4 warps x 16 query rows,
// 64-key tiles double-buffered through padded shared memory by cp.async,
// S = Q K^T and O += P V on mma.sync m16n8k16 (bf16 -> fp32), online softmax
// in registers with warp-shuffle (quad) row max/sum, exp2 with the
// log2(e)-prescaled logits. Heavy (late) query blocks are scheduled first.
//
// Backward is split so that no output is accumulated with atomics (dQ would
// otherwise be summed across key blocks in a non-deterministic order):
//   attn_bwd_dkdv: per 64-key block, sweep the causal query blocks (32 rows),
//                  recompute P^T, dV += P^T dO, dP^T = V dO^T, dK += dS^T Q;
//   attn_bwd_dq:   per 64-query block, sweep key blocks (32 keys),
//                  recompute P and dP, dQ += dS K.
// This costs 7 instead of 5 tile matmuls but keeps every gradient
// bit-reproducible. Attention is ~8% of the GPT-7B step FLOPs.
#include "common.cuh"
#include "lynx_ops_internal.h"

namespace lynx {
namespace {

constexpr float kLog2e = 1.4426950408889634f;

LYNX_DEV void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
LYNX_DEV void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
LYNX_DEV void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

LYNX_DEV void ldsm_x4(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
LYNX_DEV void ldsm_x4_t(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
LYNX_DEV void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// A fragment (16 x 16) at (r0, k0) of a row-major smem tile with pitch P.
template <int P>
LYNX_DEV void load_a(uint32_t* a, const __nv_bfloat16* s, int r0, int k0, int lane) {
  ldsm_x4(a, s + (r0 + (lane % 16)) * P + k0 + (lane / 16) * 8);
}
// B fragments for two n-blocks (n0, n0+8) x k16 from a [n][k] smem tile.
template <int P>
LYNX_DEV void load_b_nk(uint32_t* b, const __nv_bfloat16* s, int n0, int k0, int lane) {
  ldsm_x4(b, s + (n0 + (lane % 8) + (lane / 16) * 8) * P + k0 + ((lane / 8) % 2) * 8);
}
// B fragments for two n-blocks (n0, n0+8) x k16 from a [k][n] smem tile.
template <int P>
LYNX_DEV void load_b_kn(uint32_t* b, const __nv_bfloat16* s, int k0, int n0, int lane) {
  ldsm_x4_t(b, s + (k0 + (lane % 8) + ((lane / 8) % 2) * 8) * P + n0 + (lane / 16) * 8);
}
// Accumulators of n-blocks (2kk, 2kk+1) -> A fragment over k = 16 columns.
LYNX_DEV void acc_to_a(uint32_t* a, const float* c0, const float* c1) {
  a[0] = pack_bf16x2(c0[0], c0[1]);
  a[1] = pack_bf16x2(c0[2], c0[3]);
  a[2] = pack_bf16x2(c1[0], c1[1]);
  a[3] = pack_bf16x2(c1[2], c1[3]);
}

// rows x D tile from global (row pitch ld elements) into smem (pitch P), cp.async.
template <int D, int P>
LYNX_DEV void load_tile(__nv_bfloat16* s, const __nv_bfloat16* g, long long ld, int rows) {
  constexpr int CH = D / 8;
  for (int i = threadIdx.x; i < rows * CH; i += blockDim.x) {
    const int r = i / CH, c = i % CH;
    cp_async16(s + r * P + c * 8, g + r * ld + c * 8);
  }
}

template <int D>
__global__ void __launch_bounds__(128) attn_fwd_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                       __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                                                       int S, int H, float scale_log2) {
  constexpr int P = D + 8, KS = D / 16, ND = D / 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sK = sQ + 64 * P;  // [2][64*P]
  __nv_bfloat16* sV = sK + 2 * 64 * P;
  const int qb = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane / 4, t = lane % 4;
  const long long ld = 3LL * H * D;
  const __nv_bfloat16* gq = qkv + (static_cast<long long>(b) * S + qb * 64) * ld + h * D;
  const __nv_bfloat16* gk = qkv + static_cast<long long>(b) * S * ld + H * D + h * D;
  const __nv_bfloat16* gv = gk + H * D;

  load_tile<D, P>(sQ, gq, ld, 64);
  load_tile<D, P>(sK, gk, ld, 64);
  load_tile<D, P>(sV, gv, ld, 64);
  cp_commit();

  uint32_t qf[KS][4];
  float o[ND][4];
#pragma unroll
  for (int i = 0; i < ND; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int nkb = qb + 1;
  for (int kb = 0; kb < nkb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkb) {
      load_tile<D, P>(sK + (buf ^ 1) * 64 * P, gk + (kb + 1) * 64LL * ld, ld, 64);
      load_tile<D, P>(sV + (buf ^ 1) * 64 * P, gv + (kb + 1) * 64LL * ld, ld, 64);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) load_a<P>(qf[kk], sQ, warp * 16, kk * 16, lane);
    }
    const __nv_bfloat16* k_s = sK + buf * 64 * P;
    const __nv_bfloat16* v_s = sV + buf * 64 * P;
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int j2 = 0; j2 < 4; ++j2) {
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        uint32_t bf[4];
        load_b_nk<P>(bf, k_s, j2 * 16, kk * 16, lane);
        mma16816(s[2 * j2], qf[kk], bf[0], bf[1]);
        mma16816(s[2 * j2 + 1], qf[kk], bf[2], bf[3]);
      }
    }
    const bool diag = kb == qb;
    const int qr0 = warp * 16 + g, qr1 = qr0 + 8;
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = j * 8 + 2 * t + e;
        float v0 = s[j][e] * scale_log2, v1 = s[j][2 + e] * scale_log2;
        if (diag && key > qr0) v0 = -INFINITY;
        if (diag && key > qr1) v1 = -INFINITY;
        s[j][e] = v0;
        s[j][2 + e] = v1;
        mx0 = fmaxf(mx0, v0);
        mx1 = fmaxf(mx1, v1);
      }
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float c0 = exp2f(m0 - mx0), c1 = exp2f(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s[j][0] = exp2f(s[j][0] - mx0);
      s[j][1] = exp2f(s[j][1] - mx0);
      s[j][2] = exp2f(s[j][2] - mx1);
      s[j][3] = exp2f(s[j][3] - mx1);
      rs0 += s[j][0] + s[j][1];
      rs1 += s[j][2] + s[j][3];
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
#pragma unroll
    for (int i = 0; i < ND; ++i) {
      o[i][0] *= c0;
      o[i][1] *= c0;
      o[i][2] *= c1;
      o[i][3] *= c1;
    }
#pragma unroll
    for (int kk2 = 0; kk2 < 4; ++kk2) {
      uint32_t pa[4];
      acc_to_a(pa, s[2 * kk2], s[2 * kk2 + 1]);
#pragma unroll
      for (int n2 = 0; n2 < ND / 2; ++n2) {
        uint32_t bf[4];
        load_b_kn<P>(bf, v_s, kk2 * 16, n2 * 16, lane);
        mma16816(o[2 * n2], pa, bf[0], bf[1]);
        mma16816(o[2 * n2 + 1], pa, bf[2], bf[3]);
      }
    }
    __syncthreads();
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = 1.f / l0, inv1 = 1.f / l1;
  const long long row0 = static_cast<long long>(b) * S + qb * 64 + warp * 16 + g;
  __nv_bfloat16* o0 = out + row0 * (H * D) + h * D;
  __nv_bfloat16* o1 = o0 + 8LL * H * D;
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    *reinterpret_cast<uint32_t*>(o0 + i * 8 + 2 * t) = pack_bf16x2(o[i][0] * inv0, o[i][1] * inv0);
    *reinterpret_cast<uint32_t*>(o1 + i * 8 + 2 * t) = pack_bf16x2(o[i][2] * inv1, o[i][3] * inv1);
  }
  if (t == 0) {
    float* lrow = lse + (static_cast<long long>(b) * H + h) * S + qb * 64 + warp * 16 + g;
    lrow[0] = (m0 + log2f(l0)) / kLog2e;
    lrow[8] = (m1 + log2f(l1)) / kLog2e;
  }
}

// Dvec[b,h,s] = sum_d dO * O
template <int D>
__global__ void attn_bwd_pre_kernel(const __nv_bfloat16* __restrict__ out, const __nv_bfloat16* __restrict__ dout,
                                    float* __restrict__ dvec, const float* __restrict__ lse,
                                    float* __restrict__ lse2, int B, int S, int H) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(B) * S * H) return;
  const int h = static_cast<int>(idx % H);
  const long long tok = idx / H;
  const int s = static_cast<int>(tok % S), b = static_cast<int>(tok / S);
  const BF8* o = reinterpret_cast<const BF8*>(out + tok * H * D + h * D);
  const BF8* d = reinterpret_cast<const BF8*>(dout + tok * H * D + h * D);
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < D / 8; ++c) {
    float a[8], e[8];
    bf8_to_f(o[c], a);
    bf8_to_f(d[c], e);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += a[j] * e[j];
  }
  const long long vi = (static_cast<long long>(b) * H + h) * S + s;
  dvec[vi] = acc;
  if (lse2) lse2[vi] = lse[vi] * kLog2e;  // log2-domain LSE for the tcgen05 kernels
}

// Coalesced variant for D in {64, 128}: one warp per token row, lanes stream the
// row's 16-byte chunks; each head's D/8 chunks sit in a lane segment reduced by shuffles.
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_pre_rows_kernel(const __nv_bfloat16* __restrict__ out,
                                                                const __nv_bfloat16* __restrict__ dout,
                                                                float* __restrict__ dvec,
                                                                const float* __restrict__ lse,
                                                                float* __restrict__ lse2, int B, int S, int H) {
  constexpr int kSeg = D / 8;  // lanes per head (8 or 16)
  const long long tok = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (tok >= static_cast<long long>(B) * S) return;
  const int s = static_cast<int>(tok % S), b = static_cast<int>(tok / S);
  const BF8* o = reinterpret_cast<const BF8*>(out + tok * H * D);
  const BF8* d = reinterpret_cast<const BF8*>(dout + tok * H * D);
  const int nit = H * kSeg / 32;
  for (int it = 0; it < nit; ++it) {
    const int c = it * 32 + lane;
    float a[8], e[8], acc = 0.f;
    bf8_to_f(o[c], a);
    bf8_to_f(d[c], e);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += a[j] * e[j];
#pragma unroll
    for (int off = kSeg / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane % kSeg == 0) {
      const int h = c / kSeg;
      const long long vi = (static_cast<long long>(b) * H + h) * S + s;
      dvec[vi] = acc;
      if (lse2) lse2[vi] = lse[vi] * kLog2e;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(128) attn_bwd_dkdv_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                            const __nv_bfloat16* __restrict__ dout,
                                                            const float* __restrict__ lse,
                                                            const float* __restrict__ dvec,
                                                            __nv_bfloat16* __restrict__ dqkv, int S, int H,
                                                            float scale, float scale_log2) {
  constexpr int P = D + 8, KS = D / 16, ND = D / 8, BQ = 32;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sV = sK + 64 * P;
  __nv_bfloat16* sQ = sV + 64 * P;       // [2][BQ*P]
  __nv_bfloat16* sdO = sQ + 2 * BQ * P;  // [2][BQ*P]
  float* sL = reinterpret_cast<float*>(sdO + 2 * BQ * P);  // [2][BQ] lse*log2e
  float* sDv = sL + 2 * BQ;                                // [2][BQ]
  const int kb = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane / 4, t = lane % 4;
  const long long ld = 3LL * H * D, ldo = static_cast<long long>(H) * D;
  const long long tok0 = static_cast<long long>(b) * S;
  const __nv_bfloat16* gq = qkv + tok0 * ld + h * D;
  const __nv_bfloat16* gk = gq + H * D + kb * 64LL * ld;
  const __nv_bfloat16* gv = gk + H * D;
  const __nv_bfloat16* gdo = dout + tok0 * ldo + h * D;
  const float* gl = lse + (static_cast<long long>(b) * H + h) * S;
  const float* gd = dvec + (static_cast<long long>(b) * H + h) * S;

  auto load_q = [&](int qt, int buf) {
    load_tile<D, P>(sQ + buf * BQ * P, gq + qt * BQ * ld, ld, BQ);
    load_tile<D, P>(sdO + buf * BQ * P, gdo + qt * BQ * ldo, ldo, BQ);
    if (threadIdx.x < BQ) {
      sL[buf * BQ + threadIdx.x] = gl[qt * BQ + threadIdx.x] * kLog2e;
      sDv[buf * BQ + threadIdx.x] = gd[qt * BQ + threadIdx.x];
    }
  };
  load_tile<D, P>(sK, gk, ld, 64);
  load_tile<D, P>(sV, gv, ld, 64);
  const int qt0 = kb * 64 / BQ, nqt = S / BQ;
  load_q(qt0, 0);
  cp_commit();

  float dk[ND][4], dv[ND][4];
#pragma unroll
  for (int i = 0; i < ND; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int key0 = kb * 64 + warp * 16 + g, key1 = key0 + 8;

  for (int qt = qt0; qt < nqt; ++qt) {
    const int buf = (qt - qt0) & 1;
    if (qt + 1 < nqt) {
      __syncthreads();  // sL/sDv of the other buffer are free
      load_q(qt + 1, buf ^ 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const __nv_bfloat16* q_s = sQ + buf * BQ * P;
    const __nv_bfloat16* do_s = sdO + buf * BQ * P;
    const float* l_s = sL + buf * BQ;
    const float* d_s = sDv + buf * BQ;
    // S^T = K Q^T : 16 keys x 32 queries (4 n-blocks)
    float st[4][4], dpt[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[j][e] = dpt[j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      uint32_t ka[4], va[4];
      load_a<P>(ka, sK, warp * 16, kk * 16, lane);
      load_a<P>(va, sV, warp * 16, kk * 16, lane);
#pragma unroll
      for (int j2 = 0; j2 < 2; ++j2) {
        uint32_t bq[4], bd[4];
        load_b_nk<P>(bq, q_s, j2 * 16, kk * 16, lane);
        load_b_nk<P>(bd, do_s, j2 * 16, kk * 16, lane);
        mma16816(st[2 * j2], ka, bq[0], bq[1]);
        mma16816(st[2 * j2 + 1], ka, bq[2], bq[3]);
        mma16816(dpt[2 * j2], va, bd[0], bd[1]);
        mma16816(dpt[2 * j2 + 1], va, bd[2], bd[3]);
      }
    }
    // P^T and dS^T
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int ql = j * 8 + 2 * t + e;
        const int q = qt * BQ + ql;
        float p0 = exp2f(st[j][e] * scale_log2 - l_s[ql]);
        float p1 = exp2f(st[j][2 + e] * scale_log2 - l_s[ql]);
        if (q < key0) p0 = 0.f;
        if (q < key1) p1 = 0.f;
        st[j][e] = p0;
        st[j][2 + e] = p1;
        dpt[j][e] = p0 * (dpt[j][e] - d_s[ql]);
        dpt[j][2 + e] = p1 * (dpt[j][2 + e] - d_s[ql]);
      }
    }
    // dV += P^T dO ; dK += dS^T Q   (k = 32 queries -> 2 k-steps)
#pragma unroll
    for (int kq = 0; kq < 2; ++kq) {
      uint32_t pa[4], sa[4];
      acc_to_a(pa, st[2 * kq], st[2 * kq + 1]);
      acc_to_a(sa, dpt[2 * kq], dpt[2 * kq + 1]);
#pragma unroll
      for (int n2 = 0; n2 < ND / 2; ++n2) {
        uint32_t bd[4], bq[4];
        load_b_kn<P>(bd, do_s, kq * 16, n2 * 16, lane);
        load_b_kn<P>(bq, q_s, kq * 16, n2 * 16, lane);
        mma16816(dv[2 * n2], pa, bd[0], bd[1]);
        mma16816(dv[2 * n2 + 1], pa, bd[2], bd[3]);
        mma16816(dk[2 * n2], sa, bq[0], bq[1]);
        mma16816(dk[2 * n2 + 1], sa, bq[2], bq[3]);
      }
    }
  }
  const long long r0 = tok0 + key0;
  __nv_bfloat16* dk0 = dqkv + r0 * ld + H * D + h * D;
  __nv_bfloat16* dk1 = dk0 + 8 * ld;
  __nv_bfloat16* dv0 = dk0 + H * D;
  __nv_bfloat16* dv1 = dv0 + 8 * ld;
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    *reinterpret_cast<uint32_t*>(dk0 + i * 8 + 2 * t) = pack_bf16x2(dk[i][0] * scale, dk[i][1] * scale);
    *reinterpret_cast<uint32_t*>(dk1 + i * 8 + 2 * t) = pack_bf16x2(dk[i][2] * scale, dk[i][3] * scale);
    *reinterpret_cast<uint32_t*>(dv0 + i * 8 + 2 * t) = pack_bf16x2(dv[i][0], dv[i][1]);
    *reinterpret_cast<uint32_t*>(dv1 + i * 8 + 2 * t) = pack_bf16x2(dv[i][2], dv[i][3]);
  }
}

template <int D>
__global__ void __launch_bounds__(128) attn_bwd_dq_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                          const __nv_bfloat16* __restrict__ dout,
                                                          const float* __restrict__ lse,
                                                          const float* __restrict__ dvec,
                                                          __nv_bfloat16* __restrict__ dqkv, int S, int H, float scale,
                                                          float scale_log2) {
  constexpr int P = D + 8, KS = D / 16, ND = D / 8, BK = 32;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sdO = sQ + 64 * P;
  __nv_bfloat16* sK = sdO + 64 * P;     // [2][BK*P]
  __nv_bfloat16* sV = sK + 2 * BK * P;  // [2][BK*P]
  const int qb = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane / 4, t = lane % 4;
  const long long ld = 3LL * H * D, ldo = static_cast<long long>(H) * D;
  const long long tok0 = static_cast<long long>(b) * S;
  const __nv_bfloat16* gq = qkv + (tok0 + qb * 64) * ld + h * D;
  const __nv_bfloat16* gk = qkv + tok0 * ld + H * D + h * D;
  const __nv_bfloat16* gv = gk + H * D;
  const __nv_bfloat16* gdo = dout + (tok0 + qb * 64) * ldo + h * D;
  const int q0 = qb * 64 + warp * 16 + g, q1 = q0 + 8;
  const float* gl = lse + (static_cast<long long>(b) * H + h) * S;
  const float* gd = dvec + (static_cast<long long>(b) * H + h) * S;
  const float lq0 = gl[q0] * kLog2e, lq1 = gl[q1] * kLog2e;
  const float dq0v = gd[q0], dq1v = gd[q1];

  load_tile<D, P>(sQ, gq, ld, 64);
  load_tile<D, P>(sdO, gdo, ldo, 64);
  load_tile<D, P>(sK, gk, ld, BK);
  load_tile<D, P>(sV, gv, ld, BK);
  cp_commit();

  float dq[ND][4];
#pragma unroll
  for (int i = 0; i < ND; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
  const int nkt = (qb * 64 + 64) / BK;
  for (int kt = 0; kt < nkt; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nkt) {
      load_tile<D, P>(sK + (buf ^ 1) * BK * P, gk + (kt + 1) * BK * ld, ld, BK);
      load_tile<D, P>(sV + (buf ^ 1) * BK * P, gv + (kt + 1) * BK * ld, ld, BK);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const __nv_bfloat16* k_s = sK + buf * BK * P;
    const __nv_bfloat16* v_s = sV + buf * BK * P;
    float s[4][4], dp[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[j][e] = dp[j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      uint32_t qa[4], da[4];
      load_a<P>(qa, sQ, warp * 16, kk * 16, lane);
      load_a<P>(da, sdO, warp * 16, kk * 16, lane);
#pragma unroll
      for (int j2 = 0; j2 < 2; ++j2) {
        uint32_t bk[4], bv[4];
        load_b_nk<P>(bk, k_s, j2 * 16, kk * 16, lane);
        load_b_nk<P>(bv, v_s, j2 * 16, kk * 16, lane);
        mma16816(s[2 * j2], qa, bk[0], bk[1]);
        mma16816(s[2 * j2 + 1], qa, bk[2], bk[3]);
        mma16816(dp[2 * j2], da, bv[0], bv[1]);
        mma16816(dp[2 * j2 + 1], da, bv[2], bv[3]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = kt * BK + j * 8 + 2 * t + e;
        float p0 = exp2f(s[j][e] * scale_log2 - lq0);
        float p1 = exp2f(s[j][2 + e] * scale_log2 - lq1);
        if (key > q0) p0 = 0.f;
        if (key > q1) p1 = 0.f;
        s[j][e] = p0 * (dp[j][e] - dq0v);
        s[j][2 + e] = p1 * (dp[j][2 + e] - dq1v);
      }
    }
#pragma unroll
    for (int kk2 = 0; kk2 < 2; ++kk2) {
      uint32_t sa[4];
      acc_to_a(sa, s[2 * kk2], s[2 * kk2 + 1]);
#pragma unroll
      for (int n2 = 0; n2 < ND / 2; ++n2) {
        uint32_t bk[4];
        load_b_kn<P>(bk, k_s, kk2 * 16, n2 * 16, lane);
        mma16816(dq[2 * n2], sa, bk[0], bk[1]);
        mma16816(dq[2 * n2 + 1], sa, bk[2], bk[3]);
      }
    }
    __syncthreads();
  }
  __nv_bfloat16* d0 = dqkv + (tok0 + q0) * ld + h * D;
  __nv_bfloat16* d1 = d0 + 8 * ld;
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    *reinterpret_cast<uint32_t*>(d0 + i * 8 + 2 * t) = pack_bf16x2(dq[i][0] * scale, dq[i][1] * scale);
    *reinterpret_cast<uint32_t*>(d1 + i * 8 + 2 * t) = pack_bf16x2(dq[i][2] * scale, dq[i][3] * scale);
  }
}

template <int D>
int fwd_launch(const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, int B, int S, int H, cudaStream_t s) {
  constexpr int P = D + 8;
  const int smem = (64 * P + 4 * 64 * P) * 2;
  auto k = attn_fwd_kernel<D>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const float scale_log2 = kLog2e / sqrtf(static_cast<float>(D));
  k<<<dim3(S / 64, H, B), 128, smem, s>>>(qkv, out, lse, S, H, scale_log2);
  return check_launch("attention_fwd");
}

template <int D>
int bwd_launch(const __nv_bfloat16* qkv, const __nv_bfloat16* out, const __nv_bfloat16* dout, const float* lse,
               __nv_bfloat16* dqkv, float* dvec, int B, int S, int H, cudaStream_t s) {
  constexpr int P = D + 8;
  const long long rows = static_cast<long long>(B) * S * H;
  const bool tc = attention_tc_supported(S, D);
  float* lse2 = tc ? dvec + rows : nullptr;
  if ((D == 64 || D == 128) && (H * D / 8) % 32 == 0) {
    const long long threads = static_cast<long long>(B) * S * 32;
    attn_bwd_pre_rows_kernel<D><<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(out, dout, dvec, lse,
                                                                                          lse2, B, S, H);
  } else {
    attn_bwd_pre_kernel<D><<<static_cast<unsigned>((rows + 255) / 256), 256, 0, s>>>(out, dout, dvec, lse, lse2,
                                                                                    B, S, H);
  }
  if (tc) {
    if (int rc = check_launch("attention_bwd_pre")) return rc;
    return attention_bwd_tc(qkv, dout, lse2, dvec, dqkv, B, S, H, D, s);
  }
  const float scale = 1.f / sqrtf(static_cast<float>(D));
  const float scale_log2 = scale * kLog2e;
  const int smem_kv = (2 * 64 * P + 4 * 32 * P) * 2 + 4 * 32 * 4;
  auto k1 = attn_bwd_dkdv_kernel<D>;
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv);
  k1<<<dim3(S / 64, H, B), 128, smem_kv, s>>>(qkv, dout, lse, dvec, dqkv, S, H, scale, scale_log2);
  const int smem_q = (2 * 64 * P + 4 * 32 * P) * 2;
  auto k2 = attn_bwd_dq_kernel<D>;
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q);
  k2<<<dim3(S / 64, H, B), 128, smem_q, s>>>(qkv, dout, lse, dvec, dqkv, S, H, scale, scale_log2);
  return check_launch("attention_bwd", 3);
}

}  // namespace

int attention_fwd(const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, int B, int S, int H, int D,
                  cudaStream_t s) {
  if (S % 64) return set_error("attention: seq must be a multiple of 64", kValidation);
  if (attention_tc_supported(S, D)) return attention_fwd_tc(qkv, out, lse, B, S, H, D, s);
  switch (D) {
    case 64: return fwd_launch<64>(qkv, out, lse, B, S, H, s);
    case 96: return fwd_launch<96>(qkv, out, lse, B, S, H, s);
    case 112: return fwd_launch<112>(qkv, out, lse, B, S, H, s);
    case 128: return fwd_launch<128>(qkv, out, lse, B, S, H, s);
  }
  return set_error("attention: head_dim must be 64, 96, 112 or 128", kValidation);
}

size_t attention_bwd_workspace(int B, int S, int H) { return 2 * static_cast<size_t>(B) * S * H * sizeof(float); }

int attention_bwd(const __nv_bfloat16* qkv, const __nv_bfloat16* out, const __nv_bfloat16* dout, const float* lse,
                  __nv_bfloat16* dqkv, float* workspace, int B, int S, int H, int D, cudaStream_t s) {
  if (S % 64) return set_error("attention: seq must be a multiple of 64", kValidation);
  switch (D) {
    case 64: return bwd_launch<64>(qkv, out, dout, lse, dqkv, workspace, B, S, H, s);
    case 96: return bwd_launch<96>(qkv, out, dout, lse, dqkv, workspace, B, S, H, s);
    case 112: return bwd_launch<112>(qkv, out, dout, lse, dqkv, workspace, B, S, H, s);
    case 128: return bwd_launch<128>(qkv, out, dout, lse, dqkv, workspace, B, S, H, s);
  }
  return set_error("attention: head_dim must be 64, 96, 112 or 128", kValidation);
}

}  // namespace lynx
