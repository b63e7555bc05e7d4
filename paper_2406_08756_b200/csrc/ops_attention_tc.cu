// Causal attention on tcgen05 tensor cores (head_dim 64 / 96 / 112 / 128, seq % 128 == 0).
// A head of D columns occupies ceil(D / 64) 128-B swizzle atoms in shared memory (the last atom
// of D = 96 / 112 is loaded whole by TMA and only its first D % 64 columns are read: QK^T runs
// D / 16 K steps, the D-wide MMAs have N = D); epilogues move D columns in 32 / 16-column pieces.
//
// Same contract and layouts as ops_attention.cu (qkv [T, 3*H*D] = [Q|K|V],
// out [T, H*D], lse [B, H, S] natural log; backward writes dQ|dK|dV with the
// qkv layout, deterministically). Every CTA is warp-specialised:
//   warp 0      TMA producer (cp.async.bulk.tensor, 128-B swizzled tiles),
//   warp 1      single-thread tcgen05.mma issuer, completion via tcgen05.commit,
//   warp 2      TMEM allocator (512 columns),
//   warps 4..7  "row" warps: one thread per TMEM lane (= one tile row) doing
//               the softmax / gradient elementwise work between the MMAs and
//               the epilogue.
// The row warps hand bf16 P / dS tiles to the tensor core through tensor
// memory: they overwrite the fp32 S / dP columns they just read with packed
// bf16 pairs (tcgen05.st) and the MMA reads its A operand from TMEM
// (tcgen05.mma [d], [a_tmem], b_desc) — no shared-memory round trip and no
// generic -> async proxy fence on the row warps' critical path.
//
// Forward  (per 128-query tile, 128-key tiles double-buffered):
//   S_j = Q K_j^T -> TMEM (2 buffers, S_{j+1} runs while softmax j works),
//   P_j = exp2(S_j*c - m) -> smem, O += P_j V_j (TMEM accumulator).
//   Online softmax with lazy rescaling: O / l are rescaled only when a warp's
//   running max grows by more than 2^8 (P stays <= 256, exact in fp32 sums).
// Backward dK/dV (per 128-key tile, 64-query tiles double-buffered):
//   S^T = K Q^T, dP^T = V dO^T -> TMEM; P^T, dS^T = P^T o (dP^T - D) -> smem;
//   dV += P^T dO, dK += dS^T Q (TMEM accumulators, scaled once at the end).
// Backward dQ (per 128-query tile, 64-key tiles double-buffered):
//   S = Q K^T, dP = dO V^T -> TMEM; dS -> smem; dQ += dS K.
// dQ is its own kernel (7 tile MMAs per tile pair instead of 5) so that no
// gradient is accumulated with atomics: results are bit-reproducible.
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "lynx_ops_internal.h"

namespace lynx {
namespace gemm {
bool make_map(CUtensorMap* m, const void* base, long long inner, long long outer, long long ld, int box_inner,
              int box_outer);
int num_sms();
}
namespace attn_tc {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescale = 8.f;  // log2 units
constexpr int kAtom = 128;       // bytes per swizzled row (64 bf16)
constexpr int kDefaultPoly = 0;  // see poly_every()
constexpr int kDefaultBwdWG = 2;  // see bwd_warpgroups(): 4 measured no faster (profiles/r02_attention.md)

LYNX_DEV void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
LYNX_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
LYNX_DEV void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
LYNX_DEV void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// kCols consecutive 32-bit TMEM columns of this thread's lane (16 or 32).
template <int kCols>
LYNX_DEV void tmem_ld_cols(uint32_t taddr, uint32_t* r) {
  if constexpr (kCols == 32) tmem_ld32(taddr, r);
  else tmem_ld16(taddr, r);
}
template <int kCols>
LYNX_DEV void tmem_st_cols(uint32_t taddr, const uint32_t* r) {
  if constexpr (kCols == 16) tmem_st16(taddr, r);
  else tmem_st8(taddr, r);
}
// Row-warpgroup split of a 64-column (query or key) tile: warpgroup wg of kWG owns columns
// [wg * 64 / kWG, (wg + 1) * 64 / kWG) and packs its bf16 results (half as many 32-bit columns) at the
// start of that range — never into columns another warpgroup still reads. K step kk (16 columns) of
// the A-from-TMEM MMA then sits at:
template <int kWG>
LYNX_DEV constexpr uint32_t packed_col(int kk) {
  constexpr int CW = 64 / kWG;
  return static_cast<uint32_t>((16 * kk / CW) * CW + (16 * kk % CW) / 2);
}

// D[tmem] (+)= A[tmem] * B[smem]^T: A (128 rows x 16 K, bf16 pairs packed per 32-bit TMEM cell,
// one row per lane, 8 columns per K step) is read from tensor memory, so a row warp can hand
// its P / dS tile to the tensor core with tcgen05.st — no shared-memory round trip and no
// generic -> async proxy fence.
LYNX_DEV void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t desc_b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(desc_b), "r"(idesc), "r"(accumulate));
}

// 1-D bulk copy global -> shared, completing on an mbarrier (16-B aligned, size % 16 == 0).
LYNX_DEV void bulk_load(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

LYNX_DEV uint8_t* align1k(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~static_cast<uintptr_t>(1023));
}

// K-major operand whose rows are 128-B swizzled atoms of `atom_bytes` (rows x 128 B);
// K step kk (16 elements) lives in atom kk/4 at +32 B per step.
LYNX_DEV uint64_t kmaj(uint32_t base, int kk, uint32_t atom_bytes) {
  return umma_desc_sw128(base + (kk >> 2) * atom_bytes + (kk & 3) * 32, 16, 1024);
}
// MN-major operand stored [K rows][64-element MN atoms of atom_bytes]; K step kk = 16 rows.
LYNX_DEV uint64_t mnmaj(uint32_t base, int kk, uint32_t atom_bytes) {
  return umma_desc_sw128(base + kk * 2048, atom_bytes, 1024);
}

// 4 consecutive fp32 from shared memory.
LYNX_DEV float4 lds128(const void* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

LYNX_DEV float u2f(uint32_t v) { return __uint_as_float(v); }
// MUFU.EX2 without the denormal-range fix-up exp2f carries (arguments here are <= 8; underflow -> 0).
LYNX_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA / ALU pipes (no MUFU): round-to-nearest split x = j + f by the 1.5 * 2^23 trick,
// 2^f by a cubic fitted on [-0.5, 0.5] (relative error < 1.2e-4, far below the bf16 rounding of P),
// 2^j added to the exponent bits. x is clamped at -125 (ex2.approx.ftz flushes below -126 to 0; the
// clamped value contributes < 2^-125 to sums of terms >= 1). Used for a fixed share of the softmax
// exponentials so that the MUFU and FMA pipes share the row warps' work.
LYNX_DEV float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05459282f, f, 0.24221784f), f, 0.6933686f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}

// Columns [c0, c1) (multiples of 16) of this thread's TMEM lane, in 32- then 16-column pieces:
// f(col, values, count) sees the fp32 bits of `count` consecutive columns starting at `col`.
template <class F>
LYNX_DEV void tmem_cols(uint32_t taddr, int c0, int c1, F&& f) {
  int c = c0;
  for (; c + 32 <= c1; c += 32) {
    uint32_t o[32];
    tmem_ld32(taddr + c, o);
    tmem_ld_wait();
    f(c, o, 32);
  }
  if (c < c1) {
    uint32_t o[32];
    tmem_ld16(taddr + c, o);
    tmem_ld_wait();
    f(c, o, 16);
  }
}

// Per-tile event timeline of CTA (0,0,0) for kernel tuning: build with -DLYNX_ATTN_TRACE
// (LYNX_BUILD_TRACE=1 python -m paper_2406_08756_b200.build); compiled out otherwise.
#ifdef LYNX_ATTN_TRACE
__device__ long long g_atrace[16][64];
#define ATRACE(tag, j)                                                              \
  do {                                                                              \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64)          \
      g_atrace[tag][j] = clock64();                                                 \
  } while (0)
#define ATRACE_DUMP(n)                                                              \
  do {                                                                              \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0)  \
      for (int t_ = 0; t_ < 16; ++t_)                                                \
        for (int j_ = 0; j_ < (n) && j_ < 64; ++j_)                                 \
          printf("T %d %d %lld\n", t_, j_, g_atrace[t_][j_]);                       \
  } while (0)
#else
#define ATRACE(tag, j) \
  do {                 \
  } while (0)
#define ATRACE_DUMP(n) \
  do {                 \
  } while (0)
#endif

// ============================================================== forward
template <int D>
struct FwdL {
  static constexpr int kAtoms = (D + 63) / 64;
  static constexpr int kTile = 128 * kAtoms * 64 * 2;  // one 128-row x D tile (ceil(D/64) atoms of 16 KB)
  static constexpr int kQ = 0, kK = kTile, kV = 3 * kTile, kBar = 5 * kTile;  // P lives in TMEM
  static constexpr int kBytes = kBar + 128 + 1024;
};

template <int D, int kPoly>  // kPoly > 0: every kPoly-th softmax exponential on the FMA pipe (ex2_poly)
__global__ void __launch_bounds__(256, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap map_qkv, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ lse, int S, int H, float scale_log2) {
  using L = FwdL<D>;
  constexpr int kA = L::kAtoms;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
  // K and V stages have their own barriers: K_j is released once S_j is computed, so the
  // load of K_{j+2} overlaps PV_j instead of waiting for it.
  // p_full is double-buffered like S: with one barrier, a row warp that ran ahead to tile j+1 (S(j+1)
  // is issued early) arrived again before a slower warp's tile-j arrival, completed tile j's phase
  // early and let PV(j) read that warp's stale P rows (a rare, timing-dependent race).
  uint64_t *q_full = bar, *k_full = bar + 1, *k_empty = bar + 3, *v_full = bar + 5, *v_empty = bar + 7,
           *s_full = bar + 9, *p_full = bar + 11, *pv_done = bar + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 14);
  const int qb = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n = qb + 1, HD = H * D, row0 = b * S;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
      mbar_init(s_full + i, 1);
      mbar_init(p_full + i, 128);
    }
    mbar_init(pv_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S buffers at columns 0 / 128, O at 256

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&map_qkv);
      mbar_arrive_expect_tx(q_full, L::kTile);
      for (int a = 0; a < kA; ++a)
        tma_load_2d(&map_qkv, q_full, smem + L::kQ + a * 16384, h * D + 64 * a, row0 + qb * 128, kEvictFirst);
      for (int j = 0; j < n; ++j) {
        const int st = j & 1;
        if (j >= 2) mbar_wait(k_empty + st, ((j >> 1) - 1) & 1);
        mbar_arrive_expect_tx(k_full + st, L::kTile);
        for (int a = 0; a < kA; ++a)
          tma_load_2d(&map_qkv, k_full + st, smem + L::kK + st * L::kTile + a * 16384, HD + h * D + 64 * a,
                      row0 + j * 128, kEvictLast);
        if (j >= 2) mbar_wait(v_empty + st, ((j >> 1) - 1) & 1);
        mbar_arrive_expect_tx(v_full + st, L::kTile);
        for (int a = 0; a < kA; ++a)
          tma_load_2d(&map_qkv, v_full + st, smem + L::kV + st * L::kTile + a * 16384, 2 * HD + h * D + 64 * a,
                      row0 + j * 128, kEvictLast);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idS = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idO = umma_idesc_bf16(128, D, false, true);
      const uint32_t sQ = smem_u32(smem + L::kQ), sK = smem_u32(smem + L::kK), sV = smem_u32(smem + L::kV);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        mbar_wait(k_full + st, (j >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16(tmem + st * 128, kmaj(sQ, kk, 16384), kmaj(sK + st * L::kTile, kk, 16384), idS, kk > 0);
        umma_commit(s_full + st);
        umma_commit(k_empty + st);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      if (n > 1) issue_s(1);
      for (int j = 0; j < n; ++j) {
        const int st = j & 1;
        mbar_wait(v_full + st, (j >> 1) & 1);
        mbar_wait(p_full + st, (j >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_f16_ts(tmem + 256, tmem + st * 128 + kk * 8, mnmaj(sV + st * L::kTile, kk, 16384), idO,
                      (j | kk) != 0);  // A = P(j), packed bf16 over S(j) in TMEM
        umma_commit(pv_done);
        umma_commit(v_empty + st);
        if (j + 2 < n) issue_s(j + 2);
      }
    }
  } else if (warp >= 4) {
    const int r = (warp - 4) * 32 + lane;
    const uint32_t lanes = static_cast<uint32_t>((warp - 4) * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < n; ++j) {
      const int st = j & 1;
      mbar_wait(s_full + st, (j >> 1) & 1);
      tc_fence_after();
      float x[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tmem + lanes + st * 128 + c * 32, reinterpret_cast<uint32_t*>(x + c * 32));
      tmem_ld_wait();
      if (j == qb) {  // diagonal tile: causal mask (warp-uniform branch)
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i > r) x[i] = -INFINITY;
      }
      // 8 independent max / sum chains: a single 128-long dependent chain costs ~4 cycles per
      // element on the one row warp each SM sub-partition runs.
      float mv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mv[i] = x[i];
#pragma unroll
      for (int i = 8; i < 128; ++i) mv[i & 7] = fmaxf(mv[i & 7], x[i]);
      const float mt = fmaxf(fmaxf(fmaxf(mv[0], mv[1]), fmaxf(mv[2], mv[3])), fmaxf(fmaxf(mv[4], mv[5]), fmaxf(mv[6], mv[7])));
      const float m_new = fmaxf(m_run, mt * scale_log2);
      const bool need = __any_sync(0xffffffffu, m_new > m_run + kRescale);
      float corr = 1.f;
      if (need) {
        corr = exp2f(m_run - m_new);
        m_run = m_new;
      }
      float rv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < 128; ++i) {
        const float a = fmaf(x[i], scale_log2, -m_run);
        x[i] = (kPoly > 0 && i % (kPoly > 0 ? kPoly : 1) == (kPoly > 0 ? kPoly : 1) - 1) ? ex2_poly(a) : ex2(a);
        rv[i & 7] += x[i];
      }
      const float rs = ((rv[0] + rv[1]) + (rv[2] + rv[3])) + ((rv[4] + rv[5]) + (rv[6] + rv[7]));
      l_run = l_run * corr + rs;
      // O is rescaled (rarely) after PV(j-1) completes. P(j) needs no wait: PV(j-2), the last
      // reader of TMEM buffer st, completed before S(j) (tensor-pipe order). pv_done can be at
      // most at phase j here (PV(j) needs this tile's P), so skipping waits is safe.
      if (j > 0 && need) {
        mbar_wait(pv_done, (j - 1) & 1);
        tc_fence_after();
        if (need) {
          tmem_cols(tmem + lanes + 256, 0, D, [&](int c, uint32_t* o, int cnt) {
            for (int i = 0; i < cnt; ++i) o[i] = __float_as_uint(u2f(o[i]) * corr);
            if (cnt == 32)
              tmem_st32(tmem + lanes + 256 + c, o);
            else
              tmem_st16(tmem + lanes + 256 + c, o);
          });
          tmem_st_wait();
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t packed[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) packed[i] = pack_bf16x2(x[32 * c + 2 * i], x[32 * c + 2 * i + 1]);
        tmem_st16(tmem + lanes + st * 128 + c * 16, packed);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(p_full + st);
    }
    mbar_wait(pv_done, (n - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l_run;
    const int q = qb * 128 + r;
    BF8* orow = reinterpret_cast<BF8*>(out + static_cast<long long>(row0 + q) * HD + h * D);
    tmem_cols(tmem + lanes + 256, 0, D, [&](int c, const uint32_t* o, int cnt) {
      float f[32];
      for (int i = 0; i < cnt; ++i) f[i] = u2f(o[i]) * inv;
      for (int i = 0; i < cnt / 8; ++i) orow[c / 8 + i] = f_to_bf8(f + 8 * i);
    });
    lse[(static_cast<long long>(b) * H + h) * S + q] = (m_run + log2f(l_run)) / kLog2e;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ============================================================== forward, two query tiles per CTA
// Query tiles 2p and 2p+1 share each K / V tile; two softmax warpgroups (warps 4-7: tile 0, warps
// 8-11: tile 1) each own one tile's S / P and O in TMEM (S_t at columns 128 t, O_t at 256 + 128 t).
// The MMA warp ping-pongs: PV_0(j), S_0(j+1), PV_1(j), S_1(j+1) — while one warpgroup's softmax of
// tile j runs, the tensor core works for the other — so every SM sub-partition has two softmax warps
// to hide the TMEM-load / MUFU latencies that bound the one-tile kernel (tensor pipe ~39 % there).
// Per-row arithmetic, warp-to-row mapping and the lazy-rescale decisions are those of
// attn_fwd_tc_kernel, so O and lse are bit-identical to it.
//
// Persistent (like the backward kernels): grid = min(work items, SMs); work item w = (tile pair, head,
// batch), head-major with the pair rotated by the head (dq_item). The K / V ring runs on across items;
// the next item's Q tiles are loaded as soon as the current item's last S MMAs completed; O leaves
// through a 16-KB shared-memory staging tile per warpgroup with coalesced stores.
template <int D>
struct Fwd2L {
  static constexpr int kTile = FwdL<D>::kTile;
  static constexpr int kQ = 0, kK = 2 * kTile, kV = 4 * kTile, kOut = 6 * kTile;  // kOut: 2 x 128 rows x 128 B
  static constexpr int kBar = kOut + 2 * 16384;
  static constexpr int kBytes = kBar + 256 + 1024;
  static_assert(kBytes <= 232448, "exceeds the 227 KB of shared memory per CTA");
};

struct FwdItem {
  int pair, h, b, n0, n1;  // n0 / n1: key tiles of query tile 2 pair / 2 pair + 1 (0: absent)
};
LYNX_DEV FwdItem fwd_item(int w, int np, int n_qt, int H) {
  const int hb = w / np;
  FwdItem it;
  it.pair = (w % np + hb) % np;
  it.h = hb % H;
  it.b = hb / H;
  it.n0 = 2 * it.pair + 1;
  it.n1 = 2 * it.pair + 1 < n_qt ? 2 * it.pair + 2 : 0;
  return it;
}

template <int D, int kPoly>  // kPoly: as attn_fwd_tc_kernel (every kPoly-th exponential on the FMA pipe)
__global__ void __launch_bounds__(384, 1)
    attn_fwd2_tc_kernel(const __grid_constant__ CUtensorMap map_qkv, __nv_bfloat16* __restrict__ out,
                        float* __restrict__ lse, int S, int H, int B, float scale_log2) {
  using L = Fwd2L<D>;
  constexpr int kA = FwdL<D>::kAtoms;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t *q_full = bar, *q_free = bar + 1, *k_full = bar + 2, *k_empty = bar + 4, *v_full = bar + 6,
           *v_empty = bar + 8, *s_full = bar + 10, *p_full = bar + 12, *pv_done = bar + 14,
           *p_full_b = bar + 16;  // s / p / pv: per tile; p_full: P columns 0-63, p_full_b: 64-127
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 18);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_qt = S / 128, np = (n_qt + 1) / 2, n_items = np * H * B;
  const int HD = H * D;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_free, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
      mbar_init(s_full + i, 1);
      mbar_init(p_full + i, 128);
      mbar_init(p_full_b + i, 128);
      mbar_init(pv_done + i, 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Register split by warpgroup (setmaxnreg, executed at the top of each role): the control warpgroup
  // (TMA, MMA, TMEM) gives registers to the two softmax warpgroups, whose 128-column rows need them:
  // 128 x 72 + 256 x 216 = the 168 x 384 the launch allocates.

  if (warp == 0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
    if (elect_one()) {
      tma_prefetch_desc(&map_qkv);
      int g = 0, k = 0;  // K / V tile counter over this CTA's items, item counter
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
        const FwdItem it = fwd_item(w, np, n_qt, H);
        const int row0 = it.b * S, nq = it.n1 ? 2 : 1, n = it.n1 ? it.n1 : it.n0;
        if (k > 0) mbar_wait(q_free, (k - 1) & 1);  // the previous item's last S MMAs completed
        mbar_arrive_expect_tx(q_full, nq * L::kTile);
        for (int t = 0; t < nq; ++t)
          for (int a = 0; a < kA; ++a)
            tma_load_2d(&map_qkv, q_full, smem + L::kQ + t * L::kTile + a * 16384, it.h * D + 64 * a,
                        row0 + (2 * it.pair + t) * 128, kEvictFirst);
        for (int j = 0; j < n; ++j, ++g) {
          const int st = g & 1;
          if (g >= 2) mbar_wait(k_empty + st, ((g >> 1) - 1) & 1);
          mbar_arrive_expect_tx(k_full + st, L::kTile);
          for (int a = 0; a < kA; ++a)
            tma_load_2d(&map_qkv, k_full + st, smem + L::kK + st * L::kTile + a * 16384, HD + it.h * D + 64 * a,
                        row0 + j * 128, kEvictLast);
          if (g >= 2) mbar_wait(v_empty + st, ((g >> 1) - 1) & 1);
          mbar_arrive_expect_tx(v_full + st, L::kTile);
          for (int a = 0; a < kA; ++a)
            tma_load_2d(&map_qkv, v_full + st, smem + L::kV + st * L::kTile + a * 16384, 2 * HD + it.h * D + 64 * a,
                        row0 + j * 128, kEvictLast);
        }
      }
    }
  } else if (warp == 1) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
    if (elect_one()) {
      constexpr uint32_t idS = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idO = umma_idesc_bf16(128, D, false, true);
      const uint32_t sQ = smem_u32(smem + L::kQ), sK = smem_u32(smem + L::kK), sV = smem_u32(smem + L::kV);
      int g = 0, k = 0, cp0 = 0, cp1 = 0;  // K / V tiles, items, P hand-offs of query tile 0 / 1
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
        const FwdItem it = fwd_item(w, np, n_qt, H);
        const int n0 = it.n0, n1 = it.n1, n = n1 ? n1 : n0;
        auto issue_s = [&](int t, int j) {  // S_t(j) = Q_t K_j^T
          const int st = (g + j) & 1;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            umma_f16(tmem + t * 128, kmaj(sQ + t * L::kTile, kk, 16384), kmaj(sK + st * L::kTile, kk, 16384), idS,
                     kk > 0);
          umma_commit(s_full + t);
          if (k == 0) ATRACE(t ? 7 : 0, j);
        };
        auto issue_pv = [&](int t, int j) {  // O_t += P_t(j) V_j, P packed bf16 over S_t in TMEM
          // in two halves: keys 0-63 as soon as the softmax handed them over, while it computes 64-127
          const int st = (g + j) & 1;
          const uint32_t ph = (t ? cp1 : cp0) & 1;
          if (t) ++cp1; else ++cp0;
          mbar_wait(p_full + t, ph);
          if (k == 0) ATRACE(t ? 6 : 1, j);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_f16_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, mnmaj(sV + st * L::kTile, kk, 16384), idO,
                        (j | kk) != 0);
          mbar_wait(p_full_b + t, ph);
          tc_fence_after();
#pragma unroll
          for (int kk = 4; kk < 8; ++kk)
            umma_f16_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, mnmaj(sV + st * L::kTile, kk, 16384), idO, 1u);
          umma_commit(pv_done + t);
        };
        auto wait_k = [&](int j) {
          mbar_wait(k_full + ((g + j) & 1), ((g + j) >> 1) & 1);
          tc_fence_after();
        };
        mbar_wait(q_full, k & 1);
        wait_k(0);
        issue_s(0, 0);
        if (n1 > 0) issue_s(1, 0);
        if (n == 1) umma_commit(q_free);
        umma_commit(k_empty + (g & 1));
        for (int j = 0; j < n; ++j) {
          const int st = (g + j) & 1;
          mbar_wait(v_full + st, ((g + j) >> 1) & 1);
          tc_fence_after();
          if (j < n0) issue_pv(0, j);
          if (j + 1 < n) wait_k(j + 1);
          if (j + 1 < n0) issue_s(0, j + 1);
          if (j < n1) issue_pv(1, j);
          umma_commit(v_empty + st);
          if (j + 1 < n1) issue_s(1, j + 1);
          if (j + 2 == n) umma_commit(q_free);  // the item's last S MMAs are issued: Q may be replaced
          if (j + 1 < n) umma_commit(k_empty + ((g + j + 1) & 1));
        }
        g += n;
      }
    }
  } else if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 216;");
    const int t = (warp - 4) / 4;  // query tile of this warpgroup (warp w reads TMEM lanes 32 (w % 4) ...)
    const int r = (warp % 4) * 32 + lane, tr = threadIdx.x - 128 - 128 * t;  // tile row, thread in warpgroup
    const uint32_t lanes = static_cast<uint32_t>((warp % 4) * 32) << 16;
    const uint32_t s_col = tmem + lanes + t * 128, o_col = tmem + lanes + 256 + t * 128;
    uint8_t* stg = smem + L::kOut + t * 16384;  // this warpgroup's O staging: 128 rows x 64 columns
    int c = 0, k = 0;                           // S_t tiles consumed, items
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
      const FwdItem it = fwd_item(w, np, n_qt, H);
      const int nt = t ? it.n1 : it.n0;
      if (nt == 0) continue;
      const int qb = 2 * it.pair + t;
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < nt; ++j, ++c) {
        mbar_wait(s_full + t, c & 1);
        if (k == 0 && warp % 4 == 0 && lane == 0) ATRACE(t ? 4 : 2, j);
        tc_fence_after();
        float x[128];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) tmem_ld32(s_col + cc * 32, reinterpret_cast<uint32_t*>(x + cc * 32));
        tmem_ld_wait();
        if (j == qb) {  // diagonal tile: causal mask (warp-uniform branch)
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i > r) x[i] = -INFINITY;
        }
        float mv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mv[i] = x[i];
#pragma unroll
        for (int i = 8; i < 128; ++i) mv[i & 7] = fmaxf(mv[i & 7], x[i]);
        const float mt =
            fmaxf(fmaxf(fmaxf(mv[0], mv[1]), fmaxf(mv[2], mv[3])), fmaxf(fmaxf(mv[4], mv[5]), fmaxf(mv[6], mv[7])));
        const float m_new = fmaxf(m_run, mt * scale_log2);
        const bool need = __any_sync(0xffffffffu, m_new > m_run + kRescale);
        float corr = 1.f;
        if (need) {
          corr = exp2f(m_run - m_new);
          m_run = m_new;
        }
        if (j > 0 && need) {  // O_t rescale after PV_t(j-1) completes (PV_t(j) needs this tile's P)
          mbar_wait(pv_done + t, (c - 1) & 1);
          tc_fence_after();
          tmem_cols(o_col, 0, D, [&](int col, uint32_t* o, int cnt) {
            for (int i = 0; i < cnt; ++i) o[i] = __float_as_uint(u2f(o[i]) * corr);
            if (cnt == 32)
              tmem_st32(o_col + col, o);
            else
              tmem_st16(o_col + col, o);
          });
          tmem_st_wait();
        }
        // P in two halves (keys 0-63, then 64-127), each handed to the MMA warp as soon as it is in TMEM;
        // per-element math and the row-sum chains are those of the one-tile kernel (bit-identical)
        float rv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int half = 0; half < 2; ++half) {
#pragma unroll
          for (int i = 64 * half; i < 64 * half + 64; ++i) {
            const float a = fmaf(x[i], scale_log2, -m_run);
            x[i] = (kPoly > 0 && i % (kPoly > 0 ? kPoly : 1) == (kPoly > 0 ? kPoly : 1) - 1) ? ex2_poly(a) : ex2(a);
            rv[i & 7] += x[i];
          }
#pragma unroll
          for (int cc = 2 * half; cc < 2 * half + 2; ++cc) {
            uint32_t packed[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) packed[i] = pack_bf16x2(x[32 * cc + 2 * i], x[32 * cc + 2 * i + 1]);
            tmem_st16(s_col + cc * 16, packed);
          }
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(half ? p_full_b + t : p_full + t);
        }
        const float rs = ((rv[0] + rv[1]) + (rv[2] + rv[3])) + ((rv[4] + rv[5]) + (rv[6] + rv[7]));
        l_run = l_run * corr + rs;
        if (k == 0 && warp % 4 == 0 && lane == 0) ATRACE(t ? 5 : 3, j);
      }
      mbar_wait(pv_done + t, (c - 1) & 1);
      tc_fence_after();
      // O_t / l -> bf16 through the staging tile (row r's 16-B chunk ch at r * 128 + (ch ^ (r % 8)) * 16),
      // 64 columns per round, then coalesced 16-B stores (8 threads per 128-B row piece). The next item's
      // first PV_t (which overwrites O_t) waits for this warpgroup's first P hand-off, i.e. after this.
      const float inv = 1.f / l_run;
      const long long orow0 = static_cast<long long>(it.b) * S + qb * 128;
      for (int c0 = 0; c0 < D; c0 += 64) {
        const int cw = D - c0 < 64 ? D - c0 : 64, nch = cw / 8;
        tmem_cols(o_col, c0, c0 + cw, [&](int col, const uint32_t* o, int cnt) {
          float f[32];
          for (int i = 0; i < cnt; ++i) f[i] = u2f(o[i]) * inv;
          for (int i = 0; i < cnt / 8; ++i)
            *reinterpret_cast<BF8*>(stg + r * 128 + ((((col - c0) / 8 + i) ^ (r & 7)) * 16)) = f_to_bf8(f + 8 * i);
        });
        asm volatile("bar.sync %0, 128;" ::"r"(2 + t) : "memory");
        for (int i = tr; i < 128 * nch; i += 128) {
          const int rr = i / nch, ch = i % nch;
          const BF8 v = *reinterpret_cast<const BF8*>(stg + rr * 128 + ((ch ^ (rr & 7)) * 16));
          reinterpret_cast<BF8*>(out + (orow0 + rr) * HD + it.h * D + c0)[ch] = v;
        }
        asm volatile("bar.sync %0, 128;" ::"r"(2 + t) : "memory");  // staging read: reusable
      }
      lse[(static_cast<long long>(it.b) * H + it.h) * S + qb * 128 + r] = (m_run + log2f(l_run)) / kLog2e;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  ATRACE_DUMP(16);
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ============================================================== forward, 64-key blocks, P apart from S
// The two-tile kernel's per-tile chain is serial: P_t(j) overwrites S_t(j) in TMEM, so S_t(j+1) can only
// be issued after PV_t(j) has read P_t(j), and each tile alternates ~2200 cycles of softmax with ~1100
// of its own MMAs (a clock64 trace: 3600-cycle period per 128 keys for 2048 cycles of tensor work).
// Here each tile keeps a separate P region: S_t (64 columns, one 64-key block), P_t (32 packed
// columns) and O_t (D columns) fit twice into 512 columns. A softmax warp releases S_t as soon as its
// tcgen05.ld completed, so S_t(j+1) runs while it computes P_t(j); every tile has its own MMA issuer
// thread (warps 1 and 3; tcgen05.commit tracks the issuing thread's MMAs), so neither tile's MMAs wait
// behind the other's. K / V blocks of 64 rows, 4-stage ring released by both issuers.
// Online softmax per 64-key block with the same lazy rescale rule as attn_fwd_tc_kernel.
template <int D>
struct Fwd3L {
  static constexpr int kAtoms = (D + 63) / 64;
  static constexpr int kQT = 128 * kAtoms * 64 * 2;  // Q tile, 128 rows
  static constexpr int kBT = 64 * kAtoms * 64 * 2;   // K or V block, 64 rows
  static constexpr int kStages = D <= 64 ? 8 : 4;
  static constexpr int kQ = 0, kK = 2 * kQT, kV = kK + kStages * kBT, kBar = kV + kStages * kBT;
  static constexpr int kBytes = kBar + 256 + 1024;
  static_assert(kBytes <= 232448, "exceeds the 227 KB of shared memory per CTA");
};

template <int D>
__global__ void __launch_bounds__(384, 1)
    attn_fwd3_tc_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                        __nv_bfloat16* __restrict__ out, float* __restrict__ lse, int S, int H, float scale_log2) {
  using L = Fwd3L<D>;
  constexpr int kA = L::kAtoms, NS = L::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t *q_full = bar, *kv_full = bar + 1, *kv_empty = kv_full + NS, *s_full = kv_empty + NS,
           *s_free = s_full + 2, *p_full = s_free + 2, *pv_done = p_full + 2;  // s / p / pv: one per tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);
  const int pair = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_qt = S / 128;
  const bool has1 = 2 * pair + 1 < n_qt;
  // 64-key blocks per tile: query tile qb attends blocks 0 .. 2 qb + 1
  const int n0 = 4 * pair + 2, n1 = has1 ? 4 * pair + 4 : 0, n = has1 ? n1 : n0;
  const int HD = H * D, row0 = b * S;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, has1 ? 2 : 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_free + i, 128);
      mbar_init(p_full + i, 128);
      mbar_init(pv_done + i, 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // TMEM: S_t at 64 t, P_t at 128 + 32 t, O_t at 256 + 128 t.
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (elect_one()) {
      mbar_arrive_expect_tx(q_full, (has1 ? 2 : 1) * L::kQT);
      for (int t = 0; t < (has1 ? 2 : 1); ++t)
        for (int a = 0; a < kA; ++a)
          tma_load_2d(&map_q, q_full, smem + L::kQ + t * L::kQT + a * 16384, h * D + 64 * a,
                      row0 + (2 * pair + t) * 128, kEvictFirst);
      for (int j = 0; j < n; ++j) {
        const int st = j % NS;
        if (j >= NS) mbar_wait(kv_empty + st, ((j / NS) - 1) & 1);
        mbar_arrive_expect_tx(kv_full + st, 2 * L::kBT);
        for (int a = 0; a < kA; ++a) {
          tma_load_2d(&map_kv, kv_full + st, smem + L::kK + st * L::kBT + a * 8192, HD + h * D + 64 * a,
                      row0 + j * 64, kEvictLast);
          tma_load_2d(&map_kv, kv_full + st, smem + L::kV + st * L::kBT + a * 8192, 2 * HD + h * D + 64 * a,
                      row0 + j * 64, kEvictLast);
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    const int t = warp == 3;
    const int nt = t ? n1 : n0;
    if (nt > 0 && elect_one()) {
      constexpr uint32_t idS = umma_idesc_bf16(128, 64, false, false);
      constexpr uint32_t idO = umma_idesc_bf16(128, D, false, true);
      const uint32_t sQ = smem_u32(smem + L::kQ + t * L::kQT), sK = smem_u32(smem + L::kK),
                     sV = smem_u32(smem + L::kV);
      const uint32_t s_tm = tmem + 64 * t, p_tm = tmem + 128 + 32 * t, o_tm = tmem + 256 + 128 * t;
      auto issue_pv = [&](int j) {  // O_t += P_t(j) V_j
        const int st = j % NS;
        mbar_wait(p_full + t, j & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_f16_ts(o_tm, p_tm + kk * 8, mnmaj(sV + st * L::kBT, kk, 8192), idO, (j | kk) != 0);
        umma_commit(pv_done + t);
        umma_commit(kv_empty + st);
      };
      mbar_wait(q_full, 0);
      for (int j = 0; j < nt; ++j) {
        const int st = j % NS;
        mbar_wait(kv_full + st, (j / NS) & 1);
        if (j > 0) mbar_wait(s_free + t, (j - 1) & 1);
        ATRACE(t ? 4 : 0, j);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16(s_tm, kmaj(sQ, kk, 16384), kmaj(sK + st * L::kBT, kk, 8192), idS, kk > 0);
        umma_commit(s_full + t);
        if (j > 0) issue_pv(j - 1);
        if (j > 0) ATRACE(t ? 5 : 1, j - 1);
      }
      issue_pv(nt - 1);
    }
  } else if (warp == 2) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    const int t = (warp - 4) / 4;
    if (t == 0 || has1) {
      const int qb = 2 * pair + t, nt = t ? n1 : n0;
      const int r = (warp % 4) * 32 + lane;
      const uint32_t lanes = static_cast<uint32_t>((warp % 4) * 32) << 16;
      const uint32_t s_col = tmem + lanes + 64 * t, p_col = tmem + lanes + 128 + 32 * t,
                     o_col = tmem + lanes + 256 + 128 * t;
      const int q = qb * 128 + r;
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < nt; ++j) {
        mbar_wait(s_full + t, j & 1);
        if (warp % 4 == 0 && lane == 0) ATRACE(t ? 6 : 2, j);
        tc_fence_after();
        float x[64];
        tmem_ld32(s_col, reinterpret_cast<uint32_t*>(x));
        tmem_ld32(s_col + 32, reinterpret_cast<uint32_t*>(x + 32));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(s_free + t);  // S_t(j + 1) may overwrite the block now
        if (j >= 2 * qb) {  // the two blocks that meet the diagonal (warp-uniform branch)
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (j * 64 + i > q) x[i] = -INFINITY;
        }
        float mv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mv[i] = x[i];
#pragma unroll
        for (int i = 8; i < 64; ++i) mv[i & 7] = fmaxf(mv[i & 7], x[i]);
        const float mt =
            fmaxf(fmaxf(fmaxf(mv[0], mv[1]), fmaxf(mv[2], mv[3])), fmaxf(fmaxf(mv[4], mv[5]), fmaxf(mv[6], mv[7])));
        const float m_new = fmaxf(m_run, mt * scale_log2);
        const bool need = __any_sync(0xffffffffu, m_new > m_run + kRescale);
        float corr = 1.f;
        if (need) {
          corr = exp2f(m_run - m_new);
          m_run = m_new;
        }
        float rv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          x[i] = ex2(fmaf(x[i], scale_log2, -m_run));
          rv[i & 7] += x[i];
        }
        const float rs = ((rv[0] + rv[1]) + (rv[2] + rv[3])) + ((rv[4] + rv[5]) + (rv[6] + rv[7]));
        l_run = l_run * corr + rs;
        uint32_t packed[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) packed[i] = pack_bf16x2(x[2 * i], x[2 * i + 1]);
        if (j > 0) {  // PV_t(j-1) read P_t(j-1) and wrote O_t
          mbar_wait(pv_done + t, (j - 1) & 1);
          tc_fence_after();
          if (need) {
            tmem_cols(o_col, 0, D, [&](int c, uint32_t* o, int cnt) {
              for (int i = 0; i < cnt; ++i) o[i] = __float_as_uint(u2f(o[i]) * corr);
              if (cnt == 32)
                tmem_st32(o_col + c, o);
              else
                tmem_st16(o_col + c, o);
            });
          }
        }
        tmem_st32(p_col, packed);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full + t);
        if (warp % 4 == 0 && lane == 0) ATRACE(t ? 7 : 3, j);
      }
      mbar_wait(pv_done + t, (nt - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l_run;
      BF8* orow = reinterpret_cast<BF8*>(out + static_cast<long long>(row0 + q) * HD + h * D);
      tmem_cols(o_col, 0, D, [&](int c, const uint32_t* o, int cnt) {
        float f[32];
        for (int i = 0; i < cnt; ++i) f[i] = u2f(o[i]) * inv;
        for (int i = 0; i < cnt / 8; ++i) orow[c / 8 + i] = f_to_bf8(f + 8 * i);
      });
      lse[(static_cast<long long>(b) * H + h) * S + q] = (m_run + log2f(l_run)) / kLog2e;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  ATRACE_DUMP(n);
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ============================================================== forward, CTA pair (cta_group::2), D = 128
// Two CTAs of a cluster (two SMs) own query tiles 2p (rank 0) and 2p + 1 (rank 1); the leader issues
// M = 256 MMAs over both: S = Q K_j^T with each CTA's Q tile as its half of A and each CTA holding half
// of K_j's 128 keys (B is split along N), O += P V_j with P from each CTA's TMEM and each CTA holding
// half of V_j's D columns. Per CTA this halves the K / V shared-memory traffic of an S MMA (6 KB per
// 64-cycle instruction instead of 8 KB per 64 cycles) and frees TMEM: two 128-column S buffers, a
// separate 64-column P and the 128-column O fit in 512, so S(j+1) is computed while the softmax of S(j)
// runs and P(j) never overwrites S — the per-tile softmax -> PV -> S chain of the two-tile kernel is
// gone. Each CTA's 128 x 128 score tile is split over two softmax warpgroups (64 key columns each,
// row max exchanged through shared memory), so each SM sub-partition has two warps issuing
// exponentials: 1024 MUFU cycles per tile per SM against 1024 tensor cycles.
// Query tile 2p needs one key tile less than 2p + 1: rank 0 writes P = 0 for it.
struct Fwd4L {
  static constexpr int kQT = 128 * 128 * 2;   // Q tile: 2 atoms of 16 KB
  static constexpr int kKH = 64 * 128 * 2;    // K half: 64 keys x 128 columns (2 atoms of 8 KB)
  static constexpr int kVH = 128 * 64 * 2;    // V half: 128 keys x 64 columns (1 atom of 16 KB)
  static constexpr int kStage = kKH + kVH;
  static constexpr int kStages = 4;
  static constexpr int kQ = 0, kKV = kQT, kOut = kKV + kStages * kStage;  // kOut: 2 x 16 KB O staging
  static constexpr int kRed = kOut + 2 * 16384;                          // row max / sum exchange: 2 x 2 x 128 f32
  static constexpr int kBar = kRed + 2 * 2 * 128 * 4;
  static constexpr int kBytes = kBar + 256 + 1024;
  static_assert(kBytes <= 232448, "exceeds the 227 KB of shared memory per CTA");
};
constexpr uint32_t kPeerMask2 = 0xFEFFFFFFu;  // shared::cluster address of the leader's copy
LYNX_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
LYNX_DEV void cluster_sync2() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Relaxed remote arrive: the .release.cluster form compiles to MEMBAR.ALL.GPU, ~1000 cycles on the
// softmax's critical path. What an arrival here hands over is TMEM (S read / P written), and those
// tcgen05.ld / st have completed (wait::ld / wait::st) before the local arrivals this one forwards.
LYNX_DEV void arrive_leader2(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerMask2)
               : "memory");
}
LYNX_DEV void tma_load_pair(const void* desc, uint64_t* bar, void* smem, int c0, int c1, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar) & kPeerMask2), "r"(c0), "r"(c1), "l"(hint)
      : "memory");
}
LYNX_DEV void umma_pair_ss(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
LYNX_DEV void umma_pair_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
LYNX_DEV void commit_pair(uint64_t* bar) {  // arrive on `bar` in both CTAs when the leader's MMAs complete
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

template <int kPoly>  // every kPoly-th exponential on the FMA pipe (ex2_poly), 0: none
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    attn_fwd4_tc_kernel(const __grid_constant__ CUtensorMap map128, const __grid_constant__ CUtensorMap map64,
                        __nv_bfloat16* __restrict__ out, float* __restrict__ lse, int S, int H, float scale_log2) {
  using L = Fwd4L;
  constexpr int D = 128, NS = L::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t *q_full = bar, *kv_full = bar + 1, *kv_empty = kv_full + NS, *s_full = kv_empty + NS, *s_free = s_full + 2,
           *p_full = s_free + 2, *pv_done = p_full + 1, *s_free_loc = pv_done + 1, *p_full_loc = s_free_loc + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_full_loc + 1);
  float* red = reinterpret_cast<float*>(smem + L::kRed);  // [2 buffers][2 warpgroups][128 rows]
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = gridDim.x / 2 - 1 - blockIdx.x / 2, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qt = 2 * pair + static_cast<int>(rank);  // this CTA's query tile
  const int n = 2 * pair + 2;                        // key tiles of the pair (rank 0's last one is masked out)
  const int HD = H * D, row0 = b * S;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_free + i, 2);      // one forwarded arrival per CTA (on the leader)
      mbar_init(s_free_loc + i, 8);  // this CTA's 8 softmax warps
    }
    mbar_init(p_full, 2);
    mbar_init(p_full_loc, 8);
    mbar_init(pv_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync2();
  tc_fence_after();
  // TMEM (each CTA, its own 128 rows): S[2] at 0 / 128, P at 256 (64 packed columns), O at 384.
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
    if (elect_one()) {
      if (leader) mbar_arrive_expect_tx(q_full, 2 * L::kQT);
      for (int a = 0; a < 2; ++a)
        tma_load_pair(&map128, q_full, smem + L::kQ + a * 16384, h * D + 64 * a, row0 + qt * 128, kEvictFirst);
      for (int j = 0; j < n; ++j) {
        const int st = j % NS;
        if (j >= NS) mbar_wait(kv_empty + st, ((j / NS) - 1) & 1);
        uint8_t* sk = smem + L::kKV + st * L::kStage;
        if (leader) mbar_arrive_expect_tx(kv_full + st, 2 * L::kStage);
        for (int a = 0; a < 2; ++a)  // K: keys j * 128 + 64 rank ... + 63, all 128 columns
          tma_load_pair(&map64, kv_full + st, sk + a * 8192, HD + h * D + 64 * a, row0 + j * 128 + 64 * rank,
                        kEvictLast);
        // V: all 128 keys, columns 64 rank ... + 63
        tma_load_pair(&map128, kv_full + st, sk + L::kKH, 2 * HD + h * D + 64 * rank, row0 + j * 128, kEvictLast);
      }
    }
  } else if (warp == 1) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
    if (leader && elect_one()) {
      constexpr uint32_t idS = umma_idesc_bf16(256, 128, false, false);
      constexpr uint32_t idO = umma_idesc_bf16(256, D, false, true);
      const uint32_t sQ = smem_u32(smem + L::kQ), sKV = smem_u32(smem + L::kKV);
      auto issue_s = [&](int j) {  // S(j) into buffer j & 1 (both CTAs' rows)
        const int st = j % NS;
        mbar_wait(kv_full + st, (j / NS) & 1);
        if (j >= 2) mbar_wait(s_free + (j & 1), ((j >> 1) - 1) & 1);  // the softmax read S(j - 2)
        tc_fence_after();
        const uint32_t sk = sKV + st * L::kStage;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_pair_ss(tmem + (j & 1) * 128, kmaj(sQ, kk, 16384), kmaj(sk, kk, 8192), idS, kk > 0);
        commit_pair(s_full + (j & 1));
        ATRACE(0, j);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      if (n > 1) issue_s(1);
      for (int j = 0; j < n; ++j) {
        const int st = j % NS;
        mbar_wait(p_full, j & 1);
        ATRACE(1, j);
        tc_fence_after();
        const uint32_t sv = sKV + st * L::kStage + L::kKH;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // A = P (both CTAs' TMEM), B = V half per CTA (MN-major)
          umma_pair_ts(tmem + 384, tmem + 256 + kk * 8, mnmaj(sv, kk, 16384), idO, (j | kk) != 0);
        commit_pair(pv_done);
        commit_pair(kv_empty + st);
        if (j + 2 < n) issue_s(j + 2);
      }
    }
  } else if (warp == 3) {
    // Forwarder: the softmax warps arrive on this CTA's barriers (a cluster-scope remote arrive from each
    // of them cost ~1200 cycles on their critical path); one thread passes each phase on to the leader.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
    if (elect_one()) {
      for (int j = 0; j < n; ++j) {
        mbar_wait(s_free_loc + (j & 1), (j >> 1) & 1);
        arrive_leader2(s_free + (j & 1));
        mbar_wait(p_full_loc, j & 1);
        arrive_leader2(p_full);
      }
    }
  } else if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 216;");
    const int wg = (warp - 4) / 4;  // key columns 64 wg ... + 63 of every tile
    const int r = (warp % 4) * 32 + lane, tr = threadIdx.x - 128 - 128 * wg;
    const uint32_t lanes = static_cast<uint32_t>((warp % 4) * 32) << 16;
    const uint32_t o_col = tmem + lanes + 384 + 64 * wg;  // this warpgroup's half of O
    const int q = qt * 128 + r;
    float m_run = -INFINITY, l_run = 0.f;  // l_run: this warpgroup's half of the row sum
    for (int j = 0; j < n; ++j) {
      mbar_wait(s_full + (j & 1), (j >> 1) & 1);
      if (warp % 4 == 0 && lane == 0) ATRACE(wg ? 4 : 2, j);
      tc_fence_after();
      float x[64];
      const uint32_t s_col = tmem + lanes + (j & 1) * 128 + 64 * wg;
      tmem_ld32(s_col, reinterpret_cast<uint32_t*>(x));
      tmem_ld32(s_col + 32, reinterpret_cast<uint32_t*>(x + 32));
      tmem_ld_wait();
      if (warp == 4 && lane == 0) ATRACE(8, j);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free_loc + (j & 1));
      const bool dead = j > qt;  // rank 0's extra key tile: every key is after every query
      if (j == qt) {             // diagonal tile: causal mask (warp-uniform branch)
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (64 * wg + i > r) x[i] = -INFINITY;
      }
      float mv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mv[i] = x[i];
#pragma unroll
      for (int i = 8; i < 64; ++i) mv[i & 7] = fmaxf(mv[i & 7], x[i]);
      float mt =
          fmaxf(fmaxf(fmaxf(mv[0], mv[1]), fmaxf(mv[2], mv[3])), fmaxf(fmaxf(mv[4], mv[5]), fmaxf(mv[6], mv[7])));
      float* rb = red + (j & 1) * 256;
      rb[wg * 128 + r] = mt;
      asm volatile("bar.sync 2, 256;" ::: "memory");
      mt = fmaxf(mt, rb[(1 - wg) * 128 + r]);
      if (warp == 4 && lane == 0) ATRACE(9, j);
      uint32_t packed[32];
      bool need = false;
      float corr = 1.f;
      if (dead) {
#pragma unroll
        for (int i = 0; i < 32; ++i) packed[i] = 0u;
      } else {
        const float m_new = fmaxf(m_run, mt * scale_log2);
        need = __any_sync(0xffffffffu, m_new > m_run + kRescale);
        if (need) {
          corr = exp2f(m_run - m_new);
          m_run = m_new;
        }
        float rv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const float a = fmaf(x[i], scale_log2, -m_run);
          x[i] = (kPoly > 0 && i % (kPoly > 0 ? kPoly : 1) == (kPoly > 0 ? kPoly : 1) - 1) ? ex2_poly(a) : ex2(a);
          rv[i & 7] += x[i];
        }
        const float rs = ((rv[0] + rv[1]) + (rv[2] + rv[3])) + ((rv[4] + rv[5]) + (rv[6] + rv[7]));
        l_run = l_run * corr + rs;
#pragma unroll
        for (int i = 0; i < 32; ++i) packed[i] = pack_bf16x2(x[2 * i], x[2 * i + 1]);
      }
      if (warp == 4 && lane == 0) ATRACE(10, j);
      if (j > 0) {  // PV(j - 1) read P and wrote O
        mbar_wait(pv_done, (j - 1) & 1);
        tc_fence_after();
        if (need) {
          tmem_cols(o_col, 0, 64, [&](int c, uint32_t* o, int cnt) {
            for (int i = 0; i < cnt; ++i) o[i] = __float_as_uint(u2f(o[i]) * corr);
            tmem_st32(o_col + c, o);
          });
        }
      }
      if (warp == 4 && lane == 0) ATRACE(11, j);
      tmem_st32(tmem + lanes + 256 + 32 * wg, packed);
      tmem_st_wait();
      if (warp == 4 && lane == 0) ATRACE(12, j);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full_loc);
      if (warp % 4 == 0 && lane == 0) ATRACE(wg ? 5 : 3, j);
    }
    mbar_wait(pv_done, (n - 1) & 1);
    tc_fence_after();
    // row sum = both warpgroups' halves
    red[wg * 128 + r] = l_run;  // exchange buffer 0: its last readers (tile n - 2, n even) passed tile n - 1's barrier
    asm volatile("bar.sync 2, 256;" ::: "memory");
    const float l = l_run + red[(1 - wg) * 128 + r];
    const float inv = 1.f / l;
    uint8_t* stg = smem + L::kOut + wg * 16384;
    tmem_cols(o_col, 0, 64, [&](int c, const uint32_t* o, int cnt) {
      float f[32];
      for (int i = 0; i < cnt; ++i) f[i] = u2f(o[i]) * inv;
      for (int i = 0; i < cnt / 8; ++i)
        *reinterpret_cast<BF8*>(stg + r * 128 + (((c / 8 + i) ^ (r & 7)) * 16)) = f_to_bf8(f + 8 * i);
    });
    asm volatile("bar.sync %0, 128;" ::"r"(3 + wg) : "memory");
    const long long orow0 = static_cast<long long>(row0) + qt * 128;
    for (int i = tr; i < 128 * 8; i += 128) {
      const int rr = i / 8, ch = i % 8;
      const BF8 v = *reinterpret_cast<const BF8*>(stg + rr * 128 + ((ch ^ (rr & 7)) * 16));
      reinterpret_cast<BF8*>(out + (orow0 + rr) * HD + h * D + 64 * wg)[ch] = v;
    }
    if (wg == 0) lse[(static_cast<long long>(b) * H + h) * S + q] = (m_run + log2f(l)) / kLog2e;
  }
  tc_fence_before();
  cluster_sync2();
  ATRACE_DUMP(32);
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

// ============================================================== backward dK / dV
// Persistent, like the dQ kernel: grid = min(work items, SMs), work item w = (key tile, head, batch) in
// head-major, longest-first order. K / V of the next item are loaded as soon as the current item's
// last S^T / dP^T MMAs (their only readers) completed, ~2 tile periods before the item ends; the Q / dO
// ring runs on across items. dV / dK leave through a 32-KB shared-memory staging tile with coalesced
// global stores. As one CTA per item, each item paid ~5500 cycles before its first S^T and ~3000 of
// row-per-thread stores after its last tile, against ~1500 cycles per tile.
template <int D>
struct DkvL {
  // Q / dO / lse / D ring: a stage is held from S^T(i) to dV / dK(i), about two tile periods (4 stages
  // were measured no faster than 3: the tile period is set by the smem-bound S^T / dP^T MMAs).
  static constexpr int kStages = D <= 64 ? 6 : 3;
  static constexpr int kAtoms = (D + 63) / 64;
  static constexpr int kKV = 128 * kAtoms * 64 * 2;  // K or V tile: ceil(D/64) atoms of 16 KB (128 rows)
  static constexpr int kQT = 64 * kAtoms * 64 * 2;   // Q or dO tile: ceil(D/64) atoms of 8 KB (64 rows)
  static constexpr int kK = 0, kV = kKV, kQ = 2 * kKV, kDO = kQ + kStages * kQT;
  static constexpr int kVec = kDO + kStages * kQT;  // lse2[kStages][64], dvec[kStages][64]; P^T / dS^T live in TMEM
  static constexpr int kOut = kVec + 2 * kStages * 256;  // epilogue staging: 128 rows x 256 B (XOR-swizzled)
  static constexpr int kBar = kOut + 128 * 256;
  static constexpr int kBytes = kBar + 256 + 1024;
  static_assert(kBytes <= 232448, "exceeds the 227 KB of shared memory per CTA");
};

struct DkvItem {
  int kb, h, b, n;
};
LYNX_DEV DkvItem dkv_item(int w, int nk, int S, int H) {
  const int hb = w / nk;
  DkvItem it;
  it.kb = (w % nk + hb) % nk;  // rotated by head: see dq_item
  it.h = hb % H;
  it.b = hb / H;
  it.n = S / 64 - 2 * it.kb;
  return it;
}

template <int D, int kWG>  // kWG row warpgroups (2 or 4), each owning 64 / kWG query columns of a tile
__global__ void __launch_bounds__(128 + 128 * kWG, 1)
    attn_dkdv_tc_kernel(const __grid_constant__ CUtensorMap map_kv, const __grid_constant__ CUtensorMap map_q,
                        const __grid_constant__ CUtensorMap map_do, const float* __restrict__ lse2,
                        const float* __restrict__ dvec, __nv_bfloat16* __restrict__ dqkv, int S, int H, int B,
                        float scale, float scale_log2) {
  using L = DkvL<D>;
  constexpr int kA = L::kAtoms, NS = L::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
  // pd_full is double-buffered by tile parity (see the forward kernel's p_full: one barrier let a
  // row warp's arrival for tile i+1 complete tile i's phase before a slower warp had written its
  // P^T / dS^T rows, and dV / dK of those 32 keys picked up stale values, ~3 % of runs).
  uint64_t *kv_full = bar, *kv_free = bar + 1, *q_full = bar + 2, *q_empty = q_full + NS, *s_full = q_empty + NS,
           *pd_full = s_full + 2, *fin = pd_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fin + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nk = S / 128, HD = H * D, n_items = nk * H * B;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    mbar_init(kv_free, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(pd_full + i, 128 * kWG);
    }
    mbar_init(fin, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // TMEM: S^T[2] at 0 / 64, dP^T[2] at 128 / 192, dV at 256, dK at 384.
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      int g = 0, k = 0;  // Q / dO tile counter over this CTA's items, item counter
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
        const DkvItem it = dkv_item(w, nk, S, H);
        const int row0 = it.b * S, i0 = 2 * it.kb;
        const long long vec0 = (static_cast<long long>(it.b) * H + it.h) * S;
        if (k > 0) mbar_wait(kv_free, (k - 1) & 1);  // the previous item's last S^T / dP^T completed
        mbar_arrive_expect_tx(kv_full, 2 * L::kKV);
        for (int a = 0; a < kA; ++a) {
          tma_load_2d(&map_kv, kv_full, smem + L::kK + a * 16384, HD + it.h * D + 64 * a, row0 + it.kb * 128,
                      kEvictFirst);
          tma_load_2d(&map_kv, kv_full, smem + L::kV + a * 16384, 2 * HD + it.h * D + 64 * a, row0 + it.kb * 128,
                      kEvictFirst);
        }
        for (int i = 0; i < it.n; ++i, ++g) {
          const int st = g % NS, q0 = (i0 + i) * 64;
          if (g >= NS) mbar_wait(q_empty + st, ((g / NS) - 1) & 1);
          ATRACE(0, k == 0 ? i : 64);
          mbar_arrive_expect_tx(q_full + st, 2 * L::kQT + 512);
          for (int a = 0; a < kA; ++a) {
            tma_load_2d(&map_q, q_full + st, smem + L::kQ + st * L::kQT + a * 8192, it.h * D + 64 * a, row0 + q0,
                        kEvictLast);
            tma_load_2d(&map_do, q_full + st, smem + L::kDO + st * L::kQT + a * 8192, it.h * D + 64 * a,
                        row0 + q0, kEvictLast);
          }
          bulk_load(smem + L::kVec + st * 256, lse2 + vec0 + q0, 256, q_full + st);
          bulk_load(smem + L::kVec + (NS + st) * 256, dvec + vec0 + q0, 256, q_full + st);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idS = umma_idesc_bf16(128, 64, false, false);
      constexpr uint32_t idG = umma_idesc_bf16(128, D, false, true);
      const uint32_t sK = smem_u32(smem + L::kK), sV = smem_u32(smem + L::kV), sQ = smem_u32(smem + L::kQ),
                     sDO = smem_u32(smem + L::kDO);
      auto issue_s = [&](int g) {  // S^T / dP^T of the CTA's g-th tile
        const int st = g % NS, tb = g & 1;
        mbar_wait(q_full + st, (g / NS) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          umma_f16(tmem + tb * 64, kmaj(sK, kk, 16384), kmaj(sQ + st * L::kQT, kk, 8192), idS, kk > 0);
          umma_f16(tmem + 128 + tb * 64, kmaj(sV, kk, 16384), kmaj(sDO + st * L::kQT, kk, 8192), idS, kk > 0);
        }
        umma_commit(s_full + tb);
      };
      int g = 0, k = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
        const int n = dkv_item(w, nk, S, H).n;
        mbar_wait(kv_full, k & 1);
        ATRACE(10, k);
        issue_s(g);
        issue_s(g + 1);
        if (n == 2) umma_commit(kv_free);
        for (int i = 0; i < n; ++i) {
          const int gg = g + i, st = gg % NS;
          mbar_wait(pd_full + (gg & 1), (gg >> 1) & 1);
          ATRACE(2, k == 0 ? i : 64);
          tc_fence_after();
          const uint32_t tb = static_cast<uint32_t>(gg & 1);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // A = P^T / dS^T, packed bf16 over S^T / dP^T in TMEM buffer tb
            const uint32_t ac = tb * 64 + packed_col<kWG>(kk);
            umma_f16_ts(tmem + 256, tmem + ac, mnmaj(sDO + st * L::kQT, kk, 8192), idG, (i | kk) != 0);
            umma_f16_ts(tmem + 384, tmem + 128 + ac, mnmaj(sQ + st * L::kQT, kk, 8192), idG, (i | kk) != 0);
          }
          umma_commit(q_empty + st);
          if (i + 2 < n) {
            issue_s(gg + 2);
            if (i + 3 == n) umma_commit(kv_free);  // K / V have no reader left in this item
          }
        }
        umma_commit(fin);
        ATRACE(12, k);
        g += n;
      }
    }
  } else if (warp >= 4) {
    // kWG row warpgroups split each 64-query tile's columns (warpgroup wg: columns wg * CW ...
    // + CW) on the same key rows / TMEM lanes. The work is elementwise, so they never exchange data.
    constexpr int CW = 64 / kWG;
    const int wg = (warp - 4) / 4;
    const int kr = (warp % 4) * 32 + lane;  // key row of the tile
    const uint32_t lanes = static_cast<uint32_t>((warp % 4) * 32) << 16;
    constexpr int kChunks = D / 8, kIter = (128 * kChunks + 128 * kWG - 1) / (128 * kWG);
    uint8_t* stg = smem + L::kOut;
    // dV (first half of the warpgroups) then dK (second half, scaled): TMEM -> bf16 rows in the staging
    // tile (row r's 16-B chunk c at r * 256 + (c ^ (r % 16)) * 16) -> coalesced global stores
    auto epilogue = [&](const DkvItem& it) {
      constexpr int kPer = kWG / 2, kSplit = (D / 16 + kPer - 1) / kPer * 16;
      const int part = wg % kPer;
      const int c_lo = part * kSplit < D ? part * kSplit : D, c_hi = (part + 1) * kSplit < D ? (part + 1) * kSplit : D;
      for (int pass = 0; pass < 2; ++pass) {  // 0: dV, 1: dK
        if ((wg >= kPer) == (pass == 1)) {
          const float mul = pass ? scale : 1.f;
          tmem_cols(tmem + lanes + (pass ? 384 : 256), c_lo, c_hi, [&](int c, const uint32_t* o, int cnt) {
            float f[32];
            for (int i = 0; i < cnt; ++i) f[i] = u2f(o[i]) * mul;
            for (int i = 0; i < cnt / 8; ++i)
              *reinterpret_cast<BF8*>(stg + kr * 256 + (((c / 8 + i) ^ (kr & 15)) * 16)) = f_to_bf8(f + 8 * i);
          });
        }
        asm volatile("bar.sync 1, %0;" ::"r"(128 * kWG) : "memory");
        BF8* dst = reinterpret_cast<BF8*>(dqkv + (static_cast<long long>(it.b) * S + it.kb * 128) * 3 * HD +
                                          (pass ? HD : 2 * HD) + it.h * D);
        BF8 v[kIter];
#pragma unroll
        for (int x = 0; x < kIter; ++x) {
          const int i = static_cast<int>(threadIdx.x) - 128 + x * 128 * kWG, rr = i / kChunks, cc = i % kChunks;
          if (i < 128 * kChunks) v[x] = *reinterpret_cast<const BF8*>(stg + rr * 256 + ((cc ^ (rr & 15)) * 16));
        }
#pragma unroll
        for (int x = 0; x < kIter; ++x) {
          const int i = static_cast<int>(threadIdx.x) - 128 + x * 128 * kWG, rr = i / kChunks, cc = i % kChunks;
          if (i < 128 * kChunks) dst[static_cast<long long>(rr) * (3 * HD / 8) + cc] = v[x];
        }
        asm volatile("bar.sync 1, %0;" ::"r"(128 * kWG) : "memory");  // the staging tile is read: reusable
      }
    };
    int g = 0, k = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
      const DkvItem it = dkv_item(w, nk, S, H);
      const int key = it.kb * 128 + kr, i0 = 2 * it.kb;
      if (threadIdx.x == 128) ATRACE(8, k);
      for (int i = 0; i < it.n; ++i) {
        const int gg = g + i, st = gg % NS, tb = gg & 1, q0 = (i0 + i) * 64;
        mbar_wait(q_full + st, (gg / NS) & 1);
        mbar_wait(s_full + tb, (gg >> 1) & 1);
        if (threadIdx.x == 128) ATRACE(3, k == 0 ? i : 64);
        if (threadIdx.x == 128 && i == 0) ATRACE(13, k);
        tc_fence_after();
        const float* sl = reinterpret_cast<const float*>(smem + L::kVec + st * 256) + wg * CW;
        const float* sd = reinterpret_cast<const float*>(smem + L::kVec + (NS + st) * 256) + wg * CW;
        {
          uint32_t sr[CW], dp[CW];
          tmem_ld_cols<CW>(tmem + lanes + tb * 64 + wg * CW, sr);
          tmem_ld_cols<CW>(tmem + lanes + 128 + tb * 64 + wg * CW, dp);
          tmem_ld_wait();
          float p[CW], gd[CW], lv[CW], dv[CW];
#pragma unroll
          for (int c = 0; c < CW / 4; ++c) {
            const float4 a = lds128(sl + 4 * c), d4 = lds128(sd + 4 * c);
            lv[4 * c] = a.x, lv[4 * c + 1] = a.y, lv[4 * c + 2] = a.z, lv[4 * c + 3] = a.w;
            dv[4 * c] = d4.x, dv[4 * c + 1] = d4.y, dv[4 * c + 2] = d4.z, dv[4 * c + 3] = d4.w;
          }
#pragma unroll
          for (int c = 0; c < CW; ++c) p[c] = ex2(fmaf(u2f(sr[c]), scale_log2, -lv[c]));
          if (i < 2) {  // the two 64-query tiles that meet the diagonal of this 128-key tile
#pragma unroll
            for (int c = 0; c < CW; ++c)
              if (key > q0 + wg * CW + c) p[c] = 0.f;
          }
#pragma unroll
          for (int c = 0; c < CW; ++c) gd[c] = p[c] * (u2f(dp[c]) - dv[c]);
          uint32_t pp[CW / 2], gp[CW / 2];
#pragma unroll
          for (int c = 0; c < CW / 2; ++c) {
            pp[c] = pack_bf16x2(p[2 * c], p[2 * c + 1]);
            gp[c] = pack_bf16x2(gd[2 * c], gd[2 * c + 1]);
          }
          if (threadIdx.x == 128) ATRACE(4, k == 0 ? i : 64);
          // P^T(i) / dS^T(i) overwrite S^T(i) / dP^T(i) in place, each warpgroup inside the columns it
          // read itself (packed_col): the others read the same TMEM lanes without any ordering against
          // this store (packing outside its own range once made warps read P^T instead of S^T, ~0.1 %
          // of runs). dV / dK(i-2), the last readers of buffer tb, completed before S^T(i).
          tmem_st_cols<CW / 2>(tmem + lanes + tb * 64 + wg * CW, pp);
          tmem_st_cols<CW / 2>(tmem + lanes + 128 + tb * 64 + wg * CW, gp);
          tmem_st_wait();
        }
        tc_fence_before();
        mbar_arrive(pd_full + tb);
        if (threadIdx.x == 128) ATRACE(6, k == 0 ? i : 64);
      }
      g += it.n;
      if (threadIdx.x == 128) ATRACE(7, k);
      // dV / dK complete; the next item's first dV / dK MMA (accumulate = 0) waits for this thread's first
      // hand-off of that item, i.e. after the epilogue
      mbar_wait(fin, k & 1);
      tc_fence_after();
      if (threadIdx.x == 128) ATRACE(9, k);
      epilogue(it);
      if (threadIdx.x == 128) ATRACE(11, k);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  ATRACE_DUMP(64);
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ============================================================== backward dQ
// Q and dO are the same for every key tile of a work item, so they sit in TMEM as the A operands of
// S = Q K^T and dP = dO V^T (packed bf16 pairs, one row per lane). An SS MMA of 128 x 64 x 16 reads
// 6 KB of shared memory per 32-cycle instruction, 1.5x the 128 B/clk the SM's shared memory delivers,
// so with Q / dO in shared memory S and dP ran smem-bound at ~48 cycles per instruction; from TMEM only
// the 2-KB K / V slice is read (tile period 1232 -> 975 cycles in a clock64 trace).
//
// Persistent: grid = min(work items, SMs); each CTA walks the work items (query tile, head, batch)
// blockIdx.x, + gridDim.x, ... in longest-first order. The producer TMA-loads the next item's Q / dO
// into a staging buffer while the current item runs and keeps the K / V ring going across items; the
// MMA thread moves Q / dO into TMEM with tcgen05.cp (in issue order with its MMAs, so after the
// previous item's last S / dP). As one CTA per item, each item paid ~7000 cycles of prologue (TMEM
// allocation, barriers, Q / dO and K / V loads) against ~975 cycles per key tile.
template <int D>
struct DqL {
  static constexpr int kAtoms = (D + 63) / 64;
  static constexpr int kQT = 128 * kAtoms * 64 * 2;  // Q or dO tile (128 rows): the staging buffer
  static constexpr int kKT = 64 * kAtoms * 64 * 2;   // K or V tile (64 rows)
  static constexpr int kStages = D <= 64 ? 8 : 4;    // K / V ring (see DkvL::kStages)
  static constexpr int kQ = 0, kDO = kQT, kK = 2 * kQT, kV = kK + kStages * kKT;
  static constexpr int kOut = kV + kStages * kKT;  // dQ epilogue staging: 128 rows x 256 B (XOR-swizzled chunks)
  static constexpr int kBar = kOut + 128 * 256;
  static constexpr int kBytes = kBar + 256 + 1024;
  static_assert(kBytes <= 232448, "exceeds the 227 KB of shared memory per CTA");
};

struct DqItem {
  int qb, h, b, n;
};
// Work item w: head w / nq, so the CTAs that run at the same time work on the same few heads and share
// their K / V tiles in L2 (qb-major order made every CTA stream its own head's K / V from HBM: ~4.5 GB
// per call at the 7B shape). The query tile is rotated by the head index: without it CTA c (items c,
// c + 148, ...) met only the tiles (c + 4 k) % 16 — four of the sixteen lengths, up to 43 % more work
// than another CTA — with it, (c + 13.25 k) % 16 cycles through all of them.
LYNX_DEV DqItem dq_item(int w, int nq, int H, int B) {
  const int hb = w / nq;
  DqItem it;
  it.qb = nq - 1 - (w % nq + hb) % nq;
  it.h = hb % H;
  it.b = hb / H;
  it.n = 2 * (it.qb + 1);
  return it;
}

// 128 rows x 32 bytes (16 bf16 of each row: one K step) from a K-major SW128 operand in shared memory
// into 8 TMEM columns of lanes 0-127 — the packed layout an A-from-TMEM MMA reads.
LYNX_DEV void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}

template <int D, int kWG>  // kWG row warpgroups (2 or 4), each owning 64 / kWG key columns of a tile
__global__ void __launch_bounds__(128 + 128 * kWG, 1)
    attn_dq_tc_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                      const __grid_constant__ CUtensorMap map_do, const float* __restrict__ lse2,
                      const float* __restrict__ dvec, __nv_bfloat16* __restrict__ dqkv, int S, int H, int B,
                      float scale, float scale_log2) {
  using L = DqL<D>;
  constexpr int kA = L::kAtoms, NS = L::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t *q_full = bar, *q_empty = bar + 1, *kv_full = bar + 2, *kv_empty = kv_full + NS, *s_full = kv_empty + NS,
           *ds_full = s_full + 2, *fin = ds_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fin + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nq = S / 128, HD = H * D, n_items = nq * H * B;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(ds_full + i, 128 * kWG);
    }
    mbar_init(fin, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // TMEM: S[2] at 0 / 64, dP[2] at 128 / 192, dQ at 256, Q at 384, dO at 448 (D / 2 packed columns each).
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      auto load_q = [&](int w, int k) {  // Q / dO of this CTA's k-th item into the staging buffer
        const DqItem it = dq_item(w, nq, H, B);
        if (k > 0) mbar_wait(q_empty, (k - 1) & 1);  // item k - 1's Q / dO are in TMEM
        mbar_arrive_expect_tx(q_full, 2 * L::kQT);
        for (int a = 0; a < kA; ++a) {
          tma_load_2d(&map_q, q_full, smem + L::kQ + a * 16384, it.h * D + 64 * a, it.b * S + it.qb * 128,
                      kEvictFirst);
          tma_load_2d(&map_do, q_full, smem + L::kDO + a * 16384, it.h * D + 64 * a, it.b * S + it.qb * 128,
                      kEvictFirst);
        }
      };
      load_q(blockIdx.x, 0);
      int g = 0, k = 0;  // K / V tile counter over this CTA's items, item counter
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
        const DqItem it = dq_item(w, nq, H, B);
        const int row0 = it.b * S;
        for (int j = 0; j < it.n; ++j, ++g) {
          const int st = g % NS;
          if (g >= NS) mbar_wait(kv_empty + st, ((g / NS) - 1) & 1);
          ATRACE(0, w == static_cast<int>(blockIdx.x) ? j : 64);
          mbar_arrive_expect_tx(kv_full + st, 2 * L::kKT);
          for (int a = 0; a < kA; ++a) {
            tma_load_2d(&map_kv, kv_full + st, smem + L::kK + st * L::kKT + a * 8192, HD + it.h * D + 64 * a,
                        row0 + j * 64, kEvictLast);
            tma_load_2d(&map_kv, kv_full + st, smem + L::kV + st * L::kKT + a * 8192, 2 * HD + it.h * D + 64 * a,
                        row0 + j * 64, kEvictLast);
          }
          // the next item's Q / dO once this item's copy into TMEM is done (a few tiles in)
          if (j == (it.n < 4 ? it.n - 1 : 3) && w + static_cast<int>(gridDim.x) < n_items)
            load_q(w + gridDim.x, k + 1);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idS = umma_idesc_bf16(128, 64, false, false);
      constexpr uint32_t idG = umma_idesc_bf16(128, D, false, true);
      const uint32_t sQ = smem_u32(smem + L::kQ), sDO = smem_u32(smem + L::kDO), sK = smem_u32(smem + L::kK),
                     sV = smem_u32(smem + L::kV);
      auto issue_s = [&](int g) {  // S / dP of the CTA's g-th tile
        const int st = g % NS, tb = g & 1;
        mbar_wait(kv_full + st, (g / NS) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          umma_f16_ts(tmem + tb * 64, tmem + 384 + kk * 8, kmaj(sK + st * L::kKT, kk, 8192), idS, kk > 0);
          umma_f16_ts(tmem + 128 + tb * 64, tmem + 448 + kk * 8, kmaj(sV + st * L::kKT, kk, 8192), idS, kk > 0);
        }
        umma_commit(s_full + tb);
      };
      int g = 0, k = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
        const int n = dq_item(w, nq, H, B).n;
        mbar_wait(q_full, k & 1);
        ATRACE(10, k);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {  // after the previous item's MMAs (tcgen05 issue order)
          tmem_cp_128x256b(tmem + 384 + kk * 8, kmaj(sQ, kk, 16384));
          tmem_cp_128x256b(tmem + 448 + kk * 8, kmaj(sDO, kk, 16384));
        }
        umma_commit(q_empty);
        issue_s(g);
        issue_s(g + 1);
        for (int j = 0; j < n; ++j) {
          const int gg = g + j, st = gg % NS, tb = gg & 1;
          mbar_wait(ds_full + tb, (gg >> 1) & 1);
          ATRACE(2, k == 0 ? j : 64);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // A = dS(j), packed bf16 over the S(j) columns of TMEM buffer tb
            umma_f16_ts(tmem + 256, tmem + tb * 64 + packed_col<kWG>(kk), mnmaj(sK + st * L::kKT, kk, 8192),
                        idG, (j | kk) != 0);
          umma_commit(kv_empty + st);
          if (j + 2 < n) issue_s(gg + 2);
        }
        umma_commit(fin);
        ATRACE(12, k);
        g += n;
      }
    }
  } else if (warp >= 4) {
    // kWG row warpgroups split each 64-key tile's columns, as in dK/dV.
    constexpr int CW = 64 / kWG;
    const int wg = (warp - 4) / 4;
    const int r = (warp % 4) * 32 + lane;
    const uint32_t lanes = static_cast<uint32_t>((warp % 4) * 32) << 16;
    // dQ of item w: TMEM -> scaled bf16 rows in a shared-memory staging tile (row r's 16-B chunk c at
    // r * 256 + (c ^ (r % 16)) * 16: conflict-free row-per-thread stores) -> coalesced 16-B global stores,
    // all loads of a thread issued before its stores. Written per thread straight from TMEM (one 128-B
    // row piece per thread, 32 rows per warp instruction) the stores took ~3800 cycles per item.
    constexpr int kChunks = D / 8, kIter = (128 * kChunks + 128 * kWG - 1) / (128 * kWG);
    uint8_t* stg = smem + L::kOut;
    auto epilogue = [&](int w, int k) {
      const DqItem it = dq_item(w, nq, H, B);
      constexpr int kSplit = (D / 16 + kWG - 1) / kWG * 16;  // each warpgroup stages its share of the D columns
      const int c_lo = wg * kSplit < D ? wg * kSplit : D, c_hi = (wg + 1) * kSplit < D ? (wg + 1) * kSplit : D;
      tmem_cols(tmem + lanes + 256, c_lo, c_hi, [&](int c, const uint32_t* o, int cnt) {
        float f[32];
        for (int i = 0; i < cnt; ++i) f[i] = u2f(o[i]) * scale;
        for (int i = 0; i < cnt / 8; ++i)
          *reinterpret_cast<BF8*>(stg + r * 256 + (((c / 8 + i) ^ (r & 15)) * 16)) = f_to_bf8(f + 8 * i);
      });
      if (threadIdx.x == 128) ATRACE(15, k);
      asm volatile("bar.sync 1, %0;" ::"r"(128 * kWG) : "memory");
      if (threadIdx.x == 128) ATRACE(5, k);
      BF8* dst = reinterpret_cast<BF8*>(dqkv + (static_cast<long long>(it.b) * S + it.qb * 128) * 3 * HD + it.h * D);
      BF8 v[kIter];
#pragma unroll
      for (int x = 0; x < kIter; ++x) {
        const int i = static_cast<int>(threadIdx.x) - 128 + x * 128 * kWG, rr = i / kChunks, cc = i % kChunks;
        if (i < 128 * kChunks) v[x] = *reinterpret_cast<const BF8*>(stg + rr * 256 + ((cc ^ (rr & 15)) * 16));
      }
#pragma unroll
      for (int x = 0; x < kIter; ++x) {
        const int i = static_cast<int>(threadIdx.x) - 128 + x * 128 * kWG, rr = i / kChunks, cc = i % kChunks;
        if (i < 128 * kChunks) dst[static_cast<long long>(rr) * (3 * HD / 8) + cc] = v[x];
      }
      // the next epilogue rewrites the tile only after a whole item of dS hand-offs: every row thread has
      // long finished reading it
    };
    auto vec_index = [&](int w) {
      const DqItem it = dq_item(w, nq, H, B);
      return (static_cast<long long>(it.b) * H + it.h) * S + it.qb * 128 + r;
    };
    float l2 = lse2[vec_index(blockIdx.x)], dq = dvec[vec_index(blockIdx.x)];
    int g = 0, k = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
      const DqItem it = dq_item(w, nq, H, B);
      const int q = it.qb * 128 + r;
      if (threadIdx.x == 128) ATRACE(8, k);
      // the next item's row statistics, loaded a whole item ahead (issued at the item's end they were still
      // in flight ~2600 cycles later under the K / V stream)
      const int wn = w + gridDim.x;
      float l2n = 0.f, dqn = 0.f;
      if (wn < n_items) l2n = lse2[vec_index(wn)], dqn = dvec[vec_index(wn)];
      for (int j = 0; j < it.n; ++j) {
        const int gg = g + j, st = gg & 1;
        mbar_wait(s_full + st, (gg >> 1) & 1);
        if (threadIdx.x == 128) ATRACE(3, k == 0 ? j : 64);
        if (threadIdx.x == 128 && j == 0) ATRACE(13, k);
        tc_fence_after();
        const bool diag = j >= 2 * it.qb;
        {
          uint32_t sv[CW], dp[CW];
          tmem_ld_cols<CW>(tmem + lanes + st * 64 + wg * CW, sv);
          tmem_ld_cols<CW>(tmem + lanes + 128 + st * 64 + wg * CW, dp);
          tmem_ld_wait();
          float gr[CW];
#pragma unroll
          for (int c = 0; c < CW; ++c) gr[c] = ex2(fmaf(u2f(sv[c]), scale_log2, -l2));
          if (diag) {
#pragma unroll
            for (int c = 0; c < CW; ++c)
              if (j * 64 + wg * CW + c > q) gr[c] = 0.f;
          }
#pragma unroll
          for (int c = 0; c < CW; ++c) gr[c] *= u2f(dp[c]) - dq;
          uint32_t packed[CW / 2];
#pragma unroll
          for (int c = 0; c < CW / 2; ++c) packed[c] = pack_bf16x2(gr[2 * c], gr[2 * c + 1]);
          if (threadIdx.x == 128) ATRACE(4, k == 0 ? j : 64);
          // dS(j) overwrites S(j) in place, each warpgroup inside the columns it read (packed_col; see
          // the dK/dV kernel); dQ(j-2), the last reader of this buffer, completed before S(j).
          tmem_st_cols<CW / 2>(tmem + lanes + st * 64 + wg * CW, packed);
          tmem_st_wait();
        }
        tc_fence_before();
        mbar_arrive(ds_full + st);
        if (threadIdx.x == 128) ATRACE(6, k == 0 ? j : 64);
      }
      g += it.n;
      if (threadIdx.x == 128) ATRACE(7, k);
      // this item's dQ is complete; the next item's first dQ MMA (which overwrites the accumulator) waits
      // for the dS hand-off below, i.e. after this epilogue
      mbar_wait(fin, k & 1);
      tc_fence_after();
      if (threadIdx.x == 128) ATRACE(9, k);
      epilogue(w, k);
      if (threadIdx.x == 128) ATRACE(11, k);
      l2 = l2n, dq = dqn;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  ATRACE_DUMP(64);
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ============================================================== host
// LYNX_ATTN_POLY: share of the forward softmax exponentials computed on the FMA pipe, as one in N
// (0: all on MUFU). Read once.
int poly_every() {
  static const int n = [] {
    const char* e = std::getenv("LYNX_ATTN_POLY");
    return e ? std::atoi(e) : kDefaultPoly;
  }();
  return n;
}

template <int D, int kPoly>
int fwd_poly(const CUtensorMap& m, __nv_bfloat16* out, float* lse, int B, int S, int H, cudaStream_t s) {
  auto k = attn_fwd_tc_kernel<D, kPoly>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdL<D>::kBytes);
  k<<<dim3(S / 128, H, B), 256, FwdL<D>::kBytes, s>>>(m, out, lse, S, H, kLog2e / sqrtf(static_cast<float>(D)));
  return check_launch("attention_fwd_tc");
}

// Forward kernel variant: 2 (default) = two query tiles per CTA (attn_fwd2_tc_kernel), 1 = one tile.
int g_fwd_tiles = 0;
int fwd_tiles() {
  if (g_fwd_tiles) return g_fwd_tiles;
  static const int n = [] {
    const char* e = std::getenv("LYNX_ATTN_FWD_TILES");
    const int v = e ? std::atoi(e) : 2;
    return v == 1 || v == 3 || v == 4 ? v : 2;
  }();
  return n;
}

template <int D>
int fwd(const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, int B, int S, int H, cudaStream_t s) {
  CUtensorMap m;
  const long long T = static_cast<long long>(B) * S, ld = 3LL * H * D;
  if (!gemm::make_map(&m, qkv, ld, T, ld, 64, 128)) return set_error("attention: tensor map encode failed");
  if (fwd_tiles() == 4 && D == 128 && (S / 128) % 2 == 0) {
    CUtensorMap m64;
    if (!gemm::make_map(&m64, qkv, ld, T, ld, 64, 64)) return set_error("attention: tensor map encode failed");
    const int poly = poly_every();
    auto k = poly == 2 ? attn_fwd4_tc_kernel<2> : poly == 3 ? attn_fwd4_tc_kernel<3>
             : poly == 4 ? attn_fwd4_tc_kernel<4> : attn_fwd4_tc_kernel<0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd4L::kBytes);
    k<<<dim3(S / 128, H, B), 384, Fwd4L::kBytes, s>>>(m, m64, out, lse, S, H, kLog2e / sqrtf(static_cast<float>(D)));
    return check_launch("attention_fwd_tc");
  }
  if (fwd_tiles() == 3) {
    CUtensorMap m64;
    if (!gemm::make_map(&m64, qkv, ld, T, ld, 64, 64)) return set_error("attention: tensor map encode failed");
    auto k = attn_fwd3_tc_kernel<D>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd3L<D>::kBytes);
    k<<<dim3((S / 128 + 1) / 2, H, B), 384, Fwd3L<D>::kBytes, s>>>(m, m64, out, lse, S, H,
                                                                   kLog2e / sqrtf(static_cast<float>(D)));
    return check_launch("attention_fwd_tc");
  }
  if (fwd_tiles() == 2) {
    const int poly = poly_every();
    auto k = poly == 2 ? attn_fwd2_tc_kernel<D, 2>
             : poly == 3 ? attn_fwd2_tc_kernel<D, 3>
             : poly == 4 ? attn_fwd2_tc_kernel<D, 4>
                         : attn_fwd2_tc_kernel<D, 0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2L<D>::kBytes);
    const int items = (S / 128 + 1) / 2 * H * B, grid = items < gemm::num_sms() ? items : gemm::num_sms();
    k<<<grid, 384, Fwd2L<D>::kBytes, s>>>(m, out, lse, S, H, B, kLog2e / sqrtf(static_cast<float>(D)));
    return check_launch("attention_fwd_tc");
  }
  switch (poly_every()) {
    case 2: return fwd_poly<D, 2>(m, out, lse, B, S, H, s);
    case 3: return fwd_poly<D, 3>(m, out, lse, B, S, H, s);
    case 4: return fwd_poly<D, 4>(m, out, lse, B, S, H, s);
    default: break;
  }
  auto k = attn_fwd_tc_kernel<D, 0>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdL<D>::kBytes);
  k<<<dim3(S / 128, H, B), 256, FwdL<D>::kBytes, s>>>(m, out, lse, S, H, kLog2e / sqrtf(static_cast<float>(D)));
  return check_launch("attention_fwd_tc");
}

// Row warpgroups of the backward kernels (2 or 4): attention_set_bwd_warpgroups, else LYNX_ATTN_BWD_WG,
// else kDefaultBwdWG. Both give bit-identical gradients (same MMA order, same per-element math).
int g_bwd_wg = 0;
int bwd_warpgroups() {
  if (g_bwd_wg) return g_bwd_wg;
  static const int n = [] {
    const char* e = std::getenv("LYNX_ATTN_BWD_WG");
    return e ? (std::atoi(e) == 4 ? 4 : 2) : kDefaultBwdWG;
  }();
  return n;
}

template <int D, int kWG>
int bwd_launch(const CUtensorMap& m128, const CUtensorMap& m64, const CUtensorMap& d64, const CUtensorMap& d128,
               const float* lse, const float* dvec, __nv_bfloat16* dqkv, int B, int S, int H, float scale,
               float scale_log2, cudaStream_t s) {
  auto k1 = attn_dkdv_tc_kernel<D, kWG>;
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, DkvL<D>::kBytes);
  const int items1 = S / 128 * H * B, grid1 = items1 < gemm::num_sms() ? items1 : gemm::num_sms();
  k1<<<grid1, 128 + 128 * kWG, DkvL<D>::kBytes, s>>>(m128, m64, d64, lse, dvec, dqkv, S, H, B, scale, scale_log2);
  auto k2 = attn_dq_tc_kernel<D, kWG>;
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, DqL<D>::kBytes);
  const int items = S / 128 * H * B, grid2 = items < gemm::num_sms() ? items : gemm::num_sms();
  k2<<<grid2, 128 + 128 * kWG, DqL<D>::kBytes, s>>>(m128, m64, d128, lse, dvec, dqkv, S, H, B, scale, scale_log2);
  return check_launch("attention_bwd_tc", 2);
}

template <int D>
int bwd(const __nv_bfloat16* qkv, const __nv_bfloat16* dout, const float* lse, const float* dvec,
        __nv_bfloat16* dqkv, int B, int S, int H, cudaStream_t s) {
  CUtensorMap m128, m64, d64, d128;
  const long long T = static_cast<long long>(B) * S, ld = 3LL * H * D, hd = static_cast<long long>(H) * D;
  bool ok = gemm::make_map(&m128, qkv, ld, T, ld, 64, 128) && gemm::make_map(&m64, qkv, ld, T, ld, 64, 64) &&
            gemm::make_map(&d64, dout, hd, T, hd, 64, 64) && gemm::make_map(&d128, dout, hd, T, hd, 64, 128);
  if (!ok) return set_error("attention: tensor map encode failed");
  const float scale = 1.f / sqrtf(static_cast<float>(D)), scale_log2 = scale * kLog2e;
  if (bwd_warpgroups() == 2)
    return bwd_launch<D, 2>(m128, m64, d64, d128, lse, dvec, dqkv, B, S, H, scale, scale_log2, s);
  return bwd_launch<D, 4>(m128, m64, d64, d128, lse, dvec, dqkv, B, S, H, scale, scale_log2, s);
}

int g_mode = -1;

}  // namespace attn_tc

void attention_set_mode(int mode) { attn_tc::g_mode = mode; }
void attention_set_bwd_warpgroups(int n) { attn_tc::g_bwd_wg = n == 2 || n == 4 ? n : 0; }
void attention_set_fwd_tiles(int n) { attn_tc::g_fwd_tiles = n >= 1 && n <= 4 ? n : 0; }
int attention_mode() { return attn_tc::g_mode; }
bool attention_tc_supported(int seq, int head_dim) {
  return attn_tc::g_mode != 0 && seq % 128 == 0 &&
         (head_dim == 64 || head_dim == 96 || head_dim == 112 || head_dim == 128);
}

int attention_fwd_tc(const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, int B, int S, int H, int D,
                     cudaStream_t s) {
  switch (D) {
    case 64: return attn_tc::fwd<64>(qkv, out, lse, B, S, H, s);
    case 96: return attn_tc::fwd<96>(qkv, out, lse, B, S, H, s);   // GPT-20B
    case 112: return attn_tc::fwd<112>(qkv, out, lse, B, S, H, s);  // GPT-1.3B
    case 128: return attn_tc::fwd<128>(qkv, out, lse, B, S, H, s);
    default: return set_error("attention_fwd_tc: head_dim must be 64, 96, 112 or 128", kValidation);
  }
}

int attention_bwd_tc(const __nv_bfloat16* qkv, const __nv_bfloat16* dout, const float* lse, const float* dvec,
                     __nv_bfloat16* dqkv, int B, int S, int H, int D, cudaStream_t s) {
  switch (D) {
    case 64: return attn_tc::bwd<64>(qkv, dout, lse, dvec, dqkv, B, S, H, s);
    case 96: return attn_tc::bwd<96>(qkv, dout, lse, dvec, dqkv, B, S, H, s);
    case 112: return attn_tc::bwd<112>(qkv, dout, lse, dvec, dqkv, B, S, H, s);
    case 128: return attn_tc::bwd<128>(qkv, dout, lse, dvec, dqkv, B, S, H, s);
    default: return set_error("attention_bwd_tc: head_dim must be 64, 96, 112 or 128", kValidation);
  }
}

}  // namespace lynx
