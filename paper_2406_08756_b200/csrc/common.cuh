// Shared device helpers for the sm_100a operator library: bf16 packing,
// Philox-4x32-10 counter RNG (dropout masks that replay bit-identically when a
// discarded activation is recomputed), warp reductions, and thin inline-PTX
// wrappers for mbarrier / TMA / tcgen05 (UMMA + TMEM).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define LYNX_DEV __device__ __forceinline__

namespace lynx {

// ---------------------------------------------------------------- numerics
LYNX_DEV float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
LYNX_DEV __nv_bfloat16 f2bf(float v) { return __float2bfloat16_rn(v); }

LYNX_DEV uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
LYNX_DEV float2 unpack_bf16x2(uint32_t v) {
  __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&v);
  return __bfloat1622float2(b);
}

// 8 x bf16 in one 16-byte vector.
struct alignas(16) BF8 {
  uint32_t w[4];
};
LYNX_DEV void bf8_to_f(const BF8& v, float* f) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 p = unpack_bf16x2(v.w[i]);
    f[2 * i] = p.x;
    f[2 * i + 1] = p.y;
  }
}
LYNX_DEV BF8 f_to_bf8(const float* f) {
  BF8 v;
#pragma unroll
  for (int i = 0; i < 4; ++i) v.w[i] = pack_bf16x2(f[2 * i], f[2 * i + 1]);
  return v;
}

template <class T>
LYNX_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <class T>
LYNX_DEV T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// GPT-2 tanh GeLU with every rounding pinned (explicit __fmul_rn / __fadd_rn, no FMA
// contraction): the stand-alone GeLU kernel and the FC1 GEMM epilogue that fuses it must
// produce bit-identical activations, because a recomputed GeLU may come from either.
LYNX_DEV float gelu_exact(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float x3 = __fmul_rn(__fmul_rn(x, x), x);
  const float u = __fmul_rn(k0, __fadd_rn(x, __fmul_rn(k1, x3)));
  return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.f, tanhf(u)));
}

// d gelu(x) / dx for the same tanh GeLU. tanh(u) = 1 - 2 / (1 + e^{2u}) with the MUFU exp2 and
// reciprocal (error ~1e-6, far below the bf16 output's 2^-9): the accurate tanhf made the
// FC2-dX epilogue (GeLU backward fused, one evaluation per FC1 element) longer than its main loop
// (10.5 vs 6.7 ms per GPT-7B launch). Backward only: nothing regenerated depends on it, and the
// stand-alone gelu_bwd kernel uses this same function.
LYNX_DEV float gelu_grad_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float x2 = x * x;
  const float u = k0 * fmaf(k1 * x2, x, x);
  const float e = exp2f(fminf(2.8853900817779268f * u, 126.f));  // e^{2u}, clamped (t -> 1)
  const float t = 1.f - __fdividef(2.f, 1.f + e);
  return fmaf(0.5f * x * fmaf(-t, t, 1.f), k0 * fmaf(3.f * k1, x2, 1.f), 0.5f * (1.f + t));
}

// ---------------------------------------------------------------- Philox
// Philox-4x32-10 (Salmon et al., SC'11). Counter = (element group, stream),
// key = seed. Deterministic in (seed, stream, element) only, so a forward op
// and its recomputation draw identical dropout masks.
LYNX_DEV uint4 philox4x32_10(uint4 c, uint2 k) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += W0;
    k.y += W1;
  }
  return c;
}

// Four uniform 32-bit draws for elements [4*g, 4*g+4) of stream `stream`.
LYNX_DEV uint4 philox_group(uint64_t seed, uint64_t stream, uint64_t g) {
  uint4 c = make_uint4(static_cast<uint32_t>(g), static_cast<uint32_t>(g >> 32),
                       static_cast<uint32_t>(stream), static_cast<uint32_t>(stream >> 32));
  return philox4x32_10(c, make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)));
}

// ---------------------------------------------------------------- PTX: misc
LYNX_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

LYNX_DEV uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 r;\n\t.reg .pred p;\n\t"
      "elect.sync r|p, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}\n"
      : "=r"(pred));
  return pred;
}

// ---------------------------------------------------------------- mbarrier
LYNX_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
LYNX_DEV void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
LYNX_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
LYNX_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
LYNX_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
LYNX_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}

// Polling wait without a suspend-time hint: used where the arrivals come from
// the peer CTA of a cluster (remote arrive / multicast commit / 2SM TMA).
LYNX_DEV void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- TMA
LYNX_DEV void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}
LYNX_DEV void tma_load_2d(const void* desc, uint64_t* bar, void* smem, int c0, int c1, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(hint)
      : "memory");
}
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictNormal = 0x1000000000000000ull;
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;

// ---------------------------------------------------------------- tcgen05
template <uint32_t kCols>
LYNX_DEV void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <uint32_t kCols>
LYNX_DEV void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
LYNX_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
LYNX_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, fp32 accumulate).
LYNX_DEV void umma_f16(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate));
}
// Arrive on an mbarrier once all previously issued tcgen05 ops of this thread complete.
LYNX_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread.
LYNX_DEV void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
LYNX_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 bit, 32 consecutive columns per thread.
LYNX_DEV void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// UMMA shared-memory matrix descriptor (sm_100 "version 1"), SWIZZLE_128B.
// Byte offsets are encoded >> 4. See the canonical K-/MN-major layouts in
// DESIGN.md ("GEMM operand layouts").
LYNX_DEV uint64_t umma_desc_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // version = 1 (Blackwell)
  d |= 2ull << 61;  // layout = SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::f16: bf16 x bf16 -> f32, M x N, operand majors.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N, bool a_mn_major, bool b_mn_major) {
  return (1u << 4)                       // D format f32
         | (1u << 7)                     // A format bf16
         | (1u << 10)                    // B format bf16
         | ((a_mn_major ? 1u : 0u) << 15)  // A major
         | ((b_mn_major ? 1u : 0u) << 16)  // B major
         | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

// Dropout keep threshold for probability p on 16-bit draws (keep iff draw >= threshold).
__host__ __device__ inline uint32_t drop_threshold16(float p) {
  const double t = static_cast<double>(p) * 65536.0;
  return t >= 65536.0 ? 65536u : static_cast<uint32_t>(t);
}
LYNX_DEV uint32_t drop_threshold(float p) { return drop_threshold16(p); }

// keep-mask bits for elements [8v, 8v+8) of a dropout stream (shared by the dropout kernels
// and the fused GEMM residual epilogue: a regenerated activation must draw the same mask).
// One Philox-4x32-10 call per 8 elements: element j draws the 16-bit half j % 2 (low first) of
// word j / 2 of the counter (v, stream) — half the Philox work of one 32-bit draw per element,
// which bounded the dropout-backward kernels; p is resolved to 1/65536.
LYNX_DEV uint32_t keep_bits8(uint64_t seed, uint64_t stream, long long v, uint32_t thr) {
  const uint4 a = philox_group(seed, stream, static_cast<uint64_t>(v));
  const uint32_t w[4] = {a.x, a.y, a.z, a.w};
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) bits |= (((w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu) >= thr ? 1u : 0u) << j;
  return bits;
}

}  // namespace lynx
