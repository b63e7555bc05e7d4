// tcgen05 / TMEM / TMA GEMM for sm_100a — the dense contractions of the GPT
// block (QKV, attention-output, FC1, FC2, LM head) in forward, dX and dW form.
//
//   C[M,N] (op)= A[M,K] * B[N,K]^T         bf16 inputs, fp32 accumulation in TMEM
//
// Each operand is either K-major (K contiguous) or MN-major (M resp. N
// contiguous), so the three training GEMMs need no transposes:
//   forward  Y  = X  W^T : A = X  [T,in]  K-major,  B = W [out,in] K-major
//   dX       dX = dY W   : A = dY [T,out] K-major,  B = W          MN-major
//   dW       dW = dY^T X : A = dY         MN-major, B = X [T,in]   MN-major
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer (one elected lane), 4-stage smem ring
//   warp 1      MMA issuer (one elected lane), tcgen05.mma.cta_group::1, 128xBNx16
//   warp 2      TMEM allocator (512 columns = 2 accumulator buffers)
//   warps 4..7  epilogue: tcgen05.ld -> registers -> bias / convert -> global
// The double-buffered accumulator lets tile i's epilogue overlap tile i+1's
// main loop. No split-K and no atomics: every output element is produced by
// exactly one CTA in a fixed K order, so results are bit-reproducible (the
// recompute bit-identity requirement of the north star).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "lynx_ops_internal.h"

namespace lynx {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle row of bf16
constexpr int kStages = 4;
constexpr int kThreads = 256;
// Tile raster: groups of 16 N-tiles, N fastest (group < 0). Measured on the 7B shapes, this
// halves DRAM re-reads against M-grouping (dX 21.7 -> 12.8 GB, dW 21.0 -> 13.0 GB, FC1 10.5 ->
// 6.6 GB per GEMM), and under the board power cap the saved HBM power is SM clock: +6-8%.
constexpr int kGroupM = -16;
constexpr int kStagingBytes = 4 * 2 * 4096;  // bf16 TMA-store staging: 4 epilogue warps x 2 buffers

struct Args {
  void* c;          // bf16 or f32 output
  const __nv_bfloat16* bias;  // optional, per output column (EPI_BF16 only)
  long long ldc;    // elements
  int M, N, K;
  int epi;          // EpiMode
  int group;        // raster: > 0 groups of `group` M-tiles (M fastest), < 0 groups of -group N-tiles
  uint64_t hint_a, hint_b;  // L2 cache policies of the A / B TMA loads
  uint64_t hint_c;          // L2 cache policy of the output TMA stores
  int tma_store;            // bf16 epilogue through smem + TMA store (else per-thread st.global)
  void* c2;                 // EPI_BF16_GELU second output
  const __nv_bfloat16* res;  // EPI_BF16_RESID residual
  float drop_p, drop_scale;
  uint32_t drop_thr;
  uint64_t drop_seed, drop_stream;
};

// Auxiliary-input epilogues. The 16-byte aux chunks are loaded up front (ld_aux, read-only
// path, all chunks of a round in flight together, overlapping the TMEM load) and combined here:
// loaded one by one between the staging stores, the loads serialized behind the smem writes and
// made the FC2-dX / FC2 / projection epilogues longer than their main loops.
LYNX_DEV BF8 ld_aux(const __nv_bfloat16* p) {
  BF8 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3])
               : "l"(p));
  return v;
}

// EPI_BF16_GELU_BWD on 8 outputs: dfc1 = dgelu * gelu'(fc1), fc1 = `xin` (from `res`).
LYNX_DEV BF8 gelu_bwd8(BF8 xin, const float* v) {
  float x[8], o[8];
  bf8_to_f(xin, x);
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j] = v[j] * gelu_grad_f(x[j]);
  return f_to_bf8(o);
}

// EPI_BF16_RESID on 8 outputs (columns col..col+7 of `row`): out = res + dropout(bf16(v)), res = `rin`.
LYNX_DEV BF8 resid_dropout8(const Args& args, long long row, int col, BF8 rin, const float* v) {
  float y[8], r[8], o[8];
  bf8_to_f(f_to_bf8(v), y);  // the projection output is rounded to bf16 first, as in the two-kernel path
  bf8_to_f(rin, r);
  const uint32_t keep =
      args.drop_p > 0.f ? keep_bits8(args.drop_seed, args.drop_stream, (row * args.ldc + col) / 8, args.drop_thr) : 0xFFu;
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j] = ((keep >> j) & 1u) ? __fmaf_rn(y[j], args.drop_scale, r[j]) : r[j];
  return f_to_bf8(o);
}

template <int BN>
struct Smem {
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBytes = kStages * kStageBytes + kStagingBytes + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ void tile_coords(int tile, int m_tiles, int n_tiles, int group_size, int& mt, int& nt) {
  if (group_size < 0) {  // groups of G N-tiles, N fastest inside a group
    const int G = -group_size;
    const int per_group = G * m_tiles;
    const int first_n = tile / per_group * G;
    const int gn = min(G, n_tiles - first_n);
    const int in_group = tile % per_group;
    nt = first_n + in_group % gn;
    mt = in_group / gn;
    return;
  }
  const int per_group = group_size * n_tiles;
  const int first_m = tile / per_group * group_size;
  const int gm = min(group_size, m_tiles - first_m);
  const int in_group = tile % per_group;
  mt = first_m + in_group % gm;
  nt = in_group / gm;
}

// TMEM accumulator row (this thread's output row) -> global, 32 columns per
// round: the fp32 read of the accumulate epilogue is issued before the TMEM
// load is awaited so the two latencies overlap.
template <int kCols>
LYNX_DEV void epilogue_row(const Args& args, uint32_t t_row, long long row, int n0) {
  if (args.epi >= 98) return;  // timing probes: no epilogue
#pragma unroll 1
  for (int c = 0; c < kCols; c += 32) {
    uint32_t r[32];
    float4 prev[8];
    BF8 prevb[4];
    float* outf = reinterpret_cast<float*>(args.c) + row * args.ldc + n0 + c;
    BF8* outb = reinterpret_cast<BF8*>(reinterpret_cast<__nv_bfloat16*>(args.c) + row * args.ldc + n0 + c);
    // Partial edge tiles (M or N not a tile multiple, 128-aligned): every lane still runs the
    // warp-collective TMEM load; out-of-range rows / 32-column chunks are not read or written.
    const bool in = row < args.M && n0 + c < args.N;
    if (in && args.epi == EPI_ACC_F32) {
#pragma unroll
      for (int i = 0; i < 8; ++i) prev[i] = reinterpret_cast<const float4*>(outf)[i];
    } else if (in && args.epi == EPI_ACC_BF16) {
#pragma unroll
      for (int i = 0; i < 4; ++i) prevb[i] = outb[i];
    }
    tmem_ld32(t_row + c, r);
    tmem_ld_wait();
    if (!in) continue;
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
    if (args.epi == EPI_ACC_BF16) {  // bf16 gradient accumulation (16 B / parameter model states)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float pf[8];
        bf8_to_f(prevb[i], pf);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[8 * i + j] += pf[j];
        outb[i] = f_to_bf8(v + 8 * i);
      }
      continue;
    }
    if (args.epi == EPI_ACC_F32 || args.epi == EPI_STORE_F32) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 o = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        if (args.epi == EPI_ACC_F32) {
          o.x += prev[i].x;
          o.y += prev[i].y;
          o.z += prev[i].z;
          o.w += prev[i].w;
        }
        reinterpret_cast<float4*>(outf)[i] = o;
      }
    } else {
      if (args.bias) {
        const BF8* bp = reinterpret_cast<const BF8*>(args.bias + n0 + c);
        float b[32];
#pragma unroll
        for (int i = 0; i < 4; ++i) bf8_to_f(bp[i], b + 8 * i);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += b[i];
      }
      BF8* o = reinterpret_cast<BF8*>(reinterpret_cast<__nv_bfloat16*>(args.c) + row * args.ldc + n0 + c);
      if (args.epi == EPI_BF16_RESID || args.epi == EPI_BF16_GELU_BWD) {
        BF8 aux[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) aux[i] = ld_aux(args.res + row * args.ldc + n0 + c + 8 * i);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          o[i] = args.epi == EPI_BF16_RESID ? resid_dropout8(args, row, n0 + c + 8 * i, aux[i], v + 8 * i)
                                            : gelu_bwd8(aux[i], v + 8 * i);
        continue;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) o[i] = f_to_bf8(v + 8 * i);
      if (args.epi == EPI_BF16_GELU) {
        BF8* o2 = reinterpret_cast<BF8*>(reinterpret_cast<__nv_bfloat16*>(args.c2) + row * args.ldc + n0 + c);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float t[8];
          bf8_to_f(f_to_bf8(v + 8 * i), t);  // GeLU of the bf16-rounded FC1 output, as the GeLU kernel
#pragma unroll
          for (int j = 0; j < 8; ++j) t[j] = gelu_exact(t[j]);
          o2[i] = f_to_bf8(t);
        }
      }
    }
  }
}

// bf16 epilogue through shared memory and TMA stores: each epilogue warp stages its
// 32 rows x 64 columns (SW128 layout: 16-byte chunk c of row r at c ^ (r & 7), bank-conflict
// free) in one of two 4 KB buffers and one lane issues a cp.async.bulk.tensor store of the
// box. Full 128-byte lines reach L2 (the per-thread st.global path writes 16-byte pieces).

LYNX_DEV void tma_store_2d(const CUtensorMap* desc, const void* smem, int c0, int c1, uint64_t hint) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                   reinterpret_cast<uint64_t>(desc)),
               "r"(smem_u32(smem)), "r"(c0), "r"(c1), "l"(hint)
               : "memory");
}
LYNX_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
LYNX_DEV void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
LYNX_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
LYNX_DEV void bulk_wait_all_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// EPI_BF16_RESID / EPI_BF16_GELU_BWD: the auxiliary tile (residual, or the FC1 output) comes in by
// TMA into the same 4 KB staging buffer the output leaves from (tm_c2 maps `res` with C's box):
// each lane reads its row, writes the result in place, one lane TMA-stores the box, then loads
// the next round's aux box into the other buffer. Full-line loads: the per-thread 16-byte row
// reads they replace made these epilogues longer than the main loop (FC2-dX with the GeLU
// backward: 10.5 vs 6.7 ms per GPT-7B launch). abar: this warp's two buffer barriers, aphase:
// their parities (bit b for buffer b).
template <int kCols>
LYNX_DEV void epilogue_aux_tma(const Args& args, const CUtensorMap* tm_c, const CUtensorMap* tm_aux, uint32_t t_row,
                               int row0, int n0, int lane, uint8_t* staging, int& sbuf, uint64_t* abar,
                               uint32_t& aphase) {
  const bool resid = args.epi == EPI_BF16_RESID;
  if (lane == 0) {  // round 0: the store issued from this buffer two rounds ago has read it
    bulk_wait_read1();
    mbar_arrive_expect_tx(&abar[sbuf], 4096);
    tma_load_2d(tm_aux, &abar[sbuf], staging + sbuf * 4096, n0, row0, kEvictFirst);
  }
#pragma unroll 1
  for (int c = 0; c < kCols; c += 64) {
    uint32_t r[64];
    tmem_ld32(t_row + c, r);
    tmem_ld32(t_row + c + 32, r + 32);
    uint8_t* st = staging + sbuf * 4096;
    mbar_wait(&abar[sbuf], (aphase >> sbuf) & 1u);
    aphase ^= 1u << sbuf;
    tmem_ld_wait();
    float v[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
    if (args.bias) {
      const BF8* bp = reinterpret_cast<const BF8*>(args.bias + n0 + c);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float b[8];
        bf8_to_f(bp[i], b);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[8 * i + j] += b[j];
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      BF8* q = reinterpret_cast<BF8*>(st + lane * 128 + ((i ^ (lane & 7)) << 4));
      *q = resid ? resid_dropout8(args, row0 + lane, n0 + c + 8 * i, *q, v + 8 * i) : gelu_bwd8(*q, v + 8 * i);
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tm_c, st, n0 + c, row0, args.hint_c);
      bulk_commit();
      if (c + 64 < kCols) {  // prefetch the next round's aux box into the other buffer
        bulk_wait_read1();   // ... whose store (the previous round) has been read
        mbar_arrive_expect_tx(&abar[sbuf ^ 1], 4096);
        tma_load_2d(tm_aux, &abar[sbuf ^ 1], staging + (sbuf ^ 1) * 4096, n0 + c + 64, row0, kEvictFirst);
      }
    }
    sbuf ^= 1;
  }
}

template <int kCols>
LYNX_DEV void epilogue_tile_tma(const Args& args, const CUtensorMap* tm_c, const CUtensorMap* tm_c2, uint32_t t_row,
                                int row0, int n0, int lane, uint8_t* staging, int& sbuf) {
  const bool gelu = args.epi == EPI_BF16_GELU;
  const bool aux_in = args.epi == EPI_BF16_RESID || args.epi == EPI_BF16_GELU_BWD;
#pragma unroll 1
  for (int c = 0; c < kCols; c += 64) {
    uint32_t r[64];
    tmem_ld32(t_row + c, r);
    tmem_ld32(t_row + c + 32, r + 32);
    BF8 aux[8];
    if (aux_in) {  // all 8 chunks in flight while the TMEM load completes
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        // auxiliary inputs are read only in range (the TMA store clips partial edge tiles)
        const bool in = row0 + lane < args.M && n0 + c + 8 * i < args.N;
        aux[i] = in ? ld_aux(args.res + static_cast<long long>(row0 + lane) * args.ldc + n0 + c + 8 * i)
                    : BF8{{0u, 0u, 0u, 0u}};
      }
    }
    tmem_ld_wait();
    float v[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
    if (args.bias) {
      const BF8* bp = reinterpret_cast<const BF8*>(args.bias + n0 + c);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float b[8];
        bf8_to_f(bp[i], b);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[8 * i + j] += b[j];
      }
    }
    if (gelu) {  // both buffers per round: c in buffer 0, gelu(c) in buffer 1
      if (lane == 0) bulk_wait_all_read();
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const BF8 cv = f_to_bf8(v + 8 * i);
        *reinterpret_cast<BF8*>(staging + lane * 128 + ((i ^ (lane & 7)) << 4)) = cv;
        float t[8];
        bf8_to_f(cv, t);  // GeLU of the bf16-rounded FC1 output, exactly as the GeLU kernel computes it
#pragma unroll
        for (int j = 0; j < 8; ++j) t[j] = gelu_exact(t[j]);
        *reinterpret_cast<BF8*>(staging + 4096 + lane * 128 + ((i ^ (lane & 7)) << 4)) = f_to_bf8(t);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tm_c, staging, n0 + c, row0, args.hint_c);
        tma_store_2d(tm_c2, staging + 4096, n0 + c, row0, args.hint_c);
        bulk_commit();
      }
      continue;
    }
    uint8_t* st = staging + sbuf * 4096;
    if (lane == 0) bulk_wait_read1();  // the store issued from this buffer two rounds ago has read it
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      *reinterpret_cast<BF8*>(st + lane * 128 + ((i ^ (lane & 7)) << 4)) =
          args.epi == EPI_BF16_RESID      ? resid_dropout8(args, row0 + lane, n0 + c + 8 * i, aux[i], v + 8 * i)
          : args.epi == EPI_BF16_GELU_BWD ? gelu_bwd8(aux[i], v + 8 * i)
                                          : f_to_bf8(v + 8 * i);
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tm_c, st, n0 + c, row0, args.hint_c);
      bulk_commit();
    }
    sbuf ^= 1;
  }
}

template <bool kAMN, bool kBMN, int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_c2, Args args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  using S = Smem<BN>;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + kStages * S::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + kStagingBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  uint64_t* aux_bar = tmem_empty + 3;  // 4 epilogue warps x 2 aux-load barriers (after the TMEM slot)

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int m_tiles = args.M / BM;
  const int n_tiles = args.N / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int k_blocks = args.K / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 4);  // one elected lane per epilogue warp
    }
    for (int b = 0; b < 8; ++b) mbar_init(&aux_bar[b], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_base_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int mt, nt;
        tile_coords(tile, m_tiles, n_tiles, args.group, mt, nt);
        const int m0 = mt * BM, n0 = nt * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::kStageBytes;
          uint8_t* sb = sa + S::kABytes;
          if (args.epi == 98) {  // timing probe: MMA pipeline without operand traffic
            mbar_arrive(&full[stage]);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          mbar_arrive_expect_tx(&full[stage], S::kStageBytes);
          const int k0 = kb * BK;
          if constexpr (!kAMN) {
            tma_load_2d(&tm_a, &full[stage], sa, k0, m0, args.hint_a);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(&tm_a, &full[stage], sa + j * (64 * BK * 2), m0 + 64 * j, k0, args.hint_a);
          }
          if constexpr (!kBMN) {
            tma_load_2d(&tm_b, &full[stage], sb, k0, n0, args.hint_b);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(&tm_b, &full[stage], sb + j * (64 * BK * 2), n0 + 64 * j, k0, args.hint_b);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, kAMN, kBMN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < k_blocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(smem + stage * S::kStageBytes);
          const uint32_t sb = sa + S::kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: advance 16 elements (32 B) inside the swizzled 128-B row.
            // MN-major: advance 16 K-rows (16 x 128 B) -> two 1024-B swizzle atoms.
            const uint64_t da = kAMN ? umma_desc_sw128(sa + k * 2048, 64 * BK * 2, 1024)
                                     : umma_desc_sw128(sa + k * 32, 16, 1024);
            const uint64_t db = kBMN ? umma_desc_sw128(sb + k * 2048, 64 * BK * 2, 1024)
                                     : umma_desc_sw128(sb + k * 32, 16, 1024);
            umma_f16(d_tmem, da, db, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (kb == k_blocks - 1) umma_commit(&tmem_full[acc]);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;  // == warp % 4: TMEM lane quadrant
    const bool tma_out = (args.epi == EPI_BF16 || args.epi == EPI_BF16_GELU || args.epi == EPI_BF16_RESID ||
                          args.epi == EPI_BF16_GELU_BWD) &&
                         args.tma_store;
    const bool aux_tma = tma_out && args.tma_store == 2;  // aux input by TMA (tm_c2 maps `res`)
    uint32_t aphase = 0;
    uint8_t* my_staging = staging + ew * 8192;
    int sbuf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int mt, nt;
      tile_coords(tile, m_tiles, n_tiles, args.group, mt, nt);
      const int row = mt * BM + ew * 32 + lane;
      const int n0 = nt * BN;
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN;
      if (tma_out)
        if (aux_tma)
          epilogue_aux_tma<BN>(args, &tm_c, &tm_c2, t_row, mt * BM + ew * 32, n0, lane, my_staging, sbuf,
                               aux_bar + 2 * ew, aphase);
        else
          epilogue_tile_tma<BN>(args, &tm_c, &tm_c2, t_row, mt * BM + ew * 32, n0, lane, my_staging, sbuf);
      else
        epilogue_row<BN>(args, t_row, row, n0);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  if (warp >= 4 && lane == 0) bulk_wait_all();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem_base);
}

// ---------------------------------------------------------------- 2-CTA (cta_group::2)
// A CTA pair (one cluster, two SMs of a TPC) computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (UMMA M = 256): each CTA stages its 128 rows of A
// and its 128 columns of B, the leader issues the MMA that reads both CTAs'
// shared memory, and each CTA's TMEM holds its own 128 accumulator rows.
// Per SM this moves (128 + 128) instead of (128 + 256) operand rows per
// 128 x 256 outputs — 1.5x less L2->SM traffic than the 1-CTA tile.
namespace pair {

// kSub = 1: 256 x 256 pair tile, TMEM double-buffered (the epilogue of tile i overlaps tile i+1).
// kSub = 2: 512 x 256 pair tile ("wide"): each CTA stages 256 rows of A and 128 columns of B per
// k-block and issues two M = 256 MMAs that share the B stage, so L2->SM operand traffic per
// FLOP drops by 25% (48 KB instead of 64 KB per 256x256x64 of work per CTA); the two
// accumulators fill all 512 TMEM columns, so TMEM is single-buffered.
constexpr int kTileN = 256, kHalf = 128;
template <int kSub>
struct Cfg {
  static constexpr int kRowsCTA = 128 * kSub;           // A rows staged per CTA
  static constexpr int kTileM = 2 * kRowsCTA;           // pair tile rows
  static constexpr int kABytes = kRowsCTA * BK * 2;     // per CTA
  static constexpr int kBBytes = kHalf * BK * 2;        // per CTA (half of N)
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = kSub == 1 ? 6 : 4;
  static constexpr int kAcc = 2 / kSub;                  // TMEM accumulator buffers
  static constexpr int kSmemBytes = kStages * kStageBytes + kStagingBytes + 1024 + 256;
};
constexpr int kSmemBytes = Cfg<1>::kSmemBytes;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;
#ifdef LYNX_PAIR_SPIN
#define PAIR_WAIT mbar_wait_spin
#else
#define PAIR_WAIT mbar_wait  // try_wait with a suspend-time hint: waiting warps park instead of polling
#endif  // shared::cluster address of the even (leader) CTA

LYNX_DEV uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
LYNX_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
LYNX_DEV void arrive_leader(uint64_t* bar) {  // remote (or local) arrive on the leader's barrier
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerMask)
               : "memory");
}
LYNX_DEV void tma_load_2sm(const void* desc, uint64_t* bar, void* smem, int c0, int c1, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1), "l"(hint)
      : "memory");
}
LYNX_DEV void umma_f16_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
LYNX_DEV void umma_commit_pair(uint64_t* bar) {  // arrive on `bar` in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

template <bool kAMN, bool kBMN, int kSub>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                 const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_c2, Args args) {
  using C = Cfg<kSub>;
  constexpr int kStages = C::kStages, kStageBytes = C::kStageBytes, kABytes = C::kABytes, kTileM = C::kTileM;
  constexpr int kRowsCTA = C::kRowsCTA, kAcc = C::kAcc;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + kStages * kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + kStagingBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  uint64_t* aux_bar = tmem_empty + 3;  // 4 epilogue warps x 2 aux-load barriers (after the TMEM slot)

  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m_tiles = (args.M + kTileM - 1) / kTileM, n_tiles = (args.N + kTileN - 1) / kTileN;
  const int num_tiles = m_tiles * n_tiles;
  const int k_blocks = args.K / BK;
  const int cluster = blockIdx.x / 2, n_clusters = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);   // the leader's expect_tx arrival (the peer contributes bytes only)
      mbar_init(&empty[s], 1);  // the leader's multicast commit
    }
    for (int b = 0; b < kAcc; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 8);  // 4 epilogue warps x 2 CTAs
    }
    for (int b = 0; b < 8; ++b) mbar_init(&aux_bar[b], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cluster; tile < num_tiles; tile += n_clusters) {
        int mt, nt;
        tile_coords(tile, m_tiles, n_tiles, args.group, mt, nt);
        const int m0 = mt * kTileM + rank * kRowsCTA, n0 = nt * kTileN + rank * kHalf;
        for (int kb = 0; kb < k_blocks; ++kb) {
          PAIR_WAIT(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStageBytes;
          uint8_t* sb = sa + kABytes;
          if (args.epi == 98) {  // timing probe: MMA pipeline without operand traffic
            if (leader) mbar_arrive(&full[stage]);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          if (args.epi == 97) {  // timing probe: per-CTA TMA to the CTA's own barrier (leader waits on its own)
            const int k0 = kb * BK;
            if (leader) mbar_arrive_expect_tx(&full[stage], kStageBytes);
            tma_load_2d(&tm_a, &full[stage], sa, k0, m0, kEvictNormal);
            tma_load_2d(&tm_b, &full[stage], sb, k0, n0, kEvictNormal);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          // Only the leader arms the stage barrier (both CTAs' bytes). The peer's
          // complete_tx may land before the arm — the transaction count is allowed
          // to go negative while the leader's arrival is still pending — so the
          // peer needs no remote arrive (and no cluster-scope fence) per stage.
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kStageBytes);
          const int k0 = kb * BK;
          if constexpr (!kAMN) {
#pragma unroll
            for (int sub = 0; sub < kSub; ++sub)
              tma_load_2sm(&tm_a, &full[stage], sa + sub * (kHalf * BK * 2), k0, m0 + sub * kHalf, args.hint_a);
          } else {
#pragma unroll
            for (int j = 0; j < 2 * kSub; ++j)
              tma_load_2sm(&tm_a, &full[stage], sa + j * (64 * BK * 2), m0 + 64 * j, k0, args.hint_a);
          }
          if constexpr (!kBMN) {
            tma_load_2sm(&tm_b, &full[stage], sb, k0, n0, args.hint_b);
          } else {
            tma_load_2sm(&tm_b, &full[stage], sb, n0, k0, args.hint_b);
            tma_load_2sm(&tm_b, &full[stage], sb + 64 * BK * 2, n0 + 64, k0, args.hint_b);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc = umma_idesc_bf16(256, kTileN, kAMN, kBMN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = cluster; tile < num_tiles; tile += n_clusters) {
        PAIR_WAIT(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kTileN * kSub;
        for (int kb = 0; kb < k_blocks; ++kb) {
          PAIR_WAIT(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = smem_u32(smem + stage * kStageBytes);
            const uint32_t sb = sa + kABytes;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t db = kBMN ? umma_desc_sw128(sb + k * 2048, 64 * BK * 2, 1024)
                                       : umma_desc_sw128(sb + k * 32, 16, 1024);
#pragma unroll
              for (int sub = 0; sub < kSub; ++sub) {  // 128-row sub-tile `sub` of each CTA's A stage
                const uint32_t sas = sa + sub * (kHalf * BK * 2);
                const uint64_t da = kAMN ? umma_desc_sw128(sas + k * 2048, 64 * BK * 2, 1024)
                                         : umma_desc_sw128(sas + k * 32, 16, 1024);
                umma_f16_pair(d_tmem + sub * kTileN, da, db, idesc, (kb > 0 || k > 0) ? 1u : 0u);
              }
            }
            umma_commit_pair(&empty[stage]);
            if (kb == k_blocks - 1) umma_commit_pair(&tmem_full[acc]);
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (++acc == kAcc) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const bool tma_out = (args.epi == EPI_BF16 || args.epi == EPI_BF16_GELU || args.epi == EPI_BF16_RESID ||
                          args.epi == EPI_BF16_GELU_BWD) &&
                         args.tma_store;
    const bool aux_tma = tma_out && args.tma_store == 2;  // aux input by TMA (tm_c2 maps `res`)
    uint32_t aphase = 0;
    uint8_t* my_staging = staging + ew * 8192;
    int sbuf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = cluster; tile < num_tiles; tile += n_clusters) {
      int mt, nt;
      tile_coords(tile, m_tiles, n_tiles, args.group, mt, nt);
      const int n0 = nt * kTileN;
      PAIR_WAIT(&tmem_full[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int sub = 0; sub < kSub; ++sub) {
        const int row0 = mt * kTileM + rank * kRowsCTA + sub * kHalf + ew * 32;
        const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + (acc * kSub + sub) * kTileN;
        if (tma_out)
          if (aux_tma)
            epilogue_aux_tma<kTileN>(args, &tm_c, &tm_c2, t_row, row0, n0, lane, my_staging, sbuf, aux_bar + 2 * ew,
                                     aphase);
          else
            epilogue_tile_tma<kTileN>(args, &tm_c, &tm_c2, t_row, row0, n0, lane, my_staging, sbuf);
        else
          epilogue_row<kTileN>(args, t_row, row0 + lane, n0);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(&tmem_empty[acc]);
      if (++acc == kAcc) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  if (warp >= 4 && lane == 0) bulk_wait_all();
  tc_fence_before();
  cluster_sync();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(512));
}

}  // namespace pair

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 tensor map: `inner` contiguous elements per row, `outer` rows,
// row pitch `ld` elements, box {box_inner, box_outer}, 128-B swizzle.
bool make_map(CUtensorMap* m, const void* base, long long inner, long long outer, long long ld, int box_inner,
              int box_outer) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Tile raster group (L2 reuse); LYNX_GEMM_GROUP overrides the default for experiments.
int group_size() {
  static int g = [] {
    const char* e = std::getenv("LYNX_GEMM_GROUP");
    const int v = e ? std::atoi(e) : 0;
    return v != 0 ? v : kGroupM;
  }();
  return g;
}

// L2 policies of the A / B operand loads; LYNX_GEMM_HINT="ab" with a, b in {n, f, l}
// (evict_normal / evict_first / evict_last) overrides the default for experiments.
// L2 policies, LYNX_GEMM_HINT="<A><B><C>" with n(ormal) / l(ast) / f(irst). Default: normal loads,
// evict-first output stores (the 2-4 GB an epilogue writes then no longer pushes operand tiles out of
// L2: FC1 forward DRAM reads 5.1 -> 4.35 GB per launch, ncu).
uint64_t cache_hint(int operand) {
  static const char* e = std::getenv("LYNX_GEMM_HINT");
  const char c = (e && e[0] && e[1] && (operand < 2 || e[2])) ? e[operand] : (operand == 2 ? 'f' : 'n');
  return c == 'l' ? kEvictLast : (c == 'f' ? kEvictFirst : kEvictNormal);
}

// bf16 epilogue via TMA stores (default on; LYNX_GEMM_TMA_STORE=0 selects per-thread stores).
// LYNX_GEMM_AUX_TMA=0: the residual / FC1 input of the aux epilogues read per thread instead of by TMA.
bool aux_tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LYNX_GEMM_AUX_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool tma_store_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LYNX_GEMM_TMA_STORE");
    return !(e && e[0] == '0');
  }();
  return on;
}

Args make_args(const GemmDesc& g, bool tma_out) {
  Args a{g.c, g.bias, g.ldc, g.M, g.N, g.K, g.epi, group_size(), cache_hint(0), cache_hint(1), cache_hint(2),
         tma_out ? 1 : 0, g.c2,
         g.res, g.drop_p, g.drop_p > 0.f ? 1.f / (1.f - g.drop_p) : 1.f, 0u, g.drop_seed, g.drop_stream};
  a.drop_thr = drop_threshold16(g.drop_p);  // the dropout kernels' threshold (common.cuh)
  return a;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <bool kAMN, bool kBMN, int BN>
int launch(const GemmDesc& g, cudaStream_t stream, int max_ctas) {
  CUtensorMap ma, mb;
  // A: K-major -> rows = M, row = K contiguous.  MN-major -> rows = K, row = M contiguous.
  bool ok = kAMN ? make_map(&ma, g.a, g.M, g.K, g.lda, 64, BK) : make_map(&ma, g.a, g.K, g.M, g.lda, BK, BM);
  ok = ok && (kBMN ? make_map(&mb, g.b, g.N, g.K, g.ldb, 64, BK) : make_map(&mb, g.b, g.K, g.N, g.ldb, BK, BN));
  if (!ok) return set_error("cuTensorMapEncodeTiled failed (alignment or driver entry point)");
  auto kern = gemm_kernel<kAMN, kBMN, BN>;
  const int smem = Smem<BN>::kBytes;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_set = true;
  }
  CUtensorMap mc = ma, mc2 = ma;
  const bool bf16_out =
      g.epi == EPI_BF16 || g.epi == EPI_BF16_GELU || g.epi == EPI_BF16_RESID || g.epi == EPI_BF16_GELU_BWD;
  bool tma_out = bf16_out && tma_store_enabled() && make_map(&mc, g.c, g.N, g.M, g.ldc, 64, 32);
  if (tma_out && g.epi == EPI_BF16_GELU) tma_out = make_map(&mc2, g.c2, g.N, g.M, g.ldc, 64, 32);
  const bool aux_tma = tma_out && (g.epi == EPI_BF16_RESID || g.epi == EPI_BF16_GELU_BWD) && aux_tma_enabled() &&
                       make_map(&mc2, g.res, g.N, g.M, g.ldc, 64, 32);
  Args args = make_args(g, tma_out);
  if (aux_tma) args.tma_store = 2;
  const int tiles = (g.M / BM) * (g.N / BN);
  int grid = tiles < num_sms() ? tiles : num_sms();
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  kern<<<grid, kThreads, smem, stream>>>(ma, mb, mc, mc2, args);
  return check_launch("gemm_tcgen05");
}

template <bool kAMN, bool kBMN, int kSub>
int launch_pair(const GemmDesc& g, cudaStream_t stream, int max_ctas) {
  using C = pair::Cfg<kSub>;
  CUtensorMap ma, mb;
  // each CTA loads kSub 128-row boxes of A and a 128-column half of the pair's 256 B columns
  bool ok = kAMN ? make_map(&ma, g.a, g.M, g.K, g.lda, 64, BK) : make_map(&ma, g.a, g.K, g.M, g.lda, BK, pair::kHalf);
  ok = ok && (kBMN ? make_map(&mb, g.b, g.N, g.K, g.ldb, 64, BK) : make_map(&mb, g.b, g.K, g.N, g.ldb, BK, pair::kHalf));
  if (!ok) return set_error("cuTensorMapEncodeTiled failed (alignment or driver entry point)");
  auto kern = pair::gemm2_kernel<kAMN, kBMN, kSub>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    attr_set = true;
  }
  CUtensorMap mc = ma, mc2 = ma;
  const bool bf16_out =
      g.epi == EPI_BF16 || g.epi == EPI_BF16_GELU || g.epi == EPI_BF16_RESID || g.epi == EPI_BF16_GELU_BWD;
  bool tma_out = bf16_out && tma_store_enabled() && make_map(&mc, g.c, g.N, g.M, g.ldc, 64, 32);
  if (tma_out && g.epi == EPI_BF16_GELU) tma_out = make_map(&mc2, g.c2, g.N, g.M, g.ldc, 64, 32);
  const bool aux_tma = tma_out && (g.epi == EPI_BF16_RESID || g.epi == EPI_BF16_GELU_BWD) && aux_tma_enabled() &&
                       make_map(&mc2, g.res, g.N, g.M, g.ldc, 64, 32);
  Args args = make_args(g, tma_out);
  if (aux_tma) args.tma_store = 2;
  const int tiles = ((g.M + C::kTileM - 1) / C::kTileM) * ((g.N + pair::kTileN - 1) / pair::kTileN);
  int clusters = num_sms() / 2;
  if (max_ctas > 0) clusters = max_ctas / 2 > 0 ? max_ctas / 2 : 1;
  if (tiles < clusters) clusters = tiles;
  kern<<<2 * clusters, kThreads, C::kSmemBytes, stream>>>(ma, mb, mc, mc2, args);
  return check_launch("gemm_tcgen05_pair");
}

template <int kSub>
int dispatch_pair(const GemmDesc& g, cudaStream_t stream, int max_ctas) {
  if (!g.a_mn && !g.b_mn) return launch_pair<false, false, kSub>(g, stream, max_ctas);
  if (!g.a_mn && g.b_mn) return launch_pair<false, true, kSub>(g, stream, max_ctas);
  if (g.a_mn && !g.b_mn) return launch_pair<true, false, kSub>(g, stream, max_ctas);
  return launch_pair<true, true, kSub>(g, stream, max_ctas);
}

}  // namespace gemm

namespace {
// -1 (default): the wide 512x256 CTA-pair kernel for K >= 8192, else the 256x256 pair kernel for
// K-major A, else the single-CTA kernel (pair kernels accept 128-aligned edge tiles). 0: single-CTA only.
// 1: 256x256 pair wherever the shape allows. 2: wide pair, then 256x256 pair, then single.
// LYNX_GEMM_MODE sets the initial mode (experiments).
int g_gemm_mode = [] {
  const char* e = std::getenv("LYNX_GEMM_MODE");
  return e ? std::atoi(e) : -1;
}();
}

void gemm_set_mode(int mode) { g_gemm_mode = mode; }

int gemm_run(const GemmDesc& g, cudaStream_t stream, int max_ctas) {
  using namespace gemm;
  if (g.M % BM || g.K % BK || g.M <= 0 || g.N <= 0 || g.K <= 0)
    return set_error("gemm: M must be a multiple of 128 and K of 64");
  if (g.N % 128) return set_error("gemm: N must be a multiple of 128");
  const bool bf16_out = g.epi == EPI_BF16 || g.epi == EPI_ACC_BF16 || g.epi == EPI_BF16_GELU || g.epi == EPI_BF16_RESID ||
                        g.epi == EPI_BF16_GELU_BWD;
  if (g.epi == EPI_BF16_GELU && !g.c2) return set_error("gemm: the GeLU epilogue needs a second output");
  if ((g.epi == EPI_BF16_RESID || g.epi == EPI_BF16_GELU_BWD) && !g.res)
    return set_error("gemm: this epilogue needs its auxiliary input");
  if ((bf16_out && g.ldc % 8) || (!bf16_out && g.ldc % 4))
    return set_error("gemm: ldc must keep 16-byte row alignment");
  const int mode = g_gemm_mode;
  // CTA-pair kernels take 128-aligned M and N; partial edge tiles are zero-filled by TMA on load
  // and clipped by the TMA store / bounds-checked in the direct epilogue (e.g. the LM head's
  // logits, N = V = 50304 = 196.5 x 256).
  auto tiles_of = [&](int tm) { return ((g.M + tm - 1) / tm) * ((g.N + pair::kTileN - 1) / pair::kTileN); };
  // The wide tile pays a non-overlapped epilogue per tile (TMEM single-buffered), so by
  // default it is used for long reductions only (K >= 8192: FC2 forward, FC1/QKV dX, all dW),
  // where it measures 6-11% faster under the power cap (less L2->SM traffic).
  if ((mode == 2 || (mode == -1 && g.K >= 8192)) && tiles_of(pair::Cfg<2>::kTileM) >= 64)
    return dispatch_pair<2>(g, stream, max_ctas);
  // MN-major A with a short reduction (the LM head's weight gradient per 4096-token chunk):
  // the pair kernel measures 10% faster than the single-CTA one under the power cap
  // (tools/gemm_sustained.py headdw: 1.32 vs 1.46 ms).
  const bool want_pair = mode == 1 || mode == 2 || mode == -1;
  if (want_pair && tiles_of(pair::Cfg<1>::kTileM) >= 32) return dispatch_pair<1>(g, stream, max_ctas);
  const bool wide = g.N % 256 == 0;
#define LYNX_GEMM_CASE(AMN, BMN)                                                             \
  if (g.a_mn == AMN && g.b_mn == BMN)                                                         \
    return wide ? launch<AMN, BMN, 256>(g, stream, max_ctas) : launch<AMN, BMN, 128>(g, stream, max_ctas);
  LYNX_GEMM_CASE(false, false)
  LYNX_GEMM_CASE(false, true)
  LYNX_GEMM_CASE(true, false)
  LYNX_GEMM_CASE(true, true)
#undef LYNX_GEMM_CASE
  return set_error("gemm: bad operand majors");
}

}  // namespace lynx
