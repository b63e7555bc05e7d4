// TMEM read / write bandwidth per SM on this GPU: W warps per CTA (one CTA per SM) each issue
// tcgen05.ld.32x32b.x32 (or .st) in a loop; prints bytes per SM clock. Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2406_08756_b200/csrc tmem_bw.cu -o tmem_bw && ./tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

using namespace lynx;

template <int MODE>  // 0 = ld x32 + wait each, 1 = 2 x ld x32 then wait, 2 = st x32, 3 = ld x32 + st x16 (attention-like)
__global__ void __launch_bounds__(512, 1) bw(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot + (static_cast<uint32_t>((warp % 4) * 32) << 16);
  const int col0 = (warp / 4) * 32 % 512;
  uint32_t acc = 0;
  uint32_t r[32], q[32];
  for (int i = 0; i < 32; ++i) q[i] = i;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t c = static_cast<uint32_t>((col0 + it * 64) % 512);
    if constexpr (MODE == 0) {
      tmem_ld32(tmem + c, r);
      tmem_ld_wait();
      #pragma unroll
      for (int k = 0; k < 32; ++k) acc += r[k];
    } else if constexpr (MODE == 1) {
      tmem_ld32(tmem + c, r);
      tmem_ld32(tmem + ((c + 32) % 512), q);
      tmem_ld_wait();
      #pragma unroll
      for (int k = 0; k < 32; ++k) acc += r[k] ^ q[k];
    } else if constexpr (MODE == 2) {
      q[0] = it;
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + c),
          "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]), "r"(q[4]), "r"(q[5]), "r"(q[6]), "r"(q[7]), "r"(q[8]), "r"(q[9]),
          "r"(q[10]), "r"(q[11]), "r"(q[12]), "r"(q[13]), "r"(q[14]), "r"(q[15]), "r"(q[16]), "r"(q[17]), "r"(q[18]),
          "r"(q[19]), "r"(q[20]), "r"(q[21]), "r"(q[22]), "r"(q[23]), "r"(q[24]), "r"(q[25]), "r"(q[26]), "r"(q[27]),
          "r"(q[28]), "r"(q[29]), "r"(q[30]), "r"(q[31])
          : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x % 32 == 0) atomicMax(cyc, static_cast<unsigned long long>(t1 - t0));
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(slot);
}

template <int MODE>
void run(int warps) {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 4096);
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(cyc, 0, 8);
    bw<MODE><<<148, warps * 32>>>(iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("err %s\n", cudaGetErrorString(e)); return; }
  }
  unsigned long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_ld = MODE == 1 ? 8192.0 : 4096.0;  // bytes per warp per iteration
  printf("mode %d warps %2d: %.1f B/clk/SM  (%.1f clk per warp-iteration)\n", MODE, warps,
         per_ld * iters * warps / c, static_cast<double>(c) / iters);
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 12, 16}) run<0>(w);
  for (int w : {4, 8, 16}) run<1>(w);
  for (int w : {4, 8, 16}) run<2>(w);
  return 0;
}
