// Issue rate of the softmax instruction mix per SM sub-partition: MUFU.EX2, F2FP (cvt.rn.bf16x2.f32),
// FFMA, and ex2 interleaved with F2FP. One CTA per SM, W warps, 8 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 xu_rate.cu -o xu_rate && ./xu_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(int iters, unsigned long long* cyc, float* sink) {
  float x[8];
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) x[i] = 0.001f * (threadIdx.x + i), u[i] = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (MODE == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      } else if constexpr (MODE == 1) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[(i + 1) & 7]));
        u[i] ^= r;
        x[i] = __uint_as_float(u[i] | 0x3f800000u);
      } else if constexpr (MODE == 2) {
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(x[i]));
      } else {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(r) : "f"(x[i]));
        u[i] += r;
      }
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x % 32 == 0) atomicMax(cyc, static_cast<unsigned long long>(t1 - t0));
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i] + u[i];
  if (s == 1.2345f) sink[threadIdx.x] = s;
}

template <int MODE>
void run(int warps, const char* what) {
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 4096 * 4);
  const int iters = 2048;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(cyc, 0, 8);
    k<MODE><<<148, warps * 32>>>(iters, cyc, sink);
    cudaDeviceSynchronize();
  }
  unsigned long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double inst = 8.0 * iters * warps / 4;  // warp-instructions (of the measured kind) per SMSP
  printf("%-14s warps %2d: %.3f warp-inst/clk/SMSP (%.2f clk each)\n", what, warps, inst / c, c / inst);
}

int main() {
  for (int w : {4, 8, 16, 32}) run<0>(w, "ex2");
  for (int w : {4, 8, 16, 32}) run<1>(w, "cvt.bf16x2");
  for (int w : {8, 16, 32}) run<2>(w, "ffma");
  for (int w : {8, 16, 32}) run<3>(w, "ex2+cvt");
  return 0;
}
