// Experiment: MUFU.EX2 throughput on B200 for f32, f16x2 and bf16x2 operands
// (elements per SM per clock), one warp-instruction stream per variant.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

template <int V>
__global__ void k(uint32_t *out, int iters, long long *clk) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = 0x3c003c00u ^ (threadIdx.x * 7 + i);   // small values
  if (V == 0)
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(-0.001f * (float)(threadIdx.x + i));
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (V == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[i]));
      if (V == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r[i]));
      if (V == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r[i]));
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  uint32_t *out; long long *clk;
  cudaMalloc(&out, 148 * 1024 * 4 * 8);
  cudaMalloc(&clk, 8);
  const int iters = 4096;
  const char *names[3] = {"ex2.approx.ftz.f32", "ex2.approx.f16x2", "ex2.approx.ftz.bf16x2"};
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      int threads = 1024;
      if (v == 0) k<0><<<148, threads>>>(out, iters, clk);
      if (v == 1) k<1><<<148, threads>>>(out, iters, clk);
      if (v == 2) k<2><<<148, threads>>>(out, iters, clk);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      const double ops = (double)threads * iters * 16;   // lane-ops per SM
      const double elems = ops * (v == 0 ? 1 : 2);
      if (rep) printf("%-24s %8.2f lane-ops/clk/SM  %8.2f elements/clk/SM\n", names[v], ops / c, elems / c);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
