// Experiment: throughput of the prefill softmax's exp stage (the instruction mix of
// sm_exp_pack: per column pair FFMA2 + FADD2 + 2 MUFU.EX2 + F2FP + 2 FHADD.BF16) with W warps
// per SM sub-partition, and with pieces of the mix removed, in exps per clock per SMSP.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp_mix exp_mix.cu
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2(float x) {
  float r;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ uint32_t pack(float lo, float hi) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void addbf(float &a, float &b, uint32_t u) {
  asm volatile("{\n .reg .b16 lo, hi;\n mov.b32 {lo, hi}, %2;\n add.rn.f32.bf16 %0, lo, %0;\n add.rn.f32.bf16 %1, hi, %1;\n}"
               : "+f"(a), "+f"(b) : "r"(u));
}

// V: 0 full mix, 1 no FHADD, 2 no F2FP/FHADD, 3 MUFU only, 4 full mix without FFMA2/FADD2
template <int V>
__global__ void k(uint32_t *out, int iters, long long *clk) {
  float s[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) s[i] = -0.01f * (float)((threadIdx.x + 3 * i) & 255);
  float sl2 = 1.4426950f, mu = 2.f;
  float l0 = 0.f, l1 = 0.f;
  uint32_t sink = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    sl2 += 1e-9f;
    const float2 sv = make_float2(sl2, sl2), nm = make_float2(-(384.f + mu), -(384.f + mu));
#pragma unroll
    for (int e = 0; e < 128; e += 2) {
      float2 x;
      if (V == 4 || V == 3) {
        x = make_float2(s[e] * 1.0f, s[e + 1]);
        x.x = s[e] + sl2;   // one FADD keeps the input iteration-dependent
        x.y = s[e + 1] + sl2;
      } else {
        const float2 t = __ffma2_rn(make_float2(s[e], s[e + 1]), sv, make_float2(384.f, 384.f));
        x = __fadd2_rn(t, nm);
      }
      const float px = ex2(x.x), py = ex2(x.y);
      if (V == 3 || V == 2) {
        sink ^= __float_as_uint(px) ^ __float_as_uint(py);
      } else {
        const uint32_t pk = pack(px, py);
        if (V == 1)
          sink ^= pk;
        else
          addbf(l0, l1, pk);
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink ^ __float_as_uint(l0 + l1);
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  uint32_t *out;
  long long *clk;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&clk, 8);
  const int iters = 256;
  const char *names[5] = {"full mix", "no FHADD", "no F2FP, no FHADD", "MUFU only (+1 FADD)", "full mix w/o FFMA2/FADD2"};
  for (int v = 0; v < 5; ++v)
    for (int w = 1; w <= 3; ++w) {
      const int threads = 128 * w;   // w warps per SMSP
      for (int rep = 0; rep < 2; ++rep) {
        switch (v) {
          case 0: k<0><<<148, threads>>>(out, iters, clk); break;
          case 1: k<1><<<148, threads>>>(out, iters, clk); break;
          case 2: k<2><<<148, threads>>>(out, iters, clk); break;
          case 3: k<3><<<148, threads>>>(out, iters, clk); break;
          case 4: k<4><<<148, threads>>>(out, iters, clk); break;
        }
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        const double exps_per_smsp = (double)w * 32 * 128 * iters;
        if (rep) printf("%-28s warps/SMSP %d  %6.2f exps/clk/SMSP  (%5.0f clk per 4096 exps)\n", names[v], w,
                        exps_per_smsp / c, 4096.0 * c / exps_per_smsp);
      }
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
