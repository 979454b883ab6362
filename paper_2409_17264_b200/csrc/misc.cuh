// misc.cuh — K1 kv_append, K5 LSE merge, K6 HBM read probe.
#pragma once
#include "common.cuh"

namespace medha {

// K1: scatter n new token-major rows [n][h_kv][D] into the
// head-major shard [h_kv][hstride][D] at local token `len` (through the page table when
// the shard is paged).  One 16-byte vector per thread.
// cp_n > 0 (decode_step_host): the same launch also copies cp_n 16-byte vectors cp_src -> cp_dst
// (the step's query, read straight from mapped pinned host memory).
__global__ void kv_append_kernel(const uint4 *__restrict__ k_new, const uint4 *__restrict__ v_new,
                                 uint4 *__restrict__ k, uint4 *__restrict__ v, int64_t n, int32_t h_kv,
                                 int32_t vec_per_row, int64_t hstride, int64_t len,
                                 const int32_t *__restrict__ pt, int32_t psl,
                                 const uint4 *__restrict__ cp_src, uint4 *__restrict__ cp_dst, int64_t cp_n) {
  // no early trigger: a following decode may read K/V rows (and the staged query) before its
  // own grid dependency resolves, so it may start only after every CTA has written and fenced
  // them (the trigger at the end)
  pdl_wait();
#ifdef MEDHA_DECODE_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) g_ltrace[g_ltrace_n & 63][3] = gtimer();
#endif
  const int64_t total = n * h_kv * vec_per_row;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cp_n; i += (int64_t)gridDim.x * blockDim.x)
    cp_dst[i] = cp_src[i];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / vec_per_row;          // row = t*h_kv + h
    const int32_t e = (int32_t)(i - row * vec_per_row);
    const int64_t t = row / h_kv;
    const int32_t h = (int32_t)(row - t * h_kv);
    int64_t j = len + t;                      // logical token; pool row when paged
    if (pt) j = ((int64_t)pt[j >> psl] << psl) | (j & ((1ll << psl) - 1));
    const int64_t dst = ((int64_t)h * hstride + j) * vec_per_row + e;
    k[dst] = k_new[i];
    v[dst] = v_new[i];
  }
  // the rows (and the staged query) are performed at gpu scope before a dependent decode
  // may start its early, pre-wait reads of them
  __threadfence();
  __syncthreads();
  pdl_launch_dependents();
}

// K5 ("combined using online-softmax"): part r starts at
// parts + r*part_stride and holds o [rows][D] then lse [rows] (natural log);
// part_stride = rows*(D+1) for the packed ABI layout (>= that for padded workspaces).  One warp per row; parts are
// combined in order r = 0..P-1, so the result does not depend on which rank runs it.
template <int D>
__global__ void lse_merge_kernel(const float *__restrict__ parts, int32_t P, int64_t rows, int64_t part_stride,
                                 float *__restrict__ o_out, float *__restrict__ lse_out,
                                 __nv_bfloat16 *__restrict__ o_bf16) {
  constexpr int PER = D / 32;  // floats per lane: d = lane + 32 i (coalesced; parts are packed, no alignment beyond 4 B)
  constexpr int U = 8;         // parts whose o rows are loaded together (latency hiding)
  pdl_wait();
  pdl_launch_dependents();
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  // lane r (and r + 32) holds part r's lse (P <= 64)
  const float *lse_col = parts + rows * D + row;
  const float l0 = (lane < P) ? lse_col[(int64_t)lane * part_stride] : -INFINITY;
  const float l1 = (lane + 32 < P) ? lse_col[(int64_t)(lane + 32) * part_stride] : -INFINITY;
  float M = fmaxf(l0, l1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float acc[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) acc[i] = 0.f;
  float lse = -INFINITY;
  if (M != -INFINITY) {
    float s = __expf(l0 - M) + __expf(l1 - M);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    lse = M + __logf(s);
    const float w0 = __expf(l0 - lse), w1 = __expf(l1 - lse);
    for (int r0 = 0; r0 < P; r0 += U) {
      float v[U][PER];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float *orow = parts + (int64_t)(r0 + u) * part_stride + row * D;
#pragma unroll
        for (int i = 0; i < PER; ++i) v[u][i] = (r0 + u < P) ? orow[lane + 32 * i] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = r0 + u;   // rank order 0..P-1
        const float w = __shfl_sync(0xffffffffu, (r < 32) ? w0 : w1, r & 31);
        if (r < P) {
#pragma unroll
          for (int i = 0; i < PER; ++i) acc[i] += w * v[u][i];
        }
      }
    }
  }
  float *od = o_out + row * D;
#pragma unroll
  for (int i = 0; i < PER; ++i) od[lane + 32 * i] = acc[i];
  if (o_bf16) {
    __nv_bfloat16 *ob = o_bf16 + row * D;
#pragma unroll
    for (int i = 0; i < PER; ++i) ob[lane + 32 * i] = __float2bfloat16_rn(acc[i]);
  }
  if (lse_out && lane == 0) lse_out[row] = lse;
}

// K6: read-only HBM probe (measurement aid).  Each warp streams contiguous 4 KiB
// chunks with 8 independent 16-byte loads per lane in flight.
__global__ void __launch_bounds__(256) hbm_read_probe_kernel(const uint4 *__restrict__ src, int64_t n_vec,
                                                            float *__restrict__ sink) {
  constexpr int U = 8;
  uint32_t x = 0;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_chunks = n_vec / (32 * U);
  for (int64_t ch = warp; ch < n_chunks; ch += n_warps) {
    const uint4 *p = src + ch * (32 * U) + lane;
    uint4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = ldg_stream(p + 32 * u);
#pragma unroll
    for (int u = 0; u < U; ++u) x ^= a[u].x ^ a[u].y ^ a[u].z ^ a[u].w;
  }
  for (int64_t i = n_chunks * 32 * U + warp * 32 + lane; i < n_vec; i += n_warps * 32) {
    const uint4 a = ldg_stream(src + i);
    x ^= a.x ^ a.y ^ a.z ^ a.w;
  }
  x = __reduce_xor_sync(0xffffffffu, x);
  if (lane == 0 && x == 0x9E3779B9u) sink[blockIdx.x & 4095] = 1.f;  // practically never taken
}

}  // namespace medha
