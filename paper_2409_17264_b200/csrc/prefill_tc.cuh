// prefill_tc.cuh — K2 chunked-prefill partial attention on the 5th-gen tensor cores.
// SURVEY.md §8(a) a4 (+ a5 split-KV merge via K5 when the KV range is split).
//
// P:352-366 (Eq. 3): a chunk of c query tokens attending over its KV prefix has
// arithmetic intensity c*h_q/h_kv, so it is tensor-core bound on B200 for c >= 64
// (ridge ~255 FLOP/B).  P:357-358 GQA: the G query heads of one KV head are packed
// as MMA rows, row r = t_local*G + h_in_group, so each K/V tile loaded from HBM is
// used by all G*TQ rows of the CTA (TQ = 128/G query tokens per 128-row tile).
//
// Per CTA: one 128-row query tile of one KV head and a contiguous range of
// 128-token KV tiles (split-KV).  Data path:
//   TMA (SWIZZLE_128B, 3D maps, zero fill past len / c)  -> smem Q, K[2], V[2]
//   tcgen05.mma kind::f16  S[128x128] = Q.K^T           -> TMEM cols [0,128)
//   4 softmax warps: tcgen05.ld S rows, causal/len mask, base-2 online softmax,
//       P (bf16, RNE) -> smem (SW128 K-major), conditional O rescale in TMEM
//   tcgen05.mma kind::f16  O[128xD] += P.V (V as an MN-major B operand)
//                                                       -> TMEM cols [128,128+D)
//   epilogue: tcgen05.ld O, divide by l, fp32 store (o, lse) or split partial.
// Thread 0 issues every TMA and every tcgen05.mma (single-thread issue) and
// commits MMA completion to mbarriers; K/V are double buffered so the TMA of tile
// j+1 overlaps the softmax and MMAs of tile j.
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace medha {

constexpr int kPrefillThreads = 128;
constexpr int kTileM = 128;   // query rows per CTA (TMEM lanes)
constexpr int kTileN = 128;   // KV tokens per tile

struct PrefillParams {
  float *o;        // [c][h_q][D] (n_split == 1) or ws parts [n_split][part_stride]
  float *lse;      // [c][h_q]    (n_split == 1)
  int64_t c;       // query tokens in the chunk
  int64_t len;     // valid local KV tokens
  int64_t pos0;    // absolute position of local KV token 0
  int64_t q_pos0;  // absolute position of query token 0
  int64_t rows;    // c * h_q
  int64_t part_stride;  // floats between split parts (multiple of 4, >= rows*(D+1))
  int32_t h_q;
  int32_t h_kv;
  int32_t n_split;
  int32_t tiles_per_split;
  float scale_log2;
};

template <int D>
struct PrefillLayout {
  static constexpr uint32_t kHalf = kTileM * 64 * 2;          // one [128][64] bf16 SW128 block: 16 KiB
  static constexpr uint32_t kQ = 0;
  static constexpr uint32_t kQBytes = kTileM * D * 2;
  static constexpr uint32_t kKVBytes = kTileN * D * 2;        // one K (or V) stage
  static constexpr uint32_t kK0 = kQ + kQBytes;
  static constexpr uint32_t kV0 = kK0 + 2 * kKVBytes;
  static constexpr uint32_t kP = kV0 + 2 * kKVBytes;
  static constexpr uint32_t kPBytes = kTileM * kTileN * 2;
  static constexpr uint32_t kBar = kP + kPBytes;              // 8 mbarriers + tmem slot
  static constexpr uint32_t kTotal = kBar + 128;
  static constexpr uint32_t kAlloc = kTotal + 1024;           // + alignment slack
};

template <int D, int G>
__global__ void __launch_bounds__(kPrefillThreads, 1)
    prefill_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ PrefillParams p) {
  static_assert(D == 64 || D == 128, "D");
  static_assert(kTileM % G == 0, "G");
  using L = PrefillLayout<D>;
  constexpr int TQ = kTileM / G;  // query tokens per tile
  constexpr int NH = D / 64;      // 64-wide d halves
  constexpr uint32_t kIdescS = umma_idesc_bf16(kTileM, kTileN, 0);
  constexpr uint32_t kIdescO = umma_idesc_bf16(kTileM, D, 1);

  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::kBar);
  uint64_t *bar_q = bars + 0;
  uint64_t *bar_kv = bars + 1;  // [2]
  uint64_t *bar_s = bars + 3;
  uint64_t *bar_o = bars + 4;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 6);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int m_tile = blockIdx.x, kvh = blockIdx.y, split = blockIdx.z;
  const int64_t t0 = (int64_t)m_tile * TQ;
  const int64_t t1 = min64(p.c, t0 + TQ);
  // visible local keys of the tile's last query token
  const int64_t n_kv = max64(0, min64(p.len, p.q_pos0 + t1 - 1 - p.pos0 + 1));
  const int n_tiles_total = (int)((n_kv + kTileN - 1) / kTileN);
  const int jt0 = split * p.tiles_per_split;
  const int n_tiles = max(0, min(p.tiles_per_split, n_tiles_total - jt0));

  if (tid == 0) {
    mbar_init(bar_q, 1);
    mbar_init(bar_kv + 0, 1);
    mbar_init(bar_kv + 1, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    mbar_fence_init();
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == 0) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_s = tmem;
  const uint32_t tmem_o = tmem + 128;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;

  uint8_t *sQ = smem + L::kQ;
  uint8_t *sP = smem + L::kP;
  auto sK = [&](int st) { return smem + L::kK0 + st * L::kKVBytes; };
  auto sV = [&](int st) { return smem + L::kV0 + st * L::kKVBytes; };
  auto issue_kv = [&](int li) {  // thread 0 only
    const int st = li & 1;
    const int32_t tok = (jt0 + li) * kTileN;
    mbar_arrive_expect_tx(bar_kv + st, 2 * L::kKVBytes);
#pragma unroll
    for (int hh = 0; hh < NH; ++hh) {
      tma_load_3d(sK(st) + hh * L::kHalf, &tm_k, bar_kv + st, 64 * hh, tok, kvh);
      tma_load_3d(sV(st) + hh * L::kHalf, &tm_v, bar_kv + st, 64 * hh, tok, kvh);
    }
  };

  if (tid == 0 && n_tiles > 0) {
    mbar_arrive_expect_tx(bar_q, L::kQBytes);
#pragma unroll
    for (int hh = 0; hh < NH; ++hh) tma_load_3d(sQ + hh * L::kHalf, &tm_q, bar_q, 64 * hh, kvh * G, (int32_t)t0);
    issue_kv(0);
    if (n_tiles > 1) issue_kv(1);
  }

  // row owned by this thread (TMEM lane == tid)
  const int64_t t = t0 + tid / G;
  const int h = kvh * G + tid % G;
  const bool row_valid = t < p.c;
  const int64_t j_lim = row_valid ? min64(p.q_pos0 + t - p.pos0, p.len - 1) : -1;  // last visible local key
  float m_run = -INFINITY, l_run = 0.f;

  for (int li = 0; li < n_tiles; ++li) {
    const int st = li & 1;
    // ---- S = Q K^T ------------------------------------------------------------------
    if (tid == 0) {
      if (li == 0) mbar_wait(bar_q, 0);
      mbar_wait(bar_kv + st, (li >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        const uint32_t off = (ks >> 2) * L::kHalf + (ks & 3) * 32;
        umma_f16_ss(tmem_s, umma_desc_sw128(smem_u32(sQ) + off, 16, 1024),
                    umma_desc_sw128(smem_u32(sK(st)) + off, 16, 1024), kIdescS, ks > 0);
      }
      umma_commit(bar_s);
    }
    mbar_wait(bar_s, li & 1);
    __syncwarp();
    tc_fence_after();

    // ---- softmax pass 1: masked row max --------------------------------------------
    const int64_t jb = (int64_t)(jt0 + li) * kTileN;
    const int64_t nvalid = min64(kTileN, max64(0, j_lim - jb + 1));  // valid cols [0, nvalid)
    float mx = -INFINITY;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t r[32];
      tmem_ld32(tmem_s + lane_off + 32 * q, r);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (32 * q + e < nvalid) mx = fmaxf(mx, __uint_as_float(r[e]));
    }
    const float m_new = fmaxf(m_run, mx * p.scale_log2);
    const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
    const bool need_rescale = (m_run != -INFINITY) && (m_new > m_run);
    const float alpha = need_rescale ? fast_exp2(m_run - m_new) : 1.f;

    // ---- previous PV must be done before P smem is overwritten / O is rescaled -----
    if (li > 0) {
      mbar_wait(bar_o, (li - 1) & 1);
      tc_fence_after();
      if (tid == 0 && li + 1 < n_tiles) issue_kv(li + 1);  // stage of tile li-1 is free
      __syncwarp();
    }

    // ---- softmax pass 2: P = exp2(s*scale - m) -> bf16 -> smem (SW128 K-major) -------
    float lsum = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t r[32];
      tmem_ld32(tmem_s + lane_off + 32 * q, r);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        const float p0 = (32 * q + e < nvalid) ? fast_exp2(__uint_as_float(r[e]) * p.scale_log2 - m_use) : 0.f;
        const float p1 = (32 * q + e + 1 < nvalid) ? fast_exp2(__uint_as_float(r[e + 1]) * p.scale_log2 - m_use) : 0.f;
        lsum += p0 + p1;
        pk[e >> 1] = pack_bf16x2(p0, p1);
      }
      uint8_t *half = sP + (q >> 1) * L::kHalf + tid * 128;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int ch = ((q & 1) * 4 + u) ^ (tid & 7);
        *reinterpret_cast<uint4 *>(half + ch * 16) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      }
    }
    l_run = l_run * alpha + lsum;
    m_run = m_new;

    // ---- conditional O rescale (warp-uniform decision) --------------------------------
    if (__any_sync(0xffffffffu, need_rescale)) {
#pragma unroll
      for (int q = 0; q < D / 32; ++q) {
        uint32_t r[32];
        tmem_ld32(tmem_o + lane_off + 32 * q, r);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
        tmem_st32(tmem_o + lane_off + 32 * q, r);
      }
      tmem_wait_st();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();

    // ---- O += P V ------------------------------------------------------------------
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < kTileN / 16; ++ks) {
        const uint32_t aoff = (ks >> 2) * L::kHalf + (ks & 3) * 32;
        umma_f16_ss(tmem_o, umma_desc_sw128(smem_u32(sP) + aoff, 16, 1024),
                    umma_desc_sw128(smem_u32(sV(st)) + ks * 2048, L::kHalf, 1024), kIdescO,
                    (li > 0 || ks > 0) ? 1u : 0u);
      }
      umma_commit(bar_o);
    }
  }

  // ---- epilogue --------------------------------------------------------------------------
  const bool has = (n_tiles > 0) && (l_run > 0.f);
  const float inv_l = has ? 1.f / l_run : 0.f;
  const float lse_nat = has ? (m_run + __log2f(l_run)) * kLn2 : -INFINITY;
  if (n_tiles > 0) {
    mbar_wait(bar_o, (n_tiles - 1) & 1);
    __syncwarp();
    tc_fence_after();
  }
  float *orow;
  float *lrow;
  const int64_t grow = t * p.h_q + h;
  if (p.n_split == 1) {
    orow = p.o + grow * D;
    lrow = p.lse + grow;
  } else {
    float *part = p.o + (int64_t)split * p.part_stride;
    orow = part + grow * D;
    lrow = part + p.rows * D + grow;
  }
#pragma unroll
  for (int q = 0; q < D / 32; ++q) {
    uint32_t r[32];
    if (n_tiles > 0) {
      tmem_ld32(tmem_o + lane_off + 32 * q, r);
      tmem_wait_ld();
    }
    if (row_valid) {
#pragma unroll
      for (int e = 0; e < 32; e += 4) {
        float4 v4;
        v4.x = has ? __uint_as_float(r[e]) * inv_l : 0.f;
        v4.y = has ? __uint_as_float(r[e + 1]) * inv_l : 0.f;
        v4.z = has ? __uint_as_float(r[e + 2]) * inv_l : 0.f;
        v4.w = has ? __uint_as_float(r[e + 3]) * inv_l : 0.f;
        *reinterpret_cast<float4 *>(orow + 32 * q + e) = v4;
      }
    }
  }
  if (row_valid) *lrow = lse_nat;

  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

}  // namespace medha
