// prefill_ws.cuh — K2 chunked-prefill partial attention, warp-specialised tcgen05 pipeline.
// SURVEY.md §8(a) a4 (+ a5 split-KV merge via K5 when the KV range is split).
//
// P:352-366 (Eq. 3): a chunk of c query tokens over its KV prefix has arithmetic
// intensity c*h_q/h_kv, tensor-core bound on B200 once c*G >= ~255.  P:357-358 GQA:
// the G query heads of one KV head are packed as MMA rows (row = t_local*G + h), so
// each K/V tile read from HBM feeds all rows of the CTA.
//
// One CTA = two 128-row query tiles (A, B) of one KV head and a contiguous range of
// 128-token KV tiles.  12 warps:
//   warp 0      TMA producer (one elected lane): Q_A, Q_B once; K_j, V_j through a
//               4-slot smem ring (full/empty mbarriers).
//   warp 1      MMA issuer (one elected lane), in the order
//                 S_A(0) S_B(0) | PV_A(j) S_A(j+1) PV_B(j) S_B(j+1) | ...
//               S = Q K^T (SS, K-major, SWIZZLE_128B) into TMEM; O += P V with P read
//               from TMEM (TS form; P aliases the first 64 columns of S) and V as an
//               MN-major smem operand.  tcgen05.commit -> mbarriers.
//   warp 2      TMEM allocator (512 columns: S_A | S_B | O_A | O_B).
//   warps 4-7   softmax of tile A, warps 8-11 softmax of tile B: thread = TMEM lane =
//               query row.  Two passes over S (row max, then exp2/sum/pack), P as bf16
//               back into TMEM with tcgen05.st, handed to the MMA warp in two 64-key
//               chunks (PV of keys 0-63 overlaps the exponentials of keys 64-127).  The running max is only raised when
//               it grows by more than 2^8 (exact: numerator and denominator use the
//               same stale max; p <= 256 stays finite in bf16/fp32), so O is rarely
//               rescaled; when it is, the softmax warps rescale O_X in TMEM.
// Ordering argument: the commit that publishes S_X(j+1) also covers PV_X(j) (all prior
// MMAs of the issuing thread), so once a softmax warp sees S_X(j+1) it may overwrite
// the P columns and rescale O_X.  Tile A's softmax overlaps tile B's MMAs and v.v.
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace medha {

constexpr int kWsThreads = 384;
constexpr int kWsTileM = 128;
constexpr int kWsTileN = 128;
#ifndef MEDHA_PF_ABLATE
#define MEDHA_PF_ABLATE 0       // experiment-only ablations (1: skip the softmax)
#endif
#ifndef MEDHA_PF_SLOTS128
#define MEDHA_PF_SLOTS128 4     // K/V ring slots at d = 128 (32 KiB each; 5 fit in 227 KiB)
#endif
#ifndef MEDHA_PF_SLOTS64
#define MEDHA_PF_SLOTS64 4      // K/V ring slots at d = 64 (16 KiB each)
#endif
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef MEDHA_PF_SETMAXNREG
#define MEDHA_PF_SETMAXNREG 0   // rebalance registers between warpgroups (A/B knob)
#endif
#ifndef MEDHA_PF_NREG_LO
#define MEDHA_PF_NREG_LO 80    // producer / MMA / allocator warpgroup
#endif
#ifndef MEDHA_PF_NREG_HI
#define MEDHA_PF_NREG_HI 208   // softmax warpgroups
#endif
static_assert(128 * MEDHA_PF_NREG_LO + 256 * MEDHA_PF_NREG_HI <= 168 * 384, "register file");
#ifndef MEDHA_PF_SPLIT_FMA
#define MEDHA_PF_SPLIT_FMA 1   // x = (s*scale) - m in two roundings (partition-invariant P)
#endif
#ifndef MEDHA_PF_RAW_L
#define MEDHA_PF_RAW_L 0   // normaliser: 0 rounded P via FHADD.BF16 (R20), 1 unrounded P, 2 rounded P via unpack
#endif
constexpr int kPChunks = 2;   // P handed to the MMA warp in two 64-key chunks

#ifndef MEDHA_PF_POLY_NUM      // fraction NUM/DEN of column pairs whose exp2 runs on the FMA pipe
#define MEDHA_PF_POLY_NUM 0
#endif
#ifndef MEDHA_PF_POLY_DEN
#define MEDHA_PF_POLY_DEN 3
#endif

#ifdef MEDHA_PF_TRACE
// experiment only: clock64 stamps of the hand-offs in CTA 0, per KV tile (medha_debug_pf_trace)
__device__ long long g_pf_trace[512][12];
// %globaltimer (ns) of CTA 0: [0] entry, [1] past griddepcontrol.wait, [2] S_A(0) seen,
// [3] last P of tile A stored, [4] tile A's outputs stored; [5] = clock64 at [2], [6] at [3]
__device__ long long g_pf_gt[8];
__device__ __forceinline__ long long pf_gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PF_STAMP(j, k)                                                  \
  do {                                                                  \
    if (blockIdx.x == 0 && (j) < 512) g_pf_trace[(j)][(k)] = clock64(); \
  } while (0)
#define PF_STAMP_MAX(mx)                                                                         \
  do {                                                                                           \
    if ((warp & 3) == 0 && lane == 0 && blockIdx.x == 0 && j < 512)                              \
      g_pf_trace[j][4 * x + 2] = clock64() + ((mx) > 1e30f);                                     \
  } while (0)
#else
#define PF_STAMP_MAX(mx) \
  do {                   \
  } while (0)
#define PF_STAMP(j, k) \
  do {                 \
  } while (0)
#endif

struct PrefillWsParams {
  float *o;        // [c][h_q][D] (n_split == 1) or ws parts [n_split][part_stride]
  float *lse;      // [c][h_q]    (n_split == 1)
  int64_t c;
  int64_t len;
  int64_t pos0;
  int64_t q_pos0;
  int64_t rows;         // c * h_q
  int64_t part_stride;  // floats between split parts (multiple of 4)
  int32_t h_q;
  int32_t h_kv;
  int32_t n_split;
  int32_t tiles_per_split;
  const int32_t *pt;    // page table (paged KV) or null; the K/V maps then span the pools
  int32_t psl;          // log2(page size), >= 7 when paged
  int32_t m_pairs;      // 2-tile query pairs of this chunk
  int32_t item_begin;   // first CTA of this chunk in the batch grid
  float scale_log2;
};

// A batch of prefill chunks, each over its own shard, in ONE launch (prefill-prefill
// batching).  CTA items of chunk s are [item_begin, next item_begin), ordered
// pair-fastest, then kv head, then KV split (concurrent CTAs share K/V tiles through L2).
constexpr int kPfMaxBatch = 32;
struct PrefillBatch {
  CUtensorMap maps[kPfMaxBatch][3];   // Q, K, V per chunk
  PrefillWsParams seq[kPfMaxBatch];
  int32_t n_seq;
};

template <int D>
struct WsLayout {
  static constexpr uint32_t kHalf = 128 * 64 * 2;    // [128][64] bf16 SW128 block, 16 KiB
  static constexpr uint32_t kQBytes = kWsTileM * D * 2;
  static constexpr uint32_t kSlotBytes = kWsTileN * D * 2;
  static constexpr uint32_t kQ0 = 0;
  static constexpr uint32_t kSlot0 = 2 * kQBytes;
  static constexpr int kSlots = D == 128 ? MEDHA_PF_SLOTS128 : MEDHA_PF_SLOTS64;
  static_assert(kSlots >= 4 && kSlots <= 8, "slots");
  static constexpr uint32_t kBar = kSlot0 + kSlots * kSlotBytes;
  static constexpr uint32_t kTotal = kBar + 256;
  static constexpr uint32_t kAlloc = kTotal + 1024;
};

// exp2 on the FMA pipe (FA4-style offload of the MUFU pipe): 2^x = 2^j * p(f), j = rint(x),
// f = x - j in [-0.5, 0.5], p the degree-3 minimax polynomial of 2^f (max relative error
// 7.5e-5, < 1/25 of a bf16 half-ulp).  x is clamped at -126 (2^-126 ~ 0 for P).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;            // 1.5 * 2^23: rint(x) in the low mantissa bits
  const float f = x - (t - 12582912.f);
  const float pf = fmaf(fmaf(fmaf(0.055171651f, f, 0.24261107f), f, 0.69326099f), f, 0.99992808f);
  // (bits(t) << 23) == rint(x) << 23 mod 2^32 because 0x4B400000 << 23 == 0 mod 2^32
  return __int_as_float(__float_as_int(pf) + __float_as_int(t) * 8388608);
}

// Softmax of one 128-column S row (this thread's TMEM lane), register resident: the row
// is read from TMEM once (4 x tcgen05.ld, one wait), the max and the exponentials work on
// registers, and P goes back as bf16 into TMEM columns [0, 64) (aliasing consumed S).
__device__ __forceinline__ void sm_load_row(uint32_t tS, uint32_t (&s)[128]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) tmem_ld32(tS + 32 * q, reinterpret_cast<uint32_t(&)[32]>(s[32 * q]));
  tmem_wait_ld();
}

// max of the raw logits; kMasked: only columns < nvalid count (causal diagonal / shard end)
template <bool kMasked>
__device__ __forceinline__ float sm_rowmax(const uint32_t (&s)[128], int nvalid) {
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int e = 0; e < 128; e += 2) {
    if (kMasked) {
      if (e < nvalid) m0 = fmaxf(m0, __uint_as_float(s[e]));
      if (e + 1 < nvalid) m1 = fmaxf(m1, __uint_as_float(s[e + 1]));
    } else {
      m0 = fmaxf(m0, __uint_as_float(s[e]));
      m1 = fmaxf(m1, __uint_as_float(s[e + 1]));
    }
  }
  return fmaxf(m0, m1);
}

// Packed (fp32x2) version of ex2_poly: FADD2/FFMA2 on the FMA pipe, IMAD for the
// exponent, FMNMX for the clamp - no MUFU.  Same polynomial and error as ex2_poly.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 j = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(j, make_float2(-1.f, -1.f), x);
  float2 pf = __ffma2_rn(make_float2(0.055171651f, 0.055171651f), f, make_float2(0.24261107f, 0.24261107f));
  pf = __ffma2_rn(pf, f, make_float2(0.69326099f, 0.69326099f));
  pf = __ffma2_rn(pf, f, make_float2(0.99992808f, 0.99992808f));
  return make_float2(__int_as_float(__float_as_int(pf.x) + __float_as_int(t.x) * 8388608),
                     __int_as_float(__float_as_int(pf.y) + __float_as_int(t.y) * 8388608));
}

// P = 2^(s*scale_log2 - mu) -> bf16 -> TMEM.  Returns the row sum of the bf16-ROUNDED P
// (the exact weights the PV MMA uses).  In unmasked tiles, column pairs i with
// (i % MEDHA_PF_POLY_DEN) < MEDHA_PF_POLY_NUM evaluate exp2 with ex2_poly2 on the FMA pipe
// (offloading the MUFU pipe, the softmax bottleneck: 128 ex2 per row per tile), the rest
// with MUFU.EX2.
constexpr uint32_t kPOff = 0;   // TMEM column of P inside its tile's S columns

// Quarters [Q0, Q1) of the row (32 columns each); the row sum accumulates into lsum2.
template <bool kMasked, int Q0, int Q1>
__device__ __forceinline__ void sm_exp_pack(uint32_t tS, const uint32_t (&s)[128], float sl2, float mu,
                                            int nvalid, float2 &lsum2) {
  const float2 sl2v = make_float2(sl2, sl2), nmu = make_float2(-mu, -mu);
  const float2 nmu384 = make_float2(-(384.f + mu), -(384.f + mu));   // exact: mu is an integer
#pragma unroll
  for (int q = Q0; q < Q1; ++q) {
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      const int col = 32 * q + e;
#if MEDHA_PF_SPLIT_FMA
      // t = s*scale + 1.5*2^8 rounds s*scale onto the fixed grid 2^-15 (depends on s only);
      // x = t - (1.5*2^8 + m) is then EXACT for any integer m (|x| < 2^8), so P's bf16
      // rounding does not depend on the partition's max: KVP == single GPU bit for bit
      // up to fp32 summation order (grid error <= 2^-16 in x, 1e-5 relative in P)
      const float2 t = __ffma2_rn(make_float2(__uint_as_float(s[col]), __uint_as_float(s[col + 1])), sl2v,
                                  make_float2(384.f, 384.f));
      const float2 x = __fadd2_rn(t, nmu384);
#else
      const float2 x = __ffma2_rn(make_float2(__uint_as_float(s[col]), __uint_as_float(s[col + 1])), sl2v, nmu);
#endif
      float2 pp;
      if (!kMasked && ((col >> 1) % MEDHA_PF_POLY_DEN) < MEDHA_PF_POLY_NUM) {
        pp = ex2_poly2(x);
      } else {
        pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
      }
      if (kMasked) {
        pp.x = (col < nvalid) ? pp.x : 0.f;
        pp.y = (col + 1 < nvalid) ? pp.y : 0.f;
      }
      pk[e >> 1] = pack_bf16x2(pp.x, pp.y);
#if MEDHA_PF_RAW_L == 1
      lsum2 = __fadd2_rn(lsum2, pp);   // A/B: normaliser of the unrounded P
#elif MEDHA_PF_RAW_L == 2
      lsum2 = __fadd2_rn(lsum2, make_float2(__uint_as_float(pk[e >> 1] << 16), __uint_as_float(pk[e >> 1] & 0xffff0000u)));
#else
      add_bf16x2_f32(lsum2.x, lsum2.y, pk[e >> 1]);   // rounded P, one FHADD.BF16 per element
#endif
    }
    tmem_st16(tS + kPOff + 16 * q, pk);
  }
}

// hand a completed P chunk to the MMA warp (P stores, then O rescale stores, are visible)
__device__ __forceinline__ void p_handoff(uint64_t *bar) {
  tmem_wait_st();
  tc_fence_before();
  mbar_arrive(bar);
}

template <int D, int G>
__global__ void __launch_bounds__(kWsThreads, 1)
    prefill_ws_kernel(const __grid_constant__ PrefillBatch batch) {
  static_assert(D == 64 || D == 128, "D");
  static_assert(kWsTileM % G == 0, "G");
  using L = WsLayout<D>;
  constexpr int TQ = kWsTileM / G;
  constexpr int NH = D / 64;
  constexpr uint32_t kIdescS = umma_idesc_bf16(kWsTileM, kWsTileN, 0);
  constexpr uint32_t kIdescO = umma_idesc_bf16(kWsTileM, D, 1);
#ifdef MEDHA_PF_TRACE
  const long long gt_entry = pf_gtimer();
#endif
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::kBar);
  uint64_t *bar_q = bars + 0;
  constexpr int kWsSlots = L::kSlots;
  uint64_t *bar_full = bars + 1;              // [kWsSlots]
  uint64_t *bar_empty = bar_full + kWsSlots;  // [kWsSlots]
  uint64_t *bar_s = bar_empty + kWsSlots;     // [2]
  uint64_t *bar_p = bar_s + 2;                // [2][kPChunks]
  uint64_t *bar_o = bar_p + 2 * kPChunks;   // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar_o + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  int sq = 0;
  while (sq + 1 < batch.n_seq && (int)blockIdx.x >= batch.seq[sq + 1].item_begin) ++sq;
  const PrefillWsParams &p = batch.seq[sq];
  const CUtensorMap *tmq = &batch.maps[sq][0];
  const CUtensorMap *tmk = &batch.maps[sq][1];
  const CUtensorMap *tmv = &batch.maps[sq][2];
  const int local = (int)blockIdx.x - p.item_begin;
  const int pair = local % p.m_pairs;
  const int kvh = (local / p.m_pairs) % p.h_kv;
  const int split = local / (p.m_pairs * p.h_kv);
  const int64_t t0 = (int64_t)pair * 2 * TQ;                 // first query token of tile A
  const int64_t t1 = min64(p.c, t0 + 2 * TQ);
  const int64_t n_kv = max64(0, min64(p.len, p.q_pos0 + t1 - 1 - p.pos0 + 1));
  const int n_tiles_total = (int)((n_kv + kWsTileN - 1) / kWsTileN);
  const int jt0 = split * p.tiles_per_split;
  const int n = max(0, min(p.tiles_per_split, n_tiles_total - jt0));

  if (tid == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < kWsSlots; ++i) {
      mbar_init(bar_full + i, 1);
      mbar_init(bar_empty + i, 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(bar_s + x, 1);
      for (int c = 0; c < kPChunks; ++c) mbar_init(bar_p + x * kPChunks + c, 128);
      mbar_init(bar_o + x, 1);
    }
    mbar_fence_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(tmq);
    tma_prefetch_desc(tmk);
    tma_prefetch_desc(tmv);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: the set-up above touches only this CTA's shared memory, TMEM and kernel parameters,
  // so it overlaps the previous kernel's tail; global memory (Q, K/V written by e.g.
  // kv_append, outputs read by e.g. the previous split merge) only after this wait
  pdl_wait();
  pdl_launch_dependents();    // the split merge may take SMs as this grid's last wave retires
#ifdef MEDHA_PF_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g_pf_gt[0] = gt_entry;
    g_pf_gt[1] = pf_gtimer();
  }
#endif

  uint8_t *sQ = smem + L::kQ0;
  auto slot_ptr = [&](int s) { return smem + L::kSlot0 + s * L::kSlotBytes; };

  if (warp < 4) {
#if MEDHA_PF_SETMAXNREG
  // register file rebalance (all four warps of a warpgroup execute the same instruction, inside
  // the branch so ptxas knows each region's budget): 128 x LO + 256 x HI <= 168 x 384
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(MEDHA_PF_NREG_LO) : "memory");
#endif
  if (warp == 0) {
    // ================================ TMA producer ================================
    if (lane == 0 && n > 0) {
      mbar_arrive_expect_tx(bar_q, 2 * L::kQBytes);
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int hh = 0; hh < NH; ++hh)
          tma_load_3d(sQ + x * L::kQBytes + hh * L::kHalf, tmq, bar_q, 64 * hh, kvh * G, (int32_t)(t0 + x * TQ));
      for (int it = 0; it < 2 * n; ++it) {
        const int s = it % kWsSlots;
        if (it >= kWsSlots) mbar_wait(bar_empty + s, ((it / kWsSlots) - 1) & 1);
        mbar_arrive_expect_tx(bar_full + s, L::kSlotBytes);
        int32_t tok = (jt0 + (it >> 1)) * kWsTileN;   // logical tile start; pool row when paged
        if (p.pt) tok = (__ldg(p.pt + (tok >> p.psl)) << p.psl) | (tok & ((1 << p.psl) - 1));
        const void *map = (it & 1) ? (const void *)tmv : (const void *)tmk;
#pragma unroll
        for (int hh = 0; hh < NH; ++hh) tma_load_3d(slot_ptr(s) + hh * L::kHalf, map, bar_full + s, 64 * hh, tok, kvh);
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ==================================
    if (lane == 0 && n > 0) {
      auto wait_full = [&](int it) {
        mbar_wait(bar_full + (it % kWsSlots), (it / kWsSlots) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int x, int it) {
        const uint32_t kb = smem_u32(slot_ptr(it % kWsSlots));
        const uint32_t qb = smem_u32(sQ + x * L::kQBytes);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * L::kHalf + (ks & 3) * 32;
          umma_f16_ss(tmem + x * 128, umma_desc_sw128(qb + off, 16, 1024), umma_desc_sw128(kb + off, 16, 1024),
                      kIdescS, ks > 0);
        }
      };
      // O_X += P_X V, key chunk by key chunk as the softmax hands P over
      auto issue_pv = [&](int x, int it, bool acc, int j) {
        const uint32_t vb = smem_u32(slot_ptr(it % kWsSlots));
        constexpr int kKsSplit = kWsTileN / 16 / kPChunks;
#pragma unroll
        for (int c = 0; c < kPChunks; ++c) {
          mbar_wait(bar_p + x * kPChunks + c, j & 1);
          if (c == 0) PF_STAMP(j, 8 + x);
          tc_fence_after();
#pragma unroll
          for (int ks = c ? kKsSplit : 0; ks < (c ? kWsTileN / 16 : kKsSplit); ++ks) {
            umma_f16_ts(tmem + 256 + x * 128, tmem + x * 128 + kPOff + ks * 8,
                        umma_desc_sw128(vb + ks * 2048, L::kHalf, 1024), kIdescO, (acc || ks > 0) ? 1u : 0u);
          }
        }
      };
      mbar_wait(bar_q, 0);
      tc_fence_after();
      wait_full(0);
      issue_s(0, 0);
      umma_commit(bar_s + 0);
      issue_s(1, 0);
      umma_commit(bar_s + 1);
      umma_commit(bar_empty + 0);
      for (int j = 0; j < n; ++j) {
        const int iv = 2 * j + 1, ik = 2 * j + 2;
        wait_full(iv);
        issue_pv(0, iv, j > 0, j);
        if (j == n - 1) umma_commit(bar_o + 0);
        if (j + 1 < n) {
          wait_full(ik);
          PF_STAMP(j, 10);
          issue_s(0, ik);
          umma_commit(bar_s + 0);
        }
        issue_pv(1, iv, j > 0, j);
        umma_commit(bar_empty + (iv % kWsSlots));
        if (j == n - 1) umma_commit(bar_o + 1);
        if (j + 1 < n) {
          issue_s(1, ik);
          umma_commit(bar_s + 1);
          umma_commit(bar_empty + (ik % kWsSlots));
        }
      }
    }
  }
  } else {
#if MEDHA_PF_SETMAXNREG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(MEDHA_PF_NREG_HI) : "memory");
#endif
    // ================================ softmax + epilogue ==========================
    const int x = (warp - 4) >> 2;          // 0: tile A, 1: tile B
    const int r = tid - 128 - x * 128;      // row in tile = TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_base + x * 128;
    const uint32_t tO = tmem + lane_base + 256 + x * 128;
    const int64_t tx0 = t0 + x * TQ;        // first token of this tile
    const int64_t t = tx0 + r / G;
    const int h = kvh * G + r % G;
    const bool row_valid = t < p.c;
    const int64_t lenm1 = p.len - 1;
    const int64_t j_lim = row_valid ? min64(p.q_pos0 + t - p.pos0, lenm1) : -1;
    // tiles whose last key is <= the smallest j_lim of this query tile need no mask
    const int64_t j_lim_tile = min64(p.q_pos0 + tx0 - p.pos0, lenm1);
    const float sl2 = p.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;

    for (int j = 0; j < n; ++j) {
      mbar_wait(bar_s + x, j & 1);
      if ((warp & 3) == 0 && lane == 0) PF_STAMP(j, 4 * x + 0);
#ifdef MEDHA_PF_TRACE
      if (blockIdx.x == 0 && warp == 4 && lane == 0 && j == 0) {
        g_pf_gt[2] = pf_gtimer();
        g_pf_gt[5] = clock64();
      }
#endif
      __syncwarp();
      tc_fence_after();
#if MEDHA_PF_ABLATE == 1
      // experiment only: no softmax (P = whatever S left) -- the MMA/TMA pipeline alone
      tc_fence_before();
      for (int c = 0; c < kPChunks; ++c) mbar_arrive(bar_p + x * kPChunks + c);
      l_run = 1.f;
      m_run = 0.f;
      continue;
#endif
      const int64_t jb = (int64_t)(jt0 + j) * kWsTileN;
      const bool full = (jb + kWsTileN - 1) <= j_lim_tile;
      const int nvalid = (int)min64(kWsTileN, max64(0, j_lim - jb + 1));   // valid cols [0, nvalid)
      uint32_t sreg[128];
      sm_load_row(tS, sreg);
      if ((warp & 3) == 0 && lane == 0) PF_STAMP(j, 4 * x + 1);
      float m_use = m_run, alpha = 1.f;
      bool rescale = false;
      float2 lsum2 = make_float2(0.f, 0.f);
      uint64_t *bar_pc = bar_p + x * kPChunks;
      // O rescale (PV_X(j-1) is complete: covered by the S_X(j) commit); it lands before
      // the first P chunk is handed over (the hand-off waits for all TMEM stores).  Rare;
      // 4 columns at a time (the S row is live in registers).
      auto rescale_o = [&]() {
        if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll 1
          for (int q = 0; q < D / 4; ++q) {
            uint32_t ro[4];
            tmem_ld4(tO + 4 * q, ro);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 4; ++e) ro[e] = __float_as_uint(__uint_as_float(ro[e]) * alpha);
            tmem_st4(tO + 4 * q, ro);
          }
        }
      };
      // ---- row max (unmasked tiles take a compare-free path), then P ----------------
      const float mx = full ? sm_rowmax<false>(sreg, nvalid) : sm_rowmax<true>(sreg, nvalid);
      PF_STAMP_MAX(mx);
      const float m_tile = ceilf(mx * sl2);   // integer-valued (log2 units): exact rescales
      if (m_tile > m_run + kRescaleThreshold || (m_run == -INFINITY && m_tile != -INFINITY)) {
        m_use = m_tile;
        alpha = exp2_int(m_run - m_tile);   // 0 when m_run = -inf
        rescale = (j > 0) && (m_run != -INFINITY);
      }
      rescale_o();
      // ---- P = exp2(s*scale - m) -> bf16 -> TMEM (aliasing S), handed over in chunks --
      const float mu = (m_use == -INFINITY) ? 0.f : m_use;
      if (full) {
        sm_exp_pack<false, 0, 2>(tS, sreg, sl2, mu, nvalid, lsum2);
        p_handoff(bar_pc + 0);
        sm_exp_pack<false, 2, 4>(tS, sreg, sl2, mu, nvalid, lsum2);
      } else {
        sm_exp_pack<true, 0, 2>(tS, sreg, sl2, mu, nvalid, lsum2);
        p_handoff(bar_pc + 0);
        sm_exp_pack<true, 2, 4>(tS, sreg, sl2, mu, nvalid, lsum2);
      }
      p_handoff(bar_pc + 1);
      m_run = m_use;
      const float lsum = lsum2.x + lsum2.y;
      if ((warp & 3) == 0 && lane == 0) PF_STAMP(j, 4 * x + 3);
#ifdef MEDHA_PF_TRACE
      if (blockIdx.x == 0 && warp == 4 && lane == 0 && j == n - 1) {
        g_pf_gt[3] = pf_gtimer();
        g_pf_gt[6] = clock64();
      }
#endif
      l_run = l_run * alpha + lsum;
    }

    // ---- epilogue --------------------------------------------------------------------
    const bool has = (n > 0) && (l_run > 0.f);
    const float inv_l = has ? 1.f / l_run : 0.f;
    const float lse_nat = has ? (m_run + __log2f(l_run)) * kLn2 : -INFINITY;
    if (n > 0) {
      mbar_wait(bar_o + x, 0);
      __syncwarp();
      tc_fence_after();
    }
    const int64_t grow = t * p.h_q + h;
    float *orow, *lrow;
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
      uint32_t ro[32];
      if (n > 0) {
        tmem_ld32(tO + 32 * q, ro);
        tmem_wait_ld();
      }
      if (row_valid) {
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          float4 v4;
          v4.x = has ? __uint_as_float(ro[e]) * inv_l : 0.f;
          v4.y = has ? __uint_as_float(ro[e + 1]) * inv_l : 0.f;
          v4.z = has ? __uint_as_float(ro[e + 2]) * inv_l : 0.f;
          v4.w = has ? __uint_as_float(ro[e + 3]) * inv_l : 0.f;
          *reinterpret_cast<float4 *>(orow + 32 * q + e) = v4;
        }
      }
    }
    if (row_valid) *lrow = lse_nat;
#ifdef MEDHA_PF_TRACE
    if (blockIdx.x == 0 && warp == 4 && lane == 0) g_pf_gt[4] = pf_gtimer();
#endif
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

}  // namespace medha
