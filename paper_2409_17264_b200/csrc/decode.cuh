// decode.cuh — K3 split-KV decode partial with the K4 split merge fused into the
// last CTA of every (sequence, kv head).  SURVEY.md §8(a) a3 + a5.
//
// P:178-183 "During decode, we scan the entire KV cache so far" — the kernel is
// bound by HBM: every K/V byte of the visible shard is read exactly once (GQA
// packing: the G query heads of one KV head share each loaded byte),
// and the KV range is split across CTAs inside the GPU.
//
// Data path per warp and 16-token tile (D = 128):
//   * K rows: lane (g = lane/4, c = lane%4) loads tokens g and 8+g, bytes
//     [64i + 16c, +16) for i < D/32 -> every LDG.128 of the warp covers 8 full
//     64-byte row segments (coalesced), 2 KiB of K per warp instruction group.
//   * V rows: lane (g, c) loads tokens 2c, 2c+1, 2c+8, 2c+9, bytes [16g, +16) and
//     [128 + 16g, +16) -> 8 lanes read one 128-byte row segment.
//   * S = Q.K^T and O += P.V are legacy warp MMAs (m16n8k16, bf16 in, fp32 out)
//     used as dot-product engines: the FFMA pipe could not keep up with HBM at
//     G = 8.  The head dimension is permuted identically for Q and K
//     (any permutation leaves q.k unchanged), which is what lets each lane use
//     its own 16-byte loads directly as B fragments; V fragments are built with
//     PRMT.  Query heads sit on the MMA M dimension (rows g and g+8).
//   * fp32 online softmax in base 2 (scale*log2e folded into one multiply);
//     P rounded to bf16 (RNE) before the PV MMA (reading R8).
// Work items: one (seq, kv head, split) = a FIXED token range.  The grid is persistent
// (2 CTAs per SM) and CTAs take items from an atomic queue, so faster SMs take more items
// (HBM bandwidth per SM varies by ~10%) while every item's arithmetic - and therefore the
// result - stays independent of which CTA ran it (bit-reproducible).  Per item: 4 warps
// interleave 16-token tiles; their (m, l, O) are merged through shared memory; the item
// writes a normalised (o, lse2) split partial; the CTA finishing the last split of a
// (seq, kv head) (atomic ticket) merges all splits in split order (warp-parallel).
#pragma once
#include "common.cuh"

namespace medha {

#ifdef MEDHA_DECODE_TRACE
// experiment-only instrumentation: %globaltimer per CTA at start / main-loop end / partial
// written / split merge done (read back with medha_debug_decode_trace)
__device__ unsigned long long g_decode_trace[8192][8];   // indexed by work item
#define MEDHA_TRACE(k)                                                                     \
  do {                                                                                     \
    if (threadIdx.x == 0 && item < 8192) {                                                 \
      unsigned long long t_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                              \
      g_decode_trace[item][k] = t_;                                                        \
      if (k == 0) {                                                                        \
        unsigned smid_;                                                                    \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));                                \
        g_decode_trace[item][4] = blockIdx.x;                                              \
        g_decode_trace[item][5] = smid_;                                                   \
      }                                                                                    \
    }                                                                                      \
  } while (0)
// per launch (ring of 64): [0] CTA 0 resident, [1] CTA 0 past griddepcontrol.wait, [2] last
// CTA out, [3] the preceding kv_append past its wait; g_ltrace_n counts traced launches
__device__ unsigned long long g_ltrace[64][4];
__device__ unsigned g_ltrace_n;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#else
#define MEDHA_TRACE(k) do {} while (0)
#endif

#ifndef MEDHA_DEC_PINGPONG
#define MEDHA_DEC_PINGPONG 1   // 2x-unrolled main loop with ping-pong K/V register buffers
#endif

constexpr int kDecodeMaxSeqPerLaunch = 64;
constexpr int kMaxKvpRanks = 8;
constexpr int kDecodeMaxSplits = 256;  // per (seq, kv head)
constexpr int kDecodeSplitW = 2048;    // smem floats for split weights: splits <= kDecodeSplitW / G
constexpr int kDecodeWarps = 4;
constexpr int kDecodeThreads = kDecodeWarps * 32;

struct DecodeSeq {
  const __nv_bfloat16 *k;  // [h_kv][cap][D]
  const __nv_bfloat16 *v;
  int64_t hstride;        // tokens between head planes (capacity, or pool_tokens when paged)
  const int32_t *pt;      // page table (paged KV) or null
  int32_t psl;            // log2(page size)
  int64_t n_vis;         // visible local tokens (keys 0..n_vis-1); with len_dev: an upper bound
  int64_t *len_dev;       // device-length mode (graph-capturable step): keys 0..*len_dev are
                          // visible (the token appended at *len_dev included), *len_dev += 1 at the end
  // fused kv_append (SURVEY a1 in the decode launch): the new token's rows [h_kv][D] (bf16,
  // 16-byte vectors) go to local index t_app (len_dev mode: *len_dev; dropped at or past the
  // capacity).  The item whose split owns t_app writes them into the shard; every load of
  // token t_app reads k_app / v_app instead, so no CTA reads back what another wrote.
  const uint4 *k_app;     // null: no append
  const uint4 *v_app;
  int64_t t_app;
  int64_t cap;            // capacity (logical tokens) of the shard
  int64_t safe_end;       // early start: tokens [0, safe_end) may be read before the grid dependency
  int32_t split_tokens;  // tokens per split, multiple of 64
  int32_t n_splits;      // splits per kv head
  int32_t cta_begin;     // first CTA of this sequence (CTAs ordered [kvh][split])
  int32_t slot_begin;    // first workspace slot of this sequence
};

struct DecodeParams {
  const __nv_bfloat16 *q;  // [batch][h_q][D] (this launch's first sequence at q)
  float *o;                // [batch][h_q][D]
  float *lse;              // [batch][h_q], natural log
  float *ws_o;             // [slot][G][D] normalised split outputs
  float *ws_lse;           // [slot][G] base-2 split lse
  unsigned *counters;      // [n_seq * h_kv] split tickets, then [2] work queue / exit counters
  unsigned *work;          // persistent scheduler: work[0] next item, work[1] CTAs finished
  float scale_log2;        // softmax scale * log2(e)
  int32_t n_items;         // (seq, kv head, split) work items of this launch
  int32_t n_seq;
  int32_t h_kv;
  int32_t h_q;
  int32_t early;           // early start (see decode_splitkv_kernel); 0 in device-length mode
  // ---- fused KVP exchange over NVLink.  x_world == 0: off. ----
  // The last CTA of every (seq, kv head) pushes the unit's rank partial into every rank's
  // receive slot (peer memory mapped with CUDA IPC; at world 1 the local buffer), raises
  // that rank's flag for the unit to the call's epoch (release, system scope), waits for
  // the flags of all ranks (acquire, bounded by x_timeout_ns) and merges the world's
  // partials in rank order into x_o / x_lse / x_obf.  The epoch lives in DEVICE memory
  // (*x_epoch = last completed call, advanced by the last CTA out), so a captured CUDA
  // graph replays with a fresh epoch every time.  Buffer layout of every rank (XchgLayout):
  // [2 parities][world src][x_slot floats] slots, [2][world][x_units] flags, epoch word.
  int32_t x_world;
  int32_t x_rank;
  int32_t x_units;                 // flag stride per source rank
  uint32_t x_debug;                // test hook: bit 0 = withhold this rank's pushes and flags
  int64_t x_rows;                  // rows of the packed slot layout: o [x_rows][D], lse [x_rows]
  int64_t x_slot;                  // floats per source-rank slot
  uint64_t x_timeout_ns;           // bound of the flag wait (%globaltimer)
  char *x_peer[kMaxKvpRanks];      // every rank's exchange buffer (x_peer[x_rank] = local)
  uint32_t *x_epoch;               // local device word: epoch of the last completed call
  uint32_t *x_err;                 // mapped host word: set to 1 when a flag wait times out
  float *x_o;                      // final outputs [rows][D]
  float *x_lse;                    // final lse [rows] (may be null)
  __nv_bfloat16 *x_obf;            // final bf16 outputs (may be null)
  DecodeSeq seq[kDecodeMaxSeqPerLaunch];
};

__device__ __forceinline__ void st_release_sys(uint32_t *ptr, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(ptr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *ptr) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// exchange buffer of one rank: receive slot / flags of (parity, source rank)
__device__ __forceinline__ float *xchg_slot(const DecodeParams &p, char *base, uint32_t par, int src) {
  return reinterpret_cast<float *>(base) + ((int64_t)par * p.x_world + src) * p.x_slot;
}
__device__ __forceinline__ uint32_t *xchg_flags(const DecodeParams &p, char *base, uint32_t par, int src) {
  return reinterpret_cast<uint32_t *>(base + (size_t)2 * p.x_world * p.x_slot * sizeof(float)) +
         ((int64_t)par * p.x_world + src) * p.x_units;
}

template <int D, int G>
struct __align__(16) DecodeSmem {
  float o[kDecodeWarps][G][D];   // warp partials; later the warp sums of the split merge
  float m[kDecodeWarps][G];
  float l[kDecodeWarps][G];
  float w[kDecodeSplitW];        // split (or rank) merge weights [split][G]
  unsigned ticket;
  int item;
  uint32_t epoch;                // fused exchange: this call's epoch (kept out of registers)
};

// Grid dependency (PDL), once per thread: wait until the previous kernel on the stream has
// completed and its writes are visible, then let the next kernel's CTAs start, and read the
// fused exchange's epoch (written by the previous call's last CTA).
template <int D, int G>
__device__ __forceinline__ void grid_dep_sync(const DecodeParams &p, DecodeSmem<D, G> &sm, bool &waited) {
  if (waited) return;
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) sm.epoch = (p.x_world > 0) ? *reinterpret_cast<volatile uint32_t *>(p.x_epoch) + 1u : 0u;
  waited = true;
}

// One work item: split `split` of kv head `kvh` of sequence `sidx`.
// kPaged: some sequence of the launch has a page table (a separate instantiation keeps the
// contiguous path's register allocation untouched)
template <int D, int G, bool kPaged>
__device__ __forceinline__ void decode_item(const DecodeParams &p, const int item, DecodeSmem<D, G> &sm,
                                            bool &waited) {
  constexpr int KCH = D / 32;   // 16-byte K chunks per lane per token
  constexpr int VCH = D / 64;   // 16-byte V chunks per lane per token
  constexpr int KS = D / 16;    // k-steps of the QK MMA
  constexpr int NT = D / 8;     // n-tiles of the PV MMA
  constexpr bool kHi = (G > 8); // rows g+8 carry heads 8..15

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int g = lane >> 2;
  const int c = lane & 3;

  int sidx = 0;
  while (sidx + 1 < p.n_seq && item >= p.seq[sidx + 1].cta_begin) ++sidx;
  const DecodeSeq &S = p.seq[sidx];
  const int local = item - S.cta_begin;
  const int kvh = local / S.n_splits;
  const int split = local - kvh * S.n_splits;
  const int64_t t_begin = (int64_t)split * S.split_tokens;
  // device-length mode: the visible length is read at run time (splits past it are empty:
  // o = 0, lse = -inf, which the split merge ignores)
  const int64_t n_vis = S.len_dev ? min64(S.n_vis, *S.len_dev + 1) : S.n_vis;
  const int64_t t_end = min64(t_begin + S.split_tokens, n_vis);
  // fused append: token t_app (-1: none) comes from k_app / v_app
  auto app_token = [&]() -> int64_t {
    if (!S.k_app) return -1;
    const int64_t t = S.len_dev ? *S.len_dev : S.t_app;
    return t < S.cap ? t : -1;
  };
  // the appended token is the last visible one (or lies past the split), so the tile holding
  // it is the split's last tile: the main loop runs to t_bound = that tile's start (all its
  // tiles are then fully visible) and the tile itself is loaded, patched and computed once
  // after the loop - no patch code and a single bound in the hot loop (register budget)
  int64_t t_bound;
  {
    const int64_t ta = app_token();
    t_bound = (ta >= t_begin && ta < t_end) ? (ta & ~15ll) : t_end;
  }

  const __nv_bfloat16 *kbase = S.k + (int64_t)kvh * S.hstride * D;
  const __nv_bfloat16 *vbase = S.v + (int64_t)kvh * S.hstride * D;
  // pool row of logical tile start tb (16-aligned; a page holds >= 16 tokens, so all 16
  // tokens of a tile sit in one page); the page table is tiny and L1-resident
  const int32_t *pt = S.pt;
  const int psl = S.psl;
  auto tile_row = [&](int64_t tb) -> int64_t {
    if constexpr (kPaged)
      return pt ? (((int64_t)__ldg(pt + (tb >> psl)) << psl) | (tb & ((1ll << psl) - 1))) : tb;
    return tb;
  };

  // ---- Q fragments (rows g / g+8 = heads of this group), permuted like K ------------
  uint32_t qlo[KS][2], qhi[KS][2];
  {
    const __nv_bfloat16 *qrow = p.q + ((int64_t)sidx * p.h_q + (int64_t)kvh * G) * D;
#pragma unroll
    for (int i = 0; i < KCH; ++i) {
      uint4 a = make_uint4(0, 0, 0, 0), b = make_uint4(0, 0, 0, 0);
      if (g < G) a = *reinterpret_cast<const uint4 *>(qrow + (int64_t)g * D + 32 * i + 8 * c);
      if (kHi && g + 8 < G) b = *reinterpret_cast<const uint4 *>(qrow + (int64_t)(g + 8) * D + 32 * i + 8 * c);
      qlo[2 * i][0] = a.x; qlo[2 * i][1] = a.y; qlo[2 * i + 1][0] = a.z; qlo[2 * i + 1][1] = a.w;
      qhi[2 * i][0] = b.x; qhi[2 * i][1] = b.y; qhi[2 * i + 1][0] = b.z; qhi[2 * i + 1][1] = b.w;
    }
  }

  float oacc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
  float m_lo = -INFINITY, m_hi = -INFINITY;  // running max (base 2) of rows g, g+8
  float l_lo = 0.f, l_hi = 0.f;              // thread-partial running sums

  auto load_tile = [&](int64_t tb, uint4 (&kk)[2][KCH], uint4 (&vv)[4][VCH]) {
    const int64_t row0 = tile_row(tb);
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      const int64_t tok = tb + 8 * n + g;
      const bool ok = tok < t_bound;
      const __nv_bfloat16 *src = kbase + (row0 + 8 * n + g) * D + 8 * c;
#pragma unroll
      for (int i = 0; i < KCH; ++i) kk[n][i] = ok ? ldg_stream(src + 32 * i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t tok = tb + 2 * c + (r & 1) + 8 * (r >> 1);
      const bool ok = tok < t_bound;
      const __nv_bfloat16 *src = vbase + (row0 + 2 * c + (r & 1) + 8 * (r >> 1)) * D + 8 * g;
#pragma unroll
      for (int i = 0; i < VCH; ++i) vv[r][i] = ok ? ldg_stream(src + 64 * i) : make_uint4(0, 0, 0, 0);
    }
  };

  // fused append: the tile holding the new token takes that token's fragments from k_new /
  // v_new (pointers re-read from the kernel parameters); used once per item, after the loop
  auto patch_app = [&](int64_t tb, int64_t t_app, uint4 (&kk)[2][KCH], uint4 (&vv)[4][VCH]) {
    const __nv_bfloat16 *kapp = reinterpret_cast<const __nv_bfloat16 *>(S.k_app) + (int64_t)kvh * D;
    const __nv_bfloat16 *vapp = reinterpret_cast<const __nv_bfloat16 *>(S.v_app) + (int64_t)kvh * D;
#pragma unroll
    for (int n = 0; n < 2; ++n)
      if (tb + 8 * n + g == t_app) {
#pragma unroll
        for (int i = 0; i < KCH; ++i) kk[n][i] = ldg_stream(kapp + 8 * c + 32 * i);
      }
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (tb + 2 * c + (r & 1) + 8 * (r >> 1) == t_app) {
#pragma unroll
        for (int i = 0; i < VCH; ++i) vv[r][i] = ldg_stream(vapp + 8 * g + 64 * i);
      }
  };

  // one 16-token tile: S = QK^T, online softmax, O += PV (K/V fragments in registers)
  auto compute_tile = [&](const uint4 (&kr)[2][KCH], const uint4 (&vr)[4][VCH], const int64_t tb) {
    // ---- S = Q K^T  (rows: heads g / g+8; cols: tokens 2c,2c+1 of n-tile n) ----------
    float s[2][4];
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const uint4 &kv4 = kr[n][ks >> 1];
        const uint32_t b0 = (ks & 1) ? kv4.z : kv4.x;
        const uint32_t b1 = (ks & 1) ? kv4.w : kv4.y;
        mma_bf16_16816(s[n], qlo[ks][0], qhi[ks][0], qlo[ks][1], qhi[ks][1], b0, b1);
      }
    }
    // ---- masking + online softmax (base 2) ------------------------------------------
    float mx_lo = -INFINITY, mx_hi = -INFINITY;
#pragma unroll
    for (int n = 0; n < 2; ++n) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool ok = (tb + 8 * n + 2 * c + e) < t_bound;
        s[n][e] = ok ? s[n][e] * p.scale_log2 : -INFINITY;
        s[n][2 + e] = ok ? s[n][2 + e] * p.scale_log2 : -INFINITY;
        mx_lo = fmaxf(mx_lo, s[n][e]);
        mx_hi = fmaxf(mx_hi, s[n][2 + e]);
      }
    }
    mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
    mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
    if (kHi) {
      mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
      mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
    }
    // integer-valued running max (log2 units): rescales are exact powers of two
    const float mn_lo = fmaxf(m_lo, ceilf(mx_lo));
    const float mu_lo = (mn_lo == -INFINITY) ? 0.f : mn_lo;
    const float al_lo = exp2_int(m_lo - mu_lo);  // m_lo = -inf -> 0
    m_lo = mn_lo;
    float mu_hi = 0.f, al_hi = 1.f;
    if (kHi) {
      const float mn_hi = fmaxf(m_hi, ceilf(mx_hi));
      mu_hi = (mn_hi == -INFINITY) ? 0.f : mn_hi;
      al_hi = exp2_int(m_hi - mu_hi);
      m_hi = mn_hi;
    }
    float pr[2][4];
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      pr[n][0] = fast_exp2(s[n][0] - mu_lo);
      pr[n][1] = fast_exp2(s[n][1] - mu_lo);
      pr[n][2] = kHi ? fast_exp2(s[n][2] - mu_hi) : 0.f;
      pr[n][3] = kHi ? fast_exp2(s[n][3] - mu_hi) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      oacc[j][0] *= al_lo;
      oacc[j][1] *= al_lo;
      if (kHi) {
        oacc[j][2] *= al_hi;
        oacc[j][3] *= al_hi;
      }
    }
    // ---- O += P V --------------------------------------------------------------------
    const uint32_t a0 = pack_bf16x2(pr[0][0], pr[0][1]);
    const uint32_t a1 = kHi ? pack_bf16x2(pr[0][2], pr[0][3]) : 0u;
    const uint32_t a2 = pack_bf16x2(pr[1][0], pr[1][1]);
    const uint32_t a3 = kHi ? pack_bf16x2(pr[1][2], pr[1][3]) : 0u;
    // the normaliser sums the bf16-rounded P the MMA consumes (consistent weights)
    {
      float t0 = 0.f, t1 = 0.f;
      add_bf16x2_f32(t0, t1, a0);
      add_bf16x2_f32(t0, t1, a2);
      l_lo = l_lo * al_lo + (t0 + t1);
      if (kHi) {
        float u0 = 0.f, u1 = 0.f;
        add_bf16x2_f32(u0, u1, a1);
        add_bf16x2_f32(u0, u1, a3);
        l_hi = l_hi * al_hi + (u0 + u1);
      }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int ch = j >> 3, e = j & 7;
      const uint32_t sel = (e & 1) ? 0x7632u : 0x5410u;
      const uint32_t *r0 = reinterpret_cast<const uint32_t *>(&vr[0][ch]);
      const uint32_t *r1 = reinterpret_cast<const uint32_t *>(&vr[1][ch]);
      const uint32_t *r2 = reinterpret_cast<const uint32_t *>(&vr[2][ch]);
      const uint32_t *r3 = reinterpret_cast<const uint32_t *>(&vr[3][ch]);
      const uint32_t b0 = prmt(r0[e >> 1], r1[e >> 1], sel);
      const uint32_t b1 = prmt(r2[e >> 1], r3[e >> 1], sel);
      mma_bf16_16816(oacc[j], a0, a1, a2, a3, b0, b1);
    }
  };

  MEDHA_TRACE(0);
  constexpr int64_t kStep = 16 * kDecodeWarps;
  int64_t tb = t_begin + 16 * warp;
  // early start: a tile reaching past safe_end (rows the previous kernel may still write)
  // is loaded only after the grid dependency has resolved
  // the bound relative to the split start in one 32-bit register (splits are < 2^31 tokens)
  const int32_t safe_rel = (int32_t)max64(-1, min64(S.safe_end - t_begin, (int64_t)INT32_MAX));
  auto gate = [&](int64_t t) {
    if (!waited && (int32_t)(t - t_begin) + 16 > safe_rel) grid_dep_sync<D, G>(p, sm, waited);
  };
#if MEDHA_DEC_PINGPONG
  // 2x unrolled with ping-pong register buffers: tile i+1 loads while tile i computes,
  // without copying the prefetched fragments between iterations
  uint4 kb0[2][KCH], vb0[4][VCH], kb1[2][KCH], vb1[4][VCH];
  if (tb < t_bound) {
    gate(tb);
    load_tile(tb, kb0, vb0);
  }
  while (tb < t_bound) {
    if (tb + kStep < t_bound) {
      gate(tb + kStep);
      load_tile(tb + kStep, kb1, vb1);
    }
    compute_tile(kb0, vb0, tb);
    tb += kStep;
    if (tb >= t_bound) break;
    if (tb + kStep < t_bound) {
      gate(tb + kStep);
      load_tile(tb + kStep, kb0, vb0);
    }
    compute_tile(kb1, vb1, tb);
    tb += kStep;
  }
  {
    // the appended token's tile (bounds recomputed: nothing of this was live in the loop)
    const int64_t ta = app_token();
    const int64_t te = min64(t_begin + S.split_tokens, S.len_dev ? min64(S.n_vis, *S.len_dev + 1) : S.n_vis);
    if (ta >= t_begin && ta < te && (((ta & ~15ll) - t_begin) >> 4) % kDecodeWarps == warp) {
      t_bound = te;
      gate(ta & ~15ll);
      load_tile(ta & ~15ll, kb0, vb0);
      patch_app(ta & ~15ll, ta, kb0, vb0);
      compute_tile(kb0, vb0, ta & ~15ll);
    }
  }
#else
  uint4 kr[2][KCH], vr[4][VCH];
  if (tb < t_end) load_tile(tb, kr, vr);
  for (; tb < t_end; tb += kStep) {
    uint4 kn[2][KCH], vn[4][VCH];
    const int64_t nb = tb + kStep;
    if (nb < t_end) load_tile(nb, kn, vn);
    compute_tile(kr, vr, tb);
    if (nb < t_end) {
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int i = 0; i < KCH; ++i) kr[n][i] = kn[n][i];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < VCH; ++i) vr[r][i] = vn[r][i];
    }
  }
#endif

  MEDHA_TRACE(1);
  // every global write below follows the grid dependency
  grid_dep_sync<D, G>(p, sm, waited);
  // the owner of t_app (its split, or the last split when t_app lies past the visible keys)
  // stores the new K / V rows of this kv head into the shard (never read back in this launch)
  const int64_t t_app = app_token();
  if (t_app >= 0 && split == (int)min64(t_app / S.split_tokens, S.n_splits - 1) && tid < 2 * (D / 8)) {
    const int64_t row = tile_row(t_app & ~15ll) + (t_app & 15);
    const int e = tid % (D / 8);
    uint4 *dst = reinterpret_cast<uint4 *>(const_cast<__nv_bfloat16 *>(tid < D / 8 ? kbase : vbase) + row * D) + e;
    *dst = (tid < D / 8 ? S.k_app : S.v_app)[(int64_t)kvh * (D / 8) + e];
  }
  // ---- per-warp reduction of l over the 4 lanes of a row, publish to smem --------------
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
  if (kHi) {
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);
  }
  if (c == 0) {
    if (g < G) { sm.m[warp][g] = m_lo; sm.l[warp][g] = l_lo; }
    if (kHi && g + 8 < G) { sm.m[warp][g + 8] = m_hi; sm.l[warp][g + 8] = l_hi; }
  }
  // O fragment n-tile j, element e in {0,1}: head row g (+8), d = 64*(j/8) + 8*(2c+e) + (j%8)
#pragma unroll
  for (int j = 0; j < NT; ++j) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int dd = 64 * (j >> 3) + 8 * (2 * c + e) + (j & 7);
      if (g < G) sm.o[warp][g][dd] = oacc[j][e];
      if (kHi && g + 8 < G) sm.o[warp][g + 8][dd] = oacc[j][2 + e];
    }
  }
  __syncthreads();

  // ---- CTA merge of the 4 warps: (o normalised, lse2) of this split ---------------------
  const bool single = (S.n_splits == 1);   // (never with the fused exchange: host plans >= 2)
  const int64_t slot = (int64_t)S.slot_begin + (int64_t)kvh * S.n_splits + split;
  float *dst_o = single ? (p.o + ((int64_t)sidx * p.h_q + (int64_t)kvh * G) * D) : (p.ws_o + slot * G * D);
  for (int idx = tid; idx < G * D; idx += kDecodeThreads) {
    const int row = idx / D, dd = idx - row * D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kDecodeWarps; ++w) M = fmaxf(M, sm.m[w][row]);
    float L = 0.f, acc = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kDecodeWarps; ++w) {
        const float sc = exp2_int(sm.m[w][row] - M);
        L += sm.l[w][row] * sc;
        acc += sm.o[w][row][dd] * sc;
      }
    }
    dst_o[idx] = (L > 0.f) ? acc / L : 0.f;
    if (dd == 0) {
      const float lse2 = (L > 0.f) ? M + __log2f(L) : -INFINITY;
      if (single)
        p.lse[(int64_t)sidx * p.h_q + (int64_t)kvh * G + row] = lse2 * kLn2;
      else
        p.ws_lse[slot * G + row] = lse2;
    }
  }
  MEDHA_TRACE(2);
  if (single) return;

  // ---- the CTA finishing the last split of this (seq, kv head) merges the splits --------
  __threadfence();
  __syncthreads();
  unsigned *ctr = p.counters + (int64_t)sidx * p.h_kv + kvh;
  if (tid == 0) sm.ticket = atomicAdd(ctr, 1u);
  __syncthreads();
  if (sm.ticket != (unsigned)(S.n_splits - 1)) return;
  __threadfence();
  const int64_t slot0 = (int64_t)S.slot_begin + (int64_t)kvh * S.n_splits;
  const int ns = S.n_splits;                 // <= kDecodeSplitW / G (host planner)
  for (int i = tid; i < ns * G; i += kDecodeThreads) sm.w[i] = __ldcg(p.ws_lse + slot0 * G + i);
  __syncthreads();
  // per row: M = max_s lse_s, w_s = 2^(lse_s - M) / sum_s 2^(lse_s - M)   (one warp per row)
  for (int row = warp; row < G; row += kDecodeWarps) {
    float M = -INFINITY;
    for (int s2 = lane; s2 < ns; s2 += 32) M = fmaxf(M, sm.w[s2 * G + row]);
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o2));
    float L = 0.f;
    for (int s2 = lane; s2 < ns; s2 += 32) {
      const float w = (M == -INFINITY) ? 0.f : fast_exp2(sm.w[s2 * G + row] - M);
      sm.w[s2 * G + row] = w;
      L += w;
    }
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o2);
    const float inv = (L > 0.f) ? 1.f / L : 0.f;
    for (int s2 = lane; s2 < ns; s2 += 32) sm.w[s2 * G + row] *= inv;
    if (lane == 0) {
      const float lse_r = (L > 0.f) ? (M + __log2f(L)) * kLn2 : -INFINITY;
      const int64_t orow = (int64_t)sidx * p.h_q + (int64_t)kvh * G + row;
      if (p.x_world > 0) {
        if (!(p.x_debug & 1u))
          for (int r = 0; r < p.x_world; ++r)
            xchg_slot(p, p.x_peer[r], sm.epoch & 1u, p.x_rank)[p.x_rows * D + orow] = lse_r;   // NVLink stores
      } else {
        p.lse[orow] = lse_r;
      }
    }
  }
  __syncthreads();
  // warp-parallel: warp w sums splits w, w+4, ...; lane owns float4 chunks of the G*D
  // outputs; SB splits per batch keep 4*NV*SB loads in flight (one L2 latency per batch)
  {
    constexpr int NV = (G * D / 4 + 31) / 32;   // float4 chunks per lane (1..16)
    constexpr int SB = NV >= 8 ? 2 : (NV >= 4 ? 4 : 8);
    const float4 *src0 = reinterpret_cast<const float4 *>(p.ws_o + slot0 * G * D);
    float4 acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s2 = warp; s2 < ns; s2 += kDecodeWarps * SB) {
      float4 v[SB][NV];
#pragma unroll
      for (int u = 0; u < SB; ++u)
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int ch = lane + 32 * i;
          const int ss = s2 + u * kDecodeWarps;
          v[u][i] = (ss < ns && ch < G * D / 4) ? __ldcg(src0 + (int64_t)ss * (G * D / 4) + ch)
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
      for (int u = 0; u < SB; ++u)
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int ch = lane + 32 * i;
          const int ss = s2 + u * kDecodeWarps;
          if (ss < ns && ch < G * D / 4) {
            const float w = sm.w[ss * G + (4 * ch) / D];
            acc[i].x = fmaf(w, v[u][i].x, acc[i].x);
            acc[i].y = fmaf(w, v[u][i].y, acc[i].y);
            acc[i].z = fmaf(w, v[u][i].z, acc[i].z);
            acc[i].w = fmaf(w, v[u][i].w, acc[i].w);
          }
        }
    }
    float4 *wsum = reinterpret_cast<float4 *>(&sm.o[warp][0][0]);
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (lane + 32 * i < G * D / 4) wsum[lane + 32 * i] = acc[i];
  }
  __syncthreads();
  const int64_t obase = ((int64_t)sidx * p.h_q + (int64_t)kvh * G) * D;
  for (int idx = tid; idx < G * D; idx += kDecodeThreads) {
    const float *w0 = &sm.o[0][0][0];
    constexpr int WS = G * D;   // one warp's [G][D] block
    const float o = ((w0[idx] + w0[WS + idx]) + w0[2 * WS + idx]) + w0[3 * WS + idx];   // fixed order
    if (p.x_world > 0) {
      if (!(p.x_debug & 1u))
        for (int r = 0; r < p.x_world; ++r) xchg_slot(p, p.x_peer[r], sm.epoch & 1u, p.x_rank)[obase + idx] = o;
    } else {
      p.o[obase + idx] = o;
    }
  }
  if (tid == 0) *ctr = 0u;  // leave the counter zeroed for the next call
  if (p.x_world > 0) {
    __syncthreads();
    // one system-scope fence after the barrier orders every thread's NVLink stores before
    // the flag stores (cumulativity through bar.sync)
    if (tid == 0) __threadfence_system();
    __syncthreads();
    const int unit = sidx * p.h_kv + kvh;
    if (tid < p.x_world && !(p.x_debug & 1u))
      st_release_sys(xchg_flags(p, p.x_peer[tid], sm.epoch & 1u, p.x_rank) + unit, sm.epoch);
  }
  MEDHA_TRACE(3);
}

// Fused exchange, second half: wait until every rank's partial of `unit` has arrived
// (acquire) and merge them in rank order (same formula as lse_merge_kernel).  The wait is
// bounded: after x_timeout_ns without a peer's flag (a rank that never launched, or a
// collective-contract violation) the unit's outputs become NaN, *x_err is set (the host
// reports MEDHA_ENCCL) and the kernel finishes instead of hanging the GPU.
template <int D, int G>
__device__ __forceinline__ void xchg_merge_unit(const DecodeParams &p, const int unit, DecodeSmem<D, G> &sm) {
  const int tid = threadIdx.x;
  const uint32_t epoch = sm.epoch;
  const int sidx = unit / p.h_kv, kvh = unit - sidx * p.h_kv;
  char *local = p.x_peer[p.x_rank];
  const uint32_t par = epoch & 1u;
  const float *recv = xchg_slot(p, local, par, 0);
  bool late = false;
  if (tid < p.x_world) {
    const uint32_t *f = xchg_flags(p, local, par, tid) + unit;
    if (ld_acquire_sys(f) != epoch) {
      const unsigned long long t0 = global_ns();
      unsigned spins = 0;
      while (ld_acquire_sys(f) != epoch) {
        if ((++spins & 255u) == 0 && global_ns() - t0 > p.x_timeout_ns) {
          late = true;
          break;
        }
      }
    }
  }
  const int64_t obase = ((int64_t)sidx * p.h_q + (int64_t)kvh * G) * D;
  if (__syncthreads_or(late)) {
    const float qnan = __int_as_float(0x7fc00000);
    for (int idx = tid; idx < G * D; idx += kDecodeThreads) {
      p.x_o[obase + idx] = qnan;
      if (p.x_obf) p.x_obf[obase + idx] = __float2bfloat16_rn(qnan);
    }
    if (tid < G && p.x_lse) p.x_lse[(int64_t)sidx * p.h_q + (int64_t)kvh * G + tid] = qnan;
    if (tid == 0) atomicExch_system(p.x_err, 1u);
    __syncthreads();
    return;
  }
  const int64_t lrow0 = p.x_rows * D + (int64_t)sidx * p.h_q + (int64_t)kvh * G;
  if (tid < G) {
    const int row = tid;
    float M = -INFINITY;
    for (int r = 0; r < p.x_world; ++r) M = fmaxf(M, __ldcg(recv + (int64_t)r * p.x_slot + lrow0 + row));
    float lse_f = -INFINITY;
    if (M != -INFINITY) {
      float ssum = 0.f;
      for (int r = 0; r < p.x_world; ++r) ssum += __expf(__ldcg(recv + (int64_t)r * p.x_slot + lrow0 + row) - M);
      lse_f = M + __logf(ssum);
    }
    for (int r = 0; r < p.x_world; ++r)
      sm.w[r * G + row] = (M == -INFINITY) ? 0.f : __expf(__ldcg(recv + (int64_t)r * p.x_slot + lrow0 + row) - lse_f);
    if (p.x_lse) p.x_lse[(int64_t)sidx * p.h_q + (int64_t)kvh * G + row] = lse_f;
  }
  __syncthreads();
  for (int idx = tid; idx < G * D; idx += kDecodeThreads) {
    const int row = idx / D;
    float v[kMaxKvpRanks];
#pragma unroll
    for (int r = 0; r < kMaxKvpRanks; ++r) v[r] = (r < p.x_world) ? __ldcg(recv + (int64_t)r * p.x_slot + obase + idx) : 0.f;
    float o = 0.f;
#pragma unroll
    for (int r = 0; r < kMaxKvpRanks; ++r)
      if (r < p.x_world) o += sm.w[r * G + row] * v[r];
    p.x_o[obase + idx] = o;
    if (p.x_obf) p.x_obf[obase + idx] = __float2bfloat16_rn(o);
  }
  __syncthreads();
}

template <int D, int G, bool kPaged>
__global__ void __launch_bounds__(kDecodeThreads, 2) decode_splitkv_kernel(const __grid_constant__ DecodeParams p) {
  static_assert(D == 64 || D == 128, "D");
  static_assert(G >= 1 && G <= 16, "G");
  static_assert(kDecodeMaxSplits * G <= kDecodeSplitW || G > 8, "split weights");
  __shared__ DecodeSmem<D, G> sm;
#ifdef MEDHA_DECODE_TRACE
  const unsigned long long t_entry = gtimer();
#endif
  // PDL: this grid's CTAs may be resident before the previous kernel on the stream ends.
  // Early start (p.early, host-length mode): CTA b runs its first item (b) right away and
  // streams the K/V rows below the item's safe_end before the grid dependency resolves.
  // Why that is safe: every kernel of this library triggers its dependents only after its
  // own griddepcontrol.wait (kv_append_kernel only at exit), so when this grid starts, every
  // kernel before the immediately preceding one has completed; the preceding one - if it is
  // a decode of this library - writes at most its appended row (index len - 1 of ours),
  // which is at or past safe_end = len - 1; the query is only written by foreign kernels
  // (which trigger at exit) or by kv_append_kernel.  Every global WRITE (partials, counters,
  // outputs, the appended rows, the exchange) and every read of a counter, length or epoch
  // comes after grid_dep_sync.  Otherwise (and in device-length mode) the CTA waits first.
  bool waited = false;
  if (!p.early) grid_dep_sync<D, G>(p, sm, waited);
#ifdef MEDHA_DECODE_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g_ltrace[g_ltrace_n & 63][0] = t_entry;
    g_ltrace[g_ltrace_n & 63][1] = gtimer();
  }
#endif
  // persistent: the first item is this CTA's own (grid <= items), the rest come from the
  // queue (claimed after the grid dependency: the previous launch's last CTA resets it)
  for (int first = 1;; first = 0) {
    if (!first) {
      if (threadIdx.x == 0) sm.item = (int)gridDim.x + (int)atomicAdd(p.work, 1u);
      __syncthreads();
    }
    const int item = first ? (int)blockIdx.x : sm.item;
    __syncthreads();
    if (item >= p.n_items) break;
    decode_item<D, G, kPaged>(p, item, sm, waited);
    __syncthreads();
  }
  grid_dep_sync<D, G>(p, sm, waited);
  __syncthreads();
  // fused KVP exchange: units are merged after this CTA's items (no CTA ever spins while
  // this rank still has unprocessed items, so the wait cannot deadlock)
  if (p.x_world > 0)
    for (int unit = blockIdx.x; unit < p.n_seq * p.h_kv; unit += gridDim.x) xchg_merge_unit<D, G>(p, unit, sm);
  // the last CTA out resets the queue for the next launch
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.work + 1, 1u) == gridDim.x - 1) {
      p.work[0] = 0u;
      p.work[1] = 0u;
      if (p.x_world > 0) *p.x_epoch = sm.epoch;   // every CTA has read it
      // device-length mode: every item has read the lengths; advance them for the next step
      for (int i = 0; i < p.n_seq; ++i)
        if (p.seq[i].len_dev) *p.seq[i].len_dev += 1;
#ifdef MEDHA_DECODE_TRACE
      g_ltrace[g_ltrace_n & 63][2] = gtimer();
      g_ltrace_n = g_ltrace_n + 1;
#endif
    }
  }
}

}  // namespace medha
