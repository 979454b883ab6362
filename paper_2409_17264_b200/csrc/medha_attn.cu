// medha_attn.cu — host side of libmedha_attn (C ABI declared in include/medha_attn.h).
// Validation, work planning (split-KV sizing to the SM count), TMA descriptor
// encoding, NCCL KVP communicator and the all-gather + merge orchestration.
// Every compute step runs in the kernels of decode.cuh / prefill_ws.cuh / misc.cuh.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // header-only; ranges cost a pointer check when no tool is attached

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "medha_attn.h"
#include "decode.cuh"
#include "misc.cuh"
#include "prefill_ws.cuh"

using namespace medha;

namespace {

thread_local std::string g_last_error;

// NVTX range for the host-side enqueue of one phase of the Eq. 5 / Eq. 6 decomposition
// (partial, exchange, merge), so profiler timelines group the launches by phase
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

medha_status fail(medha_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                          \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess) return fail(MEDHA_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_));   \
  } while (0)

#define LAUNCH_CHECK(what)                                                                      \
  do {                                                                                          \
    cudaError_t e_ = cudaGetLastError();                                                        \
    if (e_ != cudaSuccess) return fail(MEDHA_ECUDA, "%s launch: %s", what, cudaGetErrorString(e_)); \
  } while (0)

int getenv_flag(const char *name, int dflt) {
  const char *v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

bool supported_g(int G) { return G == 1 || G == 2 || G == 4 || G == 8 || G == 16; }
bool supported_d(int d) { return d == 64 || d == 128; }

medha_status check_shard(const medha_kv_shard *kv) {
  if (!kv) return fail(MEDHA_EINVAL, "null shard");
  if (!kv->k || !kv->v) return fail(MEDHA_EINVAL, "null shard k/v pointer");
  if (!aligned16(kv->k) || !aligned16(kv->v)) return fail(MEDHA_EINVAL, "shard k/v not 16-byte aligned");
  if (kv->h_kv <= 0 || kv->capacity < 0 || kv->len < 0) return fail(MEDHA_EINVAL, "bad shard sizes");
  if (kv->len > kv->capacity) return fail(MEDHA_ERANGE, "shard len %lld > capacity %lld", (long long)kv->len,
                                          (long long)kv->capacity);
  if (!supported_d(kv->d)) return fail(MEDHA_ENOTSUP, "head dim %d not in {64,128}", kv->d);
  if (kv->page_table) {
    const int32_t ps = kv->page_size;
    if (ps < 16 || (ps & (ps - 1))) return fail(MEDHA_EINVAL, "page_size %d not a power of two >= 16", ps);
    if (kv->capacity % ps) return fail(MEDHA_EINVAL, "capacity %lld not a multiple of page_size %d",
                                       (long long)kv->capacity, ps);
    if (kv->pool_tokens < ps || kv->pool_tokens % ps)
      return fail(MEDHA_EINVAL, "pool_tokens %lld not a positive multiple of page_size %d", (long long)kv->pool_tokens,
                  ps);
    if ((uintptr_t)kv->page_table & 3)
      return fail(MEDHA_EINVAL, "page_table not 4-byte aligned");
  }
  return MEDHA_OK;
}

int32_t log2_pow2(int32_t x) {
  int32_t l = 0;
  while ((1 << l) < x) ++l;
  return l;
}
// tokens between the head planes of a shard's K/V arrays
int64_t head_stride(const medha_kv_shard &kv) { return kv.page_table ? kv.pool_tokens : kv.capacity; }

// ---------------------------------------------------------------------------------------------
// decode
// ---------------------------------------------------------------------------------------------
constexpr int kDecodeMaxKvHeads = 64;
constexpr int kDecodeWorkWord = kDecodeMaxSeqPerLaunch * kDecodeMaxKvHeads;   // tickets [seq][kv head] before it
constexpr int kDecodeCounterWords = kDecodeWorkWord + 64;
constexpr int kDecodeCtaBudget = 4096;  // upper bound of work items (splits) per launch (workspace sizing)
#ifndef MEDHA_DEC_ITEMS
#define MEDHA_DEC_ITEMS 1        // work items per resident CTA slot (A/B on B200: 1 > 2 > 4)
#endif
#ifndef MEDHA_DEC_MIN_SPLIT
#define MEDHA_DEC_MIN_SPLIT 256  // minimum tokens per split (short contexts: more CTAs, shorter chains)
#endif

struct DecodeWs {
  unsigned *counters;
  float *ws_lse;
  float *ws_o;
  size_t bytes;
};

size_t decode_ws_layout(int32_t batch, int32_t h_q, int32_t h_kv, int32_t d, char *base, DecodeWs *out) {
  const int64_t nb = std::min<int64_t>(std::max<int32_t>(batch, 1), kDecodeMaxSeqPerLaunch);
  const int64_t G = h_kv > 0 ? h_q / h_kv : 1;
  const int64_t slots = kDecodeCtaBudget + nb * h_kv;
  size_t off = 0;
  // counters live at a FIXED place and size whatever the call shape, so the "left zeroed"
  // invariant of the header holds across calls with different batch / h_kv / d
  const size_t c_off = off;
  off = round_up(off + kDecodeCounterWords * sizeof(unsigned), 256);   // split tickets + work queue
  const size_t l_off = off;
  off = round_up(off + slots * G * sizeof(float), 256);
  const size_t o_off = off;
  off = round_up(off + slots * G * d * sizeof(float), 256);
  if (out) {
    out->counters = reinterpret_cast<unsigned *>(base + c_off);
    out->ws_lse = reinterpret_cast<float *>(base + l_off);
    out->ws_o = reinterpret_cast<float *>(base + o_off);
    out->bytes = off;
  }
  return off;
}

// Launch with programmatic dependent launch (PDL) allowed: the grid's CTAs take SMs as the
// previous kernel's CTAs retire and start work (griddepcontrol.wait) the moment it
// completes, instead of after a full launch latency.  MEDHA_PDL=0 turns it off.
template <typename... Args>
void launch_pdl(void (*kernel)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  static const bool on = getenv_flag("MEDHA_PDL", 1) != 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = on ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <int D, int G>
void launch_decode(const DecodeParams &p, int grid, cudaStream_t st) {
  bool paged = false;
  for (int i = 0; i < p.n_seq; ++i) paged |= p.seq[i].pt != nullptr;
  if (paged)
    launch_pdl(decode_splitkv_kernel<D, G, true>, dim3(grid), dim3(kDecodeThreads), 0, st, p);
  else
    launch_pdl(decode_splitkv_kernel<D, G, false>, dim3(grid), dim3(kDecodeThreads), 0, st, p);
}

template <int D>
medha_status dispatch_decode_g(int G, const DecodeParams &p, int grid, cudaStream_t st) {
  switch (G) {
    case 1: launch_decode<D, 1>(p, grid, st); break;
    case 2: launch_decode<D, 2>(p, grid, st); break;
    case 4: launch_decode<D, 4>(p, grid, st); break;
    case 8: launch_decode<D, 8>(p, grid, st); break;
    case 16: launch_decode<D, 16>(p, grid, st); break;
    default: return fail(MEDHA_ENOTSUP, "group size %d", G);
  }
  LAUNCH_CHECK("decode_splitkv_kernel");
  return MEDHA_OK;
}

// Fused-exchange settings of one decode launch (see DecodeParams::x_*); null = off.
struct DecodeXchg {
  int32_t world, rank, units;
  uint32_t debug;
  int64_t rows, slot;
  uint64_t timeout_ns;
  char *peer[kMaxKvpRanks];
  uint32_t *epoch, *err;
  float *o, *lse;
  __nv_bfloat16 *obf;
};

// len_dev (device-length mode, medha_decode_step_dev): q_pos unused; sequence b attends keys
// 0..len_dev[b] read at run time, the plan covers the shard's capacity, len_dev[b] += 1 after.
// Fused append (medha_attn_decode_append / medha_kvp_decode_append / medha_decode_step_dev):
// sequence b with app_mask[b] != 0 (app_mask == null: every sequence) appends row b of
// k_app / v_app ([batch][h_kv][d] bf16) at local index len (len_dev mode: *len_dev) in the same
// launch; the caller advances the host lengths after a successful call.
struct DecodeAppend {
  const void *k, *v;
  const int32_t *mask;   // host [batch] or null
};

medha_status decode_partial_impl(const medha_kv_shard *kvs, int32_t batch, const void *q, int32_t h_q,
                                 const int64_t *q_pos, float scale, float *o, float *lse, void *ws,
                                 size_t ws_bytes, cudaStream_t st, const DecodeXchg *x = nullptr,
                                 int64_t *len_dev = nullptr, const DecodeAppend *app = nullptr) {
  if (batch < 0) return fail(MEDHA_EINVAL, "negative batch");
  if (batch == 0) return MEDHA_OK;
  if (!kvs || !q || !(q_pos || len_dev) || !o || !lse) return fail(MEDHA_EINVAL, "null argument");
  if (batch > 4096) return fail(MEDHA_ENOTSUP, "batch %d > 4096", batch);
  if (!aligned16(q)) return fail(MEDHA_EINVAL, "q not 16-byte aligned");
  if (!(scale > 0.f)) return fail(MEDHA_EINVAL, "scale must be > 0");
  const int32_t h_kv = kvs[0].h_kv, d = kvs[0].d;
  if (h_kv > kDecodeMaxKvHeads) return fail(MEDHA_ENOTSUP, "h_kv %d > %d", h_kv, kDecodeMaxKvHeads);
  for (int b = 0; b < batch; ++b) {
    medha_status s = check_shard(&kvs[b]);
    if (s) return s;
    if (kvs[b].h_kv != h_kv || kvs[b].d != d) return fail(MEDHA_ESHAPE, "shards disagree on h_kv/d");
  }
  if (h_q <= 0 || h_q % h_kv != 0) return fail(MEDHA_EINVAL, "h_q %d not a multiple of h_kv %d", h_q, h_kv);
  const int G = h_q / h_kv;
  if (!supported_g(G)) return fail(MEDHA_ENOTSUP, "group size %d not in {1,2,4,8,16}", G);
  DecodeWs W;
  if (!ws) return fail(MEDHA_EWORKSPACE, "null workspace");
  decode_ws_layout(batch, h_q, h_kv, d, static_cast<char *>(ws), &W);
  if (ws_bytes < W.bytes) return fail(MEDHA_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, W.bytes);

  if (x && batch > kDecodeMaxSeqPerLaunch) return fail(MEDHA_ENOTSUP, "fused exchange needs batch <= 64");
  if (app) {
    if (!app->k || !app->v) return fail(MEDHA_EINVAL, "null k_new/v_new");
    if (!aligned16(app->k) || !aligned16(app->v)) return fail(MEDHA_EINVAL, "k_new/v_new not 16-byte aligned");
    if (!len_dev)
      for (int b = 0; b < batch; ++b)
        if ((!app->mask || app->mask[b]) && kvs[b].len + 1 > kvs[b].capacity)
          return fail(MEDHA_ERANGE, "append at len %lld exceeds capacity %lld (sequence %d)", (long long)kvs[b].len,
                      (long long)kvs[b].capacity, b);
  }
  const int slots = 2 * num_sms();                 // two 4-warp CTAs per SM, persistent
  const int target = MEDHA_DEC_ITEMS * slots;       // work items per launch
  const int max_splits = std::min(kDecodeMaxSplits, kDecodeSplitW / G);
  for (int b0 = 0; b0 < batch; b0 += kDecodeMaxSeqPerLaunch) {
    const int nb = std::min(kDecodeMaxSeqPerLaunch, batch - b0);
    DecodeParams p;
    memset(&p, 0, sizeof(p));
    p.q = static_cast<const __nv_bfloat16 *>(q) + (int64_t)b0 * h_q * d;
    p.o = o + (int64_t)b0 * h_q * d;
    p.lse = lse + (int64_t)b0 * h_q;
    p.ws_o = W.ws_o;
    p.ws_lse = W.ws_lse;
    p.counters = W.counters;
    p.work = W.counters + kDecodeWorkWord;
    p.scale_log2 = scale * kLog2e;
    p.n_seq = nb;
    p.h_kv = h_kv;
    p.h_q = h_q;
    static const bool early_ok = getenv_flag("MEDHA_DEC_EARLY", 1) != 0;
    p.early = (early_ok && !len_dev) ? 1 : 0;
    if (x) {
      p.x_world = x->world;
      p.x_rank = x->rank;
      p.x_units = x->units;
      p.x_debug = x->debug;
      p.x_rows = x->rows;
      p.x_slot = x->slot;
      p.x_timeout_ns = x->timeout_ns;
      for (int r = 0; r < x->world; ++r) p.x_peer[r] = x->peer[r];
      p.x_epoch = x->epoch;
      p.x_err = x->err;
      p.x_o = x->o;
      p.x_lse = x->lse;
      p.x_obf = x->obf;
    }
    int64_t total = 0;
    std::vector<int64_t> nvis(nb);
    for (int i = 0; i < nb; ++i) {
      const medha_kv_shard &kv = kvs[b0 + i];
      const bool ap = app && (!app->mask || app->mask[b0 + i]);
      nvis[i] = len_dev ? kv.capacity
                        : std::max<int64_t>(0, std::min<int64_t>(kv.len + (ap ? 1 : 0), q_pos[b0 + i] - kv.pos0 + 1));
      total += nvis[i] * h_kv;
    }
    const int64_t per_cta =
        std::max<int64_t>(MEDHA_DEC_MIN_SPLIT, round_up((size_t)cdiv(std::max<int64_t>(total, 1), target), 64));
    int cta = 0;
    for (int i = 0; i < nb; ++i) {
      const medha_kv_shard &kv = kvs[b0 + i];
      int64_t ns = std::min<int64_t>(max_splits, std::max<int64_t>(1, cdiv(nvis[i], per_cta)));
      int64_t split_tokens = std::max<int64_t>(64, (int64_t)round_up((size_t)cdiv(std::max<int64_t>(nvis[i], 1), ns), 64));
      ns = std::max<int64_t>(1, cdiv(nvis[i], split_tokens));
      if (x && ns < 2) ns = 2;  // the exchange runs in the split-merging last CTA
      if (split_tokens > INT32_MAX) return fail(MEDHA_ERANGE, "split too large");
      DecodeSeq &S = p.seq[i];
      S.k = static_cast<const __nv_bfloat16 *>(kv.k);
      S.v = static_cast<const __nv_bfloat16 *>(kv.v);
      S.hstride = head_stride(kv);
      S.pt = kv.page_table;
      S.psl = kv.page_table ? log2_pow2(kv.page_size) : 0;
      S.n_vis = nvis[i];
      S.len_dev = len_dev ? len_dev + b0 + i : nullptr;
      S.split_tokens = (int32_t)split_tokens;
      S.n_splits = (int32_t)ns;
      S.cap = kv.capacity;
      S.safe_end = len_dev ? 0 : std::max<int64_t>(0, kv.len - 1);
      if (app && (!app->mask || app->mask[b0 + i])) {
        const size_t row = (size_t)(b0 + i) * h_kv * d * 2;
        S.k_app = reinterpret_cast<const uint4 *>(static_cast<const char *>(app->k) + row);
        S.v_app = reinterpret_cast<const uint4 *>(static_cast<const char *>(app->v) + row);
        S.t_app = kv.len;
      }
      S.cta_begin = cta;
      S.slot_begin = cta;
      cta += (int)(ns * h_kv);
    }
    if (cta > kDecodeCtaBudget + nb * h_kv) return fail(MEDHA_EWORKSPACE, "split plan exceeds workspace");
    p.n_items = cta;
    const int grid = std::min(cta, slots);
    medha_status s = (d == 128) ? dispatch_decode_g<128>(G, p, grid, st) : dispatch_decode_g<64>(G, p, grid, st);
    if (s) return s;
  }
  return MEDHA_OK;
}

// ---------------------------------------------------------------------------------------------
// prefill
// ---------------------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                      const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled_t get_encode_tiled() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(ptr);
  });
  return fn;
}

medha_status make_map_3d(CUtensorMap *m, const void *base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_bytes,
                         uint64_t s2_bytes, uint32_t b0, uint32_t b1, uint32_t b2) {
  PFN_encodeTiled_t enc = get_encode_tiled();
  if (!enc) return fail(MEDHA_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1_bytes, s2_bytes};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MEDHA_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return MEDHA_OK;
}

// One chunk of a prefill batch (host side).
struct PrefillChunk {
  const medha_kv_shard *kv;
  const void *q;
  int64_t c, q_pos0;
  float *o, *lse;
};

// Batch planner.  Every CTA processes one 2-tile query pair of one kv head over a range of
// `T` KV tiles (the same T for the whole batch keeps CTA durations balanced); a chunk with
// more KV tiles is split into cdiv(kv_tiles, T) ranges merged afterwards (K5).  T is chosen
// to minimise an estimate of the makespan: waves on the SM count x T, plus the HBM time of
// writing and merging split partials.
struct PrefillBatchPlan {
  std::vector<int> m_pairs, n_split, tps;
  std::vector<int64_t> rows, part_stride;
  std::vector<size_t> ws_off;
  size_t ws_bytes = 0;
  int64_t n_items = 0;
};

PrefillBatchPlan plan_prefill_batch(const PrefillChunk *ch, int n, int32_t h_q, int32_t h_kv, int32_t d) {
  PrefillBatchPlan pl;
  const int G = std::max(1, h_q / std::max(1, h_kv));
  const int TQ = kWsTileM / std::max(1, std::min(G, kWsTileM));
  std::vector<int64_t> kv_tiles(n);
  int64_t max_tiles = 1;
  for (int i = 0; i < n; ++i) {
    pl.m_pairs.push_back((int)cdiv(std::max<int64_t>(ch[i].c, 1), 2 * TQ));
    pl.rows.push_back(ch[i].c * h_q);
    pl.part_stride.push_back((int64_t)round_up((size_t)(ch[i].c * h_q * (d + 1)), 4));
    const medha_kv_shard *kv = ch[i].kv;
    const int64_t n_kv = std::max<int64_t>(0, std::min<int64_t>(kv->len, ch[i].q_pos0 + ch[i].c - 1 - kv->pos0 + 1));
    kv_tiles[i] = std::max<int64_t>(1, cdiv(n_kv, kWsTileN));
    max_tiles = std::max(max_tiles, kv_tiles[i]);
  }
  const int sms = num_sms();
  const double t_tile_us = 1.2;   // ~2 x 1024 MMA clk per KV tile and query pair
  double best = 1e300;
  int64_t best_T = max_tiles;
  static const int max_ns = std::max(1, std::min(64, getenv_flag("MEDHA_PF_MAX_SPLITS", 64)));   // A/B knob
  for (int ns = 1; ns <= max_ns; ++ns) {
    const int64_t T = cdiv(max_tiles, ns);
    if (ns > 1 && T < 4) break;
    int64_t ctas = 0;
    double merge_us = 0.0;
    for (int i = 0; i < n; ++i) {
      const int64_t nsi = std::min<int64_t>(64, cdiv(kv_tiles[i], T));
      ctas += (int64_t)pl.m_pairs[i] * h_kv * nsi;
      if (nsi > 1) merge_us += (double)pl.rows[i] * (d + 1) * 4 * 2 * nsi / 6.0e6;
    }
    const double est = (double)cdiv(ctas, sms) * T * t_tile_us + merge_us;
    if (est < best * 0.999) {
      best = est;
      best_T = T;
    }
  }
  for (int i = 0; i < n; ++i) {
    int64_t nsi = std::min<int64_t>(64, cdiv(kv_tiles[i], best_T));
    const int64_t tpsi = cdiv(kv_tiles[i], nsi);
    nsi = cdiv(kv_tiles[i], tpsi);
    pl.n_split.push_back((int)nsi);
    pl.tps.push_back((int)tpsi);
    pl.ws_off.push_back(pl.ws_bytes);
    if (nsi > 1) pl.ws_bytes += round_up((size_t)nsi * pl.part_stride[i] * sizeof(float), 256);
    pl.n_items += (int64_t)pl.m_pairs[i] * h_kv * nsi;
  }
  return pl;
}

size_t prefill_ws_bound(int64_t c, int32_t h_q, int32_t d) {
  const int64_t rows = c * h_q;
  return round_up((size_t)64 * round_up((size_t)(rows * (d + 1)), 4) * sizeof(float), 256);
}

template <int D, int G>
medha_status launch_prefill(const PrefillBatch &b, int64_t items, cudaStream_t st) {
  using L = WsLayout<D>;
  // the dynamic shared memory opt-in is a per-device (context) attribute: set it once per
  // device, thread-safely (std::call_once per device slot)
  static std::once_flag once[64];
  static cudaError_t attr_err[64];
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(MEDHA_ENOTSUP, "device ordinal %d >= 64", dev);
  std::call_once(once[dev], [dev] {
    attr_err[dev] = cudaFuncSetAttribute(prefill_ws_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L::kAlloc);
  });
  CUDA_TRY(attr_err[dev]);
  launch_pdl(prefill_ws_kernel<D, G>, dim3((unsigned)items), dim3(kWsThreads), (size_t)L::kAlloc, st, b);
  LAUNCH_CHECK("prefill_ws_kernel");
  return MEDHA_OK;
}

template <int D>
medha_status dispatch_prefill_g(int G, const PrefillBatch &b, int64_t items, cudaStream_t st) {
  switch (G) {
    case 1: return launch_prefill<D, 1>(b, items, st);
    case 2: return launch_prefill<D, 2>(b, items, st);
    case 4: return launch_prefill<D, 4>(b, items, st);
    case 8: return launch_prefill<D, 8>(b, items, st);
    case 16: return launch_prefill<D, 16>(b, items, st);
    default: return fail(MEDHA_ENOTSUP, "group size %d", G);
  }
}

medha_status merge_impl(const float *parts, int32_t P, int64_t rows, int64_t part_stride, int32_t d, float *o_out,
                        float *lse_out, void *o_bf16, cudaStream_t st) {
  if (rows == 0) return MEDHA_OK;
  const int warps_per_block = 8;
  const int64_t blocks = cdiv(rows, warps_per_block);
  if (blocks > INT32_MAX) return fail(MEDHA_ERANGE, "too many rows");
  __nv_bfloat16 *ob = static_cast<__nv_bfloat16 *>(o_bf16);
  if (d == 128)
    launch_pdl(lse_merge_kernel<128>, dim3((unsigned)blocks), dim3(32 * warps_per_block), 0, st, parts, P, rows,
               part_stride, o_out, lse_out, ob);
  else
    launch_pdl(lse_merge_kernel<64>, dim3((unsigned)blocks), dim3(32 * warps_per_block), 0, st, parts, P, rows,
               part_stride, o_out, lse_out, ob);
  LAUNCH_CHECK("lse_merge_kernel");
  return MEDHA_OK;
}

// A batch of up to kPfMaxBatch prefill chunks (all of the same layer: h_q, h_kv, d) in
// one launch, then one K5 merge per chunk whose KV range was split.
medha_status prefill_batch_impl(const PrefillChunk *ch, int n, int32_t h_q, float scale, void *ws, size_t ws_bytes,
                                cudaStream_t st) {
  if (n <= 0) return n == 0 ? MEDHA_OK : fail(MEDHA_EINVAL, "negative batch");
  if (!(scale > 0.f)) return fail(MEDHA_EINVAL, "scale must be > 0");
  medha_status s;
  const int32_t h_kv = ch[0].kv ? ch[0].kv->h_kv : 0, d = ch[0].kv ? ch[0].kv->d : 0;
  for (int i = 0; i < n; ++i) {
    if ((s = check_shard(ch[i].kv))) return s;
    if (ch[i].kv->h_kv != h_kv || ch[i].kv->d != d) return fail(MEDHA_ESHAPE, "chunks disagree on h_kv/d");
    if (ch[i].c < 1) return fail(MEDHA_EINVAL, "chunk %d is empty", i);
    if (ch[i].c > 65536) return fail(MEDHA_ENOTSUP, "chunk %lld > 65536", (long long)ch[i].c);
    if (!ch[i].q || !ch[i].o || !ch[i].lse) return fail(MEDHA_EINVAL, "null argument (chunk %d)", i);
    if (!aligned16(ch[i].q) || !aligned16(ch[i].o)) return fail(MEDHA_EINVAL, "q/o not 16-byte aligned");
    if (head_stride(*ch[i].kv) > INT32_MAX) return fail(MEDHA_ENOTSUP, "capacity/pool > 2^31 tokens");
    if (ch[i].kv->page_table && ch[i].kv->page_size < kWsTileN)
      return fail(MEDHA_ENOTSUP, "prefill needs page_size >= %d (got %d)", kWsTileN, ch[i].kv->page_size);
  }
  if (h_q <= 0 || h_q % h_kv != 0) return fail(MEDHA_EINVAL, "h_q %d not a multiple of h_kv %d", h_q, h_kv);
  const int G = h_q / h_kv;
  if (!supported_g(G)) return fail(MEDHA_ENOTSUP, "group size %d not in {1,2,4,8,16}", G);
  size_t ws_used = 0;
  for (int b0 = 0; b0 < n; b0 += kPfMaxBatch) {
    const int nb = std::min(kPfMaxBatch, n - b0);
    PrefillBatchPlan pl = plan_prefill_batch(ch + b0, nb, h_q, h_kv, d);
    if (pl.ws_bytes > 0) {
      if (!ws || !aligned16(ws)) return fail(MEDHA_EWORKSPACE, "null/misaligned workspace");
      if (ws_used + pl.ws_bytes > ws_bytes)
        return fail(MEDHA_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, ws_used + pl.ws_bytes);
    }
    if (pl.n_items > INT32_MAX) return fail(MEDHA_ERANGE, "grid too large");
    thread_local PrefillBatch b;   // ~15 KB of kernel parameters (host-side staging, per thread)
    memset(&b, 0, sizeof(b));
    b.n_seq = nb;
    const int TQ = kWsTileM / G;
    int64_t item = 0;
    for (int i = 0; i < nb; ++i) {
      const PrefillChunk &c = ch[b0 + i];
      const medha_kv_shard *kv = c.kv;
      if ((s = make_map_3d(&b.maps[i][0], c.q, d, h_q, c.c, (uint64_t)d * 2, (uint64_t)h_q * d * 2, 64, G, TQ)))
        return s;
      // contiguous: the map ends at len (TMA zero-fills the ragged tail); paged: the map
      // spans the whole pool and the producer translates each 128-token tile through the
      // page table (rows past len inside the last page are finite by contract, masked to 0)
      const uint64_t hs = (uint64_t)head_stride(*kv);
      const uint64_t len_ext = kv->page_table ? hs : (uint64_t)std::max<int64_t>(kv->len, 1);
      if ((s = make_map_3d(&b.maps[i][1], kv->k, d, len_ext, h_kv, (uint64_t)d * 2, hs * d * 2, 64, kWsTileN, 1)))
        return s;
      if ((s = make_map_3d(&b.maps[i][2], kv->v, d, len_ext, h_kv, (uint64_t)d * 2, hs * d * 2, 64, kWsTileN, 1)))
        return s;
      PrefillWsParams &p = b.seq[i];
      const bool split = pl.n_split[i] > 1;
      p.o = split ? reinterpret_cast<float *>(static_cast<char *>(ws) + ws_used + pl.ws_off[i]) : c.o;
      p.lse = c.lse;
      p.c = c.c;
      p.len = kv->len;
      p.pos0 = kv->pos0;
      p.q_pos0 = c.q_pos0;
      p.rows = pl.rows[i];
      p.part_stride = pl.part_stride[i];
      p.h_q = h_q;
      p.h_kv = h_kv;
      p.n_split = pl.n_split[i];
      p.tiles_per_split = pl.tps[i];
      p.m_pairs = pl.m_pairs[i];
      p.pt = kv->page_table;
      p.psl = kv->page_table ? log2_pow2(kv->page_size) : 0;
      p.item_begin = (int32_t)item;
      p.scale_log2 = scale * kLog2e;
      item += (int64_t)pl.m_pairs[i] * h_kv * pl.n_split[i];
    }
    s = (d == 128) ? dispatch_prefill_g<128>(G, b, item, st) : dispatch_prefill_g<64>(G, b, item, st);
    if (s) return s;
    for (int i = 0; i < nb; ++i) {
      if (pl.n_split[i] <= 1) continue;
      const PrefillChunk &c = ch[b0 + i];
      s = merge_impl(b.seq[i].o, pl.n_split[i], pl.rows[i], pl.part_stride[i], d, c.o, c.lse, nullptr, st);
      if (s) return s;
    }
    ws_used += pl.ws_bytes;
  }
  return MEDHA_OK;
}

medha_status prefill_impl(const medha_kv_shard *kv, const void *q, int64_t c, int32_t h_q, int64_t q_pos0,
                          float scale, float *o, float *lse, void *ws, size_t ws_bytes, cudaStream_t st) {
  medha_status s = check_shard(kv);
  if (s) return s;
  if (c < 0) return fail(MEDHA_EINVAL, "negative chunk");
  if (c == 0) return MEDHA_OK;
  PrefillChunk one{kv, q, c, q_pos0, o, lse};
  return prefill_batch_impl(&one, 1, h_q, scale, ws, ws_bytes, st);
}

}  // namespace

// =============================================================================================
// C ABI
// =============================================================================================
struct medha_kvp_comm {
  ncclComm_t nccl;
  int32_t rank, world;
  // fused P2P exchange (single node, CUDA IPC; at world 1 the local buffer alone): one
  // buffer per rank holding [2 parities][world src][slot floats] receive slots +
  // [2][world][units] epoch flags + the device epoch word (medha::XchgLayout below)
  bool p2p = false;
  bool p2p_on = false;      // runtime switch (medha_kvp_comm_set_p2p)
  int device = -1;
  char *local = nullptr;    // this rank's buffer
  char *peer[kMaxKvpRanks] = {};  // every rank's buffer mapped here (peer[rank] = local)
  int64_t slot = 0;         // floats per (parity, src) slot
  int32_t units = 0;        // flags per (parity, src)
  void *agree = nullptr;    // device scratch of the set-up agreement (allocated before NCCL init)
  uint32_t *err_host = nullptr;   // mapped pinned word the decode kernel sets on a timed-out wait
  uint32_t *err_dev = nullptr;    // its device address
  uint64_t timeout_ns = 0;
  uint32_t debug = 0;       // test hook (medha_kvp_comm_debug)
  bool broken = false;      // a fused wait timed out: every later collective call fails
};

namespace {
constexpr int64_t kP2PSlotFloats = (int64_t)64 * 64 * 129;   // batch 64 x h_q 64 x (d 128 + 1)
constexpr int32_t kP2PUnits = 4096;                           // (seq, kv head) units per call
constexpr size_t kAgreeBytes = sizeof(cudaIpcMemHandle_t) * (kMaxKvpRanks + 1) + 256;

size_t p2p_flags_off(int world) { return (size_t)2 * world * kP2PSlotFloats * sizeof(float); }
size_t p2p_epoch_off(int world) { return p2p_flags_off(world) + (size_t)2 * world * kP2PUnits * sizeof(uint32_t); }
size_t p2p_bytes(int world) { return p2p_epoch_off(world) + 256; }

// Collective: allocate the receive buffer, exchange CUDA IPC handles with ncclAllGather
// and map every peer's buffer.  Every rank takes part in both agreement all-reduces
// whatever fails locally, and any failure leaves the communicator on the NCCL path.
// World 1: the local buffer alone (the kernel's push, flags and merge run as a self-loop).
void p2p_setup(medha_kvp_comm *c) {
  if (c->world > kMaxKvpRanks || getenv_flag("MEDHA_KVP_P2P", 1) == 0 || !c->agree || !c->err_dev) return;
  const size_t bytes = p2p_bytes(c->world);
  int ok = 1;
  if (cudaMalloc(&c->local, bytes) != cudaSuccess || cudaMemset(c->local, 0, bytes) != cudaSuccess) ok = 0;
  if (c->world == 1) {
    if (ok) {
      cudaDeviceSynchronize();
      c->peer[0] = c->local;
    }
  } else {
    cudaStream_t st = nullptr;
    cudaIpcMemHandle_t mine;
    memset(&mine, 0, sizeof(mine));
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) st = nullptr;
    if (!ok || !st || cudaIpcGetMemHandle(&mine, c->local) != cudaSuccess) ok = 0;
    char *slots = static_cast<char *>(c->agree);
    int *dok = reinterpret_cast<int *>(slots + sizeof(cudaIpcMemHandle_t) * (kMaxKvpRanks + 1));
    auto agree = [&](int v) {   // collective min over ranks (every rank calls it)
      cudaMemcpy(dok, &v, sizeof(int), cudaMemcpyHostToDevice);
      ncclAllReduce(dok, dok, 1, ncclInt, ncclMin, c->nccl, st);
      cudaStreamSynchronize(st);
      cudaMemcpy(&v, dok, sizeof(int), cudaMemcpyDeviceToHost);
      return v;
    };
    ok = agree(ok);
    if (ok) {
      cudaMemcpy(slots + sizeof(cudaIpcMemHandle_t) * kMaxKvpRanks, &mine, sizeof(mine), cudaMemcpyHostToDevice);
      ncclAllGather(slots + sizeof(cudaIpcMemHandle_t) * kMaxKvpRanks, slots, sizeof(cudaIpcMemHandle_t), ncclChar,
                    c->nccl, st);
      cudaStreamSynchronize(st);
      std::vector<cudaIpcMemHandle_t> hs(c->world);
      cudaMemcpy(hs.data(), slots, sizeof(cudaIpcMemHandle_t) * c->world, cudaMemcpyDeviceToHost);
      for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) {
          c->peer[r] = c->local;
          continue;
        }
        void *ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, hs[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) ok = 0;
        c->peer[r] = static_cast<char *>(ptr);
      }
      cudaGetLastError();
      ok = agree(ok);
    }
    if (st) cudaStreamDestroy(st);
  }
  if (ok) {
    c->slot = kP2PSlotFloats;
    c->units = kP2PUnits;
    c->p2p = c->p2p_on = true;
  } else {
    for (int r = 0; r < c->world; ++r)
      if (r != c->rank && c->peer[r]) cudaIpcCloseMemHandle(c->peer[r]);
    if (c->local) cudaFree(c->local);
    c->local = nullptr;
    for (int r = 0; r < kMaxKvpRanks; ++r) c->peer[r] = nullptr;
  }
  cudaGetLastError();
}

// Sticky health of a communicator: a fused wait that timed out (set by the kernel in mapped
// host memory, read here without synchronising) marks it broken for good.
medha_status comm_health(medha_kvp_comm *c) {
  if (!c->broken && c->err_host && *reinterpret_cast<volatile uint32_t *>(c->err_host) != 0u) c->broken = true;
  if (c->broken)
    return fail(MEDHA_ENCCL,
                "KVP communicator unusable: a fused-exchange wait timed out (a rank did not join a collective "
                "call, or ranks disagree on its arguments); destroy and re-create it");
  return MEDHA_OK;
}
}  // namespace

extern "C" {

const char *medha_status_str(medha_status s) {
  switch (s) {
    case MEDHA_OK: return "MEDHA_OK";
    case MEDHA_EINVAL: return "MEDHA_EINVAL";
    case MEDHA_ESHAPE: return "MEDHA_ESHAPE";
    case MEDHA_ERANGE: return "MEDHA_ERANGE";
    case MEDHA_ENOTSUP: return "MEDHA_ENOTSUP";
    case MEDHA_EWORKSPACE: return "MEDHA_EWORKSPACE";
    case MEDHA_ECUDA: return "MEDHA_ECUDA";
    case MEDHA_ENCCL: return "MEDHA_ENCCL";
    default: return "MEDHA_UNKNOWN";
  }
}

const char *medha_last_error(void) { return g_last_error.c_str(); }

int32_t medha_version(void) { return (1 << 16) | 0; }

namespace {
// kv_append, optionally with a 16-byte-vector copy riding in the same launch (decode_step_host)
medha_status kv_append_impl(medha_kv_shard *kv, const void *k_new, const void *v_new, int64_t n, const void *cp_src,
                            void *cp_dst, int64_t cp_bytes, cudaStream_t st) {
  const int32_t vec = kv->d / 8;
  const int64_t total = std::max<int64_t>(n * kv->h_kv * vec, cp_bytes / 16);
  const int threads = 256;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(cdiv(total, threads), (int64_t)num_sms() * 8));
  launch_pdl(kv_append_kernel, dim3((unsigned)blocks), dim3(threads), 0, st, static_cast<const uint4 *>(k_new),
             static_cast<const uint4 *>(v_new), static_cast<uint4 *>(kv->k), static_cast<uint4 *>(kv->v), (int64_t)n,
             kv->h_kv, vec, head_stride(*kv), kv->len, (const int32_t *)kv->page_table,
             kv->page_table ? log2_pow2(kv->page_size) : 0, static_cast<const uint4 *>(cp_src),
             static_cast<uint4 *>(cp_dst), cp_bytes / 16);
  LAUNCH_CHECK("kv_append_kernel");
  kv->len += n;
  return MEDHA_OK;
}

// Device view of a host buffer: non-null iff it is pinned and mapped into the device's
// address space (cudaHostAlloc memory under UVA, e.g. torch pin_memory()), so kernels can
// read / write it directly over the host link (zero-copy).
void *mapped_host_view(const void *h) {
  if (!h) return nullptr;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return (a.type == cudaMemoryTypeHost && a.devicePointer) ? a.devicePointer : nullptr;
}
}  // namespace

medha_status medha_kv_append(medha_kv_shard *kv, const void *k_new, const void *v_new, int64_t n, void *stream) {
  medha_status s = check_shard(kv);
  if (s) return s;
  if (n < 0) return fail(MEDHA_EINVAL, "negative n");
  if (n == 0) return MEDHA_OK;
  if (!k_new || !v_new) return fail(MEDHA_EINVAL, "null k_new/v_new");
  if (!aligned16(k_new) || !aligned16(v_new)) return fail(MEDHA_EINVAL, "k_new/v_new not 16-byte aligned");
  if (kv->len + n > kv->capacity)
    return fail(MEDHA_ERANGE, "append %lld tokens at len %lld exceeds capacity %lld", (long long)n, (long long)kv->len,
                (long long)kv->capacity);
  return kv_append_impl(kv, k_new, v_new, n, nullptr, nullptr, 0, static_cast<cudaStream_t>(stream));
}

size_t medha_decode_workspace_size(int32_t batch, int32_t h_q, int32_t h_kv, int32_t d) {
  if (batch <= 0 || h_q <= 0 || h_kv <= 0 || d <= 0) return 256;
  return decode_ws_layout(batch, h_q, h_kv, d, nullptr, nullptr);
}

medha_status medha_attn_decode_partial(const medha_kv_shard *kvs_host, int32_t batch, const void *q, int32_t h_q,
                                       const int64_t *q_pos_host, float scale, float *o, float *lse, void *ws,
                                       size_t ws_bytes, void *stream) {
  return decode_partial_impl(kvs_host, batch, q, h_q, q_pos_host, scale, o, lse, ws, ws_bytes,
                             static_cast<cudaStream_t>(stream));
}

medha_status medha_attn_decode_append(medha_kv_shard *kvs_host, int32_t batch, const void *k_new, const void *v_new,
                                      const int32_t *append_host, const void *q, int32_t h_q,
                                      const int64_t *q_pos_host, float scale, float *o, float *lse, void *ws,
                                      size_t ws_bytes, void *stream) {
  DecodeAppend app{k_new, v_new, append_host};
  medha_status s = decode_partial_impl(kvs_host, batch, q, h_q, q_pos_host, scale, o, lse, ws, ws_bytes,
                                       static_cast<cudaStream_t>(stream), nullptr, nullptr, &app);
  if (s == MEDHA_OK)
    for (int b = 0; b < batch; ++b)
      if (!append_host || append_host[b]) kvs_host[b].len += 1;
  return s;
}

size_t medha_prefill_workspace_size(int64_t c, int32_t h_q, int32_t h_kv, int32_t d) {
  (void)h_kv;
  if (c <= 0 || h_q <= 0 || d <= 0) return 256;
  return prefill_ws_bound(c, h_q, d);
}

medha_status medha_attn_prefill_chunk(const medha_kv_shard *kv, const void *q, int64_t c, int32_t h_q, int64_t q_pos0,
                                      float scale, float *o, float *lse, void *ws, size_t ws_bytes, void *stream) {
  return prefill_impl(kv, q, c, h_q, q_pos0, scale, o, lse, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

size_t medha_prefill_batch_workspace_size(int32_t n, const int64_t *c_host, int32_t h_q, int32_t d) {
  if (n <= 0 || !c_host || h_q <= 0 || d <= 0) return 256;
  size_t total = 0;
  for (int i = 0; i < n; ++i) total += prefill_ws_bound(std::max<int64_t>(c_host[i], 1), h_q, d);
  return total;
}

medha_status medha_attn_prefill_batch(const medha_prefill_chunk *chunks_host, int32_t n, int32_t h_q, float scale,
                                      void *ws, size_t ws_bytes, void *stream) {
  if (n < 0) return fail(MEDHA_EINVAL, "negative batch");
  if (n == 0) return MEDHA_OK;
  if (!chunks_host) return fail(MEDHA_EINVAL, "null chunk array");
  std::vector<PrefillChunk> ch(n);
  for (int i = 0; i < n; ++i) {
    const medha_prefill_chunk &c = chunks_host[i];
    ch[i] = PrefillChunk{c.kv, c.q, c.c, c.q_pos0, c.o, c.lse};
  }
  return prefill_batch_impl(ch.data(), n, h_q, scale, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

medha_status medha_merge_partials(const float *parts, int32_t P, int64_t rows, int32_t d, float *o_out, float *lse_out,
                                  void *o_out_bf16, void *stream) {
  if (!parts || !o_out) return fail(MEDHA_EINVAL, "null argument");
  if (P < 1 || P > 64) return fail(MEDHA_EINVAL, "P = %d not in [1, 64]", P);
  if (rows < 0) return fail(MEDHA_EINVAL, "negative rows");
  if (!supported_d(d)) return fail(MEDHA_ENOTSUP, "head dim %d", d);
  return merge_impl(parts, P, rows, rows * (d + 1), d, o_out, lse_out, o_out_bf16, static_cast<cudaStream_t>(stream));
}

// ---- KVP -------------------------------------------------------------------------------------
medha_status medha_kvp_unique_id(uint8_t id_out[128]) {
  if (!id_out) return fail(MEDHA_EINVAL, "null id");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(MEDHA_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(id_out, &id, 128);
  return MEDHA_OK;
}

medha_status medha_kvp_comm_create(const uint8_t id[128], int32_t rank, int32_t world, medha_kvp_comm **out) {
  if (!id || !out) return fail(MEDHA_EINVAL, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(MEDHA_EINVAL, "rank %d / world %d", rank, world);
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  medha_kvp_comm *c = new medha_kvp_comm();
  c->rank = rank;
  c->world = world;
  c->timeout_ns = (uint64_t)std::max(1, getenv_flag("MEDHA_KVP_TIMEOUT_MS", 30000)) * 1000000ull;
  cudaGetDevice(&c->device);
  // local resources the set-up needs are taken BEFORE the collective NCCL init, so a rank
  // that cannot get them fails before any peer is waiting on it inside a collective
  void *eh = nullptr;
  if (cudaMalloc(&c->agree, kAgreeBytes) != cudaSuccess ||
      cudaHostAlloc(&eh, 256, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    if (c->agree) cudaFree(c->agree);
    delete c;
    return fail(MEDHA_ECUDA, "kvp_comm_create: device/host allocation failed");
  }
  c->err_host = static_cast<uint32_t *>(eh);
  *c->err_host = 0u;
  void *ed = nullptr;
  if (cudaHostGetDevicePointer(&ed, eh, 0) == cudaSuccess) c->err_dev = static_cast<uint32_t *>(ed);
  cudaGetLastError();
  ncclResult_t r = ncclCommInitRank(&c->nccl, world, uid, rank);
  if (r != ncclSuccess) {
    cudaFree(c->agree);
    cudaFreeHost(eh);
    delete c;
    return fail(MEDHA_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  p2p_setup(c);
  *out = c;
  return MEDHA_OK;
}

medha_status medha_kvp_comm_destroy(medha_kvp_comm *comm) {
  if (!comm) return MEDHA_OK;
  cudaDeviceSynchronize();
  if (comm->p2p) {
    for (int r = 0; r < comm->world; ++r)
      if (r != comm->rank && comm->peer[r]) cudaIpcCloseMemHandle(comm->peer[r]);
    cudaFree(comm->local);
  }
  if (comm->agree) cudaFree(comm->agree);
  if (comm->err_host) cudaFreeHost(comm->err_host);
  ncclResult_t r = comm->broken ? ncclCommAbort(comm->nccl) : ncclCommDestroy(comm->nccl);
  delete comm;
  if (r != ncclSuccess) return fail(MEDHA_ENCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return MEDHA_OK;
}

medha_status medha_kvp_comm_status(medha_kvp_comm *comm) {
  if (!comm) return fail(MEDHA_EINVAL, "null comm");
  return comm_health(comm);
}

medha_status medha_kvp_comm_set_timeout(medha_kvp_comm *comm, uint64_t timeout_ns) {
  if (!comm) return fail(MEDHA_EINVAL, "null comm");
  if (timeout_ns == 0) return fail(MEDHA_EINVAL, "timeout must be > 0");
  comm->timeout_ns = timeout_ns;
  return MEDHA_OK;
}

medha_status medha_kvp_comm_debug(medha_kvp_comm *comm, uint32_t flags) {
  if (!comm) return fail(MEDHA_EINVAL, "null comm");
  comm->debug = flags;
  return MEDHA_OK;
}

medha_status medha_kvp_comm_info(const medha_kvp_comm *comm, int32_t *rank, int32_t *world) {
  if (!comm) return fail(MEDHA_EINVAL, "null comm");
  if (rank) *rank = comm->rank;
  if (world) *world = comm->world;
  return MEDHA_OK;
}

int32_t medha_kvp_comm_p2p(const medha_kvp_comm *comm) { return (comm && comm->p2p && comm->p2p_on) ? 1 : 0; }

medha_status medha_kvp_comm_set_p2p(medha_kvp_comm *comm, int32_t enable) {
  if (!comm) return fail(MEDHA_EINVAL, "null comm");
  if (enable && !comm->p2p) return fail(MEDHA_ENOTSUP, "peer-to-peer exchange unavailable on this communicator");
  comm->p2p_on = enable != 0;
  return MEDHA_OK;
}

static medha_status kvp_exchange_merge(medha_kvp_comm *comm, const float *send, float *recv, int64_t rows, int32_t d,
                                       float *o_out, float *lse_out, void *o_bf16, cudaStream_t st) {
  const size_t count = (size_t)rows * (d + 1);
  ncclResult_t r;
  {
    NvtxRange nv("medha/kvp/exchange (ncclAllGather)");
    r = ncclAllGather(send, recv, count, ncclFloat, comm->nccl, st);
  }
  if (r != ncclSuccess) return fail(MEDHA_ENCCL, "ncclAllGather: %s", ncclGetErrorString(r));
  ncclResult_t async_err = ncclSuccess;
  if (ncclCommGetAsyncError(comm->nccl, &async_err) == ncclSuccess && async_err != ncclSuccess &&
      async_err != ncclInProgress)
    return fail(MEDHA_ENCCL, "NCCL async error: %s", ncclGetErrorString(async_err));
  NvtxRange nv("medha/kvp/merge (lse_merge_kernel)");
  return merge_impl(recv, comm->world, rows, (int64_t)count, d, o_out, lse_out, o_bf16, st);
}

static size_t kvp_buf_bytes(int32_t world, int64_t rows, int32_t d) {
  const size_t count = (size_t)rows * (d + 1);
  return round_up(count * 4, 256) + round_up(count * 4 * (size_t)world, 256);
}

size_t medha_kvp_exchange_workspace_size(int32_t world, int64_t rows, int32_t d) {
  if (world < 1 || rows <= 0 || d <= 0) return 256;
  return round_up((size_t)rows * (d + 1) * 4 * (size_t)world, 256);
}

medha_status medha_kvp_exchange_merge(medha_kvp_comm *comm, const float *send, int64_t rows, int32_t d, float *o_out,
                                      float *lse_out, void *o_out_bf16, void *ws, size_t ws_bytes, void *stream) {
  if (!comm || !send || !o_out) return fail(MEDHA_EINVAL, "null argument");
  if (rows <= 0) return fail(MEDHA_EINVAL, "rows must be > 0");
  if (medha_status h = comm_health(comm)) return h;
  if (!supported_d(d)) return fail(MEDHA_ENOTSUP, "head dim %d", d);
  const size_t need = medha_kvp_exchange_workspace_size(comm->world, rows, d);
  if (!ws || ws_bytes < need) return fail(MEDHA_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  return kvp_exchange_merge(comm, send, static_cast<float *>(ws), rows, d, o_out, lse_out, o_out_bf16,
                            static_cast<cudaStream_t>(stream));
}

size_t medha_kvp_workspace_size(int32_t world, int32_t batch, int32_t h_q, int32_t h_kv, int32_t d) {
  if (world < 1 || batch <= 0 || h_q <= 0 || d <= 0) return 256;
  return kvp_buf_bytes(world, (int64_t)batch * h_q, d) + round_up(medha_decode_workspace_size(batch, h_q, h_kv, d), 256);
}

static medha_status kvp_decode_impl(medha_kvp_comm *comm, const medha_kv_shard *kvs_host, int32_t batch, const void *q,
                                    int32_t h_q, const int64_t *q_pos_host, float scale, float *o_out, float *lse_out,
                                    void *o_out_bf16, void *ws, size_t ws_bytes, void *stream,
                                    const DecodeAppend *app) {
  if (!comm) return fail(MEDHA_EINVAL, "null comm");
  if (medha_status h = comm_health(comm)) return h;
  if (batch <= 0 || !kvs_host) return fail(MEDHA_EINVAL, "empty batch");
  if (!o_out) return fail(MEDHA_EINVAL, "null o_out");
  const int32_t d = kvs_host[0].d, h_kv = kvs_host[0].h_kv;
  if (!supported_d(d)) return fail(MEDHA_ENOTSUP, "head dim %d", d);
  const int64_t rows = (int64_t)batch * h_q;
  const size_t need = medha_kvp_workspace_size(comm->world, batch, h_q, h_kv, d);
  if (!ws || ws_bytes < need) return fail(MEDHA_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the decode workspace (its zeroed counter block first) sits at offset 0 whatever the call
  // shape, so one workspace serves calls of different shapes; send / recv follow it
  char *base = static_cast<char *>(ws);
  const size_t count = (size_t)rows * (d + 1);
  char *dws = base;
  const size_t dws_bytes = round_up(medha_decode_workspace_size(batch, h_q, h_kv, d), 256);
  float *send = reinterpret_cast<float *>(base + dws_bytes);
  float *recv = reinterpret_cast<float *>(base + dws_bytes + round_up(count * 4, 256));
  if (comm->p2p && comm->p2p_on && batch <= kDecodeMaxSeqPerLaunch && (int64_t)count <= comm->slot &&
      (int64_t)batch * h_kv <= comm->units) {
    // fused: the decode kernel's last CTAs push the partials over NVLink and merge; the
    // epoch and the slot parity are resolved on the device (graph-replayable)
    DecodeXchg x;
    memset(&x, 0, sizeof(x));
    x.world = comm->world;
    x.rank = comm->rank;
    x.units = comm->units;
    x.rows = rows;
    x.slot = comm->slot;
    x.debug = comm->debug;
    x.timeout_ns = comm->timeout_ns;
    for (int r = 0; r < comm->world; ++r) x.peer[r] = comm->peer[r];
    x.epoch = reinterpret_cast<uint32_t *>(comm->local + p2p_epoch_off(comm->world));
    x.err = comm->err_dev;
    x.o = o_out;
    x.lse = lse_out;
    x.obf = static_cast<__nv_bfloat16 *>(o_out_bf16);
    NvtxRange nv("medha/kvp/decode: partial + NVLink exchange + merge (one kernel)");
    return decode_partial_impl(kvs_host, batch, q, h_q, q_pos_host, scale, o_out, send + rows * d, dws,
                               dws_bytes, st, &x, nullptr, app);
  }
  medha_status s;
  {
    NvtxRange nv("medha/kvp/partial (decode)");
    s = decode_partial_impl(kvs_host, batch, q, h_q, q_pos_host, scale, send, send + rows * d, dws, dws_bytes, st,
                            nullptr, nullptr, app);
  }
  if (s) return s;
  return kvp_exchange_merge(comm, send, recv, rows, d, o_out, lse_out, o_out_bf16, st);
}

medha_status medha_kvp_decode(medha_kvp_comm *comm, const medha_kv_shard *kvs_host, int32_t batch, const void *q,
                              int32_t h_q, const int64_t *q_pos_host, float scale, float *o_out, float *lse_out,
                              void *o_out_bf16, void *ws, size_t ws_bytes, void *stream) {
  return kvp_decode_impl(comm, kvs_host, batch, q, h_q, q_pos_host, scale, o_out, lse_out, o_out_bf16, ws, ws_bytes,
                         stream, nullptr);
}

medha_status medha_kvp_decode_append(medha_kvp_comm *comm, medha_kv_shard *kvs_host, int32_t batch, const void *k_new,
                                     const void *v_new, const int32_t *append_host, const void *q, int32_t h_q,
                                     const int64_t *q_pos_host, float scale, float *o_out, float *lse_out,
                                     void *o_out_bf16, void *ws, size_t ws_bytes, void *stream) {
  DecodeAppend app{k_new, v_new, append_host};
  medha_status s = kvp_decode_impl(comm, kvs_host, batch, q, h_q, q_pos_host, scale, o_out, lse_out, o_out_bf16, ws,
                                   ws_bytes, stream, &app);
  if (s == MEDHA_OK)
    for (int b = 0; b < batch; ++b)
      if (!append_host || append_host[b]) kvs_host[b].len += 1;
  return s;
}

size_t medha_kvp_prefill_workspace_size(int32_t world, int64_t c, int32_t h_q, int32_t h_kv, int32_t d) {
  if (world < 1 || c <= 0 || h_q <= 0 || d <= 0) return 256;
  return kvp_buf_bytes(world, c * h_q, d) + medha_prefill_workspace_size(c, h_q, h_kv, d);
}

medha_status medha_kvp_prefill_chunk(medha_kvp_comm *comm, const medha_kv_shard *kv, const void *q, int64_t c,
                                     int32_t h_q, int64_t q_pos0, float scale, float *o_out, float *lse_out,
                                     void *o_out_bf16, void *ws, size_t ws_bytes, void *stream) {
  if (!comm) return fail(MEDHA_EINVAL, "null comm");
  if (medha_status h = comm_health(comm)) return h;
  if (!kv) return fail(MEDHA_EINVAL, "null shard");
  if (c <= 0) return fail(MEDHA_EINVAL, "empty chunk");
  if (!o_out) return fail(MEDHA_EINVAL, "null o_out");
  const int32_t d = kv->d;
  if (!supported_d(d)) return fail(MEDHA_ENOTSUP, "head dim %d", d);
  const int64_t rows = c * h_q;
  const size_t need = medha_kvp_prefill_workspace_size(comm->world, c, h_q, kv->h_kv, d);
  if (!ws || ws_bytes < need) return fail(MEDHA_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char *base = static_cast<char *>(ws);
  const size_t count = (size_t)rows * (d + 1);
  float *send = reinterpret_cast<float *>(base);
  float *recv = reinterpret_cast<float *>(base + round_up(count * 4, 256));
  char *pws = base + kvp_buf_bytes(comm->world, rows, d);
  medha_status s;
  {
    NvtxRange nv("medha/kvp/partial (prefill chunk)");
    s = prefill_impl(kv, q, c, h_q, q_pos0, scale, send, send + rows * d, pws, ws_bytes - (size_t)(pws - base), st);
  }
  if (s) return s;
  return kvp_exchange_merge(comm, send, recv, rows, d, o_out, lse_out, o_out_bf16, st);
}

// ---- end-to-end decode step with host buffers -----------------------------------------------
size_t medha_decode_step_workspace_size(int32_t world, int32_t h_q, int32_t h_kv, int32_t d) {
  if (h_q <= 0 || h_kv <= 0 || d <= 0) return 256;
  const size_t stage = round_up((size_t)h_q * d * 2, 256) + 2 * round_up((size_t)h_kv * d * 2, 256) +
                       round_up((size_t)h_q * d * 4, 256) + round_up((size_t)h_q * 4, 256);
  // sized for the KVP call (a world-1 communicator included); >= the plain decode's
  const size_t inner = round_up(medha_kvp_workspace_size(std::max(world, 1), 1, h_q, h_kv, d), 256);
  return stage + inner;
}

}  // extern "C"

namespace {
// decode_step_host, split into the per-call-invariant part (validation of the host buffers,
// their mapped device views, workspace carving: StepSetup) and the per-step launches
// (step_run).  medha_decode_plan keeps a StepSetup across steps.
struct StepSetup {
  medha_kvp_comm *comm;
  int32_t h_q, h_kv, d;
  float scale;
  const void *q_host, *k_host, *v_host;
  float *o_host, *lse_host;
  char *inner;
  size_t inner_bytes;
  void *q_dev, *k_dev, *v_dev;
  float *o_dev, *lse_dev;
  const void *q_map, *k_map, *v_map;
  float *o_map, *l_map;
  bool zc_in_q, zc_in_kv, zc_out;
};

medha_status step_setup(medha_kvp_comm *comm, const medha_kv_shard *kv, int32_t h_q, float scale, const void *q_host,
                        const void *k_new_host, const void *v_new_host, float *o_host, float *lse_host, void *ws,
                        size_t ws_bytes, StepSetup *S) {
  medha_status s = check_shard(kv);
  if (s) return s;
  if (!q_host || !o_host) return fail(MEDHA_EINVAL, "null host buffer");
  const int32_t d = kv->d, h_kv = kv->h_kv;
  const int32_t world = comm ? comm->world : 1;
  const size_t need = medha_decode_step_workspace_size(world, h_q, h_kv, d);
  if (!ws || ws_bytes < need) return fail(MEDHA_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  memset(S, 0, sizeof(*S));
  S->comm = comm;
  S->h_q = h_q;
  S->h_kv = h_kv;
  S->d = d;
  S->scale = scale;
  S->q_host = q_host;
  S->k_host = k_new_host;
  S->v_host = v_new_host;
  S->o_host = o_host;
  S->lse_host = lse_host;
  // the inner (decode / KVP) workspace first: its counter block stays at offset 0 for any
  // shape; the staging buffers follow it
  S->inner_bytes = round_up(medha_kvp_workspace_size(std::max(world, 1), 1, h_q, h_kv, d), 256);
  S->inner = static_cast<char *>(ws);
  char *b = S->inner + S->inner_bytes;
  const size_t qb = (size_t)h_q * d * 2, kb = (size_t)h_kv * d * 2;
  S->q_dev = b;
  b += round_up(qb, 256);
  S->k_dev = b;
  b += round_up(kb, 256);
  S->v_dev = b;
  b += round_up(kb, 256);
  S->o_dev = reinterpret_cast<float *>(b);
  b += round_up((size_t)h_q * d * 4, 256);
  S->lse_dev = reinterpret_cast<float *>(b);
  // mapped (zero-copy) device views of the host buffers
  S->q_map = mapped_host_view(q_host);
  S->k_map = k_new_host ? mapped_host_view(k_new_host) : nullptr;
  S->v_map = v_new_host ? mapped_host_view(v_new_host) : nullptr;
  S->zc_in_q = S->q_map && aligned16(S->q_map) && (qb % 16 == 0);
  S->zc_in_kv = S->k_map && S->v_map && aligned16(S->k_map) && aligned16(S->v_map);
  S->o_map = static_cast<float *>(mapped_host_view(o_host));
  S->l_map = lse_host ? static_cast<float *>(mapped_host_view(lse_host)) : nullptr;
  S->zc_out = S->o_map && aligned16(S->o_map) && (!lse_host || S->l_map);
  return MEDHA_OK;
}

medha_status step_run(const StepSetup &S, medha_kv_shard *kv, int32_t append, int64_t q_pos, cudaStream_t st) {
  medha_status s;
  if (append && (!S.k_host || !S.v_host)) return fail(MEDHA_EINVAL, "null k/v host buffer");
  if (kv->h_kv != S.h_kv || kv->d != S.d) return fail(MEDHA_ESHAPE, "shard does not match the step setup");
  const size_t qb = (size_t)S.h_q * S.d * 2, kb = (size_t)S.h_kv * S.d * 2;
  // Inputs: with mapped pinned host buffers, ONE launch reads q, k_new and v_new over the
  // host link (q into the workspace, K/V appended straight into the shard); otherwise
  // cudaMemcpyAsync + kv_append.
  if (S.zc_in_q && (!append || S.zc_in_kv)) {
    if ((s = check_shard(kv))) return s;
    if (append && kv->len + 1 > kv->capacity) return fail(MEDHA_ERANGE, "append exceeds capacity");
    if ((s = kv_append_impl(kv, S.k_map, S.v_map, append ? 1 : 0, S.q_map, S.q_dev, (int64_t)qb, st))) return s;
  } else {
    CUDA_TRY(cudaMemcpyAsync(S.q_dev, S.q_host, qb, cudaMemcpyHostToDevice, st));
    if (append) {
      CUDA_TRY(cudaMemcpyAsync(S.k_dev, S.k_host, kb, cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(S.v_dev, S.v_host, kb, cudaMemcpyHostToDevice, st));
      if ((s = medha_kv_append(kv, S.k_dev, S.v_dev, 1, st))) return s;
    }
  }
  // Outputs: written by the decode kernel straight into mapped pinned host buffers
  // (visible to the host once the stream is synchronised), else staged and copied back.
  float *o_tgt = S.zc_out ? S.o_map : S.o_dev;
  float *l_tgt = S.zc_out ? (S.lse_host ? S.l_map : S.lse_dev) : S.lse_dev;
  const int64_t qp = q_pos;
  if (S.comm)
    s = medha_kvp_decode(S.comm, kv, 1, S.q_dev, S.h_q, &qp, S.scale, o_tgt, l_tgt, nullptr, S.inner, S.inner_bytes, st);
  else
    s = decode_partial_impl(kv, 1, S.q_dev, S.h_q, &qp, S.scale, o_tgt, l_tgt, S.inner, S.inner_bytes, st);
  if (s) return s;
  if (!S.zc_out) {
    CUDA_TRY(cudaMemcpyAsync(S.o_host, S.o_dev, (size_t)S.h_q * S.d * 4, cudaMemcpyDeviceToHost, st));
    if (S.lse_host) CUDA_TRY(cudaMemcpyAsync(S.lse_host, S.lse_dev, (size_t)S.h_q * 4, cudaMemcpyDeviceToHost, st));
  }
  return MEDHA_OK;
}
}  // namespace

struct medha_decode_plan {
  StepSetup setup;
};

extern "C" {

medha_status medha_decode_step_host(medha_kvp_comm *comm, medha_kv_shard *kv, int32_t append, const void *q_host,
                                    const void *k_new_host, const void *v_new_host, int32_t h_q, int64_t q_pos,
                                    float scale, float *o_host, float *lse_host, void *ws, size_t ws_bytes,
                                    void *stream) {
  StepSetup S;
  medha_status s = step_setup(comm, kv, h_q, scale, q_host, append ? k_new_host : nullptr,
                              append ? v_new_host : nullptr, o_host, lse_host, ws, ws_bytes, &S);
  if (s) return s;
  return step_run(S, kv, append, q_pos, static_cast<cudaStream_t>(stream));
}

medha_status medha_decode_plan_create(medha_kvp_comm *comm, const medha_kv_shard *kv, int32_t h_q, float scale,
                                      const void *q_host, const void *k_new_host, const void *v_new_host,
                                      float *o_host, float *lse_host, void *ws, size_t ws_bytes,
                                      medha_decode_plan **out) {
  if (!out) return fail(MEDHA_EINVAL, "null plan pointer");
  medha_decode_plan *p = new medha_decode_plan();
  medha_status s = step_setup(comm, kv, h_q, scale, q_host, k_new_host, v_new_host, o_host, lse_host, ws, ws_bytes,
                              &p->setup);
  if (s) {
    delete p;
    return s;
  }
  *out = p;
  return MEDHA_OK;
}

medha_status medha_decode_plan_step(medha_decode_plan *plan, medha_kv_shard *kv, int32_t append, int64_t q_pos,
                                    void *stream) {
  if (!plan || !kv) return fail(MEDHA_EINVAL, "null argument");
  return step_run(plan->setup, kv, append, q_pos, static_cast<cudaStream_t>(stream));
}

medha_status medha_decode_plan_destroy(medha_decode_plan *plan) {
  delete plan;
  return MEDHA_OK;
}

medha_status medha_decode_step_dev(const medha_kv_shard *kvs_host, int32_t batch, const void *k_new,
                                   const void *v_new, const void *q, int32_t h_q, int64_t *len_dev, float scale,
                                   float *o, float *lse, void *ws, size_t ws_bytes, void *stream) {
  if (batch <= 0 || batch > kDecodeMaxSeqPerLaunch) return fail(MEDHA_ENOTSUP, "batch %d not in [1, 64]", batch);
  if (!kvs_host || !k_new || !v_new || !q || !len_dev || !o || !lse) return fail(MEDHA_EINVAL, "null argument");
  if (reinterpret_cast<uintptr_t>(len_dev) & 7) return fail(MEDHA_EINVAL, "len_dev not 8-byte aligned");
  // ONE launch: the decode kernel's owner items store the new rows at *len_dev (dropped at or
  // past the capacity), every item reads the new token from k_new / v_new, the last CTA out
  // advances the lengths
  DecodeAppend app{k_new, v_new, nullptr};
  return decode_partial_impl(kvs_host, batch, q, h_q, nullptr, scale, o, lse, ws, ws_bytes,
                             static_cast<cudaStream_t>(stream), nullptr, len_dev, &app);
}

#ifdef MEDHA_DECODE_TRACE
medha_status medha_debug_decode_trace(unsigned long long *host_out /* [8192][8] */) {
  CUDA_TRY(cudaMemcpyFromSymbol(host_out, g_decode_trace, sizeof(g_decode_trace)));
  return MEDHA_OK;
}
medha_status medha_debug_launch_trace(unsigned long long *host_out /* [64][4] */, unsigned *n_out) {
  CUDA_TRY(cudaMemcpyFromSymbol(host_out, g_ltrace, sizeof(g_ltrace)));
  CUDA_TRY(cudaMemcpyFromSymbol(n_out, g_ltrace_n, sizeof(unsigned)));
  return MEDHA_OK;
}
#endif

#ifdef MEDHA_PF_TRACE
medha_status medha_debug_pf_trace(long long *host_out /* [512][12] */) {
  CUDA_TRY(cudaMemcpyFromSymbol(host_out, g_pf_trace, sizeof(g_pf_trace)));
  return MEDHA_OK;
}
medha_status medha_debug_pf_gtimer(long long *host_out /* [8] */) {
  CUDA_TRY(cudaMemcpyFromSymbol(host_out, g_pf_gt, sizeof(g_pf_gt)));
  return MEDHA_OK;
}
#endif

medha_status medha_hbm_read_probe(const void *src, size_t bytes, float *sink, void *stream) {
  if (!src || !sink) return fail(MEDHA_EINVAL, "null argument");
  if (!aligned16(src) || (bytes & 15)) return fail(MEDHA_EINVAL, "src/bytes not 16-byte aligned");
  const int64_t n_vec = (int64_t)(bytes / 16);
  const int blocks = num_sms() * 8;
  hbm_read_probe_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const uint4 *>(src), n_vec,
                                                                               sink);
  LAUNCH_CHECK("hbm_read_probe_kernel");
  return MEDHA_OK;
}

}  // extern "C"
