/*
 * medha_attn.h — C ABI of libmedha_attn: the data-parallel hot path of Medha
 * (arXiv 2409.17264), exact attention over a KV cache sharded along the
 * sequence dimension, on NVIDIA B200 (sm_100a).
 *
 * Citations: "P:n" = PAPER.md line n of the paper's LaTeX source, "S:n" = the
 * SPEC.md line n written from it (see DESIGN.md for the readings R1-R22 of the
 * places where the paper is silent).
 *
 * What the library computes (P:167-171 attention; P:597-599 KVP):
 *   for a query row (token t, query head h) with absolute position q_pos[t],
 *   kv head g = h / G (G = h_q / h_kv, reading R2), and the keys j of a shard
 *   with absolute position pos0 + j <= q_pos[t] (causal, inclusive, R3):
 *      z_j = scale * <Q[t,h,:], K[g,j,:]>,  m = max_j z_j,  l = sum_j exp(z_j - m)
 *      o   = sum_j exp(z_j - m) V[g,j,:] / l,        lse = m + ln(l)   (natural log, R5)
 *   A row with no visible key gives o = 0, lse = -inf (R7).
 *   Partials of disjoint shards merge exactly ("combined using online-softmax"):
 *      M = max_r lse_r, lse = M + ln sum_r exp(lse_r - M), o = sum_r exp(lse_r - lse) o_r,
 *   summed in rank order r = 0..P-1 so every rank gets bit-identical results (R13).
 *
 * Conventions for every entry point:
 *   - Tensor pointers are DEVICE pointers owned by the caller unless the
 *     parameter name ends in _host (then: host memory, preferably pinned).
 *   - Every call is asynchronous on `stream` (a cudaStream_t passed as void*;
 *     NULL = the legacy default stream), never synchronises the device, and never
 *     allocates device memory (except medha_kvp_comm_create, through NCCL).
 *   - Precision (R8): K, V, Q are bf16; logits, softmax, accumulation and all
 *     outputs are fp32; P is rounded to bf16 (RNE) before the P.V product.
 *   - Alignment: every device pointer must be 16-byte aligned.
 *   - Supported shapes: d in {64, 128}; G = h_q / h_kv in {1, 2, 4, 8, 16};
 *     otherwise MEDHA_ENOTSUP.
 *   - Errors are returned as a negative medha_status; nothing is launched when
 *     a call returns an error detected on the host.  medha_last_error() returns a
 *     thread-local message for the last failing call on the calling thread.
 *   - Workspaces: caller-owned device memory of at least the size the matching
 *     *_workspace_size() returns.  They must be ZERO-FILLED before their first
 *     use; every call leaves the workspace's counter region zeroed again, so a
 *     workspace can be reused (and captured in a CUDA graph) indefinitely.
 *     Two calls that run concurrently need distinct workspaces.
 *   - Thread safety: calls are reentrant for distinct outputs and workspaces.
 */
#ifndef MEDHA_ATTN_H_
#define MEDHA_ATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t medha_status;
enum {
  MEDHA_OK = 0,
  MEDHA_EINVAL = -1,     /* null pointer, misaligned pointer, h_q % h_kv != 0, negative size */
  MEDHA_ESHAPE = -2,     /* dimensions of the arguments disagree */
  MEDHA_ERANGE = -3,     /* capacity overflow, bad position, merge of all -inf rows */
  MEDHA_ENOTSUP = -4,    /* d or G outside the supported set, batch too large */
  MEDHA_EWORKSPACE = -5, /* workspace too small */
  MEDHA_ECUDA = -6,      /* a CUDA runtime/driver call failed (message has the CUDA error) */
  MEDHA_ENCCL = -7       /* an NCCL call failed or the communicator is in an error state */
};

/* Human-readable name of a status code (static string). */
const char *medha_status_str(medha_status s);
/* Detail message of the last failing call on this thread ("" if none). */
const char *medha_last_error(void);
/* ABI version, (major << 16) | minor. */
int32_t medha_version(void);

/*
 * One KVP shard of one sequence for one layer ("shards the KV cache ...
 * along the sequence dimension").  k and v are bf16
 * [h_kv][capacity][d] (head-major, each head's tokens contiguous).  Local token j
 * sits at absolute position pos0 + j; tokens j >= len are never read.
 */
typedef struct medha_kv_shard {
  void *k;            /* device, bf16 [h_kv][capacity][d] (paged: the page pool, see below) */
  void *v;            /* device, bf16 [h_kv][capacity][d] (paged: the page pool) */
  int64_t capacity;   /* logical tokens per head */
  int64_t len;        /* tokens valid per head (0 <= len <= capacity) */
  int64_t pos0;       /* absolute position of local token 0 */
  int32_t h_kv;       /* KV heads */
  int32_t d;          /* head dimension */
  /* Paged KV: when page_table != NULL, k and v are page pools bf16
   * [h_kv][pool_tokens][d] shared by many sequences, and logical token j of this shard lives
   * at pool row page_table[j / page_size] * page_size + j % page_size.  capacity must be a
   * multiple of page_size (page_table has capacity / page_size entries, device int32).
   * page_size: power of two, >= 16 for decode/append, >= 128 for prefill.  Pool rows past
   * len inside a shard's last page must hold finite values (zero-fill pools on allocation):
   * the prefill's PV MMA reads whole 128-token tiles.  Table entries are not range-checked on
 * the device: each must name a page inside the pool (pool_tokens / page_size pages) that no
 * other live shard writes.  page_table == NULL: contiguous shard,
   * page_size / pool_tokens ignored. */
  const int32_t *page_table;
  int32_t page_size;
  int32_t reserved;   /* 0 */
  int64_t pool_tokens; /* tokens per head plane of the pools (paged only) */
} medha_kv_shard;

/*
 * kv_append (P:178-183 the KV cache grows by one row per token):
 * copies k_new, v_new (device, bf16 [n][h_kv][d], token-major as produced by the
 * K/V projections) into kv->k, kv->v at local tokens [len, len+n) and, on success,
 * sets kv->len += n (host-side field).  n = 0 is a no-op.
 * Errors: MEDHA_ERANGE if len + n > capacity; MEDHA_EINVAL for null/misaligned.
 */
medha_status medha_kv_append(medha_kv_shard *kv, const void *k_new, const void *v_new,
                             int64_t n, void *stream);

/*
 * attn_decode_partial (SURVEY a3 + a5; "compute partial attention outputs
 * based on each local KV-cache shard"): for each of `batch` sequences b, the
 * single query q[b] (bf16 [batch][h_q][d]) at absolute position q_pos_host[b]
 * attends over shard kvs_host[b].  Writes o (fp32 [batch][h_q][d]) and lse (fp32
 * [batch][h_q], natural log) = the exact partial state of that shard.  The KV is
 * split across CTAs inside the GPU and the splits are merged in a
 * fixed order inside the same launch (run-to-run deterministic).
 *   kvs_host, q_pos_host: host arrays of length batch (read during the call).
 *   All shards must share h_kv and d; batch <= 4096.
 * Early start (programmatic dependent launch): the kernel may start streaming K/V rows
 * [0, len - 1) of each shard, and the query, before the kernel launched just before it on
 * the stream has completed.  Every kernel of this library allows that only after its own
 * inputs are final; a foreign kernel that calls
 * griddepcontrol.launch_dependents / cudaTriggerProgrammaticLaunchCompletion early and
 * writes those rows or q must not immediately precede this call (or set MEDHA_DEC_EARLY=0).
 */
size_t medha_decode_workspace_size(int32_t batch, int32_t h_q, int32_t h_kv, int32_t d);
medha_status medha_attn_decode_partial(const medha_kv_shard *kvs_host, int32_t batch,
                                       const void *q, int32_t h_q, const int64_t *q_pos_host,
                                       float scale, float *o, float *lse,
                                       void *ws, size_t ws_bytes, void *stream);

/*
 * attn_decode_append (SURVEY a1 + a3 + a5 in ONE launch; P:178-183 each decode step appends
 * one K/V row per sequence and then scans the whole KV): exactly medha_kv_append of row b of
 * k_new / v_new (device, bf16 [batch][h_kv][d], token-major) into shard kvs_host[b] followed
 * by medha_attn_decode_partial, for every sequence b with append_host[b] != 0 (append_host ==
 * NULL: every sequence).  The kernel item whose KV split owns the new token stores its rows;
 * every read of that token takes it from k_new / v_new, so no CTA reads data another CTA
 * wrote in the same launch.  On success kvs_host[b].len += 1 for the appending sequences.
 * Errors as medha_attn_decode_partial, plus MEDHA_ERANGE when an append would exceed a
 * shard's capacity (nothing is launched).
 */
medha_status medha_attn_decode_append(medha_kv_shard *kvs_host, int32_t batch, const void *k_new,
                                      const void *v_new, const int32_t *append_host, const void *q,
                                      int32_t h_q, const int64_t *q_pos_host, float scale, float *o,
                                      float *lse, void *ws, size_t ws_bytes, void *stream);

/*
 * attn_prefill_chunk (P:321-366 chunked prefill, Eq. 3): a chunk of c
 * query tokens q (bf16 [c][h_q][d]) at absolute positions q_pos0 .. q_pos0+c-1
 * attends causally over the shard `kv` (all of its len tokens that are visible).
 * With the tail shard after medha_kv_append of the chunk's own K/V and
 * q_pos0 = pos0 + len - c this is the chunk's full causal attention on one GPU.
 * Writes o (fp32 [c][h_q][d]) and lse (fp32 [c][h_q]).  QK^T and PV run on the
 * tcgen05 tensor cores with TMEM accumulators; K/V tiles are staged by TMA.
 * c must be >= 1 and <= 65536.
 */
size_t medha_prefill_workspace_size(int64_t c, int32_t h_q, int32_t h_kv, int32_t d);
medha_status medha_attn_prefill_chunk(const medha_kv_shard *kv, const void *q, int64_t c,
                                      int32_t h_q, int64_t q_pos0, float scale,
                                      float *o, float *lse, void *ws, size_t ws_bytes,
                                      void *stream);

/*
 * attn_prefill_batch (prefill-prefill batching): n chunks of
 * different sequences of the same layer (same h_q, h_kv, d; each chunk over its own shard
 * and its own query block), computed in ONE launch per 32 chunks with a batch-wide
 * balanced split plan; per chunk the result equals medha_attn_prefill_chunk.
 *   chunks_host: host array of n descriptors, read during the call.
 *   Workspace: medha_prefill_batch_workspace_size(n, c of every chunk, h_q, d) bytes.
 */
typedef struct medha_prefill_chunk {
  const medha_kv_shard *kv;   /* host pointer to the chunk's shard */
  const void *q;              /* device, bf16 [c][h_q][d] */
  int64_t c;                  /* query tokens (1 .. 65536) */
  int64_t q_pos0;             /* absolute position of query token 0 */
  float *o;                   /* device, fp32 [c][h_q][d] */
  float *lse;                 /* device, fp32 [c][h_q], natural log */
} medha_prefill_chunk;
size_t medha_prefill_batch_workspace_size(int32_t n, const int64_t *c_host, int32_t h_q, int32_t d);
medha_status medha_attn_prefill_batch(const medha_prefill_chunk *chunks_host, int32_t n, int32_t h_q,
                                      float scale, void *ws, size_t ws_bytes, void *stream);

/*
 * merge_partials: parts is fp32 [P][rows*(d+1)] where part r
 * holds o_r [rows][d] followed by lse_r [rows].  Writes o_out fp32 [rows][d],
 * lse_out fp32 [rows] (may be NULL) and o_out_bf16 bf16 [rows][d] (may be NULL).
 * Parts are combined in order r = 0..P-1.  1 <= P <= 64.
 * A row whose parts are all -inf yields o = 0, lse = -inf and the call returns
 * MEDHA_OK (reading R22: the condition is data-dependent and only visible
 * on the device, and the calls never synchronise, so it cannot be an error status;
 * an all-empty row is the exact merge of empty shards, R7).
 */
medha_status medha_merge_partials(const float *parts, int32_t P, int64_t rows, int32_t d,
                                  float *o_out, float *lse_out, void *o_out_bf16, void *stream);

/*
 * KVP communicator: an NCCL communicator over the P ranks
 * of one KVP group, one process per GPU.  Rank 0 calls medha_kvp_unique_id and
 * ships the 128 bytes to the other ranks out of band (the Python binding uses the
 * torch.distributed store); every rank then calls medha_kvp_comm_create with the
 * current CUDA device set to its GPU.
 */
typedef struct medha_kvp_comm medha_kvp_comm;
medha_status medha_kvp_unique_id(uint8_t id_out[128]);
medha_status medha_kvp_comm_create(const uint8_t id[128], int32_t rank, int32_t world,
                                   medha_kvp_comm **out);
medha_status medha_kvp_comm_destroy(medha_kvp_comm *comm);
medha_status medha_kvp_comm_info(const medha_kvp_comm *comm, int32_t *rank, int32_t *world);
/*
 * Fused peer-to-peer exchange (single node, NVLink).  medha_kvp_comm_create also
 * allocates a receive buffer (~2 x world x 2.1 MB + flags + an epoch word) and maps every
 * peer's buffer through CUDA IPC (a collective; skipped when MEDHA_KVP_P2P=0 or when any rank
 * fails; at world 1 the local buffer serves as its own peer).  When active, medha_kvp_decode
 * (batch <= 64) runs the exchange inside the decode kernel: the last CTA of each (sequence,
 * kv head) stores the rank partial into every rank's receive slot over NVLink, raises the
 * peers' epoch flags (release, system scope), waits for all ranks' flags (acquire) and merges
 * in rank order - no NCCL call, no merge launch.  The call's epoch is read from and advanced
 * in device memory by the kernel itself, so medha_kvp_decode may be captured in a CUDA graph
 * and replayed (every rank must replay it the same number of times).
 * medha_kvp_comm_p2p returns 1 when that path is active; medha_kvp_comm_set_p2p(comm, 0)
 * forces the NCCL all-gather + merge path (must be switched identically on all ranks).
 */
int32_t medha_kvp_comm_p2p(const medha_kvp_comm *comm);
medha_status medha_kvp_comm_set_p2p(medha_kvp_comm *comm, int32_t enable);

/*
 * Failure containment of the fused exchange.  The in-kernel wait for a peer's
 * partial is bounded by a timeout (default 30 s, env MEDHA_KVP_TIMEOUT_MS, or
 * medha_kvp_comm_set_timeout in nanoseconds).  On expiry - a rank that never launched its
 * call, e.g. after failing its own argument checks, or ranks that disagree on batch / h_q -
 * the kernel writes NaN into the affected outputs, sets an error word in mapped host memory
 * and finishes instead of hanging the GPU.  The communicator is then BROKEN for good:
 * medha_kvp_comm_status (non-blocking; meaningful once the stream has been synchronised) and
 * every later collective call on it return MEDHA_ENCCL; destroy it and create a new one.
 * medha_kvp_comm_debug(comm, 1) is a test hook: this rank's decode kernels withhold their
 * pushes and flags (so every waiting rank, itself included, times out); 0 restores normal
 * operation.
 */
medha_status medha_kvp_comm_status(medha_kvp_comm *comm);
medha_status medha_kvp_comm_set_timeout(medha_kvp_comm *comm, uint64_t timeout_ns);
medha_status medha_kvp_comm_debug(medha_kvp_comm *comm, uint32_t flags);

/*
 * kvp_decode (Eq. 5): the local partial (medha_attn_decode_partial on
 * this rank's shards), an all-gather of the packed (o ‖ lse) partials of all
 * ranks (rows*(d+1)*4 bytes per rank, independent of the KV length), and the
 * rank-ordered LSE merge.  Every rank receives the identical final o_out (fp32
 * [batch][h_q][d]), lse_out (fp32 [batch][h_q], may be NULL) and o_out_bf16 (may
 * be NULL).  Must be called by all ranks of the communicator with the same
 * batch/h_q/d (a collective).
 */
size_t medha_kvp_workspace_size(int32_t world, int32_t batch, int32_t h_q, int32_t h_kv, int32_t d);
medha_status medha_kvp_decode(medha_kvp_comm *comm, const medha_kv_shard *kvs_host, int32_t batch,
                              const void *q, int32_t h_q, const int64_t *q_pos_host, float scale,
                              float *o_out, float *lse_out, void *o_out_bf16,
                              void *ws, size_t ws_bytes, void *stream);

/*
 * kvp_decode_append: medha_kvp_decode with the new token's K/V appended in the same launch on
 * the ranks / sequences that hold it (append_host[b] != 0; typically the tail rank of each
 * sequence), as medha_attn_decode_append.  kvs_host[b].len += 1 where appended.
 */
medha_status medha_kvp_decode_append(medha_kvp_comm *comm, medha_kv_shard *kvs_host, int32_t batch,
                                     const void *k_new, const void *v_new, const int32_t *append_host,
                                     const void *q, int32_t h_q, const int64_t *q_pos_host, float scale,
                                     float *o_out, float *lse_out, void *o_out_bf16, void *ws,
                                     size_t ws_bytes, void *stream);

/*
 * kvp_exchange_merge (SURVEY a6 + a7 on their own): all-gathers this rank's packed
 * partial `send` (fp32 [rows*(d+1)]: o [rows][d] then lse [rows], e.g. written by
 * medha_attn_decode_partial with o = send, lse = send + rows*d) and merges the
 * world's partials in rank order into o_out / lse_out / o_out_bf16.  ws holds the
 * receive buffer (medha_kvp_exchange_workspace_size bytes).  medha_kvp_decode is
 * exactly medha_attn_decode_partial followed by this call.
 */
size_t medha_kvp_exchange_workspace_size(int32_t world, int64_t rows, int32_t d);
medha_status medha_kvp_exchange_merge(medha_kvp_comm *comm, const float *send, int64_t rows, int32_t d,
                                      float *o_out, float *lse_out, void *o_out_bf16,
                                      void *ws, size_t ws_bytes, void *stream);

/*
 * kvp_prefill_chunk (Eq. 6): a prefill chunk under KVP — every rank
 * attends the replicated chunk queries over its own shard (ranks whose shard holds
 * no visible key contribute (0, -inf)), then the partials are all-gathered and
 * merged in rank order.  Output as medha_attn_prefill_chunk, identical on all ranks.
 */
size_t medha_kvp_prefill_workspace_size(int32_t world, int64_t c, int32_t h_q, int32_t h_kv, int32_t d);
medha_status medha_kvp_prefill_chunk(medha_kvp_comm *comm, const medha_kv_shard *kv,
                                     const void *q, int64_t c, int32_t h_q, int64_t q_pos0,
                                     float scale, float *o_out, float *lse_out, void *o_out_bf16,
                                     void *ws, size_t ws_bytes, void *stream);

/*
 * decode_step_host (the end-to-end call a serving loop makes for one decode token
 * of one sequence, batch 1): copies q_host (bf16 [h_q][d]) and, when append != 0,
 * k_new_host / v_new_host (bf16 [h_kv][d]) host->device into the workspace,
 * appends the new token to `kv` (kv->len += 1), runs the decode attention at
 * position q_pos — locally when comm == NULL, otherwise as medha_kvp_decode — and
 * copies o (fp32 [h_q][d]) and lse (fp32 [h_q]) back into o_host / lse_host.
 * Host buffers that are pinned AND mapped into the device address space (cudaHostAlloc
 * under UVA, e.g. torch pin_memory(), 16-byte aligned) are accessed zero-copy: one
 * kv_append launch reads q, k_new, v_new over the host link and the decode kernel writes
 * o / lse straight into o_host / lse_host (no cudaMemcpyAsync); other host memory is
 * staged with cudaMemcpyAsync.  Same bytes cross the link either way.
 * Asynchronous: the host buffers are read/written while the stream executes the call
 * and the outputs are valid after the stream is synchronised.
 */
size_t medha_decode_step_workspace_size(int32_t world, int32_t h_q, int32_t h_kv, int32_t d);
medha_status medha_decode_step_host(medha_kvp_comm *comm, medha_kv_shard *kv, int32_t append,
                                    const void *q_host, const void *k_new_host,
                                    const void *v_new_host, int32_t h_q, int64_t q_pos,
                                    float scale, float *o_host, float *lse_host,
                                    void *ws, size_t ws_bytes, void *stream);

/*
 * decode plan (the per-layer object of a serving loop around medha_decode_step_host): fixes
 * the communicator (or NULL), the shard geometry (h_kv, d of `kv`), h_q, scale, the host
 * buffers and the workspace once - their validation, mapped-pointer lookups
 * (cudaPointerGetAttributes) and workspace carving happen in medha_decode_plan_create - so
 * each medha_decode_plan_step(plan, kv, append, q_pos, stream) only validates the shard and
 * launches (same work and semantics as medha_decode_step_host with those arguments; k_new /
 * v_new may be NULL in the plan when no step appends).  The plan holds no device memory;
 * the buffers it names must outlive it.  Not thread-safe per plan.
 */
typedef struct medha_decode_plan medha_decode_plan;
medha_status medha_decode_plan_create(medha_kvp_comm *comm, const medha_kv_shard *kv, int32_t h_q,
                                      float scale, const void *q_host, const void *k_new_host,
                                      const void *v_new_host, float *o_host, float *lse_host,
                                      void *ws, size_t ws_bytes, medha_decode_plan **out);
medha_status medha_decode_plan_step(medha_decode_plan *plan, medha_kv_shard *kv, int32_t append,
                                    int64_t q_pos, void *stream);
medha_status medha_decode_plan_destroy(medha_decode_plan *plan);

/*
 * decode_step_dev (device-side lengths, CUDA-graph-capturable; P:178-183
 * decode scans the whole KV, P:597-599 per-shard partial).  One decode token for each of
 * `batch` (1..64) sequences on this GPU, all lengths on the DEVICE:
 *   1. k_new / v_new (bf16 [batch][h_kv][d], device) row b is appended to shard b at local
 *      index len_dev[b] (int64 [batch], device; appends at or past the capacity are dropped);
 *      the append runs inside the decode launch (one launch per step, as
 *      medha_attn_decode_append);
 *   2. sequence b attends keys 0..len_dev[b] of its shard (its own new token included; the
 *      query is q[b], bf16 [batch][h_q][d], at position pos0 + len_dev[b]) -> o fp32
 *      [batch][h_q][d], lse fp32 [batch][h_q] (natural log);
 *   3. len_dev[b] += 1.
 * Nothing on the host depends on the lengths: the split plan is fixed from kvs_host[b].capacity
 * (splits past the current length are empty), so the same call - or a CUDA graph captured
 * from it - can be replayed step after step.  kvs_host[b].len is neither read nor updated.
 * Workspace: medha_decode_workspace_size(batch, h_q, h_kv, d), zeroed once.  Errors as
 * medha_attn_decode_partial; ENOTSUP for batch > 64.
 */
medha_status medha_decode_step_dev(const medha_kv_shard *kvs_host, int32_t batch, const void *k_new,
                                   const void *v_new, const void *q, int32_t h_q, int64_t *len_dev,
                                   float scale, float *o, float *lse, void *ws, size_t ws_bytes,
                                   void *stream);

/*
 * hbm_read_probe (measurement aid K6): streams `bytes` bytes from
 * `src` with 16-byte loads and writes one word per CTA to `sink` (>= 4096 floats)
 * so the reads cannot be elided.  Gives the same-run read-only HBM bandwidth.
 */
medha_status medha_hbm_read_probe(const void *src, size_t bytes, float *sink, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MEDHA_ATTN_H_ */
