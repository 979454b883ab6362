"""Full-size parity at the BASELINE.json configurations, on sampled outputs.

The GPU path runs on the whole workload (exact shapes and sizes the bench uses);
the fp64 oracle recomputes sampled rows (a few query rows / KV heads) over the
full key range.  The oracle streams keys through `LazyKV`, which regenerates each
block on the CPU from the counter-based generator (never from the CUDA path).
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import KVP_ABS, compare

pytestmark = pytest.mark.gpu


class LazyKV:
    """Read-only [N][d] view of one KV head of the global synthetic K or V; slices are
    generated on the CPU on demand (float32, bf16-valued)."""

    def __init__(self, seed, stream, head, n, h_kv, d):
        self.seed, self.stream, self.head, self.n, self.h_kv, self.d = seed, stream, head, n, h_kv, d
        self.shape = (n, d)

    def __getitem__(self, sl):
        a, b, _ = sl.indices(self.n)
        return synth.kv_block(self.seed, self.stream, a, b - a, self.h_kv, self.d, heads=[self.head]).float().numpy()[:, 0]


def gpu_shard(M, seed, a, b, h_kv, d, extra=0):
    """Shard with global tokens [a, b) generated on the GPU block by block."""
    sh = M.KVShard.empty(h_kv, b - a + extra, d, pos0=a)
    blk = synth.BLOCK_TOKENS
    for t in range(a, b, blk):
        m = min(blk, b - t)
        sh.k[:, t - a:t - a + m] = synth.kv_block(seed, synth.STREAM_K, t, m, h_kv, d, device="cuda").permute(1, 0, 2)
        sh.v[:, t - a:t - a + m] = synth.kv_block(seed, synth.STREAM_V, t, m, h_kv, d, device="cuda").permute(1, 0, 2)
    sh.len = b - a
    return sh


def oracle_rows(seed, q_rows, q_pos, heads, n, h_kv, d):
    """o/lse for the query rows [T][G][d] of KV heads `heads` over keys [0, n)."""
    out = []
    for i, h in enumerate(heads):
        K = LazyKV(seed, synth.STREAM_K, h, n, h_kv, d)
        V = LazyKV(seed, synth.STREAM_V, h, n, h_kv, d)
        out.append(oracle.attention_group(q_rows[i], K, V, q_pos, np.arange(n), 1 / math.sqrt(d)))
    return out


@pytest.fixture(scope="module")
def M():
    import paper_2409_17264_b200 as M
    return M


def test_config1_8b_decode_1M(M):
    """configs[1]: Llama-3 8B layer (32q/8kv, d 128), batch 1, 2^20-token KV."""
    seed, N, h_kv, G, d = 21, 1 << 20, 8, 4, 128
    sh = gpu_shard(M, seed, 0, N, h_kv, d)
    q = synth.queries(seed, 1, h_kv * G, d, amp=6.0)
    o, lse = M.attn_decode_partial([sh], q.cuda(), [N - 1])
    heads = [0, 5]
    ref = oracle_rows(seed, [q[:, h * G:(h + 1) * G].double().numpy() for h in heads], [N - 1], heads, N, h_kv, d)
    for h, (ro, rl) in zip(heads, ref):
        compare(o[:, h * G:(h + 1) * G], lse[:, h * G:(h + 1) * G], ro, rl, what=f"8B decode 1M head {h}")


def test_config1_bench_step_fused_append_1M(M):
    """configs[1] in the exact launch configuration bench.py times: ONE launch per step that
    appends the new token (position 2^20 - 1) and decodes over the 2^20 keys, repeated
    back to back so every launch after the first early-starts under the previous one
    (PDL); every step must equal the plain decode of the same keys bit for bit, and the
    oracle on sampled heads."""
    seed, N, h_kv, G, d = 23, 1 << 20, 8, 4, 128
    sh = gpu_shard(M, seed, 0, N, h_kv, d)
    ref = gpu_shard(M, seed, 0, N, h_kv, d)
    k_new = synth.kv_block(seed, synth.STREAM_K, N - 1, 1, h_kv, d, device="cuda")
    v_new = synth.kv_block(seed, synth.STREAM_V, N - 1, 1, h_kv, d, device="cuda")
    sh.k[:, N - 1] = float("nan")            # the slot the append fills: never read before it is written
    sh.v[:, N - 1] = float("nan")
    q = synth.queries(seed, 1, h_kv * G, d, amp=6.0).cuda()
    o_ref, l_ref = M.attn_decode_partial([ref], q, [N - 1])
    outs = []
    for _ in range(4):
        sh.len = N - 1
        o, lse = M.attn_decode_append([sh], k_new, v_new, q, [N - 1])
        outs.append((o, lse))
    torch.cuda.synchronize()
    for o, lse in outs:
        assert torch.equal(o, o_ref) and torch.equal(lse, l_ref)
    assert torch.equal(sh.k[:, N - 1], ref.k[:, N - 1]) and torch.equal(sh.v[:, N - 1], ref.v[:, N - 1])
    heads = [3]
    qc = q.cpu()
    ro, rl = oracle_rows(seed, [qc[:, h * G:(h + 1) * G].double().numpy() for h in heads], [N - 1], heads, N, h_kv,
                         d)[0]
    compare(outs[-1][0][:, 3 * G:4 * G], outs[-1][1][:, 3 * G:4 * G], ro, rl, what="bench step 1M head 3")


@pytest.mark.parametrize("P0,c", [(1 << 20, 256), (1 << 17, 4096)])
def test_config2_8b_prefill(M, P0, c):
    """configs[2]: Llama-3 8B chunked prefill at 128K / 1M prefix (sampled rows)."""
    seed, h_kv, G, d = 22, 8, 4, 128
    sh = gpu_shard(M, seed, 0, P0 + c, h_kv, d)
    q = synth.queries(seed + 1, c, h_kv * G, d, amp=4.0, t0=P0)
    o, lse = M.attn_prefill_chunk(sh, q.cuda(), P0)
    rows = [0, c // 2, c - 1]
    h = 3
    (ro, rl), = oracle_rows(seed, [q[rows][:, h * G:(h + 1) * G].double().numpy()], [P0 + r for r in rows], [h],
                            P0 + c, h_kv, d)
    compare(o[rows][:, h * G:(h + 1) * G], lse[rows][:, h * G:(h + 1) * G], ro, rl, what=f"8B prefill P0={P0} c={c}")


def test_config3_70b_decode_10M_kvp8(M):
    """configs[3]: Llama-3 70B layer (64q/8kv, d 128), 10*2^20-token KV sharded KVP = 8:
    the 8 rank partials (computed here on one GPU, one shard each) merged exactly equal
    the unsharded decode (1e-3, fp32) and the fp64 oracle on a sampled KV head."""
    seed, N, h_kv, G, d, P = 23, 10 * (1 << 20), 8, 8, 128, 8
    from paper_2409_17264_b200.kvp import shard_range
    q = synth.queries(seed, 1, h_kv * G, d, amp=6.0).cuda()
    rows = h_kv * G
    parts = torch.empty((P, rows * (d + 1)), dtype=torch.float32, device="cuda")
    for r in range(P):
        a, b = shard_range(N, r, P)
        sh = gpu_shard(M, seed, a, b, h_kv, d)
        o_r, l_r = M.attn_decode_partial([sh], q, [N - 1])
        parts[r, :rows * d] = o_r.reshape(-1)
        parts[r, rows * d:] = l_r.reshape(-1)
        del sh
        torch.cuda.empty_cache()
    om, lm, _ = M.merge_partials(parts, rows, d)
    om, lm = om.view(1, rows, d), lm.view(1, rows)
    whole = gpu_shard(M, seed, 0, N, h_kv, d)
    o1, l1 = M.attn_decode_partial([whole], q, [N - 1])
    del whole
    torch.cuda.empty_cache()
    assert (om - o1).abs().max().item() <= KVP_ABS
    assert (lm - l1).abs().max().item() <= KVP_ABS
    h = 6
    (ro, rl), = oracle_rows(seed, [q.cpu()[:, h * G:(h + 1) * G].double().numpy()], [N - 1], [h], N, h_kv, d)
    compare(om[:, h * G:(h + 1) * G], lm[:, h * G:(h + 1) * G], ro, rl, what="70B decode 10M KVP=8")


def test_config4_mixed_batch_kvp4(M):
    """configs[4]: 32 short decodes (4K KV, rank-local, 8 per rank) + one 512-token prefill
    chunk of a 2M-context request under KVP = 4 (2^21-token prefix sharded 4 ways, the
    chunk's own K/V on the tail rank), emulated on one GPU; the chunk's 4 partials are
    merged exactly (K5) and checked against the fp64 oracle on sampled rows."""
    seed, h_kv, G, d, P, c = 24, 8, 4, 128, 4, 512
    P0 = 1 << 21
    from paper_2409_17264_b200.kvp import shard_range
    q = synth.queries(seed + 1, c, h_kv * G, d, amp=4.0, t0=P0).cuda()
    rows = c * h_kv * G
    parts = torch.empty((P, rows * (d + 1)), dtype=torch.float32, device="cuda")
    for r in range(P):
        a, b = shard_range(P0, r, P)
        if r == P - 1:
            b = P0 + c          # the tail rank holds the chunk's own K/V
        sh = gpu_shard(M, seed, a, b, h_kv, d)
        o_r, l_r = M.attn_prefill_chunk(sh, q, P0)
        parts[r, :rows * d] = o_r.reshape(-1)
        parts[r, rows * d:] = l_r.reshape(-1)
        del sh
        torch.cuda.empty_cache()
    om, lm, _ = M.merge_partials(parts, rows, d)
    om, lm = om.view(c, h_kv * G, d), lm.view(c, h_kv * G)
    sel = [0, 511]
    h = 2
    (ro, rl), = oracle_rows(seed, [q.cpu()[sel][:, h * G:(h + 1) * G].double().numpy()], [P0 + s for s in sel], [h],
                            P0 + c, h_kv, d)
    compare(om[sel][:, h * G:(h + 1) * G], lm[sel][:, h * G:(h + 1) * G], ro, rl, what="mixed: 2M chunk KVP=4")
    # the 32 short decodes: 4096-token KVs, batched 8 per rank
    n = 4096
    for r in range(P):
        shards = [gpu_shard(M, seed + 100 + 8 * r + i, 0, n, h_kv, d) for i in range(8)]
        qd = torch.cat([synth.queries(seed + 100 + 8 * r + i, 1, h_kv * G, d, amp=6.0) for i in range(8)])
        od, ld = M.attn_decode_partial(shards, qd.cuda(), [n - 1] * 8)
        i = r % 8
        (ro, rl), = oracle_rows(seed + 100 + 8 * r + i, [qd[i:i + 1, 0:G].double().numpy()], [n - 1], [0], n, h_kv, d)
        compare(od[i:i + 1, 0:G], ld[i:i + 1, 0:G], ro, rl, what=f"mixed: short decode rank {r}")
