"""Seeded random-shape parity sweep: decode and prefill vs the fp64 oracle over ragged
lengths, shard offsets (pos0), causal cuts inside and before the shard, every supported
group size and head dimension, and batches of unequal sequences."""
import numpy as np
import pytest

import synth
from helpers import compare, make_global_kv, oracle_attention, to_shard

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import paper_2409_17264_b200 as M
    return M


@pytest.mark.parametrize("case", range(24))
def test_fuzz_decode(M, case):
    rng = np.random.default_rng(1000 + case)
    d = int(rng.choice([64, 128]))
    G = int(rng.choice([1, 2, 4, 8, 16]))
    h_kv = int(rng.choice([1, 2, 3]))
    B = int(rng.integers(1, 5))
    shards, qs, qps, refs = [], [], [], []
    for b in range(B):
        N = int(rng.integers(1, 6000))
        a = int(rng.integers(0, N))                    # shard = global tokens [a, N)
        qpos = int(rng.integers(max(0, a - 20), N))     # may precede the shard (empty)
        k, v = make_global_kv(2000 + 10 * case + b, N, h_kv, d)
        q = synth.queries(2000 + 10 * case + b, 1, h_kv * G, d, amp=float(rng.choice([1.0, 4.0, 8.0])))
        shards.append(to_shard(k, v, a, N, extra_cap=int(rng.integers(0, 50))))
        qs.append(q)
        qps.append(qpos)
        refs.append(oracle_attention(q, k, v, [qpos], (a, N)))
    import torch
    o, lse = M.attn_decode_partial(shards, torch.cat(qs).cuda(), qps)
    for b in range(B):
        compare(o[b:b + 1], lse[b:b + 1], refs[b][0], refs[b][1], what=f"fuzz decode {case}/{b}")


@pytest.mark.parametrize("case", range(6))
def test_prefill_batch_ppb(M, case):
    """Prefill-prefill batching: chunks of different sequences
    (ragged c, prefixes, shard offsets) in one launch equal the per-chunk calls and the
    oracle."""
    import torch
    rng = np.random.default_rng(5000 + case)
    d = int(rng.choice([64, 128]))
    G = int(rng.choice([1, 4, 8]))
    h_kv = int(rng.choice([1, 2]))
    n = int(rng.integers(2, 9)) if case < 5 else 40            # last case: > 32 chunks (2 launches)
    shards, qs, p0s, refs = [], [], [], []
    for i in range(n):
        c = int(rng.integers(1, 300))
        P0 = int(rng.integers(0, 5000 if case < 5 else 800))
        N = P0 + c
        a = int(rng.integers(0, min(N, P0 + 1)))
        k, v = make_global_kv(6000 + 100 * case + i, N, h_kv, d)
        q = synth.queries(6000 + 100 * case + i, c, h_kv * G, d, amp=4.0, t0=P0)
        shards.append(to_shard(k, v, a, N))
        qs.append(q.cuda())
        p0s.append(P0)
        rows = sorted(set([0, c - 1, c // 2]))
        refs.append((rows, oracle_attention(q[rows], k, v, [P0 + r for r in rows], (a, N))))
    outs = M.attn_prefill_batch(shards, qs, p0s)
    for i in range(n):
        o, lse = outs[i]
        rows, (ro, rl) = refs[i]
        compare(o[rows], lse[rows], ro, rl, what=f"ppb {case}/{i}")
        o1, l1 = M.attn_prefill_chunk(shards[i], qs[i], p0s[i])
        # same kernel; only the batch-wide split plan can differ (fp32 summation order)
        assert (o1 - o).abs().max().item() < 1e-4 and (l1 - lse).abs().max().item() < 1e-4


@pytest.mark.parametrize("case", range(16))
def test_fuzz_prefill(M, case):
    rng = np.random.default_rng(3000 + case)
    d = int(rng.choice([64, 128]))
    G = int(rng.choice([1, 2, 4, 8, 16]))
    h_kv = int(rng.choice([1, 2]))
    c = int(rng.integers(1, 400))
    P0 = int(rng.integers(0, 3000))
    N = P0 + c
    a = int(rng.integers(0, min(N, P0 + 1)))          # shard [a, N): contains the chunk's own keys
    k, v = make_global_kv(4000 + case, N, h_kv, d)
    q = synth.queries(4000 + case, c, h_kv * G, d, amp=float(rng.choice([1.0, 4.0, 8.0])), t0=P0)
    sh = to_shard(k, v, a, N, extra_cap=int(rng.integers(0, 200)))
    o, lse = M.attn_prefill_chunk(sh, q.cuda(), P0)
    rows = sorted(set([0, c - 1] + [int(x) for x in rng.integers(0, c, size=min(c, 6))]))
    ro, rl = oracle_attention(q[rows], k, v, [P0 + r for r in rows], (a, N))
    compare(o[rows], lse[rows], ro, rl, what=f"fuzz prefill {case}: c={c} P0={P0} a={a} G={G} d={d}")


@pytest.mark.parametrize("case", range(12))
def test_fuzz_decode_append_back_to_back(M, case):
    """Round-2 decode path under fuzzing: several fused append+decode launches back to back on
    one workspace (each early-starting under the previous one), random group size, head dim,
    ragged lengths, shard offsets (pos0), append masks and batch sizes; every launch must equal
    kv_append + decode_partial bit for bit, and sampled sequences the oracle."""
    import torch
    rng = np.random.default_rng(7000 + case)
    d = int(rng.choice([64, 128]))
    G = int(rng.choice([1, 2, 4, 8, 16]))
    h_kv = int(rng.choice([1, 2, 4]))
    B = int(rng.integers(1, 9))
    steps = 3
    lens = [int(rng.integers(1, 20000)) for _ in range(B)]
    starts = [int(rng.integers(0, n)) for n in lens]                  # shard = global tokens [a, N)
    masks = [[bool(rng.integers(0, 2)) or s == 0 for _ in range(B)] for s in range(steps)]
    kvs = [make_global_kv(7100 + 10 * case + b, lens[b] + steps, h_kv, d) for b in range(B)]
    a_sh = [to_shard(kvs[b][0], kvs[b][1], starts[b], lens[b], extra_cap=steps + 1) for b in range(B)]
    r_sh = [to_shard(kvs[b][0], kvs[b][1], starts[b], lens[b], extra_cap=steps + 1) for b in range(B)]
    ws = M.decode_workspace(B, h_kv * G, h_kv, d)
    outs, refs = [], []
    for s in range(steps):
        pos = [sh.pos0 + sh.len for sh in a_sh]                       # the next global position
        k_new = torch.stack([kvs[b][0][pos[b]] for b in range(B)]).cuda()
        v_new = torch.stack([kvs[b][1][pos[b]] for b in range(B)]).cuda()
        q = synth.queries(7200 + 10 * case + s, B, h_kv * G, d, amp=float(rng.choice([1.0, 4.0, 8.0]))).cuda()
        qpos = [pos[b] if masks[s][b] else pos[b] - 1 for b in range(B)]
        o, lse = M.attn_decode_append(a_sh, k_new, v_new, q, qpos, append=masks[s], ws=ws)
        outs.append((o, lse, q, qpos, [sh.len for sh in a_sh]))
    torch.cuda.synchronize()
    for s in range(steps):
        o, lse, q, qpos, _ = outs[s]
        for b in range(B):
            if masks[s][b]:
                M.kv_append(r_sh[b], kvs[b][0][r_sh[b].pos0 + r_sh[b].len:][:1].cuda(),
                            kvs[b][1][r_sh[b].pos0 + r_sh[b].len:][:1].cuda())
        o1, l1 = M.attn_decode_partial(r_sh, q, qpos)
        torch.cuda.synchronize()
        assert torch.equal(o, o1) and torch.equal(lse, l1), f"case {case} step {s}"
    b = int(rng.integers(0, B))
    o, lse, q, qpos, lens_after = outs[-1]
    n_keys = lens_after[b]
    ro, rl = oracle_attention(q[b:b + 1].cpu(), kvs[b][0], kvs[b][1], [qpos[b]],
                              (starts[b], starts[b] + n_keys))
    compare(o[b:b + 1], lse[b:b + 1], ro, rl, what=f"fuzz append {case}/{b}")
