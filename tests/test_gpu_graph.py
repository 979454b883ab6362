"""Device-side lengths and CUDA-graph replay (include/medha_attn.h
`medha_decode_step_dev`): a decode step whose append position, visible length and query
position come from a device counter, so ONE captured graph serves every step.

Each step is checked against the fp64 oracle over exactly the keys the step may see (the
prefix plus every token appended so far, its own included); the spare capacity is
NaN-poisoned, so a read past the device length would show up as a non-finite output."""
import numpy as np
import pytest
import torch

import synth
from helpers import compare, make_global_kv, oracle_attention, to_shard

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import paper_2409_17264_b200 as M
    return M


def _setup(M, lens, steps, h_kv=8, G=4, d=128, seed=61):
    ks, vs, shards = [], [], []
    for i, n in enumerate(lens):
        k, v = make_global_kv(seed + i, n + steps, h_kv, d)
        ks.append(k)
        vs.append(v)
        shards.append(to_shard(k, v, 0, n, extra_cap=steps + 3))   # capacity n + steps + 3, poisoned
    return ks, vs, shards


def _check_step(M, ks, vs, lens, t, q_step, o, lse, what):
    B = len(lens)
    for b in range(B):
        n_vis = lens[b] + t + 1
        ro, rl = oracle_attention(q_step[b:b + 1], ks[b][:n_vis], vs[b][:n_vis], [n_vis - 1])
        compare(o[b:b + 1], lse[b:b + 1], ro, rl, what=f"{what} seq {b} step {t}")


def test_decode_step_dev_eager(M):
    lens, steps, h_kv, G, d = [700, 5000, 33000], 3, 8, 4, 128
    ks, vs, shards = _setup(M, lens, steps)
    B, h_q = len(lens), h_kv * G
    len_dev = torch.tensor(lens, dtype=torch.int64, device="cuda")
    ws = M.decode_workspace(B, h_q, h_kv, d)
    o = torch.empty((B, h_q, d), device="cuda")
    lse = torch.empty((B, h_q), device="cuda")
    for t in range(steps):
        k_new = torch.stack([ks[b][lens[b] + t] for b in range(B)]).cuda()
        v_new = torch.stack([vs[b][lens[b] + t] for b in range(B)]).cuda()
        q = synth.queries(90 + t, B, h_q, d, amp=6.0)
        M.decode_step_dev(shards, k_new, v_new, q.cuda(), len_dev, o, lse, ws)
        torch.cuda.synchronize()
        assert len_dev.tolist() == [n + t + 1 for n in lens]
        _check_step(M, ks, vs, lens, t, q, o, lse, "decode_step_dev")
    # the host-side lengths are untouched; the appended rows landed at the device lengths
    assert [s.len for s in shards] == lens
    for b in range(B):
        assert torch.equal(shards[b].k[:, lens[b]:lens[b] + steps].cpu(),
                           ks[b][lens[b]:lens[b] + steps].permute(1, 0, 2))


def test_decode_step_dev_cuda_graph_replay(M):
    """Capture one step with torch.cuda.graph, then replay it: new inputs are copied into the
    captured buffers before each replay; the device counter advances by one per replay."""
    lens, steps, h_kv, G, d = [1200, 9000], 4, 8, 4, 128
    ks, vs, shards = _setup(M, lens, steps + 1, seed=71)
    B, h_q = len(lens), h_kv * G
    len_dev = torch.tensor(lens, dtype=torch.int64, device="cuda")
    ws = M.decode_workspace(B, h_q, h_kv, d)
    o = torch.empty((B, h_q, d), device="cuda")
    lse = torch.empty((B, h_q), device="cuda")
    k_in = torch.zeros((B, h_kv, d), dtype=torch.bfloat16, device="cuda")
    v_in = torch.zeros_like(k_in)
    q_in = torch.zeros((B, h_q, d), dtype=torch.bfloat16, device="cuda")

    def load(t):
        k_in.copy_(torch.stack([ks[b][lens[b] + t] for b in range(B)]))
        v_in.copy_(torch.stack([vs[b][lens[b] + t] for b in range(B)]))
        q = synth.queries(300 + t, B, h_q, d, amp=6.0)
        q_in.copy_(q)
        return q

    # step 0 eagerly on a side stream (warms up the library) ...
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        q0 = load(0)
        M.decode_step_dev(shards, k_in, v_in, q_in, len_dev, o, lse, ws)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    _check_step(M, ks, vs, lens, 0, q0, o, lse, "eager step")
    # ... then capture step 1 (capture does not execute it)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        M.decode_step_dev(shards, k_in, v_in, q_in, len_dev, o, lse, ws)
    torch.cuda.synchronize()
    assert len_dev.tolist() == [n + 1 for n in lens]
    for t in range(1, steps + 1):
        q = load(t)
        g.replay()
        torch.cuda.synchronize()
        assert len_dev.tolist() == [n + t + 1 for n in lens]
        _check_step(M, ks, vs, lens, t, q, o, lse, "graph replay")


def test_decode_step_dev_errors(M):
    sh = M.KVShard.empty(8, 64, 128)
    z = torch.zeros((1, 8, 128), dtype=torch.bfloat16, device="cuda")
    q = torch.zeros((1, 32, 128), dtype=torch.bfloat16, device="cuda")
    ws = M.decode_workspace(1, 32, 8, 128)
    o = torch.empty((1, 32, 128), device="cuda")
    lse = torch.empty((1, 32), device="cuda")
    with pytest.raises(M.MedhaError, match="EINVAL"):
        M._check(M.lib.medha_decode_step_dev(M._shards_c([sh]), 1, None, None, None, 32, None, 1.0, None, None,
                                             None, 0, None), "decode_step_dev")
    with pytest.raises(M.MedhaError, match="ENOTSUP"):
        M.decode_step_dev([sh] * 65, torch.zeros((65, 8, 128), dtype=torch.bfloat16, device="cuda"),
                          torch.zeros((65, 8, 128), dtype=torch.bfloat16, device="cuda"),
                          torch.zeros((65, 32, 128), dtype=torch.bfloat16, device="cuda"),
                          torch.zeros(65, dtype=torch.int64, device="cuda"), o, lse, ws)


@pytest.mark.parametrize("ps,G,d", [(16, 8, 128), (128, 4, 64)])
def test_decode_step_dev_paged(M, ps, G, d):
    """Device-length steps on paged shards (random page order, NaN-poisoned pool): the append
    goes through the page table at the device length, the decode sees exactly keys 0..len."""
    import math
    from test_gpu_paged import Pool, paged_shards
    rng = np.random.default_rng(ps + G)
    h_kv, steps = 2, 3
    lens = [int(rng.integers(1, 3000)) for _ in range(3)]
    need = [math.ceil((n + steps) / ps) for n in lens]
    pool = Pool(sum(need) + 4, ps, h_kv, d, float("nan"), rng)
    ks, vs, specs = [], [], []
    for b, n in enumerate(lens):
        k, v = make_global_kv(8100 + b, n + steps, h_kv, d)
        pages = pool.take(need[b])
        pool.fill(pages, k, v, 0, n)
        ks.append(k)
        vs.append(v)
        specs.append((pages, n, 0))
    shards = paged_shards(M, pool, specs)
    B, h_q = len(lens), h_kv * G
    len_dev = torch.tensor(lens, dtype=torch.int64, device="cuda")
    ws = M.decode_workspace(B, h_q, h_kv, d)
    o = torch.empty((B, h_q, d), device="cuda")
    lse = torch.empty((B, h_q), device="cuda")
    for t in range(steps):
        k_new = torch.stack([ks[b][lens[b] + t] for b in range(B)]).cuda()
        v_new = torch.stack([vs[b][lens[b] + t] for b in range(B)]).cuda()
        q = synth.queries(8200 + t, B, h_q, d, amp=4.0)
        M.decode_step_dev(shards, k_new, v_new, q.cuda(), len_dev, o, lse, ws)
        torch.cuda.synchronize()
        _check_step(M, ks, vs, lens, t, q, o, lse, f"paged decode_step_dev ps={ps}")
    assert len_dev.tolist() == [n + steps for n in lens]
