"""The KVP path on ONE GPU, so the exchange code runs
under the driver's single-GPU `pytest -m gpu`:

* a world-1 KVP communicator (medha_kvp_unique_id -> medha_kvp_comm_create(0, 1)) drives
  medha_kvp_decode through BOTH exchanges - the fused in-kernel push / epoch flags /
  parity slots / rank-ordered merge (a self-loop through the local buffer) and NCCL
  all-gather + merge kernel - plus medha_kvp_exchange_merge, medha_kvp_prefill_chunk and
  medha_decode_step_host(comm).  The merge of one part is the identity (w = e^0 = 1), so
  every KVP result must equal the plain single-GPU call BIT FOR BIT, and the oracle within
  the north_star tolerance (Eq. 5, Eq. 6).
* the device-resident epoch: a CUDA graph holding medha_kvp_decode replays with fresh
  queries and matches the eager call every time (a stale epoch would let the merge read
  the previous replay's partials);
* failure containment: a rank that withholds its push makes the bounded wait expire; the
  kernel finishes, the outputs are NaN and the communicator reports MEDHA_ENCCL;
* dynamic KVP growth ("workers are added once we exceed the worker KV-cache
  token limit") emulated with P rank shards on one GPU: every rank's prefill / decode
  partial (ranks past the sequence hold nothing, the tail rank's shard starts inside the
  chunk) merged with the K5 kernel equals the oracle and the single-shard result;
* prefill shards whose first position lies INSIDE or AFTER the query chunk (the KVP tail /
  growth case): rows with no visible key are exactly (0, -inf) (reading R7).
"""
import math

import numpy as np
import pytest
import torch

import synth
from helpers import KVP_ABS, compare, make_global_kv, oracle_attention, to_shard

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import paper_2409_17264_b200 as M
    return M


@pytest.fixture(scope="module")
def comm(M):
    c = M.KVPComm.single()
    yield c
    c.close()


def _packed(o, lse):
    """(o [..][d], lse [..]) -> the ABI's packed partial o ‖ lse (fp32)."""
    return torch.cat([o.reshape(-1), lse.reshape(-1)])


# ---- a6 + a7 + N1 at world 1 ------------------------------------------------------------
@pytest.mark.parametrize("G,d,lens", [(4, 128, [40000, 777]), (8, 128, [70000]), (1, 64, [5000, 1, 300]),
                                      (16, 64, [9000, 20000]),
                                      (4, 64, [int(x) for x in np.random.default_rng(5).integers(1, 3000, 64)])])
def test_kvp_decode_world1_fused_and_nccl(M, comm, G, d, lens):
    assert comm.world == 1 and comm.p2p, "world-1 fused self-exchange did not initialise"
    h_kv = 2
    B = len(lens)
    kvs, shards, qps = [], [], []
    for b, n in enumerate(lens):
        k, v = make_global_kv(300 + b, n, h_kv, d)
        kvs.append((k, v))
        shards.append(to_shard(k, v, 0, n))
        qps.append(n - 1 if b % 2 == 0 else n // 2)
    q = synth.queries(301, B, h_kv * G, d, amp=6.0).cuda()
    o1, l1 = M.attn_decode_partial(shards, q, qps)
    outs = []
    for _ in range(3):        # three epochs: both parities of the receive slots, and back
        o, lse, ob = M.kvp_decode(comm, shards, q, qps, want_bf16=True)
        outs.append((o.clone(), lse.clone(), ob.clone()))
    comm.set_p2p(False)
    try:
        o_n, l_n, ob_n = M.kvp_decode(comm, shards, q, qps, want_bf16=True)
    finally:
        comm.set_p2p(True)
    torch.cuda.synchronize()
    assert comm.status() == 0
    for o, lse, ob in outs + [(o_n, l_n, ob_n)]:
        assert torch.equal(o, o1) and torch.equal(lse, l1), (o - o1).abs().max().item()
        assert torch.equal(ob, o1.to(torch.bfloat16))
    for b, (k, v) in enumerate(kvs):
        ro, rl = oracle_attention(q[b:b + 1].cpu(), k, v, [qps[b]])
        compare(o1[b:b + 1], l1[b:b + 1], ro, rl, what=f"kvp world1 seq {b}")


def test_kvp_exchange_merge_world1(M, comm):
    h_kv, G, d, N = 8, 4, 128, 12345
    k, v = make_global_kv(310, N, h_kv, d)
    sh = to_shard(k, v, 0, N)
    q = synth.queries(311, 1, h_kv * G, d, amp=4.0).cuda()
    o1, l1 = M.attn_decode_partial([sh], q, [N - 1])
    rows = h_kv * G
    send = _packed(o1, l1)
    o = torch.empty((rows, d), device="cuda")
    lse = torch.empty((rows,), device="cuda")
    ob = torch.empty((rows, d), dtype=torch.bfloat16, device="cuda")
    M.kvp_exchange_merge(comm, send, rows, d, o, lse, ob)
    torch.cuda.synchronize()
    assert torch.equal(o, o1.reshape(rows, d)) and torch.equal(lse, l1.reshape(rows))
    assert torch.equal(ob, o.to(torch.bfloat16))


@pytest.mark.parametrize("c,P0,G,d", [(256, 9000, 4, 128), (64, 30000, 8, 128), (300, 1000, 1, 64)])
def test_kvp_prefill_world1(M, comm, c, P0, G, d):
    h_kv = 2
    N = P0 + c
    k, v = make_global_kv(320 + c, N, h_kv, d)
    sh = to_shard(k, v, 0, N)
    q = synth.queries(321, c, h_kv * G, d, amp=4.0, t0=P0).cuda()
    o1, l1 = M.attn_prefill_chunk(sh, q, P0)
    o, lse, ob = M.kvp_prefill_chunk(comm, sh, q, P0, want_bf16=True)
    torch.cuda.synchronize()
    assert torch.equal(o, o1) and torch.equal(lse, l1)
    assert torch.equal(ob, o1.to(torch.bfloat16))
    rows = [0, c // 2, c - 1]
    ro, rl = oracle_attention(q[rows].cpu(), k, v, [P0 + r for r in rows])
    compare(o[rows], lse[rows], ro, rl, what="kvp prefill world1")


def test_decode_step_host_world1(M, comm):
    """e2e host-buffer step through the KVP communicator (fused exchange) = without it."""
    h_kv, G, d, N = 8, 4, 128, 50000
    k, v = make_global_kv(330, N, h_kv, d)
    q = synth.queries(331, 1, h_kv * G, d, amp=6.0)
    res = []
    for use_comm in (False, True):
        sh = to_shard(k, v, 0, N - 1, extra_cap=5)
        ws = M.decode_step_workspace(1, h_kv * G, h_kv, d)
        o_h = torch.empty((h_kv * G, d), dtype=torch.float32).pin_memory()
        l_h = torch.empty((h_kv * G,), dtype=torch.float32).pin_memory()
        M.decode_step_host(comm if use_comm else None, sh, True, q[0].contiguous().pin_memory(),
                           k[N - 1].contiguous().pin_memory(), v[N - 1].contiguous().pin_memory(), N - 1, o_h, l_h,
                           ws)
        torch.cuda.synchronize()
        assert sh.len == N
        res.append((o_h.clone(), l_h.clone()))
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])
    ro, rl = oracle_attention(q, k, v, [N - 1])
    compare(res[1][0][None], res[1][1][None], ro, rl, what="decode_step_host world1")


@pytest.mark.parametrize("fused", [True, False])
def test_kvp_decode_cuda_graph_replay(M, comm, fused):
    """medha_kvp_decode captured once, replayed with new queries: the device-resident epoch
    advances on every replay, so each replay merges the partials of ITS OWN launch."""
    h_kv, G, d, N, steps = 8, 4, 128, 60000, 5
    k, v = make_global_kv(340, N, h_kv, d)
    sh = to_shard(k, v, 0, N)
    B = 2
    qps = [N - 1, N - 7]
    q_static = torch.zeros((B, h_kv * G, d), dtype=torch.bfloat16, device="cuda")
    o = torch.empty((B, h_kv * G, d), device="cuda")
    lse = torch.empty((B, h_kv * G), device="cuda")
    ws = torch.zeros(M.lib.medha_kvp_workspace_size(1, B, h_kv * G, h_kv, d), dtype=torch.uint8, device="cuda")
    comm.set_p2p(fused)
    try:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):          # warm-up outside the capture
            M.kvp_decode(comm, [sh, sh], q_static, qps, ws=ws, o=o, lse=lse)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            M.kvp_decode(comm, [sh, sh], q_static, qps, ws=ws, o=o, lse=lse)
        for t in range(steps):
            qt = synth.queries(350 + t, B, h_kv * G, d, amp=6.0).cuda()
            q_static.copy_(qt)
            g.replay()
            torch.cuda.synchronize()
            o_ref, l_ref = M.attn_decode_partial([sh, sh], qt, qps)
            torch.cuda.synchronize()
            assert torch.equal(o, o_ref) and torch.equal(lse, l_ref), f"replay {t}: {(o - o_ref).abs().max().item()}"
        del g
        assert comm.status() == 0
    finally:
        comm.set_p2p(True)


def test_fused_exchange_timeout_is_reported(M):
    """A rank that never pushes (test hook) must not hang the GPU: the bounded wait expires,
    the outputs become NaN, the communicator reports MEDHA_ENCCL and later calls fail."""
    c = M.KVPComm.single()
    try:
        assert c.p2p
        h_kv, G, d, N = 2, 4, 128, 4000
        k, v = make_global_kv(360, N, h_kv, d)
        sh = to_shard(k, v, 0, N)
        q = synth.queries(361, 1, h_kv * G, d).cuda()
        o, lse, _ = M.kvp_decode(c, [sh], q, [N - 1])        # healthy first
        torch.cuda.synchronize()
        assert c.status() == 0 and torch.isfinite(o).all()
        c.set_timeout(0.05)
        c.debug(1)
        o, lse, _ = M.kvp_decode(c, [sh], q, [N - 1])
        torch.cuda.synchronize()                              # returns: the wait is bounded
        assert c.status() == -7
        assert torch.isnan(o).all() and torch.isnan(lse).all()
        c.debug(0)
        with pytest.raises(M.MedhaError, match="MEDHA_ENCCL"):
            M.kvp_decode(c, [sh], q, [N - 1])
        # the device is still healthy: plain calls run and are correct
        o1, l1 = M.attn_decode_partial([sh], q, [N - 1])
        ro, rl = oracle_attention(q.cpu(), k, v, [N - 1])
        compare(o1, l1, ro, rl, what="after timeout")
    finally:
        c.close()


# ---- N3: dynamic KVP growth, P rank shards emulated on one GPU -----------------------------
@pytest.mark.parametrize("P,limit,G,d", [(2, 3000, 4, 128), (4, 1500, 8, 128), (8, 700, 1, 64)])
def test_kvp_growth_emulated(M, P, limit, G, d):
    """A sequence grows through the workers (rank r owns positions [r L, (r+1) L),
    kvp.KVPGrowingSequence); after every chunk, the chunk attends over all P rank shards
    (each a medha_attn_prefill_chunk partial; unused ranks and the tail rank's
    chunk-straddling shard included), the partials are merged by the K5 kernel
    (medha_merge_partials, rank order), then one decode token does the same.  Each result
    equals the oracle and, within the north_star KVP tolerance, the single-shard call."""
    from paper_2409_17264_b200.kvp import KVPGrowingSequence
    h_kv = 2
    h_q = h_kv * G
    cap = limit * P
    chunks = [int(cap * f) for f in (0.15, 0.3, 0.25, 0.2)]     # straddle the rank boundaries
    total = sum(chunks) + 1
    assert total <= cap
    k, v = make_global_kv(370 + P, total, h_kv, d)
    ranks = [KVPGrowingSequence(r, P, limit, h_kv, d) for r in range(P)]
    whole = M.KVShard.empty(h_kv, total + 8, d)
    n = 0

    def merged(parts):
        packed = torch.stack([_packed(o, l) for o, l in parts])
        rows = parts[0][1].numel()
        o_m, l_m, _ = M.merge_partials(packed, rows, d)
        return o_m.reshape(parts[0][0].shape), l_m.reshape(parts[0][1].shape)

    for ci, c in enumerate(chunks):
        kc, vc = k[n:n + c].cuda(), v[n:n + c].cuda()
        for rk in ranks:
            rk.append(kc, vc)
        M.kv_append(whole, kc, vc)
        q = synth.queries(380 + ci, c, h_q, d, amp=4.0, t0=n).cuda()
        parts = [M.attn_prefill_chunk(rk.shard, q, n) for rk in ranks]
        o_m, l_m = merged(parts)
        o1, l1 = M.attn_prefill_chunk(whole, q, n)
        torch.cuda.synchronize()
        assert (o_m - o1).abs().max().item() <= KVP_ABS and (l_m - l1).abs().max().item() <= KVP_ABS
        rows = sorted(set([0, c // 3, c - 1]))
        ro, rl = oracle_attention(q[rows].cpu(), k[:n + c], v[:n + c], [n + r for r in rows])
        compare(o_m[rows], l_m[rows], ro, rl, what=f"growth P={P} chunk {ci}")
        n += c
        active = sum(1 for rk in ranks if rk.shard.len > 0)
        assert active == math.ceil(n / limit) == ranks[0].active_workers
    # one decode token after the last chunk
    kd, vd = k[n:n + 1].cuda(), v[n:n + 1].cuda()
    for rk in ranks:
        rk.append(kd, vd)
    M.kv_append(whole, kd, vd)
    qd = synth.queries(390, 1, h_q, d, amp=6.0).cuda()
    parts = [M.attn_decode_partial([rk.shard], qd, [n]) for rk in ranks]
    o_m, l_m = merged(parts)
    o1, l1 = M.attn_decode_partial([whole], qd, [n])
    torch.cuda.synchronize()
    assert (o_m - o1).abs().max().item() <= KVP_ABS
    ro, rl = oracle_attention(qd.cpu(), k[:n + 1], v[:n + 1], [n])
    compare(o_m, l_m, ro, rl, what=f"growth P={P} decode")


# ---- prefill over shards that start inside or after the chunk ----------------------------
def _paged_copy(M, sh, ps, rng):
    """The same shard in a zero-filled page pool with a random page order."""
    n_pages = math.ceil(max(sh.capacity, 1) / ps) + 2
    h_kv, _, d = sh.k.shape
    K = torch.zeros((h_kv, n_pages * ps, d), dtype=torch.bfloat16, device="cuda")
    V = torch.zeros_like(K)
    order = [int(x) for x in rng.permutation(n_pages)]
    need = math.ceil(max(sh.len, 1) / ps)
    for i in range(need):
        m = min(ps, sh.len - i * ps)
        if m > 0:
            K[:, order[i] * ps:order[i] * ps + m] = sh.k[:, i * ps:i * ps + m]
            V[:, order[i] * ps:order[i] * ps + m] = sh.v[:, i * ps:i * ps + m]
    table = torch.tensor(order[:need], dtype=torch.int32, device="cuda")
    return M.KVShard.paged(K, V, table, ps, sh.len, sh.pos0)


_TAIL_CASES = [(G, d, c, where) for G in (1, 4, 8, 16) for d in (64, 128) for c, where in
               ((1, "after"), (64, "inside"), (300, "inside"), (1024, "after"))] + \
              [(4, 128, 1024, "inside"), (16, 64, 300, "after"), (8, 128, 64, "after"), (1, 64, 1024, "inside")]


@pytest.mark.parametrize("G,d,c,where", _TAIL_CASES)
def test_prefill_shard_starts_inside_or_after_chunk(M, G, d, c, where):
    rng = np.random.default_rng(G * 1000 + d + c)
    h_kv = 2 if G <= 4 else 1
    P0 = int(rng.integers(200, 3000))             # chunk at [P0, P0 + c)
    N = P0 + c + int(rng.integers(0, 400))        # the shard may also hold tokens past the chunk
    if where == "inside":
        a = P0 + int(rng.integers(1, c)) if c > 1 else P0
    else:
        a = P0 + c + int(rng.integers(0, 50))
    N = max(N, a + 1)
    k, v = make_global_kv(400 + G + c, N, h_kv, d)
    q = synth.queries(401 + c, c, h_kv * G, d, amp=4.0, t0=P0)
    sh = to_shard(k, v, a, N, poison=False)
    ref_o, ref_l = oracle_attention(q, k, v, list(range(P0, P0 + c)), (a, N))
    for layout in ("contiguous", "paged"):
        s = sh if layout == "contiguous" else _paged_copy(M, sh, 128 if c % 2 else 256, rng)
        o, lse = M.attn_prefill_chunk(s, q.cuda(), P0)
        torch.cuda.synchronize()
        lg = lse.cpu()
        empty = ~np.isfinite(ref_l)
        if where == "after":
            assert empty.all()
        else:
            assert empty.any() and (~empty).any()
        # rows with no visible key: exactly o = 0, lse = -inf
        assert torch.equal(o.cpu()[torch.from_numpy(empty)], torch.zeros_like(o.cpu()[torch.from_numpy(empty)]))
        assert torch.isneginf(lg[torch.from_numpy(empty)]).all()
        compare(o, lse, ref_o, ref_l, what=f"{layout} G={G} d={d} c={c} {where}")


@pytest.mark.parametrize("fused", [True, False])
def test_kvp_workspace_reused_across_shapes(M, comm, fused):
    """One zero-filled workspace serves KVP decode calls of different shapes (the header's
    "left zeroed" contract): the counter block must not move with (batch, h_q, d)."""
    big = max(M.lib.medha_kvp_workspace_size(1, b, h_kv * G, h_kv, d)
              for b, h_kv, G, d in ((1, 8, 8, 128), (3, 2, 1, 64), (2, 4, 4, 128)))
    ws = torch.zeros(big, dtype=torch.uint8, device="cuda")
    comm.set_p2p(fused)
    try:
        for i, (B, h_kv, G, d, n) in enumerate(((1, 8, 8, 128, 30000), (3, 2, 1, 64, 5000), (2, 4, 4, 128, 9000),
                                                 (1, 8, 8, 128, 30000))):
            k, v = make_global_kv(500 + i, n, h_kv, d)
            sh = to_shard(k, v, 0, n)
            q = synth.queries(501 + i, B, h_kv * G, d, amp=4.0).cuda()
            qps = [n - 1 - b for b in range(B)]
            o, lse, _ = M.kvp_decode(comm, [sh] * B, q, qps, ws=ws)
            o1, l1 = M.attn_decode_partial([sh] * B, q, qps)
            torch.cuda.synchronize()
            assert comm.status() == 0
            assert torch.equal(o, o1) and torch.equal(lse, l1), f"shape {i}"
    finally:
        comm.set_p2p(True)


@pytest.mark.parametrize("use_comm,pinned", [(False, True), (True, True), (False, False)])
def test_decode_plan_equals_decode_step_host(M, comm, use_comm, pinned):
    """medha_decode_plan_step (prepared host buffers / workspace) = medha_decode_step_host,
    step after step; pinned (zero-copy) and pageable (staged copies) host buffers."""
    h_kv, G, d, N, steps = 8, 4, 128, 30000, 3
    k, v = make_global_kv(700, N + steps, h_kv, d)
    qs = synth.queries(701, steps, h_kv * G, d, amp=6.0)
    pin = (lambda t: t.pin_memory()) if pinned else (lambda t: t)
    c = comm if use_comm else None
    res = []
    for mode in ("host", "plan"):
        sh = to_shard(k, v, 0, N, extra_cap=steps + 2)
        ws = torch.zeros(M.lib.medha_decode_step_workspace_size(1, h_kv * G, h_kv, d), dtype=torch.uint8, device="cuda")
        q_h = pin(torch.empty((h_kv * G, d), dtype=torch.bfloat16))
        k_h = pin(torch.empty((h_kv, d), dtype=torch.bfloat16))
        v_h = pin(torch.empty((h_kv, d), dtype=torch.bfloat16))
        o_h = pin(torch.empty((h_kv * G, d), dtype=torch.float32))
        l_h = pin(torch.empty((h_kv * G,), dtype=torch.float32))
        plan = M.DecodePlan(c, sh, q_h, k_h, v_h, o_h, l_h, ws) if mode == "plan" else None
        outs = []
        for t in range(steps):
            q_h.copy_(qs[t])
            k_h.copy_(k[N + t])
            v_h.copy_(v[N + t])
            if plan is None:
                M.decode_step_host(c, sh, True, q_h, k_h, v_h, N + t, o_h, l_h, ws)
            else:
                plan.step(sh, True, N + t)
            torch.cuda.synchronize()
            outs.append((o_h.clone(), l_h.clone()))
        if plan is not None:
            plan.close()
        assert sh.len == N + steps
        res.append(outs)
    for t in range(steps):
        assert torch.equal(res[0][t][0], res[1][t][0]) and torch.equal(res[0][t][1], res[1][t][1])
        ro, rl = oracle_attention(qs[t:t + 1], k[:N + t + 1], v[:N + t + 1], [N + t])
        compare(res[1][t][0][None], res[1][t][1][None], ro, rl, what=f"decode plan step {t}")


@pytest.mark.parametrize("tp,kvp", [(2, 2), (4, 2), (2, 4)])
def test_kvp_x_tp_emulated(M, tp, kvp):
    """N4 (P:509-516 KVP x TP) on one GPU: TP slices of the KV heads (each with its query heads)
    times KVP sequence shards; every (slice, rank) partial is a medha_attn_decode_partial /
    medha_attn_prefill_chunk call, the KVP merge is the K5 kernel over the ranks of a slice,
    and the slices concatenate to the single-GPU result (north_star 1e-3) and the oracle."""
    from paper_2409_17264_b200.kvp import shard_range
    h_kv, G, d, N, c = 8, 4, 128, 40000, 96
    k, v = make_global_kv(720 + tp * 10 + kvp, N, h_kv, d)
    qd = synth.queries(721, 1, h_kv * G, d, amp=6.0)
    qc = synth.queries(722, c, h_kv * G, d, amp=4.0, t0=N - c)
    whole = to_shard(k, v, 0, N)
    od1, ld1 = M.attn_decode_partial([whole], qd.cuda(), [N - 1])
    op1, lp1 = M.attn_prefill_chunk(whole, qc.cuda(), N - c)
    hs = h_kv // tp
    od = torch.empty_like(od1)
    ld = torch.empty_like(ld1)
    op = torch.empty_like(op1)
    lp = torch.empty_like(lp1)
    for t in range(tp):
        heads = slice(t * hs, (t + 1) * hs)
        qh = slice(t * hs * G, (t + 1) * hs * G)
        kt, vt = k[:, heads].contiguous(), v[:, heads].contiguous()
        parts_d, parts_p = [], []
        for r in range(kvp):
            a, b = shard_range(N, r, kvp)
            sh = to_shard(kt, vt, a, b)
            o, l = M.attn_decode_partial([sh], qd[:, qh].contiguous().cuda(), [N - 1])
            parts_d.append(torch.cat([o.reshape(-1), l.reshape(-1)]))
            o, l = M.attn_prefill_chunk(sh, qc[:, qh].contiguous().cuda(), N - c)
            parts_p.append(torch.cat([o.reshape(-1), l.reshape(-1)]))
        o, l, _ = M.merge_partials(torch.stack(parts_d), hs * G, d)
        od[:, qh], ld[:, qh] = o.view(1, hs * G, d), l.view(1, hs * G)
        o, l, _ = M.merge_partials(torch.stack(parts_p), c * hs * G, d)
        op[:, qh], lp[:, qh] = o.view(c, hs * G, d), l.view(c, hs * G)
    torch.cuda.synchronize()
    assert (od - od1).abs().max().item() <= KVP_ABS and (ld - ld1).abs().max().item() <= KVP_ABS
    assert (op - op1).abs().max().item() <= KVP_ABS and (lp - lp1).abs().max().item() <= KVP_ABS
    ro, rl = oracle_attention(qd, k, v, [N - 1])
    compare(od, ld, ro, rl, what=f"KVPxTP {tp}x{kvp} decode")
    rows = [0, c - 1]
    ro, rl = oracle_attention(qc[rows], k, v, [N - c + r for r in rows])
    compare(op[rows], lp[rows], ro, rl, what=f"KVPxTP {tp}x{kvp} prefill")
