"""Fused append + decode in one launch (SURVEY §8(a) a1 + a3 + a5; include/medha_attn.h
`medha_attn_decode_append`, `medha_kvp_decode_append`, and the one-launch
`medha_decode_step_dev`): the result must be BIT-identical to medha_kv_append followed by
medha_attn_decode_partial (same split plan, same arithmetic - only the source of the new
token's bytes differs), the new rows must land in the shard, and the oracle must agree.
The slot the new token goes to is NaN-poisoned beforehand: reading it instead of k_new /
v_new would poison the output."""
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


def _copy(M, sh):
    return M.KVShard(sh.k.clone(), sh.v.clone(), sh.len, sh.pos0)


@pytest.mark.parametrize("G,d,lens,mask", [(4, 128, [1 << 17], None), (8, 128, [40000, 3, 700], [1, 0, 1]),
                                           (1, 64, [5000, 1], None), (16, 64, [9000, 20000, 64], [0, 1, 1]),
                                           (2, 128, [300000], [1])])
def test_decode_append_equals_append_then_decode(M, G, d, lens, mask):
    h_kv = 2
    B = len(lens)
    ks, vs, shards, qps = [], [], [], []
    for b, n in enumerate(lens):
        k, v = make_global_kv(600 + b, n + 1, h_kv, d)
        ks.append(k)
        vs.append(v)
        shards.append(to_shard(k, v, 0, n, extra_cap=5))       # spare capacity NaN-poisoned
        qps.append(n)                                          # the new token's own position
    if mask is not None:
        qps = [n if m else n - 1 for n, m in zip(lens, mask)]
    k_new = torch.stack([ks[b][lens[b]] for b in range(B)]).cuda()
    v_new = torch.stack([vs[b][lens[b]] for b in range(B)]).cuda()
    q = synth.queries(610, B, h_kv * G, d, amp=6.0).cuda()
    ref = [_copy(M, s) for s in shards]
    for b in range(B):
        if mask is None or mask[b]:
            M.kv_append(ref[b], k_new[b:b + 1], v_new[b:b + 1])
    o1, l1 = M.attn_decode_partial(ref, q, qps)
    o2, l2 = M.attn_decode_append(shards, k_new, v_new, q, qps, append=mask)
    torch.cuda.synchronize()
    assert [s.len for s in shards] == [s.len for s in ref]
    assert torch.equal(o1, o2) and torch.equal(l1, l2), (o1 - o2).abs().max().item()
    for b in range(B):
        n = shards[b].len
        assert torch.equal(shards[b].k[:, :n], ref[b].k[:, :n]) and torch.equal(shards[b].v[:, :n], ref[b].v[:, :n])
        ro, rl = oracle_attention(q[b:b + 1].cpu(), ks[b][:n], vs[b][:n], [qps[b]])
        compare(o2[b:b + 1], l2[b:b + 1], ro, rl, what=f"decode_append seq {b}")


@pytest.mark.parametrize("ps,n", [(64, 5000), (64, 4096), (16, 4095), (256, 1)])
def test_decode_append_paged(M, ps, n):
    """Paged shard: the owner item stores the new rows through the page table (incl. a new
    token that opens a new page, n % ps == 0)."""
    h_kv, G, d = 2, 4, 128
    rng = np.random.default_rng(7)
    k, v = make_global_kv(620, n + 1, h_kv, d)
    n_pages = (n + 1 + ps - 1) // ps + 1
    order = [int(x) for x in rng.permutation(n_pages + 3)[:n_pages]]
    K = torch.full((h_kv, (n_pages + 3) * ps, d), float("nan"), dtype=torch.bfloat16)
    V = torch.full_like(K, float("nan"))
    for i, pg in enumerate(order):
        m = max(0, min(ps, n - i * ps))
        if m:
            K[:, pg * ps:pg * ps + m] = k[i * ps:i * ps + m].permute(1, 0, 2)
            V[:, pg * ps:pg * ps + m] = v[i * ps:i * ps + m].permute(1, 0, 2)
    sh = M.KVShard.paged(K.cuda(), V.cuda(), torch.tensor(order, dtype=torch.int32, device="cuda"), ps, n, 0)
    q = synth.queries(621, 1, h_kv * G, d, amp=6.0).cuda()
    o, lse = M.attn_decode_append([sh], k[n:n + 1].cuda(), v[n:n + 1].cuda(), q, [n])
    torch.cuda.synchronize()
    assert sh.len == n + 1
    row = order[n // ps] * ps + n % ps
    assert torch.equal(sh.k[:, row].cpu(), k[n]) and torch.equal(sh.v[:, row].cpu(), v[n])
    ro, rl = oracle_attention(q.cpu(), k, v, [n])
    compare(o, lse, ro, rl, what="decode_append paged")


def test_decode_append_full_shard_is_erange(M):
    h_kv, d = 2, 64
    k, v = make_global_kv(630, 100, h_kv, d)
    sh = to_shard(k, v, 0, 100, extra_cap=0)
    q = synth.queries(631, 1, h_kv * 4, d).cuda()
    with pytest.raises(M.MedhaError, match="MEDHA_ERANGE"):
        M.attn_decode_append([sh], k[:1].cuda(), v[:1].cuda(), q, [100])
    assert sh.len == 100


def test_kvp_decode_append_world1(M):
    comm = M.KVPComm.single()
    try:
        h_kv, G, d = 8, 4, 128
        lens = [70000, 1234]
        B = len(lens)
        ks, vs, a_sh, b_sh = [], [], [], []
        for b, n in enumerate(lens):
            k, v = make_global_kv(640 + b, n + 1, h_kv, d)
            ks.append(k)
            vs.append(v)
            a_sh.append(to_shard(k, v, 0, n, extra_cap=3))
            b_sh.append(to_shard(k, v, 0, n, extra_cap=3))
        k_new = torch.stack([ks[b][lens[b]] for b in range(B)]).cuda()
        v_new = torch.stack([vs[b][lens[b]] for b in range(B)]).cuda()
        q = synth.queries(641, B, h_kv * G, d, amp=6.0).cuda()
        o1, l1 = M.attn_decode_append(a_sh, k_new, v_new, q, lens)
        o2, l2, _ = M.kvp_decode_append(comm, b_sh, k_new, v_new, q, lens)
        torch.cuda.synchronize()
        assert [s.len for s in b_sh] == [n + 1 for n in lens]
        # fused exchange plans >= 2 splits per sequence; weights of a lone split are exactly 1
        assert (o1 - o2).abs().max().item() <= 1e-6 and (l1 - l2).abs().max().item() <= 1e-6
        for b in range(B):
            ro, rl = oracle_attention(q[b:b + 1].cpu(), ks[b], vs[b], [lens[b]])
            compare(o2[b:b + 1], l2[b:b + 1], ro, rl, what=f"kvp_decode_append seq {b}")
    finally:
        comm.close()


def test_decode_append_batch_over_64(M):
    """> 64 sequences: two launches on one workspace (both early-started); still equal to
    kv_append + decode_partial and the appended rows land in every shard."""
    h_kv, G, d, B = 2, 4, 64, 70
    rng = np.random.default_rng(11)
    lens = [int(x) for x in rng.integers(1, 3000, size=B)]
    ks, vs, a_sh, r_sh = [], [], [], []
    for b, n in enumerate(lens):
        k, v = make_global_kv(900 + b, n + 1, h_kv, d)
        ks.append(k)
        vs.append(v)
        a_sh.append(to_shard(k, v, 0, n, extra_cap=2))
        r_sh.append(to_shard(k, v, 0, n, extra_cap=2))
    k_new = torch.stack([ks[b][lens[b]] for b in range(B)]).cuda()
    v_new = torch.stack([vs[b][lens[b]] for b in range(B)]).cuda()
    q = synth.queries(901, B, h_kv * G, d, amp=4.0).cuda()
    for b in range(B):
        M.kv_append(r_sh[b], k_new[b:b + 1], v_new[b:b + 1])
    o1, l1 = M.attn_decode_partial(r_sh, q, lens)
    o2, l2 = M.attn_decode_append(a_sh, k_new, v_new, q, lens)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    for b in (0, 63, 64, B - 1):
        n = lens[b] + 1
        assert torch.equal(a_sh[b].k[:, :n], r_sh[b].k[:, :n])
        ro, rl = oracle_attention(q[b:b + 1].cpu(), ks[b], vs[b], [lens[b]])
        compare(o2[b:b + 1], l2[b:b + 1], ro, rl, what=f"batch>64 seq {b}")
