"""Paged KV cache (include/medha_attn.h `page_table`): shards whose tokens live in
pages of a shared pool, in a random page order, must give the SAME bits as the contiguous
layout (same split plan, same arithmetic, only the addresses differ) and match the oracle.

Decode pools are NaN-poisoned everywhere a shard does not own valid tokens (decode must not
read them); prefill pools are zero-filled, as the header's contract requires."""
import math

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


class Pool:
    """CPU staging of a page pool [h_kv][n_pages * ps][d] handed out in a random order."""

    def __init__(self, n_pages, ps, h_kv, d, fill, rng):
        self.ps = ps
        self.k = torch.full((h_kv, n_pages * ps, d), fill, dtype=torch.bfloat16)
        self.v = torch.full((h_kv, n_pages * ps, d), fill, dtype=torch.bfloat16)
        self.free = [int(x) for x in rng.permutation(n_pages)]

    def take(self, n_pages):
        pages, self.free = self.free[:n_pages], self.free[n_pages:]
        return pages

    def fill(self, pages, k_tok, v_tok, a, b):
        """Write global tokens [a, b) into the shard's pages (local token j = global a + j)."""
        ps = self.ps
        for i, pg in enumerate(pages):
            lo = a + i * ps
            m = max(0, min(ps, b - lo))
            if m:
                self.k[:, pg * ps:pg * ps + m] = k_tok[lo:lo + m].permute(1, 0, 2)
                self.v[:, pg * ps:pg * ps + m] = v_tok[lo:lo + m].permute(1, 0, 2)


def paged_shards(M, pool, specs):
    """specs: list of (pages, length, pos0) -> KVShard.paged over the pool moved to the GPU."""
    K, V = pool.k.cuda(), pool.v.cuda()
    return [M.KVShard.paged(K, V, torch.tensor(pages, dtype=torch.int32, device="cuda"), pool.ps, n, a)
            for pages, n, a in specs]


@pytest.mark.parametrize("ps,G,d", [(16, 8, 128), (64, 4, 128), (256, 1, 64), (128, 16, 64), (1024, 8, 128)])
def test_paged_decode_matches_contiguous(M, ps, G, d):
    rng = np.random.default_rng(ps * 7 + G)
    h_kv, B = 2, 4
    lens = [int(rng.integers(1, 9000)) for _ in range(B)]
    starts = [int(rng.integers(0, n)) for n in lens]          # shard = global tokens [a, N)
    pages_needed = [math.ceil((n - a) / ps) + int(rng.integers(0, 3)) for n, a in zip(lens, starts)]
    pool = Pool(sum(pages_needed) + 5, ps, h_kv, d, float("nan"), rng)
    kvs, specs, refs, qs, qps = [], [], [], [], []
    for b in range(B):
        N, a = lens[b], starts[b]
        k, v = make_global_kv(7000 + b, N, h_kv, d)
        pages = pool.take(pages_needed[b])
        pool.fill(pages, k, v, a, N)
        specs.append((pages, N - a, a))
        kvs.append(to_shard(k, v, a, N, extra_cap=pages_needed[b] * ps - (N - a)))
        q = synth.queries(7100 + b, 1, h_kv * G, d, amp=4.0)
        qp = int(rng.integers(a, N))
        qs.append(q)
        qps.append(qp)
        refs.append(oracle_attention(q, k, v, [qp], (a, N)))
    paged = paged_shards(M, pool, specs)
    q = torch.cat(qs).cuda()
    o_p, l_p = M.attn_decode_partial(paged, q, qps)
    o_c, l_c = M.attn_decode_partial(kvs, q, qps)
    torch.cuda.synchronize()
    assert torch.equal(o_p, o_c) and torch.equal(l_p, l_c), "paged decode differs from contiguous"
    for b in range(B):
        compare(o_p[b:b + 1], l_p[b:b + 1], refs[b][0], refs[b][1], what=f"paged decode ps={ps} b={b}")


@pytest.mark.parametrize("ps,G,d,c", [(128, 8, 128, 300), (256, 4, 64, 77), (128, 1, 128, 1), (512, 16, 128, 129)])
def test_paged_prefill_matches_contiguous(M, ps, G, d, c):
    rng = np.random.default_rng(ps + c)
    h_kv, n = 2, 3
    pool_pages, specs, chunks = 0, [], []
    for i in range(n):
        P0 = int(rng.integers(0, 4000))
        N = P0 + c
        a = int(rng.integers(0, P0 + 1))
        chunks.append((P0, N, a))
        pool_pages += math.ceil((N - a) / ps) + 1
    pool = Pool(pool_pages + 3, ps, h_kv, d, 0.0, rng)
    contig, qs, refs = [], [], []
    for i, (P0, N, a) in enumerate(chunks):
        k, v = make_global_kv(7200 + i, N, h_kv, d)
        pages = pool.take(math.ceil((N - a) / ps) + 1)
        pool.fill(pages, k, v, a, N)
        specs.append((pages, N - a, a))
        contig.append(to_shard(k, v, a, N))
        q = synth.queries(7300 + i, c, h_kv * G, d, amp=4.0, t0=P0)
        qs.append(q.cuda())
        rows = sorted(set([0, c - 1, c // 2]))
        refs.append((rows, oracle_attention(q[rows], k, v, [P0 + r for r in rows], (a, N))))
    paged = paged_shards(M, pool, specs)
    p0s = [P0 for P0, _, _ in chunks]
    outs_p = M.attn_prefill_batch(paged, qs, p0s)
    outs_c = M.attn_prefill_batch(contig, qs, p0s)
    for i in range(n):
        (op, lp), (oc, lc) = outs_p[i], outs_c[i]
        assert torch.equal(op, oc) and torch.equal(lp, lc), f"paged prefill {i} differs from contiguous"
        rows, (ro, rl) = refs[i]
        compare(op[rows], lp[rows], ro, rl, what=f"paged prefill ps={ps} chunk={i}")
        o1, l1 = M.attn_prefill_chunk(paged[i], qs[i], p0s[i])
        assert (o1 - op).abs().max().item() < 1e-4 and (l1 - lp).abs().max().item() < 1e-4


def test_paged_append_then_decode(M):
    """K1 scatters through the page table: appending in ragged pieces across page boundaries
    into a paged shard gives the same cache (read back through the table) and the same decode
    as the contiguous shard."""
    rng = np.random.default_rng(77)
    h_kv, d, G, ps, N = 2, 128, 4, 16, 1000
    k, v = make_global_kv(7400, N, h_kv, d)
    pool = Pool(math.ceil(N / ps) + 8, ps, h_kv, d, float("nan"), rng)
    pages = pool.take(math.ceil(N / ps))
    (sh_p,) = paged_shards(M, pool, [(pages, 0, 0)])
    sh_c = M.KVShard.empty(h_kv, N, d)
    t = 0
    while t < N:
        m = min(N - t, int(rng.integers(1, 70)))
        kn, vn = k[t:t + m].cuda(), v[t:t + m].cuda()
        M.kv_append(sh_p, kn, vn)
        M.kv_append(sh_c, kn, vn)
        t += m
    assert sh_p.len == N == sh_c.len
    rows = torch.tensor([pg * ps + j for pg in pages for j in range(ps)][:N], device="cuda")
    assert torch.equal(sh_p.k[:, rows], sh_c.k) and torch.equal(sh_p.v[:, rows], sh_c.v)
    q = synth.queries(7401, 1, h_kv * G, d).cuda()
    o_p, l_p = M.attn_decode_partial([sh_p], q, [N - 1])
    o_c, l_c = M.attn_decode_partial([sh_c], q, [N - 1])
    assert torch.equal(o_p, o_c) and torch.equal(l_p, l_c)


def test_paged_argument_errors(M):
    h_kv, d = 1, 64
    K = torch.zeros((h_kv, 256, d), dtype=torch.bfloat16, device="cuda")
    pt = torch.arange(4, dtype=torch.int32, device="cuda")
    q = torch.zeros((1, 8, d), dtype=torch.bfloat16, device="cuda")
    bad = M.KVShard.paged(K, K, pt, 48, 10)                         # not a power of two
    with pytest.raises(M.MedhaError, match="EINVAL"):
        M.attn_decode_partial([bad], q, [9])
    small = M.KVShard.paged(K, K, pt, 64, 10)                       # prefill needs >= 128
    with pytest.raises(M.MedhaError, match="ENOTSUP"):
        M.attn_prefill_chunk(small, q, 0)
    over = M.KVShard.paged(K, K, pt, 64, 10)
    over.len = 257                                                  # len > 4 pages x 64
    with pytest.raises(M.MedhaError, match="ERANGE"):
        M.attn_decode_partial([over], q, [9])
