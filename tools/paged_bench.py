"""Paged vs contiguous KV: 8B decode over 2^20 tokens and a c = 1024 prefill chunk
over a 128K prefix, with the pages in a random order, on one GPU."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2409_17264_b200 as M  # noqa: E402
from paper_2409_17264_b200 import accounting as acc  # noqa: E402

H_Q, H_KV, D = 32, 8, 128


def timeit(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def contiguous(n):
    sh = M.KVShard.empty(H_KV, n, D)
    for t in range(0, n, synth.BLOCK_TOKENS):
        m = min(synth.BLOCK_TOKENS, n - t)
        sh.k[:, t:t + m] = synth.kv_block(1, 1, t, m, H_KV, D, device="cuda").permute(1, 0, 2)
        sh.v[:, t:t + m] = synth.kv_block(1, 2, t, m, H_KV, D, device="cuda").permute(1, 0, 2)
    sh.len = n
    return sh


def paged_copy(sh, ps, seed=0):
    """The same tokens in a pool whose pages are a random permutation."""
    n_pages = (sh.len + ps - 1) // ps
    g = torch.Generator().manual_seed(seed)
    perm = torch.randperm(n_pages, generator=g).to(torch.int32)
    pk = torch.zeros((H_KV, n_pages * ps, D), dtype=torch.bfloat16, device="cuda")
    pv = torch.zeros_like(pk)
    src = torch.arange(n_pages * ps, device="cuda").clamp_max(sh.len - 1)
    dst = (perm.cuda().long()[:, None] * ps + torch.arange(ps, device="cuda")[None]).reshape(-1)
    keep = torch.arange(n_pages * ps, device="cuda") < sh.len
    pk[:, dst[keep]] = sh.k[:, src[keep]]
    pv[:, dst[keep]] = sh.v[:, src[keep]]
    return M.KVShard.paged(pk, pv, perm.cuda(), ps, sh.len, sh.pos0)


n = 1 << 20
sh = contiguous(n)
q = synth.queries(1, 1, H_Q, D, device="cuda", amp=4.0)
by = acc.decode_bytes(n, H_KV, D)
o_c, l_c = M.attn_decode_partial([sh], q, [n - 1])
t_c = timeit(lambda: M.attn_decode_partial([sh], q, [n - 1]))
print(json.dumps({"op": "decode", "layout": "contiguous", "ms": round(t_c, 4), "GBps": round(by / t_c / 1e6, 1)}), flush=True)
for ps in (16, 64, 256, 4096):
    pg = paged_copy(sh, ps)
    o_p, l_p = M.attn_decode_partial([pg], q, [n - 1])
    same = bool(torch.equal(o_p, o_c) and torch.equal(l_p, l_c))
    t_p = timeit(lambda: M.attn_decode_partial([pg], q, [n - 1]))
    print(json.dumps({"op": "decode", "layout": f"paged ps={ps}", "ms": round(t_p, 4), "GBps": round(by / t_p / 1e6, 1),
                      "bit_identical": same}), flush=True)
    del pg
    torch.cuda.empty_cache()

P0, c = 1 << 17, 1024
sh.len = P0 + c
qp = synth.queries(8, c, H_Q, D, device="cuda", t0=P0)
fl = acc.prefill_chunk_flops(c, P0, H_Q, D)
o_c, l_c = M.attn_prefill_chunk(sh, qp, P0)
t_c = timeit(lambda: M.attn_prefill_chunk(sh, qp, P0), iters=10, warm=3)
print(json.dumps({"op": "prefill c=1024 @128K", "layout": "contiguous", "ms": round(t_c, 4),
                  "tflops": round(fl / t_c / 1e9, 1)}), flush=True)
for ps in (128, 1024):
    pg = paged_copy(sh, ps)
    o_p, l_p = M.attn_prefill_chunk(pg, qp, P0)
    same = bool(torch.equal(o_p, o_c) and torch.equal(l_p, l_c))
    t_p = timeit(lambda: M.attn_prefill_chunk(pg, qp, P0), iters=10, warm=3)
    print(json.dumps({"op": "prefill c=1024 @128K", "layout": f"paged ps={ps}", "ms": round(t_p, 4),
                      "tflops": round(fl / t_p / 1e9, 1), "bit_identical": same}), flush=True)
    del pg
    torch.cuda.empty_cache()
