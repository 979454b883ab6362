"""Prefill-prefill batching: n short chunks of different sequences
(each attending over its own 128K-token prefix) in one launch vs one launch per chunk."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2409_17264_b200 as M  # noqa: E402
from paper_2409_17264_b200 import accounting as acc  # noqa: E402

H_Q, H_KV, D = 32, 8, 128


def timeit(fn, iters=10, warm=3):
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


for P0, n, c in ((4096, 8, 64), (4096, 16, 256), (16384, 8, 128), (1 << 17, 8, 64), (1 << 17, 16, 64)):
    shards, qs = [], []
    for i in range(n):
        sh = M.KVShard.empty(H_KV, P0 + c, D)
        for t in range(0, P0 + c, synth.BLOCK_TOKENS):
            m = min(synth.BLOCK_TOKENS, P0 + c - t)
            sh.k[:, t:t + m] = synth.kv_block(100 + i, 1, t, m, H_KV, D, device="cuda").permute(1, 0, 2)
            sh.v[:, t:t + m] = synth.kv_block(100 + i, 2, t, m, H_KV, D, device="cuda").permute(1, 0, 2)
        sh.len = P0 + c
        shards.append(sh)
        qs.append(synth.queries(200 + i, c, H_Q, D, device="cuda", t0=P0))
    fl = n * acc.prefill_chunk_flops(c, P0, H_Q, D)
    t_sep = timeit(lambda: [M.attn_prefill_chunk(shards[i], qs[i], P0) for i in range(n)])
    t_bat = timeit(lambda: M.attn_prefill_batch(shards, qs, [P0] * n))
    print(json.dumps({"chunks": n, "c": c, "prefix": P0, "separate_ms": round(t_sep, 4), "batched_ms": round(t_bat, 4),
                      "separate_tflops": round(fl / t_sep / 1e9, 1), "batched_tflops": round(fl / t_bat / 1e9, 1),
                      "speedup": round(t_sep / t_bat, 3)}), flush=True)
    del shards, qs
    torch.cuda.empty_cache()
