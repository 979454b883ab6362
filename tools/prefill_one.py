"""Run one chunked-prefill configuration a few times (for ncu captures)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2409_17264_b200 as M

ap = argparse.ArgumentParser()
ap.add_argument("--prefix", type=int, default=1 << 17)
ap.add_argument("--c", type=int, default=1024)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--hq", type=int, default=32)
a = ap.parse_args()
H_KV, D = 8, 128
n = a.prefix + a.c
sh = M.KVShard.empty(H_KV, n, D)
for t in range(0, n, 65536):
    m = min(65536, n - t)
    sh.k[:, t:t + m] = synth.kv_block(1, 1, t, m, H_KV, D, device="cuda").permute(1, 0, 2)
    sh.v[:, t:t + m] = synth.kv_block(1, 2, t, m, H_KV, D, device="cuda").permute(1, 0, 2)
sh.len = n
q = synth.queries(8, a.c, a.hq, D, device="cuda")
for _ in range(a.iters):
    o, l = M.attn_prefill_chunk(sh, q, a.prefix)
torch.cuda.synchronize()
print("ok", float(o.abs().mean()))
