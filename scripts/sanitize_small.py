"""Tiny invocations of every kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch, synth
import paper_2409_17264_b200 as M
from helpers import make_global_kv, to_shard
for (N, h_kv, G, d) in [(4161, 1, 4, 64), (300, 2, 8, 128), (77, 1, 16, 128), (1000, 2, 1, 64)]:
    k, v = make_global_kv(1, N, h_kv, d)
    q = synth.queries(1, 3, h_kv * G, d, amp=4.0).cuda()
    sh = to_shard(k, v, 0, N, poison=False)
    M.attn_decode_partial([sh, sh, sh], q, [N - 1, N // 2, 0])
    c = min(64, N)
    M.attn_prefill_chunk(sh, synth.queries(2, c, h_kv * G, d).cuda(), N - c)
    M.attn_prefill_chunk(sh, synth.queries(2, 5, h_kv * G, d).cuda(), 0)
    sh2 = M.KVShard.empty(h_kv, 40, d)
    M.kv_append(sh2, k[:33].cuda(), v[:33].cuda())
    parts = torch.randn((3, 7 * (d + 1)), device="cuda")
    M.merge_partials(parts, 7, d, want_bf16=True)
    torch.cuda.synchronize()
print("sanitize OK")
