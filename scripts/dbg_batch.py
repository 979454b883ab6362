import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch, synth
import paper_2409_17264_b200 as M
from helpers import make_global_kv, to_shard
h_kv, G, d = 1, 4, 64
k, v = make_global_kv(77, 600, h_kv, d)
for B in (1, 2, 63, 64, 65, 70):
    q = synth.queries(77, B, h_kv * G, d, amp=4.0).cuda()
    lens = [10 + 7 * i for i in range(B)]
    shards = [to_shard(k, v, 0, n) for n in lens]
    o, l = M.attn_decode_partial(shards, q, [n - 1 for n in lens])
    o, l = o.clone(), l.clone()
    bad = []
    for i in range(B):
        o1, l1 = M.attn_decode_partial([shards[i]], q[i:i+1], [lens[i] - 1])
        if not torch.equal(o1[0], o[i]): bad.append((i, float((o1[0]-o[i]).abs().max())))
    print("B", B, "bad", bad[:8], len(bad), flush=True)
