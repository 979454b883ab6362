"""Decode bandwidth vs GQA group size G (h_kv = 8, d = 128, 2^20 tokens, batch 1), same box.
    python tools/decode_g_sweep.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
import paper_2409_17264_b200 as M

H_KV, D, N = 8, 128, 1 << 20
sh = bench.build_shard(M, 0, 1, N, H_KV, D)
for G in (1, 2, 4, 8, 16):
    q = synth.queries(1, 1, H_KV * G, D, device="cuda", amp=4.0)
    o = torch.empty((1, H_KV * G, D), device="cuda")
    lse = torch.empty((1, H_KV * G), device="cuda")
    ws = M.decode_workspace(1, H_KV * G, H_KV, D)
    best = 1e9
    for rep in range(3):
        for _ in range(5):
            M.attn_decode_partial([sh], q, [N - 1], o=o, lse=lse, ws=ws)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(30):
            M.attn_decode_partial([sh], q, [N - 1], o=o, lse=lse, ws=ws)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 30)
    print(json.dumps({"G": G, "h_q": H_KV * G, "us": round(best * 1e3, 1), "GBps": round(N * H_KV * D * 4 / (best * 1e-3) / 1e9, 1)}), flush=True)
