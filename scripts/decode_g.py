"""Decode kernel GB/s vs group size G on the same KV (same bytes, different G)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, bench
import paper_2409_17264_b200 as M
from decode_micro_helpers import timeit  # noqa
for n in (1 << 20, 10 * (1 << 20) // 8):
    sh = bench.build_shard(M, 0, 1, n, 8, 128)
    res = {}
    for G in (1, 2, 4, 8, 16):
        q = synth.queries(1, 1, 8 * G, 128, device="cuda", amp=4.0)
        o = torch.empty((1, 8 * G, 128), device="cuda"); l = torch.empty((1, 8 * G), device="cuda")
        ws = M.decode_workspace(1, 8 * G, 8, 128)
        t = timeit(lambda: M.attn_decode_partial([sh], q, [n - 1], o=o, lse=l, ws=ws))
        res[G] = (round(t, 1), round(n * 8 * 512 / t / 1e3, 1))
    print(json.dumps({"tokens": n, "G: (us, GB/s)": res}), flush=True)
    del sh; torch.cuda.empty_cache()
