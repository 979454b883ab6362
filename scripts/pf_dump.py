"""Dump prefill-chunk outputs of the loaded library (MEDHA_LIB_PATH selects a variant) for a
bit-for-bit comparison between kernel variants:  python scripts/pf_dump.py OUT.pt"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import synth
import paper_2409_17264_b200 as M
out = {}
sh = bench.build_range(M, 0, 131072 + 4096, 8, 128)
for amp in (1.0, 6.0):                 # amp 6: peaked logits, the max grows often (redo path)
    for P0, c in ((0, 300), (4096, 64), (65536, 1024), (131072 - 2048, 2048), (131072, 4096)):
        q = synth.queries(7, c, 32, 128, amp=amp).cuda()
        sh.len = P0 + c
        o, l = M.attn_prefill_chunk(sh, q, P0)
        out[(amp, P0, c)] = (o.cpu(), l.cpu())
torch.cuda.synchronize()
torch.save(out, sys.argv[1])
print("dumped", len(out), "cases to", sys.argv[1])
