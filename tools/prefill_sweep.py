"""Prefill-chunk TFLOP/s sweep (configs[2]) using bench.py's measurement code.
    python tools/prefill_sweep.py [prefixes] [chunks] [label]
MEDHA_LIB_PATH selects an experiment variant of the library (same-box A/B)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2409_17264_b200 as M
pre = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "131072,1048576").split(",")]
cs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "64,256,1024,4096").split(",")]
label = sys.argv[3] if len(sys.argv) > 3 else os.path.basename(M.LIB_PATH)
sh = bench.build_shard(M, 0, 1, max(pre) + max(cs), bench.H_KV, bench.D)
clk = bench.ClockSampler(torch.cuda.current_device()); clk.start()
res = bench.bench_prefill(M, sh, pre, cs, iters=10, warm=3)
c = clk.stop()
for r in res:
    r["lib"] = label
    print(json.dumps(r), flush=True)
print(json.dumps({"lib": label, "clocks": c}), flush=True)
