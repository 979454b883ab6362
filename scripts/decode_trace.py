"""Experiment: per-CTA timeline of the decode kernel (build/dtrace.so, MEDHA_DECODE_TRACE)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
import paper_2409_17264_b200 as M
for n in (1 << 20, 1 << 18, 1 << 17):
    sh = bench.build_shard(M, 0, 1, n, 8, 128)
    q = synth.queries(1, 1, 32, 128, device="cuda", amp=4.0)
    o = torch.empty((1, 32, 128), device="cuda"); l = torch.empty((1, 32), device="cuda")
    ws = M.decode_workspace(1, 32, 8, 128)
    for _ in range(5): M.attn_decode_partial([sh], q, [n - 1], o=o, lse=l, ws=ws)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); M.attn_decode_partial([sh], q, [n - 1], o=o, lse=l, ws=ws); b.record(); torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (8192 * 8))()
    M.lib.medha_debug_decode_trace(buf)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 8).astype(np.int64)
    used = t[:296]
    t0 = used[:, 0].min()
    st, loop, part = (used[:, 0] - t0) / 1e3, (used[:, 1] - t0) / 1e3, (used[:, 2] - t0) / 1e3
    fin = used[:, 3][used[:, 3] > t0]
    print(json.dumps({"tokens": n, "event_us": round(a.elapsed_time(b) * 1e3, 1),
        "start_us": [round(float(x), 2) for x in np.percentile(st, [0, 50, 100])],
        "loop_end_us": [round(float(x), 2) for x in np.percentile(loop, [0, 10, 50, 90, 100])],
        "partial_us": [round(float(x), 2) for x in np.percentile(part, [0, 50, 100])],
        "merge_done_us": [round(float((x - t0) / 1e3), 2) for x in sorted(fin)[-8:]]}), flush=True)
    del sh; torch.cuda.empty_cache()
