"""Experiment: where the decode kernel's fixed per-launch cost goes (persistent item queue).
Needs a library built with -DMEDHA_DECODE_TRACE=1 (MEDHA_LIB_PATH=build/dtrace.so).
Per item: %globaltimer at item start / main-loop end / partial written / split merge done,
the CTA and the SM; per size, the launch's CUDA-event time against the traced span."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2409_17264_b200 as M  # noqa: E402

for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1048576,262144,131072").split(",")]:
    sh = bench.build_shard(M, 0, 1, n, 8, 128)
    q = synth.queries(1, 1, 32, 128, device="cuda", amp=4.0)
    o = torch.empty((1, 32, 128), device="cuda")
    lse = torch.empty((1, 32), device="cuda")
    ws = M.decode_workspace(1, 32, 8, 128)
    for _ in range(5):
        M.attn_decode_partial([sh], q, [n - 1], o=o, lse=lse, ws=ws)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    M.attn_decode_partial([sh], q, [n - 1], o=o, lse=lse, ws=ws)
    b.record()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (8192 * 8))()
    M.lib.medha_debug_decode_trace(buf)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 8).astype(np.int64)
    valid = t[:, 0] > 0
    last = t[valid, 0].max()
    it = t[valid & (t[:, 0] > last - 5_000_000)]          # items of the last launch (within 5 ms)
    t0 = it[:, 0].min()
    start = (it[:, 0] - t0) / 1e3
    loop_end = (it[:, 1] - t0) / 1e3
    part = (it[:, 2] - t0) / 1e3
    merge = (it[it[:, 3] > t0, 3] - t0) / 1e3
    dur = loop_end - start
    cta = it[:, 4]
    cta_end = {}
    for c, e in zip(cta, part):
        cta_end[c] = max(cta_end.get(c, 0), e)
    ends = np.array(sorted(cta_end.values()))
    span = max(part.max(), merge.max() if len(merge) else 0)
    print(json.dumps({
        "tokens": n, "items": int(len(it)), "ctas": int(len(cta_end)), "event_us": round(a.elapsed_time(b) * 1e3, 1),
        "traced_span_us": round(float(span), 2),
        "first_wave_start_us": [round(float(x), 2) for x in np.percentile(np.sort(start)[:len(cta_end)], [0, 50, 100])],
        "item_dur_us": [round(float(x), 2) for x in np.percentile(dur, [0, 10, 50, 90, 100])],
        "loop_to_partial_us": round(float(np.median(part - loop_end)), 2),
        "cta_last_end_us": [round(float(x), 2) for x in np.percentile(ends, [0, 10, 50, 90, 100])],
        "merge_done_us": [round(float(x), 2) for x in sorted(merge)[-4:]],
    }), flush=True)
    del sh
    torch.cuda.empty_cache()
