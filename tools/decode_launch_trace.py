"""Experiment: where a pipelined decode step's time goes between kernels (needs a library built
with -DMEDHA_DECODE_TRACE=1, MEDHA_LIB_PATH=build/dtrace.so).  Runs `steps` back-to-back steps
of (kv_append of one token + decode) as bench.py does and prints, per step, %globaltimer
offsets (us): previous decode's last CTA out -> kv_append past its wait -> decode CTA 0
resident -> CTA 0 past griddepcontrol.wait -> last CTA out; plus the CUDA-event step time."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench, synth
import paper_2409_17264_b200 as M
steps = 20
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1048576,262144,131072").split(",")]:
    sh = bench.build_shard(M, 0, 1, n, 8, 128, extra_cap=steps + 8)
    q = synth.queries(1, 1, 32, 128, device="cuda", amp=4.0)
    kn = torch.randn(1, 8, 128, device="cuda").to(torch.bfloat16)
    o = torch.empty((1, 32, 128), device="cuda")
    lse = torch.empty((1, 32), device="cuda")
    ws = M.decode_workspace(1, 32, 8, 128)
    base = sh.len

    def step():
        sh.len = base
        M.kv_append(sh, kn, kn)
        M.attn_decode_partial([sh], q, [sh.len - 1], o=o, lse=lse, ws=ws)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (64 * 4))()
    cnt = ctypes.c_uint(0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    M.lib.medha_debug_launch_trace(buf, ctypes.byref(cnt))
    n0 = cnt.value
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    M.lib.medha_debug_launch_trace(buf, ctypes.byref(cnt))
    t = np.frombuffer(buf, dtype=np.uint64).reshape(64, 4).astype(np.int64)
    idx = [(n0 + i) % 64 for i in range(steps)]
    prev_end = [t[(n0 + i - 1) % 64, 2] for i in range(steps)]
    rows = []
    for i, k in enumerate(idx):
        pe = prev_end[i]
        rows.append([(t[k, 3] - pe) / 1e3, (t[k, 0] - pe) / 1e3, (t[k, 1] - pe) / 1e3, (t[k, 2] - pe) / 1e3])
    r = np.median(np.array(rows[1:]), axis=0)
    print(json.dumps({"tokens": n, "event_step_us": round(a.elapsed_time(b) * 1e3 / steps, 2),
                      "median_us_after_prev_decode_end": {"kv_append_past_wait": round(r[0], 2),
                      "decode_cta0_resident": round(r[1], 2), "decode_cta0_past_wait": round(r[2], 2),
                      "decode_last_cta_out (= step period)": round(r[3], 2)}}), flush=True)
    del sh
    torch.cuda.empty_cache()
