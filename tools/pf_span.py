"""Experiment: where a pipelined prefill call's time goes outside CTA 0's KV loop (needs a library
built with -DMEDHA_PF_TRACE=1).  20 back-to-back calls; for the last: %globaltimer of CTA 0 at
entry, past griddepcontrol.wait, S_A(0) seen, last P stored, outputs stored, and the SM clock
over the loop; beside the per-call period from CUDA events."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
import paper_2409_17264_b200 as M
for P0, c in ((131072, 64), (131072, 256), (131072, 1024)):
    sh = bench.build_range(M, 0, P0 + c, 8, 128)
    q = synth.queries(3, c, 32, 128, device="cuda")
    o = torch.empty((c, 32, 128), device="cuda")
    lse = torch.empty((c, 32), device="cuda")
    for _ in range(3):
        M.attn_prefill_chunk(sh, q, P0, o=o, lse=lse)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        M.attn_prefill_chunk(sh, q, P0, o=o, lse=lse)
    b.record()
    torch.cuda.synchronize()
    g = (ctypes.c_longlong * 8)()
    M.lib.medha_debug_pf_gtimer(g)
    t = list(g)
    period = a.elapsed_time(b) / 20 * 1e3
    mhz = (t[6] - t[5]) / max(1, (t[3] - t[2])) * 1e3
    print(f"P0={P0} c={c}: period {period:.1f} us | CTA0: entry->past wait {(t[1]-t[0])/1e3:.2f}, ->S_A(0) {(t[2]-t[1])/1e3:.2f}, "
          f"loop {(t[3]-t[2])/1e3:.1f}, ->outputs stored {(t[4]-t[3])/1e3:.2f} us; SM clock in loop {mhz:.0f} MHz", flush=True)
