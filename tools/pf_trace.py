"""Experiment: hand-off timeline of the prefill kernel's CTA 0 (needs a library built with
-DMEDHA_PF_TRACE=1, MEDHA_LIB_PATH=build/pftrace.so).  clock64 stamps per KV tile j:
softmax X in {A, B}: S_X(j) seen, S row loaded, row max done, P stored (just before arrive);
MMA warp: P_A(j) seen, P_B(j) seen, K(j+1) ready (just before S_A(j+1) is issued)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench, synth
import paper_2409_17264_b200 as M
for P0, c in ((131072, 64), (131072, 1024)):
    sh = bench.build_range(M, 0, P0 + c, 8, 128)
    q = synth.queries(3, c, 32, 128, device="cuda")
    for _ in range(3):
        M.attn_prefill_chunk(sh, q, P0)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * (512 * 12))()
    M.lib.medha_debug_pf_trace(buf)
    t = np.frombuffer(buf, dtype=np.int64).reshape(512, 12).copy()
    n = int((t[:, 0] > 0).sum())
    t = t[:n]
    t0 = t[0, 0]
    print(f"P0={P0} c={c}: {n} tiles traced; columns relative to S_A(0) seen, SM cycles")
    print(" j | A:S seen  ld  max  P done | B:S seen  ld  max  P done | MMA:P_A seen P_B seen | cycleA  D_A  D_B  ld  max  exp")
    for j in list(range(min(n, 6))) + list(range(n // 2, n // 2 + 6)):
        r = t[j] - t0
        cyc = (t[j + 1, 0] - t[j, 0]) if j + 1 < n else 0
        print(f"{j:3d} | {r[0]:8d} {r[1]-r[0]:4d} {r[2]-r[1]:4d} {r[3]-r[2]:5d} | {r[4]:8d} {r[5]-r[4]:4d} {r[6]-r[5]:4d} {r[7]-r[6]:5d} |"
              f" {r[8]-r[3]:5d} {r[9]-r[7]:5d} | {cyc:6d} {r[3]-r[0]:5d} {r[7]-r[4]:5d}")
    mid = t[2:n - 2]
    cyc = np.diff(t[2:n - 1, 0])
    print("median: cycle %d  D_A %d  D_B %d  ld %d  max %d  exp+store %d  A->MMA %d  B->MMA %d  B-start minus A-start %d" % (
        np.median(cyc), np.median(mid[:, 3] - mid[:, 0]), np.median(mid[:, 7] - mid[:, 4]),
        np.median(mid[:, 1] - mid[:, 0]), np.median(mid[:, 2] - mid[:, 1]), np.median(mid[:, 3] - mid[:, 2]),
        np.median(mid[:, 8] - mid[:, 3]), np.median(mid[:, 9] - mid[:, 7]), np.median(mid[:, 4] - mid[:, 0])))
    # S_A(j+1) seen minus P_A(j) seen by the MMA warp = PV_A(j) + S_A(j+1) on the tensor pipe (+ queueing behind B)
    span = int(max(t[n - 1, 3], t[n - 1, 7]) - t[0, 0])
    a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a_ev.record()
    M.attn_prefill_chunk(sh, q, P0)
    b_ev.record()
    torch.cuda.synchronize()
    print("loop span of CTA 0 (S_A(0) seen -> last P stored): %d clk; one call (prefill + split merge) %.1f us" % (
        span, a_ev.elapsed_time(b_ev) * 1e3))
    print("median S_A(j+1) seen - P_A(j) seen by MMA: %d ; S_B(j+1) seen - P_B(j) seen: %d" % (
        np.median(t[3:n - 1, 0] - t[2:n - 2, 8]), np.median(t[3:n - 1, 4] - t[2:n - 2, 9])))
