"""Where the e2e decode step (configs[1], N = 1) loses time against the device loop:
  device_pipelined  attn_decode_append back to back (the bench `value` loop)
  device_synced     the same call, stream synchronised after every step
  plan_synced       DecodePlan.step with pinned host buffers + synchronise (the bench `e2e` loop)
  plan_pipelined    DecodePlan.step back to back (host buffers, no per-step synchronise)
    python tools/e2e_anatomy.py"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
import paper_2409_17264_b200 as M

H_KV, H_Q, D, N = 8, 32, 128, 1 << 20
sh = bench.build_shard(M, 0, 1, N, H_KV, D)
L = sh.len - 1
k_new = synth.kv_block(bench.SEED, synth.STREAM_K, N - 1, 1, H_KV, D, device="cuda")
v_new = synth.kv_block(bench.SEED, synth.STREAM_V, N - 1, 1, H_KV, D, device="cuda")
q = synth.queries(bench.SEED, 1, H_Q, D, device="cuda", amp=4.0)
o = torch.empty((1, H_Q, D), device="cuda")
lse = torch.empty((1, H_Q), device="cuda")
ws = M.decode_workspace(1, H_Q, H_KV, D)
st = torch.cuda.current_stream()
q_h, k_h, v_h = q[0].cpu().pin_memory(), k_new[0].cpu().pin_memory(), v_new[0].cpu().pin_memory()
o_h = torch.empty((H_Q, D)).pin_memory()
l_h = torch.empty((H_Q,)).pin_memory()
sws = M.decode_step_workspace(1, H_Q, H_KV, D)
plan = M.DecodePlan(None, sh, q_h, k_h, v_h, o_h, l_h, sws)


def dev():
    sh.len = L
    M.attn_decode_append([sh], k_new, v_new, q, [N - 1], o=o, lse=lse, ws=ws)


def pl():
    sh.len = L
    plan.step(sh, True, N - 1, st)


res = {}
for name, fn, sync in (("device_pipelined", dev, False), ("device_synced", dev, True),
                       ("plan_synced", pl, True), ("plan_pipelined", pl, False), ("device_pipelined_again", dev, False)):
    for _ in range(5):
        fn()
        st.synchronize()
    host = 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(40):
        t = time.perf_counter()
        fn()
        host += time.perf_counter() - t
        if sync:
            st.synchronize()
    e1.record(st)
    torch.cuda.synchronize()
    res[name] = {"us_per_step": round(e0.elapsed_time(e1) / 40 * 1e3, 1), "host_us_per_call": round(host / 40 * 1e6, 1)}
plan.close()
print(json.dumps(res), flush=True)
