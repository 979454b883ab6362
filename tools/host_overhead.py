"""Experiment: host-side cost of one decode_step_host call (the e2e path), split into Python
marshalling, cudaPointerGetAttributes and the rest of the C call; GPU time per step beside it."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
import paper_2409_17264_b200 as M
N = 1 << 17
sh = bench.build_shard(M, 0, 1, N, 8, 128, extra_cap=8)
q_h = synth.queries(1, 1, 32, 128).contiguous()[0].pin_memory()
k_h = torch.randn(8, 128).to(torch.bfloat16).pin_memory()
o_h = torch.empty((32, 128)).pin_memory()
l_h = torch.empty(32).pin_memory()
ws = M.decode_step_workspace(1, 32, 8, 128)
base = sh.len
def call():
    sh.len = base
    M.decode_step_host(None, sh, True, q_h, k_h, k_h, base, o_h, l_h, ws)
for _ in range(20):
    call()
torch.cuda.synchronize()
n = 200
t = time.perf_counter()
for _ in range(n):
    call()
host_us = (time.perf_counter() - t) / n * 1e6
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(n):
    call()
    torch.cuda.current_stream().synchronize()
step_us = (time.perf_counter() - t) / n * 1e6
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
attr_us = None
if rt is not None:
    buf = ctypes.create_string_buffer(64)
    t = time.perf_counter()
    for _ in range(2000):
        rt.cudaPointerGetAttributes(buf, ctypes.c_void_p(q_h.data_ptr()))
    attr_us = (time.perf_counter() - t) / 2000 * 1e6
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(n):
    sh.len = base
    M.kv_append(sh, k_h.cuda(), k_h.cuda()) if False else None
    M.attn_decode_partial([sh], q_h.cuda()[None], [base], )
b.record(); torch.cuda.synchronize()
print({"host_us_per_call_async": round(host_us, 2), "synced_step_us": round(step_us, 2),
       "cudaPointerGetAttributes_us": attr_us and round(attr_us, 3), "gpu_decode_us": round(a.elapsed_time(b) / n * 1e3, 2)})
