"""Experiment (torchrun): per-CTA timeline of the fused KVP decode (build/dtrace.so)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
import bench, synth
import paper_2409_17264_b200 as M
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank); dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
sh = bench.build_shard(M, rank, world, 1 << 20, 8, 128)
q = synth.queries(1, 1, 32, 128, device="cuda", amp=4.0)
comm = M.KVPComm()
o = torch.empty((1, 32, 128), device="cuda"); l = torch.empty((1, 32), device="cuda")
ws = M.kvp_workspace(world, 1, 32, 8, 128)
for it in range(6):
    dist.barrier(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); M.kvp_decode(comm, [sh], q, [(1 << 20) - 1], ws=ws, o=o, lse=l); b.record(); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (8192 * 8))()
M.lib.medha_debug_decode_trace(buf)
t = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 8).astype(np.int64)[:300]
t0 = t[t[:, 0] > 0, 0].min()
rel = lambda c: sorted(((t[t[:, c] > 0, c] - t0) / 1e3).round(2).tolist())
out = {"rank": rank, "event_us": round(a.elapsed_time(b) * 1e3, 1), "loop_end_max": rel(1)[-1], "partial_max": rel(2)[-1],
       "split_merged(3)": rel(3)[-8:] if rel(3) else None, "pushed(4)": rel(4)[-8:], "fenced(5)": rel(5)[-8:], "flags_seen(6)": rel(6)[-8:]}
print(json.dumps(out), flush=True)
comm.close(); dist.destroy_process_group()
