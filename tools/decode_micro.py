"""Decode kernel time vs shard size (fixed-cost fit) and, under torchrun, the cost of
the KVP exchange (NCCL all-gather + merge) alone."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import bench
import paper_2409_17264_b200 as M

world = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))))

def timeit(fn, iters=50, warm=5):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3   # us

H_Q, H_KV, D = 32, 8, 128
q = synth.queries(1, 1, H_Q, D, device="cuda", amp=4.0)
res = {}
if rank == 0:
    sh = bench.build_shard(M, 0, 1, 1 << 20, H_KV, D)
    o = torch.empty((1, H_Q, D), device="cuda"); l = torch.empty((1, H_Q), device="cuda")
    ws = M.decode_workspace(1, H_Q, H_KV, D)
    for n in (4096, 16384, 65536, 131072, 262144, 524288, 1048576):
        sh.len = n
        t = timeit(lambda: M.attn_decode_partial([sh], q, [n - 1], o=o, lse=l, ws=ws))
        res[n] = round(t, 2)
    print(json.dumps({"decode_us_vs_tokens": res}), flush=True)
    del sh
if world > 1:
    comm = M.KVPComm()
    rows = H_Q
    send = torch.randn(rows * (D + 1), device="cuda")
    oo = torch.empty((rows, D), device="cuda"); ll = torch.empty((rows,), device="cuda")
    xws = M.exchange_workspace(world, rows, D)
    t = timeit(lambda: M.kvp_exchange_merge(comm, send, rows, D, oo, ll, ws=xws), iters=200, warm=20)
    tt = torch.tensor([t], device="cuda"); dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    if rank == 0: print(json.dumps({"world": world, "exchange_merge_us": round(tt.item(), 2)}), flush=True)
    comm.close()
    dist.destroy_process_group()
