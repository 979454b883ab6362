"""Experiment (torchrun): where the multi-GPU KVP decode step spends the time beyond the
per-rank decode kernel.  Every variant runs 30 back-to-back steps (CUDA events, max over
ranks): the rank-local decode alone, + kv_append on the tail rank, the fused-exchange
KVP decode with and without the append (two launches, or one with medha_kvp_decode_append),
and the NCCL all-gather path.  KVP_TOKENS sets the global KV length (default 2^20)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2409_17264_b200 as M  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
N = int(os.environ.get("KVP_TOKENS", 1 << 20))
H_Q, H_KV, D = 32, 8, 128
sh = bench.build_shard(M, rank, world, N, H_KV, D)
tail = rank == world - 1
q = synth.queries(1, 1, H_Q, D, device="cuda", amp=4.0)
k_new = synth.kv_block(1, 1, N - 1, 1, H_KV, D, device="cuda")
v_new = synth.kv_block(1, 2, N - 1, 1, H_KV, D, device="cuda")
len_before = sh.len - 1 if tail else sh.len
comm = M.KVPComm()
o = torch.empty((1, H_Q, D), device="cuda")
lse = torch.empty((1, H_Q), device="cuda")
dws = M.decode_workspace(1, H_Q, H_KV, D)
kws = M.kvp_workspace(world, 1, H_Q, H_KV, D)
xws = M.exchange_workspace(world, H_Q, D)
parts = torch.empty(H_Q * (D + 1), device="cuda")


def append():
    if tail:
        sh.len = len_before
        M.kv_append(sh, k_new, v_new)


def local():
    M.attn_decode_partial([sh], q, [N - 1], o=o, lse=lse, ws=dws)


def local_append():
    append()
    local()


def fused():
    M.kvp_decode(comm, [sh], q, [N - 1], ws=kws, o=o, lse=lse)


def fused_append():
    append()
    fused()


def fused_append_one_launch():
    # the tail rank's append rides in the decode launch (medha_kvp_decode_append)
    if tail:
        sh.len = len_before
    M.kvp_decode_append(comm, [sh], k_new, v_new, q, [N - 1], append=[tail], ws=kws, o=o, lse=lse)


def nccl():
    M.attn_decode_partial([sh], q, [N - 1], o=parts[:H_Q * D].view(1, H_Q, D), lse=parts[H_Q * D:].view(1, H_Q), ws=dws)
    M.kvp_exchange_merge(comm, parts, H_Q, D, o, lse, ws=xws)


def timed(fn, iters=30, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / iters
    allv = [None] * world
    dist.all_gather_object(allv, round(us, 1))
    return allv


res = {"world": world, "tokens": N}
for name, fn in (("local", local), ("local+append", local_append), ("fused", fused), ("fused+append", fused_append),
                 ("fused_append_1launch", fused_append_one_launch)):
    res[name] = timed(fn)
comm.set_p2p(False)
res["nccl"] = timed(nccl)
comm.set_p2p(True)
res["fused_again"] = timed(fused)
if rank == 0:
    print(json.dumps(res), flush=True)
comm.close()
dist.destroy_process_group()
