"""torchrun worker for the multi-GPU KVP parity test (tests/test_gpu_kvp_multi.py).

Every rank holds a contiguous slice of one global KV, receives the same
queries and runs the C-ABI KVP calls (local partial, NCCL all-gather,
rank-ordered merge).  Checks: outputs bit-identical on all ranks (R13),
within 1e-3 of the single-GPU fp32 result, and within the north_star tolerance of
the fp64 oracle; the e2e host-buffer call agrees with the device call.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import synth
    import paper_2409_17264_b200 as M
    from paper_2409_17264_b200.kvp import shard_range
    from helpers import compare, oracle_attention, to_shard

    N, h_kv, G, d = 200_000, 8, 4, 128
    k, v = synth.kv_block(11, synth.STREAM_K, 0, N, h_kv, d), synth.kv_block(11, synth.STREAM_V, 0, N, h_kv, d)
    a, b = shard_range(N, rank, world)
    sh = to_shard(k, v, a, b)
    comm = M.KVPComm()
    fails = []

    def allsame(t, what):
        g = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(g, t.contiguous())
        if not all(torch.equal(g[0], x) for x in g):
            fails.append(f"{what}: ranks differ")

    # ---- decode: Eq. 5 (fused NVLink exchange when available, and the NCCL path) -------
    q = synth.queries(11, 2, h_kv * G, d, amp=8.0)
    qp = [N - 1, N // 3]
    p2p = comm.p2p
    if world > 1 and not p2p:
        fails.append("fused P2P exchange did not initialise")
    if p2p:
        comm.set_p2p(False)
        o_n, lse_n, _ = M.kvp_decode(comm, [sh, sh], q.cuda(), qp)
        o_n, lse_n = o_n.clone(), lse_n.clone()
        comm.set_p2p(True)
        for _ in range(3):          # several epochs through the double-buffered slots
            o, lse, ob = M.kvp_decode(comm, [sh, sh], q.cuda(), qp, want_bf16=True)
        torch.cuda.synchronize()
        if (o - o_n).abs().max().item() > 1e-6 or (lse - lse_n).abs().max().item() > 1e-6:
            fails.append(f"p2p vs nccl exchange differ: {(o - o_n).abs().max().item()}")
    o, lse, ob = M.kvp_decode(comm, [sh, sh], q.cuda(), qp, want_bf16=True)
    torch.cuda.synchronize()
    allsame(o, "kvp_decode o")
    allsame(lse, "kvp_decode lse")
    if not torch.equal(ob, o.to(torch.bfloat16)):
        fails.append("bf16 output is not RNE of fp32 output")
    whole = to_shard(k, v, 0, N)
    o1, l1 = M.attn_decode_partial([whole, whole], q.cuda(), qp)
    dmax = (o - o1).abs().max().item()
    if dmax > 1e-3 or (lse - l1).abs().max().item() > 1e-3:
        fails.append(f"kvp vs single gpu {dmax}")
    if rank == 0:
        ro, rl = oracle_attention(q[:, :2 * G], k[:, :2], v[:, :2], qp)   # kv heads 0,1 (8 q heads)
        try:
            compare(o[:, :2 * G], lse[:, :2 * G], ro, rl, what=f"kvp_decode P={world}")
        except AssertionError as e:
            fails.append(str(e))

    # ---- e2e host-buffer step (decode_step_host) agrees with the device call ----------
    ws = M.decode_step_workspace(world, h_kv * G, h_kv, d)
    o_h = torch.empty((h_kv * G, d), dtype=torch.float32).pin_memory()
    l_h = torch.empty((h_kv * G,), dtype=torch.float32).pin_memory()
    tail = rank == world - 1
    sh_t = to_shard(k, v, a, b - 1 if tail else b)
    M.decode_step_host(comm, sh_t, tail, q[0].contiguous().pin_memory(),
                       k[N - 1].contiguous().pin_memory() if tail else None,
                       v[N - 1].contiguous().pin_memory() if tail else None, N - 1, o_h, l_h, ws)
    torch.cuda.synchronize()
    # (the batch-2 call above planned its KV splits for two sequences: fp32 summation order differs)
    if (o_h - o[0].cpu()).abs().max().item() > 1e-4:
        fails.append(f"decode_step_host differs from kvp_decode: {(o_h - o[0].cpu()).abs().max().item()}")

    # ---- prefill chunk under KVP: Eq. 6 ------------------------------------------------
    c = 256
    qc = synth.queries(12, c, h_kv * G, d, amp=6.0)
    op, lp, _ = M.kvp_prefill_chunk(comm, sh, qc.cuda(), N - c)
    torch.cuda.synchronize()
    allsame(op, "kvp_prefill o")
    o1p, l1p = M.attn_prefill_chunk(whole, qc.cuda(), N - c)
    dmax = (op - o1p).abs().max().item()
    if dmax > 1e-3 or (lp - l1p).abs().max().item() > 1e-3:
        fails.append(f"kvp prefill vs single gpu {dmax}")
    if rank == 0:
        rows = [0, 100, 255]
        ro, rl = oracle_attention(qc[rows][:, :G], k[:, :1], v[:, :1], [N - c + r for r in rows])
        try:
            compare(op[rows][:, :G], lp[rows][:, :G], ro, rl, what=f"kvp_prefill P={world}")
        except AssertionError as e:
            fails.append(str(e))

    comm.close()
    flag = torch.tensor([len(fails)], device="cuda")
    dist.all_reduce(flag)
    if fails:
        print(f"rank {rank} FAIL: {fails}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if flag.item() else 0)


if __name__ == "__main__":
    main()
