"""torchrun worker: SURVEY §8(f) next items on real GPUs.

* N3 dynamic KVP growth: a sequence grows chunk by chunk with a per-worker
  token limit, so the set of ranks holding tokens grows 1 -> world; after every chunk a
  KVP prefill over the current chunk and a KVP decode of the next token are checked
  against the single-GPU result (1e-3, fp32) and for bit-identity across ranks.
* N4 KVP x TP, world 4: TP = 2 head slices x KVP = 2 sequence shards; each TP
  slice has its own KVP communicator (torch.distributed sub-group); the concatenated heads
  equal the single-GPU result.
* N1 / N2 across GPUs: the one-launch KVP step (medha_kvp_decode_append, the tail rank
  appends) equals append + kvp_decode; medha_kvp_decode captured in a CUDA graph on every
  rank replays with fresh queries (device-resident epoch) and matches the eager call; and
  when one rank withholds its pushes (test hook) every rank's bounded wait expires, the
  communicator reports MEDHA_ENCCL everywhere and nothing hangs.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import synth
    import paper_2409_17264_b200 as M
    from paper_2409_17264_b200.kvp import KVPGrowingSequence, shard_range
    from helpers import to_shard

    fails = []
    h_kv, G, d = 8, 4, 128

    def allsame(t, what):
        g = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(g, t.contiguous())
        if not all(torch.equal(g[0], x) for x in g):
            fails.append(f"{what}: ranks differ")

    # ---------------- N3: dynamic KVP growth --------------------------------------------
    comm = M.KVPComm()
    L = 3000                                     # per-worker token limit
    seq = KVPGrowingSequence(rank, world, L, h_kv, d)
    total = L * world - 1
    k_all = synth.kv_block(31, synth.STREAM_K, 0, total, h_kv, d).cuda()
    v_all = synth.kv_block(31, synth.STREAM_V, 0, total, h_kv, d).cuda()
    chunk = 1200
    for a in range(0, total - 1, chunk):
        b = min(total - 1, a + chunk)
        seq.append(k_all[a:b], v_all[a:b])
        qc = synth.queries(32, b - a, h_kv * G, d, amp=4.0, t0=a).cuda()
        op, lp, _ = M.kvp_prefill_chunk(comm, seq.shard, qc, a)
        seq.append(k_all[b:b + 1], v_all[b:b + 1])          # the decode token
        qd = synth.queries(33, 1, h_kv * G, d, amp=4.0, t0=b).cuda()
        od, ld, _ = M.kvp_decode(comm, [seq.shard], qd, [b])
        torch.cuda.synchronize()
        allsame(op, f"growth prefill @{a}")
        allsame(od, f"growth decode @{b}")
        whole = to_shard(k_all.cpu(), v_all.cpu(), 0, b + 1)
        o1p, l1p = M.attn_prefill_chunk(whole, qc, a)
        o1d, l1d = M.attn_decode_partial([whole], qd, [b])
        ep = (op - o1p).abs().max().item()
        ed = (od - o1d).abs().max().item()
        if ep > 1e-3 or ed > 1e-3 or (ld - l1d).abs().max().item() > 1e-3:
            fails.append(f"growth @{b} (workers {seq.active_workers}): prefill {ep} decode {ed}")
        # roll the decode token back into the stream (next chunk starts at b)
        seq.n -= 1
        if seq.shard.pos0 <= b < seq.shard.pos0 + seq.shard.len:
            seq.shard.len -= 1
    if seq.active_workers != world:
        fails.append(f"growth reached {seq.active_workers} workers, expected {world}")
    comm.close()

    # ---------------- one-launch step, graph replay, bounded wait --------------------------
    N = 120_000
    a0, b0 = shard_range(N, rank, world)
    tail = rank == world - 1
    kg = synth.kv_block(51, synth.STREAM_K, 0, N, h_kv, d)
    vg = synth.kv_block(51, synth.STREAM_V, 0, N, h_kv, d)
    comm = M.KVPComm()
    if not comm.p2p:
        fails.append("fused exchange not initialised")
    sh_a = to_shard(kg, vg, a0, b0 - 1 if tail else b0, extra_cap=4)
    sh_b = to_shard(kg, vg, a0, b0 - 1 if tail else b0, extra_cap=4)
    kn, vn = kg[N - 1:N].cuda(), vg[N - 1:N].cuda()
    qd = synth.queries(52, 1, h_kv * G, d, amp=6.0).cuda()
    o1, l1, _ = M.kvp_decode_append(comm, [sh_a], kn, vn, qd, [N - 1], append=[tail])
    if tail:
        M.kv_append(sh_b, kn, vn)
    o2, l2, _ = M.kvp_decode(comm, [sh_b], qd, [N - 1])
    torch.cuda.synchronize()
    if (o1 - o2).abs().max().item() > 1e-6:
        fails.append(f"kvp_decode_append vs append + kvp_decode: {(o1 - o2).abs().max().item()}")
    allsame(o1, "kvp_decode_append")
    # CUDA graph replay (every rank replays the same number of times)
    ws = torch.zeros(M.lib.medha_kvp_workspace_size(world, 1, h_kv * G, h_kv, d), dtype=torch.uint8, device="cuda")
    q_st = torch.zeros_like(qd)
    og = torch.empty_like(o1)
    lg = torch.empty_like(l1)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        M.kvp_decode(comm, [sh_b], q_st, [N - 1], ws=ws, o=og, lse=lg)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        M.kvp_decode(comm, [sh_b], q_st, [N - 1], ws=ws, o=og, lse=lg)
    for t in range(4):
        qt = synth.queries(60 + t, 1, h_kv * G, d, amp=6.0).cuda()
        q_st.copy_(qt)
        g.replay()
        torch.cuda.synchronize()
        oe, le, _ = M.kvp_decode(comm, [sh_b], qt, [N - 1])
        torch.cuda.synchronize()
        if not (torch.equal(og, oe) and torch.equal(lg, le)):
            fails.append(f"graph replay {t} differs from eager kvp_decode")
    del g
    dist.barrier()
    # bounded wait: rank 0 withholds its pushes, everybody must time out and report
    comm.set_timeout(0.1)
    if rank == 0:
        comm.debug(1)
    ot, lt, _ = M.kvp_decode(comm, [sh_b], qd, [N - 1])
    torch.cuda.synchronize()
    if comm.status() != -7:
        fails.append(f"rank {rank}: status {comm.status()} after a withheld push (expected MEDHA_ENCCL)")
    try:
        M.kvp_decode(comm, [sh_b], qd, [N - 1])
        fails.append("a broken communicator accepted another call")
    except M.MedhaError:
        pass
    comm.close()
    dist.barrier()

    # ---------------- N4: KVP x TP (world 4: 2 x 2) --------------------------------------
    if world == 4:
        tp, kvp = 2, 2
        t, r = rank // kvp, rank % kvp                    # TP slice, KVP rank in the slice
        groups = [dist.new_group([tt * kvp + rr for rr in range(kvp)]) for tt in range(tp)]
        comm2 = M.KVPComm(groups[t])
        N = 50_000
        heads = list(range(t * h_kv // tp, (t + 1) * h_kv // tp))
        k = synth.kv_block(41, synth.STREAM_K, 0, N, h_kv, d)
        v = synth.kv_block(41, synth.STREAM_V, 0, N, h_kv, d)
        q = synth.queries(41, 1, h_kv * G, d, amp=6.0)
        a, b = shard_range(N, r, kvp)
        sh = to_shard(k[:, heads].contiguous(), v[:, heads].contiguous(), a, b)
        q_loc = q[:, heads[0] * G:(heads[-1] + 1) * G].contiguous().cuda()
        o, lse, _ = M.kvp_decode(comm2, [sh], q_loc, [N - 1])
        whole = to_shard(k, v, 0, N)
        o1, l1 = M.attn_decode_partial([whole], q.cuda(), [N - 1])
        e = (o - o1[:, heads[0] * G:(heads[-1] + 1) * G]).abs().max().item()
        if e > 1e-3:
            fails.append(f"KVPxTP slice {t} rank {r}: {e}")
        comm2.close()

    flag = torch.tensor([len(fails)], device="cuda")
    dist.all_reduce(flag)
    if fails:
        print(f"rank {rank} FAIL: {fails}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if flag.item() else 0)


if __name__ == "__main__":
    main()
