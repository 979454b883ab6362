"""Chunk x KVP sweep of chunked-prefill attention at 2M-10M prefixes (the
analogue of the paper's fig:kvpscaling:prefill:ttft, Eq. 6).

    python tools/kvp_prefill_sweep.py                     (KVP = 1)
    torchrun --nproc-per-node P tools/kvp_prefill_sweep.py (KVP = P)

Llama-3 8B layer shape.  Every rank holds an equal slice of the prefix; the tail rank also
holds the chunk's own K/V.  A step = the KVP prefill of one chunk (local tcgen05 partial +
NCCL all-gather of (o, lse) + rank-ordered merge); time = CUDA events, max over ranks.
Prints one JSON line per (prefix, chunk) on rank 0.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

H_Q, H_KV, D = 32, 8, 128


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import synth
    import paper_2409_17264_b200 as M
    from paper_2409_17264_b200 import accounting as acc
    from paper_2409_17264_b200.kvp import shard_range
    comm = M.KVPComm() if world > 1 else None
    prefixes = [int(x) for x in os.environ.get("SWEEP_PREFIXES", f"{2 << 20},{4 << 20},{10 << 20}").split(",")]
    chunks = [int(x) for x in os.environ.get("SWEEP_CHUNKS", "128,512,2048").split(",")]
    cmax = max(chunks)
    for P0 in prefixes:
        a, b = shard_range(P0, rank, world)
        tail = rank == world - 1
        n_local = (b - a) + (cmax if tail else 0)
        sh = M.KVShard.empty(H_KV, n_local, D, pos0=a)
        for t in range(a, b + (cmax if tail else 0), synth.BLOCK_TOKENS):
            m = min(synth.BLOCK_TOKENS, b + (cmax if tail else 0) - t)
            sh.k[:, t - a:t - a + m] = synth.kv_block(5, synth.STREAM_K, t, m, H_KV, D, device="cuda").permute(1, 0, 2)
            sh.v[:, t - a:t - a + m] = synth.kv_block(5, synth.STREAM_V, t, m, H_KV, D, device="cuda").permute(1, 0, 2)
        for c in chunks:
            sh.len = (b - a) + (c if tail else 0)
            q = synth.queries(6, c, H_Q, D, device="cuda", t0=P0)

            def step():
                if comm is None:
                    return M.attn_prefill_chunk(sh, q, P0)
                return M.kvp_prefill_chunk(comm, sh, q, P0)

            for _ in range(2):
                step()
            iters = 5
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                step()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / iters
            if world > 1:
                t_ = torch.tensor([ms], device="cuda", dtype=torch.float64)
                dist.all_reduce(t_, op=dist.ReduceOp.MAX)
                ms = t_.item()
            fl = acc.prefill_chunk_flops(c, P0, H_Q, D)
            if rank == 0:
                print(json.dumps({"kvp": world, "prefix": P0, "c": c, "ms_per_chunk": round(ms, 3),
                                  "tflops_total": round(fl / (ms * 1e-3) / 1e12, 1),
                                  "tflops_per_gpu": round(fl / (ms * 1e-3) / 1e12 / world, 1),
                                  "exchange_bytes_per_rank": c * H_Q * (D + 1) * 4 if world > 1 else 0}),
                      flush=True)
        del sh
        torch.cuda.empty_cache()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
