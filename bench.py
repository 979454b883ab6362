#!/usr/bin/env python
"""bench.py — KVP decode attention (BASELINE.json configs[1]) on 1..N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl medha|reference] [--no-extra]
    torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1, one rank per GPU)

One step = one pass of the hot path for one decode token of
a Llama-3 8B attention layer (h_q 32, h_kv 8, d 128, bf16) whose 2^20-token KV
cache is sharded over the N ranks by KVP:
  a1 kv_append of the new token's K/V on the tail rank,
  a2 the replicated query, a3+a5 split-KV decode partial (fused split merge),
  a6 NCCL all-gather of the (o, lse) partials and a7 the rank-ordered LSE merge
  (N > 1 only).
The KV is resident in HBM before the timed region (value); `e2e` times the same
step through the C ABI's decode_step_host with pinned host buffers (H2D of q and
the new K/V, D2H of o and lse inside the timed region).  Rank 0 prints ONE JSON
line.  Extra sub-objects (N = 1): prefill-chunk TFLOP/s at 128K and 1M prefix
(configs[2]) and the 70B 10M-token decode (configs[3]).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H_Q, H_KV, D = 32, 8, 128          # Llama-3 8B attention layer (Table 1 notation)
N_KV = 1 << 20                      # 1M tokens, binary (reading R10)
SEED = 1
# per-launch CUDA events bracket every EV_EVERY-th decode launch of the timed region (an
# event pair between two launches costs the step ~6 us at N = 4: measured with 1 in 5)
EV_EVERY = max(1, int(os.environ.get("MEDHA_BENCH_EVENT_EVERY", "5")))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), float(pk["bf16_tflops"]), float(pk.get("bf16_tflops_sustained", pk["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        """Start sampling and return once the first sample is in, so that nvidia-smi's own
        start-up (NVML initialisation) is over before the timed region begins."""
        import threading
        self.lines = []
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        first = threading.Event()

        def reader():
            for line in self.proc.stdout:
                self.lines.append(line)
                first.set()
            first.set()

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        first.wait(timeout=10)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=10)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=5)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(n)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun (one rank per GPU)")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def _barrier(world):
    import torch.distributed as dist
    if world > 1:
        dist.barrier()


def _max_over_ranks(x: float, world: int) -> float:
    import torch
    import torch.distributed as dist
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def build_shard(M, rank, world, n_total, h_kv, d, extra_cap=0, seed=SEED):
    """Rank r holds global tokens [r n/P, (r+1) n/P), generated on the GPU by
    the counter-based generator (same global KV for every P)."""
    return build_range(M, n_total * rank // world, n_total * (rank + 1) // world, h_kv, d, extra_cap, seed)


def build_range(M, a, b, h_kv, d, extra_cap=0, seed=SEED):
    """Shard holding global tokens [a, b) of the synthetic sequence `seed` (pos0 = a)."""
    import torch
    import synth
    n = b - a
    sh = M.KVShard.empty(h_kv, n + extra_cap, d, pos0=a)
    blk = synth.BLOCK_TOKENS
    for t in range(a, b, blk):
        m = min(blk, b - t)
        for which, dst in ((synth.STREAM_K, sh.k), (synth.STREAM_V, sh.v)):
            x = synth.kv_block(seed, which, t, m, h_kv, d, device="cuda")
            dst[:, t - a:t - a + m].copy_(x.permute(1, 0, 2))
    sh.len = n
    torch.cuda.synchronize()
    return sh


def bench_decode(args, rank, world, M):
    import torch
    import synth
    from paper_2409_17264_b200 import accounting as acc

    tail = rank == world - 1
    sh = build_shard(M, rank, world, N_KV, H_KV, D)
    # the decode token is global position N_KV-1: its K/V is the tail rank's last row,
    # re-appended every step (len reset on the host after each step)
    new_pos = N_KV - 1
    k_new = synth.kv_block(SEED, synth.STREAM_K, new_pos, 1, H_KV, D, device="cuda")
    v_new = synth.kv_block(SEED, synth.STREAM_V, new_pos, 1, H_KV, D, device="cuda")
    q = synth.queries(SEED, 1, H_Q, D, device="cuda", amp=4.0)
    len_before = sh.len - 1 if tail else sh.len
    comm = M.KVPComm() if world > 1 else None
    stream = torch.cuda.current_stream()
    rows = H_Q
    dws = M.decode_workspace(1, H_Q, H_KV, D)
    parts_send = torch.empty(rows * (D + 1), dtype=torch.float32, device="cuda")
    o_out = torch.empty((1, H_Q, D), dtype=torch.float32, device="cuda")
    lse_out = torch.empty((1, H_Q), dtype=torch.float32, device="cuda")
    xws = M.exchange_workspace(world, rows, D) if world > 1 else None
    kws = M.kvp_workspace(world, 1, H_Q, H_KV, D) if world > 1 else None
    if comm is not None and os.environ.get("MEDHA_BENCH_NCCL") == "1":
        comm.set_p2p(False)                       # A/B: NCCL all-gather + merge kernel
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ev_every = EV_EVERY if args.steps >= 2 * EV_EVERY else 1

    def step(i=None):
        # ONE launch per step and rank: the tail rank's append of the new token rides in the
        # decode launch (medha_attn_decode_append / medha_kvp_decode_append)
        if tail:
            sh.len = len_before
        e = ev[i] if (i is not None and i % ev_every == ev_every - 1) else None
        if e:
            e[0].record(stream)
        if world == 1:
            M.attn_decode_append([sh], k_new, v_new, q, [new_pos], o=o_out, lse=lse_out, ws=dws)
            if e:
                e[1].record(stream)
        elif comm.p2p:
            # decode partial + append + NVLink push + rank-ordered merge (fused exchange)
            M.kvp_decode_append(comm, [sh], k_new, v_new, q, [new_pos], append=[tail], ws=kws, o=o_out, lse=lse_out)
            if e:
                e[1].record(stream)
        else:
            o_p, l_p = parts_send[:rows * D].view(1, H_Q, D), parts_send[rows * D:].view(1, H_Q)
            M.attn_decode_append([sh], k_new, v_new, q, [new_pos], append=[tail], o=o_p, lse=l_p, ws=dws)
            if e:
                e[1].record(stream)
            M.kvp_exchange_merge(comm, parts_send, rows, D, o_out, lse_out, ws=xws)

    # the sampler is up (first sample in) before the warm-up, so its start-up never overlaps
    # the timed region
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    _barrier(world)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(args.steps):
        step(i)
    t1.record(stream)
    torch.cuda.synchronize()
    _barrier(world)
    ms_local = t0.elapsed_time(t1) / args.steps
    ms = _max_over_ranks(ms_local, world)
    timed_ev = [ev[i] for i in range(ev_every - 1, args.steps, ev_every)]
    kern_ms_local = sum(a.elapsed_time(b) for a, b in timed_ev) / len(timed_ev)
    kern_ms = _max_over_ranks(kern_ms_local, world)

    # ---- end to end through the C ABI with pinned host buffers ------------------------------
    q_h = q[0].cpu().pin_memory()
    k_h = k_new[0].cpu().pin_memory()
    v_h = v_new[0].cpu().pin_memory()
    o_h = torch.empty((H_Q, D), dtype=torch.float32).pin_memory()
    l_h = torch.empty((H_Q,), dtype=torch.float32).pin_memory()
    sws = M.decode_step_workspace(world, H_Q, H_KV, D)

    # the serving loop's prepared step (medha_decode_plan: host buffers, comm and workspace
    # resolved once; each step = the H2D-reading staging launch + the decode launch)
    plan = M.DecodePlan(comm, sh, q_h, k_h if tail else None, v_h if tail else None, o_h, l_h, sws)

    def e2e_step():
        if tail:
            sh.len = len_before
        plan.step(sh, tail, new_pos, stream)
        stream.synchronize()   # the host reads the step's result

    for _ in range(args.warmup):
        e2e_step()
    _barrier(world)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    _barrier(world)
    clk = clocks.stop()   # sampled across both timed regions (device-resident and e2e)
    e2e_ms = _max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    # parity of the e2e output against the device path (same inputs)
    e2e_diff = float((o_h - o_out[0].cpu()).abs().max())
    plan.close()

    bytes_total = acc.decode_bytes(N_KV, H_KV, D)              # all ranks together
    bytes_rank = acc.decode_bytes(sh.len, H_KV, D)
    h2d = world * (H_Q * D * 2) + 2 * H_KV * D * 2
    d2h = world * (H_Q * D * 4 + H_Q * 4)
    fused = comm is not None and comm.p2p
    launches_per_step = 1 + (1 if (world > 1 and not fused) else 0)   # rank-0 view (NCCL path: + merge kernel)
    exch = "none" if comm is None else ("fused NVLink push in the decode kernel" if fused else "NCCL all-gather + merge kernel")
    if comm is not None:
        comm.close()
    return dict(exchange=exch, ms=ms, kern_ms=kern_ms, ev_every=ev_every, bytes_total=bytes_total, bytes_rank=bytes_rank, e2e_ms=e2e_ms,
                h2d=h2d, d2h=d2h, clocks=clk, launches=launches_per_step * args.steps, e2e_diff=e2e_diff,
                o=o_out, sh=sh)


def bench_graph_decode(M, iters=50, warm=5):
    """configs[1] decode step replayed from ONE captured CUDA graph (device-side
    lengths, `medha_decode_step_dev`): graph = reset the device length to 2^20 - 1, append the
    token at it, decode over 2^20 keys (the device length then advances); same work per step
    as the eager line."""
    import torch
    import synth
    sh = build_shard(M, 0, 1, N_KV, H_KV, D)
    new_pos = N_KV - 1
    k_new = synth.kv_block(SEED, synth.STREAM_K, new_pos, 1, H_KV, D, device="cuda")
    v_new = synth.kv_block(SEED, synth.STREAM_V, new_pos, 1, H_KV, D, device="cuda")
    q = synth.queries(SEED, 1, H_Q, D, device="cuda", amp=4.0)
    len0 = torch.tensor([new_pos], dtype=torch.int64, device="cuda")
    len_dev = len0.clone()
    ws = M.decode_workspace(1, H_Q, H_KV, D)
    o = torch.empty((1, H_Q, D), dtype=torch.float32, device="cuda")
    lse = torch.empty((1, H_Q), dtype=torch.float32, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            len_dev.copy_(len0)
            M.decode_step_dev([sh], k_new, v_new, q, len_dev, o, lse, ws)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    o_eager = o.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        len_dev.copy_(len0)
        M.decode_step_dev([sh], k_new, v_new, q, len_dev, o, lse, ws)
    for _ in range(warm):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    same = bool(torch.equal(o, o_eager))
    del sh
    torch.cuda.empty_cache()
    return {"ms_per_step": round(ms, 5), "GBps": round(N_KV * H_KV * D * 2 * 2 / (ms * 1e-3) / 1e9, 1),
            "graph": "length reset (memcpy) + one decode launch with the fused append, replayed", "replays": iters,
            "output_equals_eager_call": same}


def bench_prefill(M, sh_full, prefixes, chunks, iters=5, warm=2):
    """Chunked-prefill partial on one GPU at prefix P0 (configs[2]): the chunk's own
    K/V are rows [P0, P0+c) of the same synthetic sequence (already resident)."""
    import torch
    import synth
    from paper_2409_17264_b200 import accounting as acc
    _, tf_peak, tf_sus, _ = _peaks()
    out = []
    for P0 in prefixes:
        for c in chunks:
            if P0 + c > sh_full.capacity:
                continue
            q = synth.queries(SEED + 7, c, H_Q, D, device="cuda", amp=1.0, t0=P0)
            saved = sh_full.len
            sh_full.len = P0 + c
            o = torch.empty((c, H_Q, D), dtype=torch.float32, device="cuda")
            l = torch.empty((c, H_Q), dtype=torch.float32, device="cuda")
            ws = M.prefill_workspace(c, H_Q, H_KV, D)
            for _ in range(warm):
                M.attn_prefill_chunk(sh_full, q, P0, o=o, lse=l, ws=ws)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(iters):
                M.attn_prefill_chunk(sh_full, q, P0, o=o, lse=l, ws=ws)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / iters
            fl = acc.prefill_chunk_flops(c, P0, H_Q, D)
            tfs = fl / (ms * 1e-3) / 1e12
            out.append({"prefix": P0, "c": c, "ms": round(ms, 4), "tflops": round(tfs, 1),
                        "frac_of_measured_bf16": round(tfs / tf_peak, 4),
                        "frac_of_measured_bf16_sustained": round(tfs / tf_sus, 4)})
            sh_full.len = saved
    return out


def bench_70b_decode(M, iters=5, warm=2):
    """configs[3]: Llama-3 70B (h_q 64, h_kv 8, d 128) decode at 10*2^20 tokens.
    On one GPU: the whole 40 GiB KV (P = 1) and one KVP=8 shard (1/8 of it)."""
    import torch
    import synth
    from paper_2409_17264_b200 import accounting as acc
    n = 10 * (1 << 20)
    res = {}
    for P, label in ((1, "kvp1_full"), (8, "kvp8_one_rank_shard")):
        sh = build_shard(M, P - 1, P, n, 8, 128, seed=SEED + 3)
        q = synth.queries(SEED + 3, 1, 64, 128, device="cuda", amp=4.0)
        ws = M.decode_workspace(1, 64, 8, 128)
        o = torch.empty((1, 64, 128), dtype=torch.float32, device="cuda")
        l = torch.empty((1, 64), dtype=torch.float32, device="cuda")
        for _ in range(warm):
            M.attn_decode_partial([sh], q, [n - 1], o=o, lse=l, ws=ws)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            M.attn_decode_partial([sh], q, [n - 1], o=o, lse=l, ws=ws)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / iters
        by = acc.decode_bytes(sh.len, 8, 128)
        res[label] = {"tokens_on_gpu": sh.len, "ms": round(ms, 4), "GBps": round(by / (ms * 1e-3) / 1e9, 1)}
        del sh
        torch.cuda.empty_cache()
    return res


def mixed_two_streams(M, shorts, qd, qpos_d, sh_long, q_long, p0_long, iters=5, warm=2):
    """SURVEY N2 / P:89, P:752 (prefill and decode batched together): a batch of decodes
    (one decode launch over all `shorts`) beside one prefill chunk, run (a) one after the
    other on one stream and (b) concurrently on two streams (the prefill's 1-CTA-per-SM grid
    and the decode's 2-CTA-per-SM grid then share the SMs as the block scheduler places
    them).  Returns per-step ms of both arms and the max |difference| of their outputs
    (same kernels and split plans: 0 expected)."""
    import torch
    B = len(shorts)
    c = q_long.shape[0]
    od = [torch.empty((B, H_Q, D), device="cuda") for _ in range(2)]
    ld = [torch.empty((B, H_Q), device="cuda") for _ in range(2)]
    op = [torch.empty((c, H_Q, D), device="cuda") for _ in range(2)]
    lp = [torch.empty((c, H_Q), device="cuda") for _ in range(2)]
    s_main = torch.cuda.current_stream()
    s_dec = torch.cuda.Stream()
    dws = [torch.zeros(M.lib.medha_decode_workspace_size(B, H_Q, H_KV, D), dtype=torch.uint8, device="cuda")
           for _ in range(2)]
    pws = [torch.zeros(M.lib.medha_prefill_workspace_size(c, H_Q, H_KV, D), dtype=torch.uint8, device="cuda")
           for _ in range(2)]

    def serial(k):
        M.attn_prefill_chunk(sh_long, q_long, p0_long, o=op[k], lse=lp[k], ws=pws[k])
        M.attn_decode_partial(shorts, qd, qpos_d, o=od[k], lse=ld[k], ws=dws[k])

    def concurrent(k):
        s_dec.wait_stream(s_main)
        M.attn_prefill_chunk(sh_long, q_long, p0_long, o=op[k], lse=lp[k], ws=pws[k])
        with torch.cuda.stream(s_dec):
            M.attn_decode_partial(shorts, qd, qpos_d, o=od[k], lse=ld[k], ws=dws[k], stream=s_dec)
        s_main.wait_stream(s_dec)

    res = {}
    for name, fn, k in (("one_stream", serial, 0), ("two_streams", concurrent, 1), ("one_stream_again", serial, 0)):
        for _ in range(warm):
            fn(k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_main)
        for _ in range(iters):
            fn(k)
        e1.record(s_main)
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / iters
    # the arms alone, for the sum / max bounds
    for name, fn in (("prefill_alone", lambda: M.attn_prefill_chunk(sh_long, q_long, p0_long, o=op[0], lse=lp[0],
                                                                     ws=pws[0])),
                     ("decodes_alone", lambda: M.attn_decode_partial(shorts, qd, qpos_d, o=od[0], lse=ld[0],
                                                                     ws=dws[0]))):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / iters
    serial(0)
    concurrent(1)
    torch.cuda.synchronize()
    diff = max(float((od[0] - od[1]).abs().max()), float((op[0] - op[1]).abs().max()))
    return res, diff, (od[1], ld[1], op[1], lp[1])


def bench_mixed_n2(M, iters=5, warm=2):
    """SURVEY N2 at a size where the decodes are not negligible: 32 decodes over 64K-token
    KVs (8 GiB of K/V) beside one c = 128 chunk at a 2M prefix (4.4 TFLOP), 8B shape, one GPU."""
    import torch
    import synth
    from paper_2409_17264_b200 import accounting as acc
    B, n_dec, c, P0 = 32, 1 << 16, 128, 1 << 21
    shorts = [build_range(M, 0, n_dec, H_KV, D, seed=SEED + 200 + i) for i in range(B)]
    qd = synth.queries(SEED + 201, B, H_Q, D, device="cuda", amp=4.0)
    sh_long = build_range(M, 0, P0 + c, H_KV, D, seed=SEED + 202)
    q_long = synth.queries(SEED + 203, c, H_Q, D, device="cuda", amp=1.0, t0=P0)
    t, diff, _ = mixed_two_streams(M, shorts, qd, [n_dec - 1] * B, sh_long, q_long, P0, iters, warm)
    fl = acc.prefill_chunk_flops(c, P0, H_Q, D)
    by = acc.decode_bytes(B * n_dec, H_KV, D)
    out = {"workload": f"{B} x {n_dec}-token decodes + one c={c} chunk at a {P0}-token prefix (8B shape, N=1)",
           "decode_bytes": by, "chunk_tflop": round(fl / 1e12, 3),
           "ms": {k: round(v, 4) for k, v in t.items()},
           "two_stream_speedup": round(min(t["one_stream"], t["one_stream_again"]) / t["two_streams"], 4),
           "max_abs_diff_between_arms": diff,
           "note": "parity of both arms vs the fp64 oracle: tests/test_gpu_mixed.py (same code path, smaller sizes)"}
    del shorts, sh_long
    torch.cuda.empty_cache()
    return out


def bench_mixed(M, rank, world, iters=5, warm=3):
    """configs[4], the mixed hybrid batch under KVP = 4: per rank, one 512-token prefill chunk
    of a 2M-context request over the rank's 512K-token slice (the tail rank also holds the
    chunk's own K/V, Eq. 6) plus 8 rank-local short decodes over 4K-token KVs
    (32 in all).  At N = 4 the step is measured as it runs (KVP prefill with
    all-gather + merge, then the batched decodes), max over ranks.  At N = 1 every rank's
    work is timed on this GPU in turn and the K5 merge of the four partials beside it; the
    projected KVP = 4 step is the slowest rank + the merge (the exchange, 8 MiB per rank, is
    measured only at N = 4)."""
    import torch
    import synth
    from paper_2409_17264_b200 import accounting as acc
    from paper_2409_17264_b200.kvp import shard_range
    P, c, P0, n_short = 4, 512, 1 << 21, 4096
    if world not in (1, P):
        return None
    comm = M.KVPComm() if world == P else None
    q = synth.queries(SEED + 11, c, H_Q, D, device="cuda", amp=1.0, t0=P0)
    rows = c * H_Q
    pws = M.prefill_workspace(c, H_Q, H_KV, D)
    dws = M.decode_workspace(8, H_Q, H_KV, D)
    parts = torch.empty((P, rows * (D + 1)), dtype=torch.float32, device="cuda")
    od = torch.empty((8, H_Q, D), dtype=torch.float32, device="cuda")
    ld = torch.empty((8, H_Q), dtype=torch.float32, device="cuda")
    per_rank = []
    for r in ([rank] if comm is not None else range(P)):
        a, b = shard_range(P0, r, P)
        if r == P - 1:
            b = P0 + c
        sh = build_range(M, a, b, H_KV, D, seed=SEED + 11)
        shorts = [build_range(M, 0, n_short, H_KV, D, seed=SEED + 100 + 8 * r + i) for i in range(8)]
        qd = synth.queries(SEED + 100 + 8 * r, 8, H_Q, D, device="cuda", amp=4.0)
        po, pl = parts[r, :rows * D].view(c, H_Q, D), parts[r, rows * D:].view(c, H_Q)

        def step():
            if comm is not None:
                M.kvp_prefill_chunk(comm, sh, q, P0)
            else:
                M.attn_prefill_chunk(sh, q, P0, o=po, lse=pl, ws=pws)
            M.attn_decode_partial(shorts, qd, [n_short - 1] * 8, o=od, lse=ld, ws=dws)

        for _ in range(warm):
            step()
        _barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            step()
        e1.record()
        torch.cuda.synchronize()
        _barrier(world)
        per_rank.append(e0.elapsed_time(e1) / iters)
        del sh, shorts
        torch.cuda.empty_cache()
    fl = acc.prefill_chunk_flops(c, P0, H_Q, D)
    _, tf_peak, _, _ = _peaks()
    roof_ms = fl / P / (tf_peak * 1e12) * 1e3
    res = {"workload": "configs[4]: 32 x 4K-token decodes (8 per rank) + one c=512 chunk at 2M prefix, KVP=4",
           "chunk_tflop": round(fl / 1e12, 3), "short_decode_bytes": acc.decode_bytes(32 * n_short, H_KV, D),
           "rank_roofline_ms": round(roof_ms, 4)}
    if comm is not None:
        ms = _max_over_ranks(per_rank[0], world)
        comm.close()
        res.update({"measured": "N=4, max over ranks", "ms_per_step": round(ms, 4),
                    "chunk_tflops": round(fl / (ms * 1e-3) / 1e12, 1), "frac_of_rank_roofline": round(roof_ms / ms, 4)})
    else:
        for _ in range(warm):
            M.merge_partials(parts, rows, D)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            M.merge_partials(parts, rows, D)
        e1.record()
        torch.cuda.synchronize()
        merge_ms = e0.elapsed_time(e1) / iters
        ms = max(per_rank) + merge_ms
        res.update({"measured": "N=1: each rank's work in turn on one GPU", "rank_ms": [round(x, 4) for x in per_rank],
                    "merge_ms": round(merge_ms, 4), "kvp4_projected_ms_excl_exchange": round(ms, 4),
                    "chunk_tflops_projected": round(fl / (ms * 1e-3) / 1e12, 1),
                    "frac_of_rank_roofline": round(roof_ms / ms, 4)})
    return res


def hbm_probe(M, nbytes=4 << 30, iters=5):
    import torch
    buf = torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda")
    buf.fill_(1.0)
    sink = torch.zeros(4096, dtype=torch.float32, device="cuda")
    M.hbm_read_probe(buf, sink)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        M.hbm_read_probe(buf, sink)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    del buf
    torch.cuda.empty_cache()
    return round(nbytes / (ms * 1e-3) / 1e9, 1)


def cpu_oracle_sample(kv_heads=1, tokens=N_KV):
    """Time the fp64 oracle as it stands on a bounded sample of the decode workload:
    `kv_heads` KV heads (G = 4 query heads each) over `tokens` keys."""
    import numpy as np
    import torch
    import oracle
    import synth
    torch.set_num_threads(os.cpu_count() or 1)
    G = H_Q // H_KV
    q = synth.queries(SEED, 1, H_Q, D, amp=4.0).double().numpy()
    total_s = 0.0
    for h in range(kv_heads):
        k = synth.kv_block(SEED, synth.STREAM_K, 0, tokens, H_KV, D, heads=[h]).float().numpy()[:, 0]
        v = synth.kv_block(SEED, synth.STREAM_V, 0, tokens, H_KV, D, heads=[h]).float().numpy()[:, 0]
        t = time.perf_counter()
        oracle.attention_group(q[:, h * G:(h + 1) * G], k, v, [tokens - 1], np.arange(tokens), 1 / math.sqrt(D))
        total_s += time.perf_counter() - t
    by = kv_heads * tokens * 2 * D * 2
    return by / total_s / 1e9, total_s


def run_reference(args):
    """--impl reference: the oracle as it stands, on the host cores, same metric/config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    sample_tokens = 1 << 18
    for _ in range(args.warmup):
        cpu_oracle_sample(1, sample_tokens)
    times, vals = [], []
    for _ in range(args.steps):
        v, s = cpu_oracle_sample(1, sample_tokens)
        vals.append(v)
        times.append(s)
    by = sample_tokens * 2 * D * 2
    val = by * len(times) / sum(times) / 1e9
    cores = os.cpu_count()
    sample = f"1 of 8 KV heads (G=4) x {sample_tokens} keys per step ({by / 2**20:.0f} MiB of K+V)"
    line = {"impl": "reference", "metric": "KVP decode attn HBM GB/s & ms/layer; prefill-chunk TFLOPS; at 1/2/4/8 B200",
            "value": round(val, 4), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * sum(times) / len(times), 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config(args.gpus),
            "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(n):
    return {"workload": f"llama3-8b attention decode, batch 1, 2^20-token KV, KVP={n}",
            "h_q": H_Q, "h_kv": H_KV, "d": D, "kv_tokens": N_KV, "batch": 1, "kvp": n,
            "parallelism": f"kvp{n}", "l2": "inputs larger than L2 (4 GiB/P of K+V per rank, no flush)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="medha", choices=["medha", "reference"])
    ap.add_argument("--no-extra", action="store_true", help="skip prefill / 70B / probe / cpu sub-measurements")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    rank, world, local = _dist_setup(args)
    import paper_2409_17264_b200 as M
    hbm_peak, tf_peak, tf_sus, peak_src = _peaks()

    r = bench_decode(args, rank, world, M)
    value = r["bytes_total"] / (r["ms"] * 1e-3) / 1e9
    achieved = r["bytes_rank"] / (r["kern_ms"] * 1e-3) / 1e9
    # DRAM bytes per launch of the decode kernel are not measurable without a profiler: the
    # value comes from the committed ncu capture named in traffic_source (same kernel, same
    # configuration), not from this run
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "decode_ncu_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get("dram_bytes_per_launch", {}).get(f"kvp{world}")
        traffic_src = "profiles/decode_ncu_traffic.json: " + str(tj.get("source_run", tj.get("source", "")))[:160]
    except Exception:
        pass
    extra = {}
    if rank == 0 and world == 1 and not args.no_extra:
        sh = r["sh"]
        extra["hbm_read_probe_GBps"] = hbm_probe(M)
    del r["sh"], r["o"]
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_extra:
        sh_p = build_shard(M, 0, 1, N_KV + 4096, H_KV, D, seed=SEED)
        extra["prefill_chunk"] = {"unit": "TFLOP/s", "peak_bf16_tflops": tf_peak, "peak_bf16_tflops_sustained": tf_sus,
                                  "peak_source": peak_src,
                                  "flops": "4 d h_q (c P0 + c(c+1)/2)",
                                  "results": bench_prefill(M, sh_p, [1 << 17, 1 << 20], [64, 256, 1024, 4096])}
        del sh_p
        torch.cuda.empty_cache()
        extra["decode_70b_10M"] = bench_70b_decode(M)
        extra["decode_cuda_graph"] = bench_graph_decode(M)
        extra["mixed_n2"] = bench_mixed_n2(M)
    if world in (1, 4) and not args.no_extra:
        mixed = bench_mixed(M, rank, world)
        if rank == 0:
            extra["mixed_c4"] = mixed
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, s = cpu_oracle_sample(2, N_KV)
        cpu = {"value": round(v, 4), "unit": "GB/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"2 of 8 KV heads (G=4 query heads each) x 2^20 keys, fp64 two-pass, {s:.1f} s"}
    if rank == 0:
        line = {
            "metric": "KVP decode attn HBM GB/s & ms/layer; prefill-chunk TFLOPS; at 1/2/4/8 B200",
            "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(r["ms"], 5), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (counter-based seeded generator, N(0,1)-like)",
            "config": _config(world),
            "roofline": {"bound": "hbm", "kernel": "decode_splitkv_kernel<128,4>", "achieved": round(achieved, 1),
                         "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                         "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                         "frac_of_read_probe": (round(achieved / extra["hbm_read_probe_GBps"], 4)
                                                if extra.get("hbm_read_probe_GBps") else None),
                         "per_launch_bytes": r["bytes_rank"], "kernel_ms": round(r["kern_ms"], 5),
                         "kernel_timing": f"CUDA events around 1 in {r['ev_every']} decode launches of the timed region"},
            "e2e": {"value": round(r["bytes_total"] / (r["e2e_ms"] * 1e-3) / 1e9, 1), "unit": "GB/s",
                    "ms_per_step": round(r["e2e_ms"], 5), "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"],
                    "api": "medha_decode_plan_step (prepared medha_decode_step_host)", "max_abs_vs_device_path": r["e2e_diff"]},
            "gpu_launches": r["launches"],
            "kvp_exchange": r["exchange"],
            "clocks": r["clocks"],
            "cpu_baseline": cpu,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
