"""Same-box decode step A/B (configs[1] shape): per-step device time of
  partial   medha_attn_decode_partial alone
  app+dec   medha_kv_append + medha_attn_decode_partial (two launches)
  fused     medha_attn_decode_append (one launch; skipped if the library predates it)
at 2^20 and 2^17 tokens (the KVP = 8 per-rank shard).  MEDHA_LIB_PATH selects the library.
    python tools/decode_ab.py [label]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
import paper_2409_17264_b200 as M

label = sys.argv[1] if len(sys.argv) > 1 else os.path.basename(M.LIB_PATH)
H_KV, H_Q, D = 8, 32, 128
for n in (1 << 20, 1 << 17):
    sh = bench.build_shard(M, 0, 1, n, H_KV, D)
    k_new = synth.kv_block(1, synth.STREAM_K, n - 1, 1, H_KV, D, device="cuda")
    v_new = synth.kv_block(1, synth.STREAM_V, n - 1, 1, H_KV, D, device="cuda")
    q = synth.queries(1, 1, H_Q, D, device="cuda", amp=4.0)
    o = torch.empty((1, H_Q, D), device="cuda")
    lse = torch.empty((1, H_Q), device="cuda")
    ws = M.decode_workspace(1, H_Q, H_KV, D)
    L = sh.len - 1
    arms = {"partial": lambda: M.attn_decode_partial([sh], q, [n - 1], o=o, lse=lse, ws=ws)}

    def app_dec():
        sh.len = L
        M.kv_append(sh, k_new, v_new)
        M.attn_decode_partial([sh], q, [n - 1], o=o, lse=lse, ws=ws)
    arms["app+dec"] = app_dec
    if hasattr(M, "attn_decode_append"):
        def fused():
            sh.len = L
            M.attn_decode_append([sh], k_new, v_new, q, [n - 1], o=o, lse=lse, ws=ws)
        arms["fused"] = fused

        def fused_noapp():        # same call, append flag off (no owner write, no redirect)
            sh.len = L + 1
            M.attn_decode_append([sh], k_new, v_new, q, [n - 1], append=[False], o=o, lse=lse, ws=ws)
        arms["fused_noapp"] = fused_noapp

        def partial_lenreset():   # plain decode with the host length rewritten every step
            sh.len = L + 1
            M.attn_decode_partial([sh], q, [n - 1], o=o, lse=lse, ws=ws)
        arms["partial_lenreset"] = partial_lenreset
    if os.environ.get("AB_REVERSE") == "1":
        arms = dict(reversed(list(arms.items())))
    res = {}
    for rep in range(3):
        for name, fn in arms.items():
            for _ in range(10):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(100):
                fn()
            b.record()
            torch.cuda.synchronize()
            res.setdefault(name, []).append(a.elapsed_time(b) / 100 * 1e3)
    sh.len = L + 1
    print(json.dumps({"lib": label, "tokens": n, "us_per_step_min_of_3": {k: round(min(v), 2) for k, v in res.items()},
                      "GBps": {k: round(n * H_KV * D * 4 / (min(v) * 1e-6) / 1e9, 1) for k, v in res.items()}}), flush=True)
    del sh
    torch.cuda.empty_cache()
