"""Mixed hybrid batch ("prefill and decode to be batched together",
P:752 mixed batching): a decode batch beside a prefill chunk, on one stream and on two
concurrent streams (bench.py `mixed_n2` times the same code at 32 x 64K decodes + c = 128 at
2M).  Both arms must give identical outputs and match the fp64 oracle."""
import pytest

import bench
import synth
from helpers import compare, make_global_kv, oracle_attention, to_shard

pytestmark = pytest.mark.gpu


def test_mixed_one_vs_two_streams():
    import paper_2409_17264_b200 as M
    B, n_dec, c, P0 = 6, 9000, 64, 40000
    H_KV, H_Q, D = bench.H_KV, bench.H_Q, bench.D
    kvs = [make_global_kv(800 + i, n_dec, H_KV, D) for i in range(B)]
    shorts = [to_shard(k, v, 0, n_dec) for k, v in kvs]
    qd = synth.queries(810, B, H_Q, D, amp=6.0)
    kl, vl = make_global_kv(811, P0 + c, H_KV, D)
    sh_long = to_shard(kl, vl, 0, P0 + c)
    ql = synth.queries(812, c, H_Q, D, amp=4.0, t0=P0)
    qpos = [n_dec - 1 - 3 * i for i in range(B)]
    t, diff, (od, ld, op, lp) = bench.mixed_two_streams(M, shorts, qd.cuda(), qpos, sh_long, ql.cuda(), P0, iters=2,
                                                         warm=1)
    assert diff == 0.0
    assert all(v > 0 for v in t.values())
    for i in (0, B - 1):
        k, v = kvs[i]
        ro, rl = oracle_attention(qd[i:i + 1][:, :8], k[:, :2], v[:, :2], [qpos[i]])   # kv heads 0-1
        compare(od[i:i + 1, :8], ld[i:i + 1, :8], ro, rl, what=f"mixed decode {i}")
    rows = [0, c - 1]
    ro, rl = oracle_attention(ql[rows][:, :4], kl[:, :1], vl[:, :1], [P0 + r for r in rows])
    compare(op[rows][:, :4], lp[rows][:, :4], ro, rl, what="mixed prefill")
