"""CPU, world_size 2 (gloo): the KVP host logic — NCCL unique-id bootstrap over the
process group, the sequence partition, and the rank-ordered exchange + merge
orchestration (oracle partials standing in for the GPU partials)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2409_17264_b200.kvp import exchange_unique_id, shard_range
        uid = exchange_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert all(i == ids[0] for i in ids) and len(uid) == 128 and any(uid)
        N, h_kv, G, d = 1000, 2, 4, 32
        a, b = shard_range(N, rank, world)
        k = synth.kv_block(5, synth.STREAM_K, 0, N, h_kv, d).double().numpy()
        v = synth.kv_block(5, synth.STREAM_V, 0, N, h_kv, d).double().numpy()
        qq = synth.queries(5, 3, h_kv * G, d, amp=4.0).double().numpy()
        qp = [N - 1, 600, 250]               # rank 1 has no visible key for 250/600 when P=2
        o_r, l_r = oracle.partial(qq, k, v, qp, (a, b))
        packed = torch.from_numpy(np.concatenate([o_r.reshape(-1), l_r.reshape(-1)]))
        gathered = [torch.empty_like(packed) for _ in range(world)]
        dist.all_gather(gathered, packed)
        rows = 3 * h_kv * G
        parts = [(g[:rows * d].numpy().reshape(3, h_kv * G, d), g[rows * d:].numpy().reshape(3, h_kv * G))
                 for g in gathered]
        om, lm = oracle.merge(parts)
        ref_o, ref_l = oracle.attention(qq, k, v, qp)
        np.testing.assert_allclose(om, ref_o, rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(lm, ref_l, rtol=1e-12)
        q.put((rank, "ok", (a, b)))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


def test_kvp_host_logic_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    res.sort()
    assert all(r[1] == "ok" for r in res), res
    assert [r[2] for r in res] == [(0, 500), (500, 1000)]


def test_shard_range_partitions_exactly():
    from paper_2409_17264_b200.kvp import shard_range
    for n in (1, 7, 1 << 20, 10 * (1 << 20) + 3):
        for P in (1, 2, 3, 4, 8):
            rs = [shard_range(n, r, P) for r in range(P)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(P - 1))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_growth_placement():
    from paper_2409_17264_b200.kvp import growth_placement
    assert growth_placement(0, 100, 4) == [(0, 0)] * 4
    assert growth_placement(250, 100, 4) == [(0, 100), (100, 200), (200, 250), (250, 250)]
    assert growth_placement(400, 100, 4)[-1] == (300, 400)
    with pytest.raises(ValueError):
        growth_placement(401, 100, 4)
    # the placement is a contiguous partition of [0, n) for every n (exact merge, I1)
    for n in range(0, 401, 7):
        rs = growth_placement(n, 100, 4)
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(rs[i][1] == rs[i + 1][0] for i in range(3))
