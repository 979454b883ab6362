"""CPU tests of the input generator and of the work accounting (paper pins)."""
import json
import math
import os

import torch

import synth
from paper_2409_17264_b200 import accounting as acc

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_synth_is_counter_based_and_block_independent():
    full = synth.kv_block(3, synth.STREAM_K, 0, 300, 8, 64)
    part = synth.kv_block(3, synth.STREAM_K, 100, 150, 8, 64)
    assert torch.equal(full[100:250], part)
    sub = synth.kv_block(3, synth.STREAM_K, 100, 150, 8, 64, heads=[5])
    assert torch.equal(sub[:, 0], full[100:250, 5])
    assert not torch.equal(full, synth.kv_block(4, synth.STREAM_K, 0, 300, 8, 64))
    assert not torch.equal(full, synth.kv_block(3, synth.STREAM_V, 0, 300, 8, 64))


def test_synth_distribution():
    x = synth.kv_block(1, synth.STREAM_K, 0, 4096, 8, 128).float()
    assert abs(x.mean().item()) < 0.01
    assert abs(x.std().item() - 1.0) < 0.01
    assert x.abs().max().item() <= 3.46
    # large flat indices (> 2^32) still hash (10M-token 70B KV spans 2^33.3 elements)
    big = synth.values_bf16(1, 1, torch.arange(2**34, 2**34 + 4096, dtype=torch.int64))
    assert abs(big.float().std().item() - 1.0) < 0.05


def test_synth_amp_is_exact_power_of_two_scaling():
    a = synth.queries(2, 3, 4, 64)
    b = synth.queries(2, 3, 4, 64, amp=4.0)
    assert torch.equal(a.float() * 4, b.float())


def test_golden_paper_accounting():
    """tests/golden/paper_accounting.json: numbers the paper prints (cited there)."""
    with open(os.path.join(GOLDEN, "paper_accounting.json")) as f:
        g = json.load(f)
    kv = g["kv_cache_70b_1M"]
    n = kv["n_tokens"]
    assert acc.kv_bytes(n, kv["h_kv"], kv["d"]) * kv["layers"] == kv["bytes"]
    assert kv["bytes"] == 320 * 2**30            # P:164 "320 GB" is exactly 320 GiB at n = 2^20
    for ex in g["chunk_intensity"]:
        assert acc.chunk_intensity(ex["c"], ex["h_q"], ex["h_kv"]) == ex["intensity"]


def test_pair_accounting_sums_to_eq1():
    """Sum over chunks of exact pairs = n(n+1)/2 for any chunk size, so the
    per-chunk FLOPs sum to Eq. 1 + O(n) (S:100 invariant, exact here)."""
    for n in (1, 97, 4096, 10000):
        for c in (1, 32, 64, 256, 4096):
            tot = sum(acc.visible_pairs(min(c, n - a), a) for a in range(0, n, c))
            assert tot == n * (n + 1) // 2
            fl = sum(acc.prefill_chunk_flops(min(c, n - a), a, 32, 128) for a in range(0, n, c))
            assert fl - acc.eq1_flops(n, 32, 128) == 4 * 128 * 32 * n // 2  # 2n d h_q exactly


def test_eq3_intensity_independent_of_position():
    """Eq. 3: FLOPs/bytes of chunk i approach c h_q/h_kv for any i (large prefix)."""
    for c in (64, 256, 4096):
        for P0 in (2**17, 2**20):
            fl = acc.prefill_chunk_flops(c, P0, 32, 128)
            by = acc.kv_bytes(P0 + c, 8, 128)
            assert math.isclose(fl / by, acc.chunk_intensity(c, 32, 8), rel_tol=0.02)
