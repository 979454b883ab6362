"""Shared test helpers: build seeded inputs, run the product path and the oracle.

Inputs come from synth (counter-based, identical on CPU and GPU); the oracle
gets CPU-generated copies, never anything produced by the CUDA path.
"""
from __future__ import annotations

import math

import numpy as np
import torch

import synth

# north_star tolerances (BASELINE.json): GPU vs fp64 oracle on bf16 inputs
MAX_ABS = 2e-2
MEAN_ABS = 2e-3
# LSE bound: the normaliser sums the bf16-rounded P the MMA consumes
# (reading R8), each p within a relative 2^-9 of exact, so |ln l~ - ln l| <= -ln(1 - 2^-9)
# = 1.955e-3; plus the error of the fp32 tensor-core accumulation of the d-term logits,
# observed <= 1.6e-3 at |z| <= 30 (amp-8 queries) -> 2e-3 allowance.
LSE_ABS = 4e-3
KVP_ABS = 1e-3        # KVP merge vs single-GPU, fp32 outputs


def make_global_kv(seed, N, h_kv, d, amp_k=1.0):
    """Token-major bf16 K, V [N][h_kv][d] on the CPU."""
    k = synth.kv_block(seed, synth.STREAM_K, 0, N, h_kv, d, amp=amp_k)
    v = synth.kv_block(seed, synth.STREAM_V, 0, N, h_kv, d)
    return k, v


def to_shard(k_tok, v_tok, a, b, pos0=None, extra_cap=37, poison=True, device="cuda"):
    """Shard holding global tokens [a, b) (head-major), with poisoned spare capacity."""
    from paper_2409_17264_b200 import KVShard
    n = b - a
    h_kv, d = k_tok.shape[1], k_tok.shape[2]
    cap = n + extra_cap
    K = torch.full((h_kv, cap, d), float("nan") if poison else 0.0, dtype=torch.bfloat16)
    V = torch.full((h_kv, cap, d), float("nan") if poison else 0.0, dtype=torch.bfloat16)
    K[:, :n] = k_tok[a:b].permute(1, 0, 2)
    V[:, :n] = v_tok[a:b].permute(1, 0, 2)
    return KVShard(K.to(device), V.to(device), n, a if pos0 is None else pos0)


def oracle_attention(q_tok, k_tok, v_tok, q_pos, key_range=None, scale=None):
    import oracle
    if key_range is not None:
        a, b = key_range
        return oracle.partial(q_tok.double().numpy(), k_tok.float().numpy(), v_tok.float().numpy(), q_pos, (a, b),
                              scale=scale)
    return oracle.attention(q_tok.double().numpy(), k_tok.float().numpy(), v_tok.float().numpy(), q_pos, scale=scale)


def compare(o_gpu, lse_gpu, o_ref, lse_ref, max_abs=MAX_ABS, mean_abs=MEAN_ABS, lse_abs=LSE_ABS, what=""):
    o_gpu = o_gpu.detach().double().cpu().numpy()
    lse_gpu = lse_gpu.detach().double().cpu().numpy()
    assert o_gpu.shape == o_ref.shape, (o_gpu.shape, o_ref.shape)
    assert np.all(np.isfinite(o_gpu)), f"{what}: non-finite output"
    err = np.abs(o_gpu - o_ref)
    fin = np.isfinite(lse_ref)
    assert np.array_equal(fin, np.isfinite(lse_gpu)), f"{what}: -inf pattern of lse differs"
    assert np.all(o_gpu[~fin] == 0.0), f"{what}: empty rows must be exactly 0"
    lerr = np.abs(lse_gpu[fin] - lse_ref[fin]) if fin.any() else np.zeros(1)
    msg = f"{what}: max_abs={err.max():.3e} mean_abs={err.mean():.3e} lse_max={lerr.max():.3e}"
    assert err.max() <= max_abs, msg
    assert err.mean() <= mean_abs, msg
    assert lerr.max() <= lse_abs, msg
    return float(err.max()), float(err.mean()), float(lerr.max())


def default_scale(d):
    return 1.0 / math.sqrt(d)
