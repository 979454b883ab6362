"""Seeded synthetic inputs shared by the tests, the oracle checks and bench.py.

This module holds NO attention arithmetic.  It is a counter-based generator:
every value is a pure function of (seed, stream, flat index), so any block of
the global KV (any token range, any head) can be produced independently, on
the CPU for the oracle and on the GPU for the product path, with bit-identical
results.  That is what lets the KVP shards of every degree P see the same
global KV and lets the oracle regenerate exactly the block
it needs without copying anything back from the CUDA path.

Generator (identical on CPU and CUDA because it uses only int64 integer ops,
one correctly rounded fp32 multiply and one RNE fp32->bf16 conversion):
  h  = mix32(mix32(lo32(i) ^ key(seed, stream)) ^ mix32(hi32(i) ^ key2))
  x  = (byte0(h) + byte1(h) + byte2(h) + byte3(h) - 510) * (1/sqrt(21845))
  value = bf16_rne(x * amp)          (amp a power of two; default 1)
x is an Irwin-Hall(4) approximation of N(0, 1): mean 0, variance 1, |x| <= 3.45.

Layouts: the global KV is token-major [N][h_kv][d]; the flat index of element
(tok, h, e) is (tok*h_kv + h)*d + e.  Queries are [T][h_q][d] with their own
stream.  Streams: K = 1, V = 2, Q = 3, new-token K/V = 4/5.
"""
from __future__ import annotations

import torch

__all__ = ["STREAM_K", "STREAM_V", "STREAM_Q", "values_bf16", "kv_block", "queries",
           "hnd", "BLOCK_TOKENS"]

STREAM_K, STREAM_V, STREAM_Q = 1, 2, 3
BLOCK_TOKENS = 65536            # generation granularity (per 64K-token block)
_M32 = 0xFFFFFFFF
_SCALE = 1.0 / (21845.0 ** 0.5)  # 1/sd of a sum of four uniform bytes


def _mix32_int(x: int) -> int:
    x &= _M32
    x ^= x >> 16
    x = (x * 0x7FEB352D) & _M32
    x ^= x >> 15
    x = (x * 0x68E31DA5) & _M32
    x ^= x >> 16
    return x


def _mix32(x: torch.Tensor) -> torch.Tensor:
    # int64 tensor in [0, 2^32); multipliers < 2^31 keep every product < 2^63.
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & _M32
    x = x ^ (x >> 15)
    x = (x * 0x68E31DA5) & _M32
    x = x ^ (x >> 16)
    return x


def _hash(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    key = _mix32_int(seed * 0x9E3779B1 + stream * 0x85EBCA77 + 0x165667B1)
    key2 = _mix32_int(key ^ 0x27D4EB2F)
    lo = idx & _M32
    hi = idx >> 32
    return _mix32(_mix32(lo ^ key) ^ _mix32(hi ^ key2))


def values_bf16(seed: int, stream: int, idx: torch.Tensor, amp: float = 1.0) -> torch.Tensor:
    """bf16 values for int64 flat indices ``idx`` (any shape, any device)."""
    h = _hash(seed, stream, idx)
    s = (h & 255) + ((h >> 8) & 255) + ((h >> 16) & 255) + (h >> 24) - 510
    x = s.to(torch.float32) * torch.tensor(_SCALE * amp, dtype=torch.float32, device=idx.device)
    return x.to(torch.bfloat16)


def kv_block(seed: int, stream: int, tok0: int, ntok: int, h_kv: int, d: int,
             heads=None, device="cpu", amp: float = 1.0) -> torch.Tensor:
    """Rows [tok0, tok0+ntok) of the global K (stream 1) or V (stream 2).

    Returns a token-major bf16 tensor [ntok][len(heads)][d] (heads default: all).
    """
    if heads is None:
        heads = list(range(h_kv))
    tok = torch.arange(tok0, tok0 + ntok, dtype=torch.int64, device=device)
    hh = torch.as_tensor(list(heads), dtype=torch.int64, device=device)
    e = torch.arange(d, dtype=torch.int64, device=device)
    idx = ((tok[:, None, None] * h_kv + hh[None, :, None]) * d) + e[None, None, :]
    return values_bf16(seed, stream, idx, amp)


def queries(seed: int, T: int, h_q: int, d: int, device="cpu", amp: float = 1.0,
            stream: int = STREAM_Q, t0: int = 0) -> torch.Tensor:
    """Query rows [T][h_q][d] bf16 (amp > 1 gives peaked logits)."""
    tok = torch.arange(t0, t0 + T, dtype=torch.int64, device=device)
    idx = ((tok[:, None, None] * h_q + torch.arange(h_q, device=device)[None, :, None]) * d
           + torch.arange(d, device=device)[None, None, :])
    return values_bf16(seed, stream, idx, amp)


def hnd(x_tok_major: torch.Tensor) -> torch.Tensor:
    """[n][h][d] -> contiguous [h][n][d] (the shard layout)."""
    return x_tok_major.permute(1, 0, 2).contiguous()
