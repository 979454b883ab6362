"""Algorithmic work accounting for the hot path (measurement only, no attention math).

The bench divides these ALGORITHMIC figures by measured kernel times to report
GB/s and TFLOP/s; they never feed the computation itself.

* Eq. 1: F_a(n) = 2 n^2 d h_q for a whole causal prefill.  We count
  the exact number of visible (query, key) pairs instead: each pair costs
  2d FLOPs for q.k and 2d for p.v per query head, i.e. 4 d h_q per pair of
  tokens.  sum over pairs = n(n+1)/2, so 4 d h_q n(n+1)/2 = 2n^2 d h_q + O(n)
  (reading R11 in DESIGN.md).
* Eq. 2: M_kv(n) = 4 n d h_kv = R_a(n) bytes per layer for 2-byte
  K and V (2 tensors x 2 B).
* Eq. 3: chunk intensity I_cp = c h_q / h_kv (reading R12: i is
  the chunk index).
"""
from __future__ import annotations

__all__ = ["visible_pairs", "prefill_chunk_flops", "kv_bytes", "decode_bytes",
           "chunk_intensity", "eq1_flops"]


def visible_pairs(c: int, prefix: int) -> int:
    """Exact causal (query, key) pairs of a chunk of c tokens after `prefix`
    cached tokens, inclusive of each query's own key: c*prefix + c(c+1)/2."""
    return c * prefix + c * (c + 1) // 2


def prefill_chunk_flops(c: int, prefix: int, h_q: int, d: int) -> int:
    """4 d h_q FLOPs per visible pair (2d for QK^T, 2d for PV), one layer."""
    return 4 * d * h_q * visible_pairs(c, prefix)


def eq1_flops(n: int, h_q: int, d: int) -> int:
    """Eq. 1 verbatim: F_a(n) = 2 n^2 d h_q."""
    return 2 * n * n * d * h_q


def kv_bytes(n: int, h_kv: int, d: int, elem_bytes: int = 2) -> int:
    """Eq. 2: M_kv(n) = 4 n d h_kv for 2-byte elements (K and V), one layer."""
    return 2 * n * d * h_kv * elem_bytes


def decode_bytes(n_keys: int, h_kv: int, d: int, batch_q_bytes: int = 0) -> int:
    """Algorithmic HBM bytes of one decode attention over n_keys cached tokens:
    the K and V reads of Eq. 2 (R_a(n) = M_kv(n)) plus the (tiny) query bytes."""
    return kv_bytes(n_keys, h_kv, d) + batch_q_bytes


def chunk_intensity(c: int, h_q: int, h_kv: int) -> float:
    """Eq. 3: I_cp = 4ic^2 d h_q / (4icd h_kv) = c h_q / h_kv."""
    return c * h_q / h_kv
