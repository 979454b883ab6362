"""fp64 CPU oracle for KV-sharded exact attention (Medha, arXiv 2409.17264).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2409_17264_b200``) never imports it and
shares no code with it: no kernels, headers, helpers, constants or pre/post
processing.

Citations: ``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n.

What it computes (the plain definition):

* Attention (§2.1 "each token attends to all prior tokens, involving
  two matrix multiplications: (1) query and key tensors to obtain the attention
  matrix and (2) attention matrix with value tensors"), causal and inclusive of
  the query's own position (reading R3), softmax scale ``s`` passed in
  (reading R1: 1/sqrt(d) by default), GQA head map ``kv_head = h // G``
  (reading R2, "8 query heads share one KV head").
* Per-shard partial attention (§3.4 "KVP shards the KV cache ...
  along the sequence dimension ... replicate the Q token(s) ... compute partial
  attention outputs based on each local KV-cache shard"), returned as
  (normalised o, natural-log lse) (readings R5, R6).
* The exact merge of partials (§3.4 "combined using online-softmax").

Every value is computed in float64 from inputs that are already bf16-rounded
(the caller converts bf16 -> float64 exactly).  Softmax is the textbook
two-pass form (max, then exp/sum); there is no running rescale, i.e. no shared
algorithm with the GPU online softmax.

Blocking: for very long key ranges (1M-10M keys) the logits ``z_j`` are
computed block by block (each ``z_j`` is an independent dot product, so this is
not a reordering of any sum), and sum_j w_j V_j is accumulated block by block
(a regrouping of an fp64 sum; its effect, ~1e-16 relative, is far below every
tolerance used against the GPU).  Nothing else is blocked, fused or reordered.

Parity pins (tests/test_oracle_*.py): brute force with math.fsum on tiny
inputs, torch fp64 SDPA with an explicit bottom-right mask, closed forms
(K = 0 => prefix mean; needle), invariants I1-I13 of SURVEY.md §8(c).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "attention_group",
    "attention",
    "partial",
    "merge",
    "NEG_INF",
]

NEG_INF = float("-inf")

# Key block for the streaming dot products: 65536 keys x 128 dims x 8 B = 64 MiB.
_BLOCK = 65536


def _as_f64(x) -> np.ndarray:
    """bf16-valued input (float32 / float64 / torch tensor) -> float64 exactly."""
    if hasattr(x, "detach"):  # torch tensor; .double() of bf16/fp32 is exact
        x = x.detach().double().cpu().numpy()
    return np.asarray(x, dtype=np.float64)


def attention_group(q, k, v, q_pos, key_pos, scale: float, block: int = _BLOCK):
    """Exact causal attention of G query heads that share ONE KV head.

    P:167-171 (attention), P:357-358 (GQA sharing), SURVEY §8(c) definition:
        z_j = s * sum_k Q[t,h,k] K[j,k]    for j with key_pos[j] <= q_pos[t]
        m = max_j z_j;  w_j = exp(z_j - m);  l = sum_j w_j
        O[t,h,:] = sum_j w_j V[j,:] / l;    LSE[t,h] = m + ln l
        (no visible key => O = 0, LSE = -inf; reading R7)

    Args:
      q:       [T][G][d] query rows (bf16-valued).
      k, v:    [N][d] keys / values of this KV head (bf16-valued); may be float32
               to save memory - converted to float64 block by block.
      q_pos:   [T] absolute positions of the query tokens.
      key_pos: [N] absolute positions of the keys (non-decreasing).
      scale:   softmax scale s.
    Returns:
      (o [T][G][d] float64, lse [T][G] float64, natural log).
    """
    q = _as_f64(q)
    T, G, d = q.shape
    q_pos = np.asarray(q_pos, dtype=np.int64).reshape(T)
    key_pos = np.asarray(key_pos, dtype=np.int64)
    N = key_pos.shape[0]
    if k.shape[0] != N or v.shape[0] != N or k.shape[-1] != d or v.shape[-1] != d:
        raise ValueError("dimension mismatch")
    o = np.zeros((T, G, d), dtype=np.float64)
    lse = np.full((T, G), NEG_INF, dtype=np.float64)
    for t in range(T):
        # keys are sorted by position, so the visible set is a prefix
        n_vis = int(np.searchsorted(key_pos, q_pos[t], side="right"))
        if n_vis == 0:
            continue
        # pass 1: logits z [n_vis][G]
        z = np.empty((n_vis, G), dtype=np.float64)
        for a in range(0, n_vis, block):
            b = min(n_vis, a + block)
            z[a:b] = scale * (_as_f64(k[a:b]) @ q[t].T)
        m = z.max(axis=0)                      # [G]
        w = np.exp(z - m)                      # [n_vis][G]
        l = w.sum(axis=0)                      # [G]
        # pass 2: weighted sum of values
        acc = np.zeros((G, d), dtype=np.float64)
        for a in range(0, n_vis, block):
            b = min(n_vis, a + block)
            acc += w[a:b].T @ _as_f64(v[a:b])
        o[t] = acc / l[:, None]
        lse[t] = m + np.log(l)
    return o, lse


def attention(q, k, v, q_pos, key_pos=None, scale: float | None = None):
    """Exact GQA causal attention over a whole (unsharded) KV.

    Args:
      q:  [T][h_q][d]; k, v: [N][h_kv][d] (token-major, as in P:178-183 the KV
          cache of n tokens has h_kv heads of dimension d).
      q_pos: [T] absolute positions; key_pos: [N] (default 0..N-1).
      scale: default 1/sqrt(d) (reading R1).
    Returns (o [T][h_q][d], lse [T][h_q]).
    """
    T, h_q, d = q.shape
    N, h_kv, dk = k.shape
    if dk != d or v.shape != k.shape or h_q % h_kv != 0:
        raise ValueError("dimension mismatch")
    G = h_q // h_kv                       # reading R2: kv_head = h // G
    if key_pos is None:
        key_pos = np.arange(N, dtype=np.int64)
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    q64 = _as_f64(q)
    o = np.zeros((T, h_q, d), dtype=np.float64)
    lse = np.full((T, h_q), NEG_INF, dtype=np.float64)
    for g in range(h_kv):
        og, lg = attention_group(q64[:, g * G:(g + 1) * G, :], k[:, g, :], v[:, g, :],
                                 q_pos, key_pos, scale)
        o[:, g * G:(g + 1) * G, :] = og
        lse[:, g * G:(g + 1) * G] = lg
    return o, lse


def partial(q, k, v, q_pos, shard, key_pos=None, scale: float | None = None):
    """Partial attention of replicated queries over one contiguous KV shard.

    P:597-598: the shard is the key index range [a, b) of the global KV; the
    result is the exact attention restricted to those keys, as (o, lse)
    (reading R6; an empty or fully masked shard gives o = 0, lse = -inf, R7).
    """
    a, b = shard
    N = k.shape[0]
    if key_pos is None:
        key_pos = np.arange(N, dtype=np.int64)
    key_pos = np.asarray(key_pos, dtype=np.int64)
    return attention(q, k[a:b], v[a:b], q_pos, key_pos[a:b], scale)


def merge(parts):
    """Exact merge of partial attention states ("combined using online-softmax").

    parts: sequence of (o [..., d], lse [...]) with identical shapes.
        M   = max_r lse_r
        LSE = M + ln sum_r exp(lse_r - M)
        O   = sum_r exp(lse_r - LSE) * o_r
    A row whose parts all have lse = -inf merges to (0, -inf) (reading R7).
    """
    if len(parts) == 0:
        raise ValueError("empty list")
    os_ = [_as_f64(p[0]) for p in parts]
    ls_ = [_as_f64(p[1]) for p in parts]
    for o_r, l_r in zip(os_, ls_):
        if o_r.shape != os_[0].shape or l_r.shape != ls_[0].shape or o_r.shape[:-1] != l_r.shape:
            raise ValueError("shape mismatch")
    L = np.stack(ls_)                      # [P][...]
    O = np.stack(os_)                      # [P][...][d]
    M = L.max(axis=0)
    empty = np.isneginf(M)
    M_safe = np.where(empty, 0.0, M)
    s = np.exp(L - M_safe).sum(axis=0)
    with np.errstate(divide="ignore"):
        lse = np.where(empty, NEG_INF, M_safe + np.log(np.where(empty, 1.0, s)))
    wts = np.exp(L - np.where(empty, 0.0, lse))   # exp(-inf) = 0 for empty parts
    wts = np.where(empty[None], 0.0, wts)
    o = (wts[..., None] * O).sum(axis=0)
    return o, lse
