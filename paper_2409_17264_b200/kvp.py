"""KVP host-side helpers: the sequence partition of the KV cache over the
ranks of a KVP group and the NCCL unique-id bootstrap over torch.distributed.

No attention arithmetic here; the device work is in libmedha_attn.
"""
from __future__ import annotations

import ctypes

__all__ = ["shard_range", "exchange_unique_id", "growth_placement", "KVPGrowingSequence"]


def shard_range(n_total: int, rank: int, world: int):
    """Contiguous token slice [a, b) of rank `rank` (reading R14: equal slices
    [r N/P, (r+1) N/P); any contiguous partition is exact)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"rank {rank} / world {world}")
    return n_total * rank // world, n_total * (rank + 1) // world


def exchange_unique_id(group=None) -> bytes:
    """Rank 0 of `group` creates the 128-byte NCCL unique id (medha_kvp_unique_id) and
    broadcasts it over the process group (any backend, gloo included)."""
    import torch.distributed as dist
    from . import lib, _check
    rank = dist.get_rank(group)
    buf = (ctypes.c_uint8 * 128)()
    if rank == 0:
        _check(lib.medha_kvp_unique_id(buf), "kvp_unique_id")
    obj = [bytes(buf)]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def growth_placement(n_tokens: int, token_limit: int, world: int):
    """Dynamic KVP worker allocation ("Each request starts with one worker, and
    workers are added once we exceed the worker KV-cache token limit"): rank r holds the
    absolute tokens [r L, min((r+1) L, n)); ranks past ceil(n / L) hold nothing yet.
    Returns [(a, b)] per rank (empty ranges as (a, a))."""
    if token_limit < 1 or world < 1:
        raise ValueError("token_limit and world must be >= 1")
    if n_tokens > token_limit * world:
        raise ValueError(f"{n_tokens} tokens exceed {world} workers x {token_limit}")
    out = []
    for r in range(world):
        a = min(n_tokens, r * token_limit)
        b = min(n_tokens, (r + 1) * token_limit)
        out.append((a, b))
    return out


class KVPGrowingSequence:
    """One sequence's KV under dynamic KVP growth on this rank (every rank of the KVP
    group holds one instance).  Rank r owns the absolute positions [r L, (r+1) L); new
    tokens are appended in order by whichever rank owns their positions (a chunk that
    crosses a boundary is split), so the worker set grows as the sequence does.  Ranks
    that own no token yet contribute the empty partial (o = 0, lse = -inf, reading R7)
    to the exact merge.  Collective-free on the append path: every rank sees the same
    token stream and keeps only its own positions."""

    def __init__(self, rank: int, world: int, token_limit: int, h_kv: int, d: int, device=None):
        from . import KVShard
        self.rank, self.world, self.limit = rank, world, token_limit
        self.n = 0                                     # global tokens so far
        self.shard = KVShard.empty(h_kv, token_limit, d, pos0=rank * token_limit, device=device)

    @property
    def active_workers(self) -> int:
        return max(1, -(-self.n // self.limit))

    def append(self, k_new, v_new, stream=None) -> None:
        """Append token-major [n][h_kv][d] rows (the same rows on every rank)."""
        from . import kv_append
        m = k_new.shape[0]
        if self.n + m > self.limit * self.world:
            raise ValueError("sequence exceeds the KVP group's capacity")
        lo, hi = self.rank * self.limit, (self.rank + 1) * self.limit
        a, b = max(lo, self.n), min(hi, self.n + m)
        if a < b:
            kv_append(self.shard, k_new[a - self.n:b - self.n].contiguous(), v_new[a - self.n:b - self.n].contiguous(),
                      stream=stream)
        self.n += m
