"""KVP host-side helpers: the sequence partition of the KV cache over the
ranks of a KVP group and the NCCL unique-id bootstrap over torch.distributed.

No attention arithmetic here; the device work is in libmedha_attn.
"""
from __future__ import annotations

import ctypes

__all__ = ["shard_range", "exchange_unique_id"]


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
