"""Thin Python binding of libmedha_attn (C ABI in include/medha_attn.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  PyTorch supplies device memory (tensor.data_ptr()), the current
stream and the process group used to ship the NCCL unique id.  There is no CPU
or PyTorch fallback: if the extension is missing, importing this package
raises.

Names follow the C ABI: kv_append, attn_decode_partial,
attn_prefill_chunk, merge_partials, kvp_decode, kvp_prefill_chunk,
decode_step_host.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import List, Optional, Sequence

import torch

__all__ = ["lib", "MedhaError", "KVShard", "kv_append", "attn_decode_partial", "attn_decode_append",
           "kvp_decode_append", "attn_prefill_chunk", "DecodePlan",
           "merge_partials", "KVPComm", "kvp_decode", "kvp_exchange_merge", "exchange_workspace", "kvp_prefill_chunk", "decode_step_host",
           "hbm_read_probe", "decode_workspace", "prefill_workspace", "kvp_workspace", "LIB_PATH"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmedha_attn.so")
if os.environ.get("MEDHA_LIB_PATH"):          # experiment variants built by build.py --out=...
    LIB_PATH = os.environ["MEDHA_LIB_PATH"]
if not os.path.exists(LIB_PATH):
    raise ImportError(f"libmedha_attn.so not built at {LIB_PATH}; run `python -m paper_2409_17264_b200.build` "
                      "(there is no CPU fallback)")
lib = ctypes.CDLL(LIB_PATH)


class _Shard(ctypes.Structure):
    _fields_ = [("k", ctypes.c_void_p), ("v", ctypes.c_void_p), ("capacity", ctypes.c_int64),
                ("len", ctypes.c_int64), ("pos0", ctypes.c_int64), ("h_kv", ctypes.c_int32),
                ("d", ctypes.c_int32), ("page_table", ctypes.c_void_p), ("page_size", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("pool_tokens", ctypes.c_int64)]


_vp, _i32, _i64, _f32, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_size_t
_P = ctypes.POINTER


def _sig(name, restype, *argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = list(argtypes)
    return fn


_sig("medha_status_str", ctypes.c_char_p, _i32)
_sig("medha_last_error", ctypes.c_char_p)
_sig("medha_version", _i32)
_sig("medha_kv_append", _i32, _P(_Shard), _vp, _vp, _i64, _vp)
_sig("medha_decode_workspace_size", _sz, _i32, _i32, _i32, _i32)
_sig("medha_attn_decode_partial", _i32, _P(_Shard), _i32, _vp, _i32, _P(_i64), _f32, _vp, _vp, _vp, _sz, _vp)
_sig("medha_prefill_workspace_size", _sz, _i64, _i32, _i32, _i32)
_sig("medha_attn_prefill_chunk", _i32, _P(_Shard), _vp, _i64, _i32, _i64, _f32, _vp, _vp, _vp, _sz, _vp)
_sig("medha_merge_partials", _i32, _vp, _i32, _i64, _i32, _vp, _vp, _vp, _vp)
_sig("medha_kvp_unique_id", _i32, _vp)
_sig("medha_kvp_comm_create", _i32, _vp, _i32, _i32, _P(_vp))
_sig("medha_kvp_comm_destroy", _i32, _vp)
_sig("medha_kvp_comm_info", _i32, _vp, _P(_i32), _P(_i32))
_sig("medha_kvp_comm_p2p", _i32, _vp)
_sig("medha_kvp_comm_set_p2p", _i32, _vp, _i32)
_sig("medha_kvp_comm_status", _i32, _vp)
_sig("medha_kvp_comm_set_timeout", _i32, _vp, ctypes.c_uint64)
_sig("medha_kvp_comm_debug", _i32, _vp, ctypes.c_uint32)
_sig("medha_kvp_workspace_size", _sz, _i32, _i32, _i32, _i32, _i32)
_sig("medha_kvp_decode", _i32, _vp, _P(_Shard), _i32, _vp, _i32, _P(_i64), _f32, _vp, _vp, _vp, _vp, _sz, _vp)
_sig("medha_kvp_exchange_workspace_size", _sz, _i32, _i64, _i32)
_sig("medha_kvp_exchange_merge", _i32, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _sz, _vp)
_sig("medha_kvp_prefill_workspace_size", _sz, _i32, _i64, _i32, _i32, _i32)
_sig("medha_kvp_prefill_chunk", _i32, _vp, _P(_Shard), _vp, _i64, _i32, _i64, _f32, _vp, _vp, _vp, _vp, _sz, _vp)
_sig("medha_decode_step_workspace_size", _sz, _i32, _i32, _i32, _i32)
_sig("medha_decode_step_host", _i32, _vp, _P(_Shard), _i32, _vp, _vp, _vp, _i32, _i64, _f32, _vp, _vp, _vp, _sz,
     _vp)
_sig("medha_attn_decode_append", _i32, _P(_Shard), _i32, _vp, _vp, _vp, _vp, _i32, _P(_i64), _f32, _vp, _vp, _vp, _sz, _vp)
_sig("medha_kvp_decode_append", _i32, _vp, _P(_Shard), _i32, _vp, _vp, _vp, _vp, _i32, _P(_i64), _f32, _vp, _vp, _vp,
     _vp, _sz, _vp)
_sig("medha_decode_step_dev", _i32, _P(_Shard), _i32, _vp, _vp, _vp, _i32, _vp, _f32, _vp, _vp, _vp, _sz, _vp)
_sig("medha_hbm_read_probe", _i32, _vp, _sz, _vp, _vp)


class MedhaError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        name = lib.medha_status_str(status).decode()
        detail = lib.medha_last_error().decode()
        super().__init__(f"{where}: {name} ({status}): {detail}")


def _check(status: int, where: str):
    if status != 0:
        raise MedhaError(status, where)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:   # raw handle of the current stream, without building a Stream object
        return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch.cuda.current_device()))
    return ctypes.c_void_p(stream.cuda_stream)


def _need_cuda(t: torch.Tensor, name: str, dtype=None):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


class KVShard:
    """One KVP shard of one sequence: bf16 k, v [h_kv][capacity][d] on the GPU.

    Local token j holds absolute position pos0 + j; `len` tokens are valid.
    Paged: `KVShard.paged(pool_k, pool_v, page_table, page_size)` — k, v are
    page pools [h_kv][pool_tokens][d] shared by many shards and local token j lives at pool
    row page_table[j // page_size] * page_size + j % page_size (include/medha_attn.h).
    """

    def __init__(self, k: torch.Tensor, v: torch.Tensor, length: int = 0, pos0: int = 0):
        _need_cuda(k, "k", torch.bfloat16)
        _need_cuda(v, "v", torch.bfloat16)
        if k.shape != v.shape or k.dim() != 3:
            raise ValueError("k, v must both be [h_kv][capacity][d]")
        self.k, self.v = k, v
        self.h_kv, self.capacity, self.d = k.shape
        self.len = int(length)
        self.pos0 = int(pos0)
        self.page_table, self.page_size, self.pool_tokens = None, 0, 0

    @classmethod
    def empty(cls, h_kv: int, capacity: int, d: int, pos0: int = 0, device=None):
        k = torch.empty((h_kv, capacity, d), dtype=torch.bfloat16, device=device or "cuda")
        v = torch.empty_like(k)
        return cls(k, v, 0, pos0)

    @classmethod
    def paged(cls, pool_k: torch.Tensor, pool_v: torch.Tensor, page_table: torch.Tensor, page_size: int,
              length: int = 0, pos0: int = 0):
        sh = cls(pool_k, pool_v, length, pos0)
        _need_cuda(page_table, "page_table", torch.int32)
        sh.page_table, sh.page_size, sh.pool_tokens = page_table, int(page_size), sh.capacity
        sh.capacity = page_table.numel() * int(page_size)
        return sh

    def c(self) -> _Shard:
        pt = self.page_table
        return _Shard(self.k.data_ptr(), self.v.data_ptr(), self.capacity, self.len, self.pos0, self.h_kv, self.d,
                      None if pt is None else pt.data_ptr(), self.page_size, 0, self.pool_tokens)


def _shards_c(shards: Sequence[KVShard]):
    arr = (_Shard * len(shards))()
    for i, s in enumerate(shards):
        arr[i] = s.c()
    return arr


def _scale(scale, d):
    return float(scale) if scale is not None else 1.0 / math.sqrt(d)


_WS = {}


def _workspace(kind: str, nbytes: int, device, stream=None) -> torch.Tensor:
    """Cached zero-initialised workspace (the library leaves counters zeroed), one per
    (kind, device, stream): calls that may run concurrently on different streams must not
    share a workspace (include/medha_attn.h)."""
    dev = torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    sid = stream.cuda_stream if stream is not None else torch._C._cuda_getCurrentRawStream(idx)
    key = (kind, idx, sid)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def decode_workspace(batch, h_q, h_kv, d, device=None, stream=None):
    return _workspace("decode", lib.medha_decode_workspace_size(batch, h_q, h_kv, d), device or "cuda", stream)


def prefill_workspace(c, h_q, h_kv, d, device=None, stream=None):
    return _workspace("prefill", lib.medha_prefill_workspace_size(c, h_q, h_kv, d), device or "cuda", stream)


def kvp_workspace(world, batch, h_q, h_kv, d, device=None, stream=None):
    return _workspace("kvp", lib.medha_kvp_workspace_size(world, batch, h_q, h_kv, d), device or "cuda", stream)


def kv_append(shard: KVShard, k_new: torch.Tensor, v_new: torch.Tensor, stream=None) -> None:
    """K1: append token-major bf16 [n][h_kv][d] rows at shard.len (shard.len += n)."""
    _need_cuda(k_new, "k_new", torch.bfloat16)
    _need_cuda(v_new, "v_new", torch.bfloat16)
    n = k_new.shape[0]
    c = shard.c()
    _check(lib.medha_kv_append(ctypes.byref(c), _ptr(k_new), _ptr(v_new), n, _stream(stream)), "kv_append")
    shard.len = c.len


def attn_decode_partial(shards: Sequence[KVShard], q: torch.Tensor, q_pos: Sequence[int], scale=None,
                        o: Optional[torch.Tensor] = None, lse: Optional[torch.Tensor] = None,
                        ws: Optional[torch.Tensor] = None, stream=None):
    """K3+K4: decode partial (o fp32 [B][h_q][d], lse fp32 [B][h_q]) of each sequence over its shard."""
    _need_cuda(q, "q", torch.bfloat16)
    B, h_q, d = q.shape
    if len(shards) != B or len(q_pos) != B:
        raise ValueError("need one shard and one q_pos per sequence")
    if o is None:
        o = torch.empty((B, h_q, d), dtype=torch.float32, device=q.device)
    if lse is None:
        lse = torch.empty((B, h_q), dtype=torch.float32, device=q.device)
    h_kv = shards[0].h_kv
    if ws is None:
        ws = decode_workspace(B, h_q, h_kv, d, q.device, stream)
    qp = (ctypes.c_int64 * B)(*[int(x) for x in q_pos])
    _check(lib.medha_attn_decode_partial(_shards_c(shards), B, _ptr(q), h_q, qp, _scale(scale, d), _ptr(o),
                                         _ptr(lse), _ptr(ws), ws.numel(), _stream(stream)), "attn_decode_partial")
    return o, lse


def _append_mask(shards, append):
    if append is None:
        return None
    if len(append) != len(shards):
        raise ValueError("need one append flag per sequence")
    return (ctypes.c_int32 * len(shards))(*[1 if a else 0 for a in append])


def attn_decode_append(shards: Sequence[KVShard], k_new: torch.Tensor, v_new: torch.Tensor, q: torch.Tensor,
                       q_pos: Sequence[int], append: Optional[Sequence[bool]] = None, scale=None,
                       o: Optional[torch.Tensor] = None, lse: Optional[torch.Tensor] = None,
                       ws: Optional[torch.Tensor] = None, stream=None):
    """K1 + K3 + K4 in one launch: append row b of k_new / v_new (bf16 [B][h_kv][d]) to
    shards[b] (where append[b], default all) and decode; shard.len advances."""
    _need_cuda(q, "q", torch.bfloat16)
    _need_cuda(k_new, "k_new", torch.bfloat16)
    _need_cuda(v_new, "v_new", torch.bfloat16)
    B, h_q, d = q.shape
    if len(shards) != B or len(q_pos) != B:
        raise ValueError("need one shard and one q_pos per sequence")
    if o is None:
        o = torch.empty((B, h_q, d), dtype=torch.float32, device=q.device)
    if lse is None:
        lse = torch.empty((B, h_q), dtype=torch.float32, device=q.device)
    if ws is None:
        ws = decode_workspace(B, h_q, shards[0].h_kv, d, q.device, stream)
    arr = _shards_c(shards)
    qp = (ctypes.c_int64 * B)(*[int(x) for x in q_pos])
    _check(lib.medha_attn_decode_append(arr, B, _ptr(k_new), _ptr(v_new), _append_mask(shards, append), _ptr(q), h_q,
                                        qp, _scale(scale, d), _ptr(o), _ptr(lse), _ptr(ws), ws.numel(),
                                        _stream(stream)), "attn_decode_append")
    for i, sh in enumerate(shards):
        sh.len = arr[i].len
    return o, lse


def attn_prefill_chunk(shard: KVShard, q: torch.Tensor, q_pos0: int, scale=None, o=None, lse=None, ws=None,
                       stream=None):
    """K2: chunk of c query tokens (bf16 [c][h_q][d]) at positions q_pos0.. over the shard."""
    _need_cuda(q, "q", torch.bfloat16)
    c, h_q, d = q.shape
    if o is None:
        o = torch.empty((c, h_q, d), dtype=torch.float32, device=q.device)
    if lse is None:
        lse = torch.empty((c, h_q), dtype=torch.float32, device=q.device)
    if ws is None:
        ws = prefill_workspace(c, h_q, shard.h_kv, d, q.device, stream)
    sh = shard.c()
    _check(lib.medha_attn_prefill_chunk(ctypes.byref(sh), _ptr(q), c, h_q, int(q_pos0), _scale(scale, d), _ptr(o),
                                        _ptr(lse), _ptr(ws), ws.numel(), _stream(stream)), "attn_prefill_chunk")
    return o, lse


class _PrefillChunk(ctypes.Structure):
    _fields_ = [("kv", ctypes.POINTER(_Shard)), ("q", ctypes.c_void_p), ("c", ctypes.c_int64),
                ("q_pos0", ctypes.c_int64), ("o", ctypes.c_void_p), ("lse", ctypes.c_void_p)]


_sig("medha_prefill_batch_workspace_size", _sz, _i32, _P(_i64), _i32, _i32)
_sig("medha_attn_prefill_batch", _i32, _P(_PrefillChunk), _i32, _i32, _f32, _vp, _sz, _vp)


def attn_prefill_batch(shards: Sequence[KVShard], qs: Sequence[torch.Tensor], q_pos0s: Sequence[int], scale=None,
                       ws=None, stream=None):
    """Prefill-prefill batching: chunk i (bf16 [c_i][h_q][d]) at positions
    q_pos0s[i].. over shards[i], all chunks in one launch.  Returns [(o_i, lse_i)]."""
    n = len(shards)
    if len(qs) != n or len(q_pos0s) != n:
        raise ValueError("need one shard, one query block and one q_pos0 per chunk")
    h_q, d = qs[0].shape[1], qs[0].shape[2]
    outs = []
    arr = (_PrefillChunk * n)()
    keep = []
    for i, (sh, q, p0) in enumerate(zip(shards, qs, q_pos0s)):
        _need_cuda(q, f"q[{i}]", torch.bfloat16)
        c = q.shape[0]
        o = torch.empty((c, h_q, d), dtype=torch.float32, device=q.device)
        lse = torch.empty((c, h_q), dtype=torch.float32, device=q.device)
        cs = sh.c()
        keep.append(cs)
        arr[i] = _PrefillChunk(ctypes.pointer(cs), q.data_ptr(), c, int(p0), o.data_ptr(), lse.data_ptr())
        outs.append((o, lse))
    if ws is None:
        cs_arr = (ctypes.c_int64 * n)(*[q.shape[0] for q in qs])
        ws = _workspace("prefill_batch", lib.medha_prefill_batch_workspace_size(n, cs_arr, h_q, d), qs[0].device,
                        stream)
    _check(lib.medha_attn_prefill_batch(arr, n, h_q, _scale(scale, d), _ptr(ws), ws.numel(), _stream(stream)),
           "attn_prefill_batch")
    return outs


def merge_partials(parts: torch.Tensor, rows: int, d: int, want_bf16: bool = False, stream=None):
    """K5: parts fp32 [P][rows*(d+1)] (o then lse per part) -> (o [rows][d], lse [rows], o_bf16|None)."""
    _need_cuda(parts, "parts", torch.float32)
    P = parts.shape[0]
    o = torch.empty((rows, d), dtype=torch.float32, device=parts.device)
    lse = torch.empty((rows,), dtype=torch.float32, device=parts.device)
    ob = torch.empty((rows, d), dtype=torch.bfloat16, device=parts.device) if want_bf16 else None
    _check(lib.medha_merge_partials(_ptr(parts), P, rows, d, _ptr(o), _ptr(lse), _ptr(ob), _stream(stream)),
           "merge_partials")
    return o, lse, ob


class KVPComm:
    """NCCL communicator of one KVP group, bootstrapped over torch.distributed.

    Rank 0 creates the 128-byte NCCL unique id and ships it through the
    process group (works with gloo or nccl); every rank then creates the
    communicator on its current CUDA device.
    """

    def __init__(self, group=None, _single=False):
        if _single:       # a one-rank group, no process group needed (KVPComm.single())
            self.rank, self.world = 0, 1
            uid = (ctypes.c_uint8 * 128)()
            _check(lib.medha_kvp_unique_id(uid), "kvp_unique_id")
        else:
            import torch.distributed as dist
            from .kvp import exchange_unique_id
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
            uid = (ctypes.c_uint8 * 128).from_buffer_copy(exchange_unique_id(group))
        h = ctypes.c_void_p()
        _check(lib.medha_kvp_comm_create(uid, self.rank, self.world, ctypes.byref(h)), "kvp_comm_create")
        self.handle = h

    @classmethod
    def single(cls) -> "KVPComm":
        """A KVP group of one rank on the current device (world 1): the full KVP path
        (fused self-exchange or NCCL all-gather of one part, then the merge) on one GPU."""
        return cls(_single=True)

    def status(self) -> int:
        """medha_kvp_comm_status: 0, or MEDHA_ENCCL (-7) once a fused-exchange wait timed out."""
        return int(lib.medha_kvp_comm_status(self.handle))

    def set_timeout(self, seconds: float) -> None:
        """Bound of the in-kernel wait for peers' partials (default 30 s)."""
        _check(lib.medha_kvp_comm_set_timeout(self.handle, int(seconds * 1e9)), "kvp_comm_set_timeout")

    def debug(self, flags: int) -> None:
        """Test hook (medha_kvp_comm_debug): 1 = this rank withholds its exchange pushes."""
        _check(lib.medha_kvp_comm_debug(self.handle, int(flags)), "kvp_comm_debug")

    @property
    def p2p(self) -> bool:
        """True when kvp_decode runs the fused NVLink exchange inside the decode kernel."""
        return bool(lib.medha_kvp_comm_p2p(self.handle))

    def set_p2p(self, enable: bool) -> None:
        """Switch between the fused NVLink exchange and NCCL all-gather + merge (collective:
        call identically on every rank)."""
        _check(lib.medha_kvp_comm_set_p2p(self.handle, int(bool(enable))), "kvp_comm_set_p2p")

    def close(self):
        if self.handle:
            _check(lib.medha_kvp_comm_destroy(self.handle), "kvp_comm_destroy")
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def kvp_decode(comm: KVPComm, shards: Sequence[KVShard], q: torch.Tensor, q_pos: Sequence[int], scale=None,
               want_bf16=False, ws=None, stream=None, o=None, lse=None):
    """Eq. 5: local partial + exchange (fused NVLink push inside the decode kernel when
    comm.p2p, else NCCL all-gather + merge kernel) + rank-ordered LSE merge; identical on
    all ranks."""
    _need_cuda(q, "q", torch.bfloat16)
    B, h_q, d = q.shape
    if o is None:
        o = torch.empty((B, h_q, d), dtype=torch.float32, device=q.device)
    if lse is None:
        lse = torch.empty((B, h_q), dtype=torch.float32, device=q.device)
    ob = torch.empty((B, h_q, d), dtype=torch.bfloat16, device=q.device) if want_bf16 else None
    if ws is None:
        ws = kvp_workspace(comm.world, B, h_q, shards[0].h_kv, d, q.device, stream)
    qp = (ctypes.c_int64 * B)(*[int(x) for x in q_pos])
    _check(lib.medha_kvp_decode(comm.handle, _shards_c(shards), B, _ptr(q), h_q, qp, _scale(scale, d), _ptr(o),
                                _ptr(lse), _ptr(ob), _ptr(ws), ws.numel(), _stream(stream)), "kvp_decode")
    return o, lse, ob


def kvp_decode_append(comm: KVPComm, shards: Sequence[KVShard], k_new: torch.Tensor, v_new: torch.Tensor,
                      q: torch.Tensor, q_pos: Sequence[int], append: Optional[Sequence[bool]] = None, scale=None,
                      want_bf16=False, ws=None, stream=None, o=None, lse=None):
    """kvp_decode with the new token appended in the same launch where append[b] (default
    all; typically this rank holds sequence b's tail)."""
    _need_cuda(q, "q", torch.bfloat16)
    _need_cuda(k_new, "k_new", torch.bfloat16)
    _need_cuda(v_new, "v_new", torch.bfloat16)
    B, h_q, d = q.shape
    if o is None:
        o = torch.empty((B, h_q, d), dtype=torch.float32, device=q.device)
    if lse is None:
        lse = torch.empty((B, h_q), dtype=torch.float32, device=q.device)
    ob = torch.empty((B, h_q, d), dtype=torch.bfloat16, device=q.device) if want_bf16 else None
    if ws is None:
        ws = kvp_workspace(comm.world, B, h_q, shards[0].h_kv, d, q.device, stream)
    arr = _shards_c(shards)
    qp = (ctypes.c_int64 * B)(*[int(x) for x in q_pos])
    _check(lib.medha_kvp_decode_append(comm.handle, arr, B, _ptr(k_new), _ptr(v_new), _append_mask(shards, append),
                                       _ptr(q), h_q, qp, _scale(scale, d), _ptr(o), _ptr(lse), _ptr(ob), _ptr(ws),
                                       ws.numel(), _stream(stream)), "kvp_decode_append")
    for i, sh in enumerate(shards):
        sh.len = arr[i].len
    return o, lse, ob


def exchange_workspace(world, rows, d, device=None, stream=None):
    return _workspace(f"xchg{world}", lib.medha_kvp_exchange_workspace_size(world, rows, d), device or "cuda", stream)


def kvp_exchange_merge(comm: KVPComm, send: torch.Tensor, rows: int, d: int, o_out: torch.Tensor,
                       lse_out: Optional[torch.Tensor] = None, o_bf16: Optional[torch.Tensor] = None, ws=None,
                       stream=None) -> None:
    """a6 + a7: all-gather this rank's packed (o, lse) partial and merge in rank order."""
    _need_cuda(send, "send", torch.float32)
    if ws is None:
        ws = exchange_workspace(comm.world, rows, d, send.device, stream)
    _check(lib.medha_kvp_exchange_merge(comm.handle, _ptr(send), rows, d, _ptr(o_out), _ptr(lse_out), _ptr(o_bf16),
                                        _ptr(ws), ws.numel(), _stream(stream)), "kvp_exchange_merge")


def kvp_prefill_chunk(comm: KVPComm, shard: KVShard, q: torch.Tensor, q_pos0: int, scale=None, want_bf16=False,
                      ws=None, stream=None):
    """Eq. 6: prefill chunk under KVP (each rank over its shard, then all-gather + merge)."""
    _need_cuda(q, "q", torch.bfloat16)
    c, h_q, d = q.shape
    o = torch.empty((c, h_q, d), dtype=torch.float32, device=q.device)
    lse = torch.empty((c, h_q), dtype=torch.float32, device=q.device)
    ob = torch.empty((c, h_q, d), dtype=torch.bfloat16, device=q.device) if want_bf16 else None
    if ws is None:
        ws = _workspace("kvp_prefill", lib.medha_kvp_prefill_workspace_size(comm.world, c, h_q, shard.h_kv, d),
                        q.device, stream)
    sh = shard.c()
    _check(lib.medha_kvp_prefill_chunk(comm.handle, ctypes.byref(sh), _ptr(q), c, h_q, int(q_pos0), _scale(scale, d),
                                       _ptr(o), _ptr(lse), _ptr(ob), _ptr(ws), ws.numel(), _stream(stream)),
           "kvp_prefill_chunk")
    return o, lse, ob


def decode_step_host(comm: Optional[KVPComm], shard: KVShard, append: bool, q_host: torch.Tensor,
                     k_host: Optional[torch.Tensor], v_host: Optional[torch.Tensor], q_pos: int,
                     o_host: torch.Tensor, lse_host: Optional[torch.Tensor], ws: torch.Tensor, scale=None,
                     stream=None) -> None:
    """End-to-end decode step with host (pinned) buffers; async on the stream."""
    h_q, d = q_host.shape
    sh = shard.c()
    _check(lib.medha_decode_step_host(comm.handle if comm is not None else None, ctypes.byref(sh), int(bool(append)),
                                      _ptr(q_host), _ptr(k_host), _ptr(v_host), h_q, int(q_pos), _scale(scale, d),
                                      _ptr(o_host), _ptr(lse_host), _ptr(ws), ws.numel(), _stream(stream)),
           "decode_step_host")
    shard.len = sh.len


_sig("medha_decode_plan_create", _i32, _vp, _P(_Shard), _i32, _f32, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _P(_vp))
_sig("medha_decode_plan_step", _i32, _vp, _P(_Shard), _i32, _i64, _vp)
_sig("medha_decode_plan_destroy", _i32, _vp)


class DecodePlan:
    """Prepared decode_step_host (include/medha_attn.h `medha_decode_plan_*`): the host
    buffers, communicator, shard geometry and workspace are resolved once; each step() is
    one C call that launches the step (no per-step pointer queries or argument re-checks
    beyond the shard).  The tensors passed here must stay alive with the plan; step() takes
    the same shard (its len advances) every time."""

    def __init__(self, comm: Optional["KVPComm"], shard: KVShard, q_host: torch.Tensor,
                 k_host: Optional[torch.Tensor], v_host: Optional[torch.Tensor], o_host: torch.Tensor,
                 lse_host: Optional[torch.Tensor], ws: torch.Tensor, scale=None):
        h_q, d = q_host.shape
        self._keep = (comm, q_host, k_host, v_host, o_host, lse_host, ws)
        self._sh = shard.c()
        h = ctypes.c_void_p()
        _check(lib.medha_decode_plan_create(comm.handle if comm is not None else None, ctypes.byref(self._sh), h_q,
                                            _scale(scale, d), _ptr(q_host), _ptr(k_host), _ptr(v_host), _ptr(o_host),
                                            _ptr(lse_host), _ptr(ws), ws.numel(), ctypes.byref(h)), "decode_plan_create")
        self.handle = h
        self._step = lib.medha_decode_plan_step
        self._shref = ctypes.byref(self._sh)

    def step(self, shard: KVShard, append: bool, q_pos: int, stream=None) -> None:
        """One decode step (async on the stream; outputs valid after it is synchronised)."""
        sh = self._sh                # the plan's shard struct: same k / v / capacity / pos0
        sh.len = shard.len
        rc = self._step(self.handle, self._shref, 1 if append else 0, q_pos, _stream(stream))
        if rc:
            raise MedhaError(rc, "decode_plan_step")
        shard.len = sh.len

    def close(self):
        if self.handle:
            lib.medha_decode_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def decode_step_workspace(world, h_q, h_kv, d, device=None, stream=None):
    return _workspace(f"step{world}", lib.medha_decode_step_workspace_size(world, h_q, h_kv, d), device or "cuda",
                      stream)


def decode_step_dev(shards: Sequence[KVShard], k_new: torch.Tensor, v_new: torch.Tensor, q: torch.Tensor,
                    len_dev: torch.Tensor, o: torch.Tensor, lse: torch.Tensor, ws: torch.Tensor, scale=None,
                    stream=None) -> None:
    """Graph-capturable decode step with device-side lengths (include/medha_attn.h): append
    k_new/v_new [B][h_kv][d] at len_dev[b], attend keys 0..len_dev[b], then len_dev += 1.
    Host shard lengths are neither read nor updated."""
    _need_cuda(k_new, "k_new", torch.bfloat16)
    _need_cuda(v_new, "v_new", torch.bfloat16)
    _need_cuda(q, "q", torch.bfloat16)
    _need_cuda(len_dev, "len_dev", torch.int64)
    B, h_q, d = q.shape
    arr = _shards_c(shards)
    _check(lib.medha_decode_step_dev(arr, B, _ptr(k_new), _ptr(v_new), _ptr(q), h_q, _ptr(len_dev), _scale(scale, d),
                                     _ptr(o), _ptr(lse), _ptr(ws), ws.numel(), _stream(stream)), "decode_step_dev")


def hbm_read_probe(src: torch.Tensor, sink: torch.Tensor, stream=None) -> None:
    _check(lib.medha_hbm_read_probe(_ptr(src), src.numel() * src.element_size(), _ptr(sink), _stream(stream)),
           "hbm_read_probe")
