"""CPU-only checks of the C ABI library: it builds, loads without a GPU, and
exports every function include/medha_attn.h declares (no compute calls)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "medha_attn.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(medha_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for want in ("medha_kv_append", "medha_attn_prefill_chunk", "medha_attn_decode_partial",
                 "medha_merge_partials", "medha_kvp_decode"):
        assert want in names


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2409_17264_b200 import LIB_PATH as path
    lib = ctypes.CDLL(path)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, f"not exported: {missing}"
    # and they are real dynamic symbols of the .so (not resolved from elsewhere)
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    for n in declared_functions():
        assert re.search(rf"\bT {n}\b", out), n


def test_status_strings_without_gpu():
    from paper_2409_17264_b200 import lib
    assert lib.medha_status_str(0) == b"MEDHA_OK"
    assert lib.medha_status_str(-7) == b"MEDHA_ENCCL"
    assert lib.medha_version() >> 16 == 1
    # workspace sizing is pure host arithmetic
    assert lib.medha_decode_workspace_size(1, 32, 8, 128) > 0
    assert lib.medha_kvp_workspace_size(8, 1, 32, 8, 128) > lib.medha_decode_workspace_size(1, 32, 8, 128)


def test_kernels_are_sm100a_and_use_tcgen05_tma():
    """The fatbin holds sm_100a SASS; the prefill kernel uses UTCHMMA (tcgen05.mma),
    LDTM/STTM (tcgen05.ld/st) and UTMALDG (TMA)."""
    from paper_2409_17264_b200 import LIB_PATH as path
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    assert "UTCHMMA" in sass or "UTCMMA" in sass
    assert "UTMALDG" in sass
    assert "LDTM" in sass
    assert "HMMA" in sass  # decode dot products


def test_shard_struct_layout_matches_binding(tmp_path):
    """The ctypes mirror of medha_kv_shard (incl. the paged-KV fields) has the header's
    size and field offsets, as compiled by the C compiler."""
    from paper_2409_17264_b200 import _Shard
    fields = [f for f, _ in _Shard._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "medha_attn.h"\nint main(void){\n'
                   + 'printf("%zu\\n", sizeof(medha_kv_shard));\n'
                   + "".join(f'printf("%zu\\n", offsetof(medha_kv_shard, {f}));\n' for f in fields) + "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got[0] == ctypes.sizeof(_Shard)
    assert got[1:] == [getattr(_Shard, f).offset for f in fields]


def test_argument_errors_are_caught_on_the_host_without_gpu():
    """Validation that precedes any CUDA call (round-2 entry points included): null or bad
    arguments return the documented status and a message; nothing is launched."""
    from paper_2409_17264_b200 import lib, _Shard
    EINVAL, ERANGE, ENOTSUP, EWS = -1, -3, -4, -5
    sh = _Shard(0, 0, 100, 10, 0, 8, 128, None, 0, 0, 0)            # null k/v pointers
    assert lib.medha_kv_append(ctypes.byref(sh), None, None, 1, None) == EINVAL
    assert b"null" in lib.medha_last_error()
    qp = (ctypes.c_int64 * 1)(5)
    assert lib.medha_attn_decode_append(ctypes.byref(sh), 1, None, None, None, None, 32, qp, 0.1, None, None, None,
                                        0, None) == EINVAL
    # a well-formed but full shard: the fused append reports ERANGE before launching
    full = _Shard(16, 16, 100, 100, 0, 8, 128, None, 0, 0, 0)
    k = (ctypes.c_uint8 * 64)()
    addr = (ctypes.addressof(k) + 15) // 16 * 16
    assert lib.medha_attn_decode_append(ctypes.byref(full), 1, addr, addr, None, addr, 32, qp, 0.1, addr, addr, addr,
                                        1 << 28, None) == ERANGE
    bad_d = _Shard(16, 16, 100, 10, 0, 8, 96, None, 0, 0, 0)        # head dim 96
    assert lib.medha_attn_decode_partial(ctypes.byref(bad_d), 1, addr, 32, qp, 0.1, addr, addr, addr, 1 << 28,
                                         None) == ENOTSUP
    plan = ctypes.c_void_p()
    assert lib.medha_decode_plan_create(None, ctypes.byref(sh), 32, 0.1, None, None, None, None, None, None, 0,
                                        ctypes.byref(plan)) == EINVAL
    good = _Shard(16, 16, 100, 10, 0, 8, 128, None, 0, 0, 0)
    assert lib.medha_decode_plan_create(None, ctypes.byref(good), 32, 0.1, addr, None, None, addr, None, addr, 16,
                                        ctypes.byref(plan)) == EWS
    assert lib.medha_decode_plan_step(None, ctypes.byref(good), 0, 5, None) == EINVAL
    assert lib.medha_kvp_comm_status(None) == EINVAL
    assert lib.medha_kvp_comm_set_timeout(None, 1) == EINVAL
    assert lib.medha_kvp_comm_debug(None, 1) == EINVAL
    assert lib.medha_kvp_decode_append(None, ctypes.byref(good), 1, addr, addr, None, addr, 32, qp, 0.1, addr, addr,
                                       None, addr, 1 << 28, None) == EINVAL
