"""Build libmedha_attn.so in-tree for sm_100a (nvcc, no JIT cache).

    python paper_2409_17264_b200/build.py [--verbose]   (the package itself needs the .so to import)

The .so lands next to this file, so it travels to the GPU box with the repo
snapshot.  NCCL comes from the torch-bundled nvidia-nccl wheel (same image on
the GPU box), linked by soname with an rpath.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmedha_attn.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl  # torch's bundled NCCL
    base = os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) else list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return [os.path.join(CSRC, "medha_attn.cu")]


def deps():
    out = [os.path.join(ROOT, "include", "medha_attn.h")]
    for f in os.listdir(CSRC):
        if f.endswith((".cu", ".cuh", ".h")):
            out.append(os.path.join(CSRC, f))
    return out


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(verbose: bool = False, force: bool = False, ptxas_v: bool = False, out: str = None,
          defines=()) -> str:
    """Build the library (default: in-tree LIB).  `out`/`defines` build an experiment
    variant elsewhere (e.g. build/variant.so with -DMEDHA_...); the product is LIB."""
    lib_path = out or LIB
    if not force and out is None and up_to_date():
        return LIB
    inc, lib = nccl_dirs()
    cmd = [NVCC, *ARCH, "-O3", "-std=c++17", "-lineinfo", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=default", "--expt-relaxed-constexpr",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
           *[f"-D{d}" for d in defines], *sources(), "-o", lib_path + ".tmp",
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}"]
    if ptxas_v:
        cmd[1:1] = ["-Xptxas", "-v"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libmedha_attn.so")
    if verbose or ptxas_v:
        sys.stderr.write(r.stdout + r.stderr)
    os.replace(lib_path + ".tmp", lib_path)
    return lib_path


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    defs = []
    for a in args:
        if a.startswith("--out="):
            out = os.path.abspath(a[6:])
            os.makedirs(os.path.dirname(out), exist_ok=True)
        elif a.startswith("-D"):
            defs.append(a[2:])
    print(build(verbose="--verbose" in args, force=True, ptxas_v="--ptxas" in args, out=out, defines=defs))
