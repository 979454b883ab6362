#!/bin/bash
# build_variant.sh <git-rev> <out.so> [-DFOO=1 ...]: build libmedha_attn from the csrc of <git-rev> (same-box A/B)
set -e
rev=$1; out=$2; shift 2
tmp=$(mktemp -d)
git archive "$rev" paper_2409_17264_b200/csrc include | tar -x -C "$tmp"
NCCL=$(python -c "import nvidia.nccl,os;print(list(nvidia.nccl.__path__)[0])")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -shared -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I "$tmp/include" -I "$tmp/paper_2409_17264_b200/csrc" -I "$NCCL/include" "$@" \
  "$tmp/paper_2409_17264_b200/csrc/medha_attn.cu" -o "$out" -L "$NCCL/lib" -l:libnccl.so.2 -Xlinker -rpath,"$NCCL/lib"
rm -rf "$tmp"; echo "$out"
