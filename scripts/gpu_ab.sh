# same-box A/B of experiment variants: bash scripts/gpu_ab.sh build/v_a.so build/v_b.so ...
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for v in "$@"; do
  MEDHA_LIB_PATH=$PWD/$v timeout -s KILL 300 python scripts/prefill_sweep.py 131072,1048576 64,256,1024,4096 $(basename $v) 2>&1 | grep -v Warn
done
