python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for v in "$@"; do
  MEDHA_LIB_PATH=$PWD/$v timeout -s KILL 300 python scripts/decode_micro.py 2>/dev/null | sed "s/^/$(basename $v) /"
done
