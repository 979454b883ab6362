python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for v in dec_i1 dec_i2 dec_i3 dec_i1 dec_i2 dec_i3; do echo "== $v"; MEDHA_LIB_PATH=$PWD/build/$v.so timeout -s KILL 300 python scripts/decode_micro.py 2>&1 | grep decode_us; done
