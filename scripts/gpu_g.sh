python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
cd scripts
for v in dec_pp0 dec_pp1 dec_pp0 dec_pp1; do echo "== $v"; MEDHA_LIB_PATH=$PWD/../build/$v.so timeout -s KILL 300 python decode_g.py | head -1; done
