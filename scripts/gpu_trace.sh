python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
MEDHA_LIB_PATH=$PWD/build/dtrace.so timeout -s KILL 300 python scripts/decode_trace.py 2>&1 | grep tokens
