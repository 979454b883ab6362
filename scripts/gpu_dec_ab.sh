python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_dec.log 2>&1; echo pytest rc=$?; tail -n 2 gpurun_out/pytest_dec.log
for v in "$@"; do echo "== $v"; MEDHA_LIB_PATH=$PWD/$v timeout -s KILL 300 python scripts/decode_micro.py 2>&1 | grep decode_us; done
MEDHA_LIB_PATH=$PWD/build/dtrace.so timeout -s KILL 300 python scripts/decode_trace.py 2>&1 | grep tokens
