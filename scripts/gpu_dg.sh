python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -k "decode or kvp or needle" > gpurun_out/pytest_dg.log 2>&1; echo pytest rc=$?; tail -n 1 gpurun_out/pytest_dg.log
for v in dg_100_1 dg_85_1 dg_85_2 dg_70_2 dg_100_1 dg_85_1 dg_85_2 dg_70_2; do echo "== $v"; MEDHA_LIB_PATH=$PWD/build/$v.so timeout -s KILL 300 python scripts/decode_micro.py 2>&1 | grep decode_us; done
