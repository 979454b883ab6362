python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
MEDHA_LIB_PATH=$PWD/build/v_split.so timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_paged.py -q -x -k "prefill or ppb" > gpurun_out/split_tests.log 2>&1; rc=$?; echo tests rc=$rc; tail -n 5 gpurun_out/split_tests.log
if [ $rc -eq 0 ]; then bash scripts/gpu_ab2.sh 131072,1048576 64,256,1024,4096 build/v_base.so build/v_split.so build/v_base.so build/v_split.so; fi
