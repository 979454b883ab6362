set -x
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_paged.py -x -q > gpurun_out/pytest_paged.log 2>&1; echo paged rc=$?
timeout -s KILL 900 python -m pytest tests -m "gpu and not multigpu" -q -x --ignore=tests/test_gpu_fullsize.py > gpurun_out/pytest_gpu.log 2>&1; echo gpu rc=$?
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -5 gpurun_out/pytest_paged.log gpurun_out/pytest_gpu.log; cut -c1-600 gpurun_out/bench.json
