mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_paged.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_paged.log 2>&1; echo pytest rc=$?
timeout -s KILL 300 python scripts/paged_bench.py > gpurun_out/paged_bench.jsonl 2> gpurun_out/paged_bench.err; echo paged_bench rc=$?
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-extra --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -n 3 gpurun_out/pytest_paged.log; cat gpurun_out/paged_bench.jsonl; tail -n 3 gpurun_out/paged_bench.err; cut -c1-300 gpurun_out/bench.json
