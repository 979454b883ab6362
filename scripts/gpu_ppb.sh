python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -q -x -k "prefill or ppb or smoke" > gpurun_out/pytest_ppb.log 2>&1; echo rc=$?
grep -E "passed|failed|Error|error" gpurun_out/pytest_ppb.log | head -8
timeout -s KILL 300 python scripts/prefill_sweep.py 131072,1048576 64,256,1024,4096 2>&1 | grep -v Warn
