python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_fuzz.py -q > gpurun_out/pytest_fuzz.log 2>&1; echo rc=$?
grep -E "passed|failed|AssertionError|Error" gpurun_out/pytest_fuzz.log | head -12
