python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_kvp_multi.py -q > gpurun_out/pytest_multi_ext.log 2>&1; echo rc=$?
grep -E "passed|failed|FAIL" gpurun_out/pytest_multi_ext.log | cut -c1-400 | head
