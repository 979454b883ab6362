python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
nproc; free -g | head -2
( time timeout -s KILL 1500 python -m pytest tests/test_gpu_fullsize.py -q -x --durations=10 ) > gpurun_out/pytest_full.log 2>&1; echo pytest rc=$?
tail -n 20 gpurun_out/pytest_full.log
