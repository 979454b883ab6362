python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all3.log 2>&1; echo pytest rc=$?
tail -n 30 gpurun_out/pytest_all3.log
