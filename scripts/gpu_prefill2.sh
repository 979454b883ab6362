python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests -m gpu -q -k "prefill or smoke or I9 or last_prefill" -x > gpurun_out/pytest_prefill2.log 2>&1; echo pytest rc=$?
tail -n 30 gpurun_out/pytest_prefill2.log
timeout -s KILL 300 python scripts/prefill_sweep.py > gpurun_out/prefill_sweep2.log 2>&1; echo sweep rc=$?
cat gpurun_out/prefill_sweep2.log | tail -n 12
