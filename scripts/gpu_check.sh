set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout -s KILL 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not prefill" > gpurun_out/pytest_decode.log 2>&1; echo pytest decode rc=$?
timeout -s KILL 600 python -m pytest tests -m gpu -q -k "prefill" > gpurun_out/pytest_prefill.log 2>&1; echo pytest prefill rc=$?
tail -5 gpurun_out/smoke.log gpurun_out/pytest_decode.log gpurun_out/pytest_prefill.log
