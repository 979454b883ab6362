python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python scripts/prefill_one.py --prefix 131072 --c 1024 > gpurun_out/plain_pre.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:prefill_ws -s 1 -c 1 -o gpurun_out/r01_prefill_v2_128k python scripts/prefill_one.py --prefix 131072 --c 1024 > gpurun_out/ncu_pre2.log 2>&1; echo ncu1 rc=$?
python scripts/prefill_one.py --prefix 1048576 --c 1024 > gpurun_out/plain_pre1m.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:prefill_ws -s 1 -c 1 -o gpurun_out/r01_prefill_v2_1m python scripts/prefill_one.py --prefix 1048576 --c 1024 > gpurun_out/ncu_pre3.log 2>&1; echo ncu2 rc=$?
