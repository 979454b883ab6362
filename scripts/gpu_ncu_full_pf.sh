mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python scripts/prefill_one.py --prefix 131072 --c 1024 > gpurun_out/plain_pre.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:prefill_ws -s 1 -c 1 -o gpurun_out/r01_final_prefill_full python scripts/prefill_one.py --prefix 131072 --c 1024 > gpurun_out/ncu_pre.log 2>&1; echo ncu-pre rc=$?
