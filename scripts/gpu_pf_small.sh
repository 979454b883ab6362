python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python scripts/prefill_one.py --prefix 131072 --c 64 --iters 5 > gpurun_out/plain_pre64.log 2>&1 && \
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches_pre64.csv python scripts/prefill_one.py --prefix 131072 --c 64 --iters 5 > /dev/null 2>&1; echo rc=$?
grep -E "medha" gpurun_out/launches_pre64.csv | awk -F'","' '{print $5, $13, $15}' | tail -12
