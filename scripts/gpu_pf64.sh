# c = 64 at a 128K prefix: launch list (prefill vs split merge) + one full ncu capture
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python scripts/prefill_one.py --prefix 131072 --c 64 --iters 5 > gpurun_out/plain64.log 2>&1 || exit 1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/pf64_launches.csv python scripts/prefill_one.py --prefix 131072 --c 64 --iters 5 > /dev/null 2>&1; echo launches rc=$?
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:prefill_ws -s 2 -c 1 -o gpurun_out/pf64_full python scripts/prefill_one.py --prefix 131072 --c 64 --iters 3 > gpurun_out/ncu64.log 2>&1; echo ncu rc=$?
