python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?
python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/plain_short.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo ncu-list rc=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:decode_splitkv -s 3 -c 1 -o gpurun_out/r01_decode_full_v2 python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/ncu_dec2.log 2>&1; echo ncu-full rc=$?
python scripts/prefill_one.py --prefix 131072 --c 1024 > gpurun_out/plain_pre.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:prefill_ws -s 1 -c 1 -o gpurun_out/r01_prefill_v3_128k python scripts/prefill_one.py --prefix 131072 --c 1024 > gpurun_out/ncu_pre4.log 2>&1; echo ncu-pre rc=$?
