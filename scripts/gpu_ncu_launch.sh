mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/plain_launch.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_splitkv|kv_append|prefill_ws|lse_merge" -c 200 --csv --log-file gpurun_out/r01_final_launches.csv python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
timeout -s KILL 300 python bench.py --no-extra --no-cpu --steps 20 --warmup 5 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?; cut -c1-200 gpurun_out/bench_q.json; python -c "import json; d=json.load(open('gpurun_out/bench_q.json')); print(d['roofline'])"
