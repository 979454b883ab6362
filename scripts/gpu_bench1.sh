python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench1.json; tail -n 20 gpurun_out/bench1.err
timeout -s KILL 300 python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/plain_short.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
