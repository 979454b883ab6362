# ncu evidence for the refreshed round-1 code: launch list of the default bench, full captures of decode and prefill
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -k "growing_max or step_host" > gpurun_out/r1b_newtests.log 2>&1; echo newtests rc=$?; tail -n 2 gpurun_out/r1b_newtests.log
python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/plain_launch.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_splitkv|kv_append|prefill_ws|lse_merge" -c 200 --csv --log-file gpurun_out/r01b_launches.csv python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo ncu-list rc=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:decode_splitkv -s 3 -c 1 -o gpurun_out/r01b_decode_full python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/ncu_dec.log 2>&1; echo ncu-dec rc=$?
python scripts/prefill_one.py --prefix 131072 --c 1024 > gpurun_out/plain_pre.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:prefill_ws -s 1 -c 1 -o gpurun_out/r01b_prefill_full python scripts/prefill_one.py --prefix 131072 --c 1024 > gpurun_out/ncu_pre.log 2>&1; echo ncu-pre rc=$?
for f in r01b_decode_full r01b_prefill_full; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/$f.raw.csv 2>/dev/null; done
rm -f gpurun_out/pf_*.pt
