mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/plain_dec.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:decode_splitkv -s 2 -c 1 -o gpurun_out/r01_final_decode_full python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/ncu_dec.log 2>&1; echo ncu-dec rc=$?
