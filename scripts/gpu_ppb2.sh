python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 300 python scripts/ppb_bench.py 2>&1 | grep chunks | tee gpurun_out/ppb_bench.jsonl
