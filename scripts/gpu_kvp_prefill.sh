python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python scripts/kvp_prefill_sweep.py > gpurun_out/kvp_prefill_p1.jsonl 2>gpurun_out/kvp_prefill_p1.err; echo p1 rc=$?
for N in 2 4; do timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N scripts/kvp_prefill_sweep.py > gpurun_out/kvp_prefill_p$N.jsonl 2>gpurun_out/kvp_prefill_p$N.err; echo p$N rc=$?; done
cat gpurun_out/kvp_prefill_p*.jsonl
