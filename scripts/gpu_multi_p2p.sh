python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
NG=$(nvidia-smi -L | wc -l)
timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 tests/kvp_worker.py > gpurun_out/kvp_worker.log 2>&1; echo worker rc=$?
grep FAIL gpurun_out/kvp_worker.log | head -3
for N in 2 4; do
  [ $N -gt $NG ] && continue
  for mode in fused nccl; do
    if [ $mode = nccl ]; then export MEDHA_BENCH_NCCL=1; else unset MEDHA_BENCH_NCCL; fi
    timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N bench.py --gpus $N --steps 200 --warmup 20 > gpurun_out/bench_${mode}_n$N.json 2>/dev/null; echo N=$N $mode rc=$?
    grep -o '"value": [0-9.]*\|"ms_per_step": [0-9.]*\|"kernel_ms": [0-9.]*\|"kvp_exchange": "[a-zA-Z -]*"' gpurun_out/bench_${mode}_n$N.json | tr '\n' ' '; echo
  done
done
