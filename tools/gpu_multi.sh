#!/bin/bash
# Multi-GPU evidence (run under `gpurun --gpus N`): the multigpu pytest workers, bench.py at
# N = 1, 2, 4 (as the driver launches it) and the KVP step breakdown at 2^20 and 2^17 x P tokens.
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_kvp_multi.py -q -m gpu > gpurun_out/pytest_multi.log 2>&1
echo "pytest multi rc=$?"; grep -E "passed|failed" gpurun_out/pytest_multi.log | tail -n 2
for n in 1 2 4; do
  [ $n -gt $N ] && continue
  if [ $n -eq 1 ]; then
    timeout -s KILL 600 python bench.py --no-cpu --steps 50 --warmup 10 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
  else
    timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + n)) bench.py --gpus $n --steps 50 --warmup 10 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  fi
  echo "bench n=$n rc=$?"
done
for n in 2 4; do
  [ $n -gt $N ] && continue
  for tok in 1048576 $((131072 * n)); do
    KVP_TOKENS=$tok timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29600 + n)) tools/kvp_breakdown.py 2>/dev/null | grep world >> gpurun_out/kvp_breakdown.jsonl
  done
done
cat gpurun_out/kvp_breakdown.jsonl
