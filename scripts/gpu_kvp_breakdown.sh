python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for n in 2 4; do
  timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n scripts/kvp_breakdown.py 2>&1 | grep '"world"'
  KVP_TOKENS=262144 timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n scripts/kvp_breakdown.py 2>&1 | grep '"world"'
done
