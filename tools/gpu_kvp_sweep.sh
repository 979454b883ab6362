#!/bin/bash
# SURVEY N4 chunk x KVP prefill sweep at P = 1, 2, 4 (run under `gpurun --gpus 4`)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
rm -f gpurun_out/kvp_prefill_sweep.jsonl
timeout -s KILL 900 python tools/kvp_prefill_sweep.py 2>/dev/null | grep '{' >> gpurun_out/kvp_prefill_sweep.jsonl
for p in 2 4; do
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $p --master-addr 127.0.0.1 \
    --master-port $((29700 + p)) tools/kvp_prefill_sweep.py 2>/dev/null | grep '{' >> gpurun_out/kvp_prefill_sweep.jsonl
done
cat gpurun_out/kvp_prefill_sweep.jsonl
