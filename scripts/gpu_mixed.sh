mkdir -p gpurun_out
timeout -s KILL 400 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench1 rc=$?
timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench4 rc=$?
python -c "
import json
for f in ('gpurun_out/bench1.json','gpurun_out/bench4.json'):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['value'], d.get('mixed_c4'))
    except Exception as e: print(f, 'ERR', e)
"
tail -3 gpurun_out/bench1.err gpurun_out/bench4.err
