python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for ev in 1 1000 1 1000; do
  MEDHA_BENCH_EVENT_EVERY=$ev timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29704 bench.py --gpus 4 --no-extra > gpurun_out/ev.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ev.json').read().strip().splitlines()[-1]); print('every=$ev', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"
done
MEDHA_BENCH_EVENT_EVERY=1 timeout -s KILL 300 python bench.py --no-extra --no-cpu > gpurun_out/ev1.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/ev1.json').read().strip().splitlines()[-1]); print('N1 every=1', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"
MEDHA_BENCH_EVENT_EVERY=1000 timeout -s KILL 300 python bench.py --no-extra --no-cpu > gpurun_out/ev1.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/ev1.json').read().strip().splitlines()[-1]); print('N1 every=1000', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"
