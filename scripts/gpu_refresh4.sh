# round-1 refresh on 4 GPUs: multi-GPU tests, bench N = 1 (full line), 2, 4, reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_kvp_multi.py -q > gpurun_out/r1c_multi4.log 2>&1; echo multi rc=$?; tail -n 2 gpurun_out/r1c_multi4.log
timeout -s KILL 900 python bench.py > gpurun_out/r1c_n1.json 2> gpurun_out/r1c_n1.err; echo n1 rc=$?
for n in 2 4; do
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2990$n bench.py --gpus $n > gpurun_out/r1c_n$n.json 2> gpurun_out/r1c_n$n.err; echo n$n rc=$?
done
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1c_ref_n1.json 2> gpurun_out/r1c_ref_n1.err; echo ref rc=$?
python - <<'P'
import json
for n in (1,2,4):
    try:
        d=json.loads(open(f'gpurun_out/r1c_n{n}.json').read().strip().splitlines()[-1])
        print(n, d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], (d.get('mixed_c4') or {}).get('ms_per_step'))
    except Exception as e: print(n, 'ERR', e)
P
tail -c 300 gpurun_out/r1c_ref_n1.json
