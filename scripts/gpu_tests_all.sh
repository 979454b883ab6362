python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -n 3 gpurun_out/smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_all.log
timeout -s KILL 600 python bench.py --no-cpu --steps 100 --warmup 10 > gpurun_out/bench_q.json 2>/dev/null; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['value'], d.get('hbm_read_probe_GBps'), d['decode_70b_10M'])
for r in d['prefill_chunk']['results']: print(r['prefix'], r['c'], r['tflops'], r['frac_of_measured_bf16'])"
