python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests -q -x -m "gpu" --ignore=tests/test_gpu_fullsize.py > gpurun_out/pdl_tests.log 2>&1; echo tests rc=$?; tail -n 3 gpurun_out/pdl_tests.log
for pdl in 0 1 0 1; do
  MEDHA_PDL=$pdl timeout -s KILL 300 python bench.py --no-extra --no-cpu > gpurun_out/pdl.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/pdl.json').read().strip().splitlines()[-1]); print('N1 pdl=$pdl', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['value'])"
done
for pdl in 0 1 0 1; do
  MEDHA_PDL=$pdl timeout -s KILL 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2960$pdl scripts/kvp_breakdown.py 2>&1 | grep '"world"' | sed "s/^/pdl=$pdl /"
done
