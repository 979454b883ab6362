python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests -q -x -m "gpu and not multigpu" --ignore=tests/test_gpu_fullsize.py > gpurun_out/pdl_tests.log 2>&1; echo tests rc=$?; tail -n 2 gpurun_out/pdl_tests.log
for pdl in 0 1 0 1; do
  MEDHA_PDL=$pdl timeout -s KILL 300 python scripts/prefill_sweep.py 131072,1048576 64,256,1024,4096 pdl$pdl 2>&1 | grep -v Warn | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(d['lib'], d.get('prefix'), d.get('c'), d.get('tflops'), d.get('clocks',''))"
done
