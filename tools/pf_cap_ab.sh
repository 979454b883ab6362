python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cap in 64 1 4 8 64 1 4 8; do
  MEDHA_PF_MAX_SPLITS=$cap timeout -s KILL 200 python tools/prefill_sweep.py 1048576,131072 64,256,1024,4096 cap$cap 2>&1 | grep -v Warn | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    print(d.get('lib'), d.get('prefix'), d.get('c'), d.get('tflops'), d.get('clocks', ''))"
done
