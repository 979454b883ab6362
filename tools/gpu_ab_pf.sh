# same-box prefill A/B over variants (sweep only, 128K and 1M, all chunk sizes)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for v in "$@"; do
  MEDHA_LIB_PATH=$PWD/$v timeout -s KILL 300 python tools/prefill_sweep.py ${PF_PREFIXES:-131072} ${PF_CHUNKS:-64,1024,4096} $(basename $v) 2>&1 | grep -v Warn | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    print(d.get('lib'), d.get('prefix'), d.get('c'), d.get('tflops'), d.get('clocks', ''))"
done
