# same-box A/B on a reduced sweep: bash scripts/gpu_ab2.sh prefixes chunks lib1.so lib2.so ...
pre=$1; cs=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for v in "$@"; do
  MEDHA_LIB_PATH=$PWD/$v timeout -s KILL 300 python scripts/prefill_sweep.py $pre $cs $(basename $v) 2>&1 | grep -v Warn | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(d['lib'], d.get('prefix'), d.get('c'), d.get('tflops'), d.get('clocks',''))"
done
