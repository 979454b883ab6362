# same-box A/B of prefill softmax variants + bit-identity of outputs vs the baseline variant
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for v in "$@"; do
  MEDHA_LIB_PATH=$PWD/$v timeout -s KILL 120 python scripts/pf_dump.py gpurun_out/pf_$(basename $v .so).pt 2>&1 | tail -1
done
python - "$@" <<'PY'
import sys, torch, os
base = torch.load(f"gpurun_out/pf_{os.path.basename(sys.argv[1])[:-3]}.pt")
for v in sys.argv[2:]:
    o = torch.load(f"gpurun_out/pf_{os.path.basename(v)[:-3]}.pt")
    same = all(torch.equal(o[k][0], base[k][0]) and torch.equal(o[k][1], base[k][1]) for k in base)
    dmax = max((o[k][0] - base[k][0]).abs().max().item() for k in base)
    print(v, "bit-identical" if same else "DIFFERS", "max|dO| =", dmax)
PY
rm -f gpurun_out/pf_*.pt
for v in "$@" $1; do
  MEDHA_LIB_PATH=$PWD/$v timeout -s KILL 300 python scripts/prefill_sweep.py ${PF_PREFIXES:-131072,1048576} ${PF_CHUNKS:-64,256,1024,4096} $(basename $v) 2>&1 | grep -v Warn
done
