#!/bin/bash
# The round's evidence run on one GPU (gpurun): smoke, pytest -m gpu, bench.py, the ncu launch
# list of the bench step and one `ncu --set full` capture each of the decode kernel (bench
# step) and the prefill kernel (128K prefix, c = 64 and c = 1024).  Outputs in gpurun_out/.
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout -s KILL 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 2 gpurun_out/smoke.log
if [ "${SKIP_PYTEST:-0}" != 1 ]; then
  timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/pytest_gpu.log
fi
timeout -s KILL 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:medha:: -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-extra --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:decode_splitkv -s 3 -c 1 -f \
  -o gpurun_out/decode_full python bench.py --no-extra --no-cpu --steps 5 --warmup 3 > gpurun_out/ncu_decode.log 2>&1; echo "ncu decode rc=$?"
for c in 1024 64; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:prefill_ws -s 1 -c 1 -f \
    -o gpurun_out/prefill_c$c python tools/prefill_one.py --prefix 131072 --c $c > gpurun_out/ncu_prefill_c$c.log 2>&1
  echo "ncu prefill c=$c rc=$?"
done
ls gpurun_out
