python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 300 python scripts/decode_micro.py 2>&1 | grep decode_us
MEDHA_LIB_PATH=$PWD/build/dtrace.so timeout -s KILL 300 python scripts/decode_trace.py 2>&1 | grep tokens
NG=$(nvidia-smi -L | wc -l)
for N in 1 2 4; do
  [ $N -gt $NG ] && continue
  if [ $N = 1 ]; then timeout -s KILL 600 python bench.py --no-extra --no-cpu --steps 200 --warmup 20 > gpurun_out/scale_n$N.json 2> gpurun_out/scale_n$N.err;
  else timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --steps 200 --warmup 20 > gpurun_out/scale_n$N.json 2> gpurun_out/scale_n$N.err; fi
  echo N=$N rc=$?; grep -o '"value": [0-9.]*\|"ms_per_step": [0-9.]*\|"frac": [0-9.]*\|"kernel_ms": [0-9.]*' gpurun_out/scale_n$N.json | tr '\n' ' '; echo
done
