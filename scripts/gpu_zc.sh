# zero-copy decode_step_host: parity tests + same-box e2e A/B (old library = memcpy staging)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -k "step_host or decode_vs_oracle" > gpurun_out/zc_pytest.log 2>&1; echo pytest rc=$?; tail -n 2 gpurun_out/zc_pytest.log
timeout -s KILL 900 python -m pytest tests/test_gpu_kvp_multi.py -q -x > gpurun_out/zc_multi.log 2>&1; echo multi rc=$?; tail -n 2 gpurun_out/zc_multi.log
NG=$(nvidia-smi -L | wc -l)
for lib in "" build/a0.so ""; do
  for N in 1 $NG; do
    if [ $N = 1 ]; then MEDHA_LIB_PATH=${lib:+$PWD/$lib} timeout -s KILL 600 python bench.py --no-extra --no-cpu --steps 100 --warmup 10 > gpurun_out/zc.json 2> gpurun_out/zc.err;
    else MEDHA_LIB_PATH=${lib:+$PWD/$lib} timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2964$N bench.py --gpus $N --steps 100 --warmup 10 > gpurun_out/zc.json 2> gpurun_out/zc.err; fi
    echo "lib=${lib:-new} N=$N rc=$?" $(python -c "
import json; d=json.loads(open('gpurun_out/zc.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], d['e2e'].get('max_abs_vs_device_path'))")
  done
done
