python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_kvp_multi.py -q -x > gpurun_out/pytest_multi.log 2>&1; echo pytest multi rc=$?
tail -n 30 gpurun_out/pytest_multi.log
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo bench2 rc=$?
cat gpurun_out/bench_n2.json; tail -n 5 gpurun_out/bench_n2.err
