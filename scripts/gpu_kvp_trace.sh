python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
MEDHA_LIB_PATH=$PWD/build/dtrace.so timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 scripts/kvp_trace.py 2>&1 | grep rank
