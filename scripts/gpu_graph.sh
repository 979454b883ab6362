python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests/test_gpu_graph.py tests/test_abi_exports.py -q -x > gpurun_out/graph_tests.log 2>&1; echo graph tests rc=$?; tail -n 15 gpurun_out/graph_tests.log
timeout -s KILL 300 python -c "
import sys, json; sys.argv=['bench.py']
import bench, torch
import paper_2409_17264_b200 as M
print(json.dumps(bench.bench_graph_decode(M)))
" 2>&1 | tail -3
