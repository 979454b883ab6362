python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 120 python -m pytest tests/test_gpu_parity.py -q -x -k "large_batch" 2>&1 | tail -3
timeout -s KILL 120 python -m pytest tests/test_gpu_parity.py -q -x -k "mixed_lengths or large_batch" 2>&1 | tail -3
timeout -s KILL 120 python -m pytest tests/test_gpu_parity.py -q -x -k "decode_vs_oracle or large_batch" 2>&1 | tail -3
