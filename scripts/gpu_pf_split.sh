python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_kvp_multi.py -q -k "ext" > gpurun_out/pytest_multi_ext.log 2>&1; echo rc=$?
grep -E "passed|failed|FAIL" gpurun_out/pytest_multi_ext.log | cut -c1-300 | head -4
for v in pf_split0 pf_split1 pf_split0 pf_split1; do MEDHA_LIB_PATH=$PWD/build/$v.so timeout -s KILL 300 python scripts/prefill_sweep.py 131072,1048576 64,256,1024,4096 $v 2>&1 | grep -v Warn; done
