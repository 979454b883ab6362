PF_PREFIXES=131072 PF_CHUNKS=64,1024,4096 bash scripts/gpu_pf_opt_ab.sh "$@"
for t in th1; do echo "== trace $t"; MEDHA_LIB_PATH=$PWD/build/$t.so python scripts/pf_trace.py 2>&1 | grep -E "median|P0=131072 c=1024" | head -3; done
