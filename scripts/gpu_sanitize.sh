python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python scripts/sanitize_small.py > gpurun_out/san_plain.log 2>&1 || { echo plain failed; exit 1; }
timeout -s KILL 900 compute-sanitizer --tool $1 --target-processes all python scripts/sanitize_small.py > gpurun_out/sanitize_$1.log 2>&1; echo $1 rc=$?
grep -E "ERROR SUMMARY|sanitize OK|Invalid|Race|hazard" gpurun_out/sanitize_$1.log | head -10
