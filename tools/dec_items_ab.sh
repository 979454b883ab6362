#!/bin/bash
# same-box decode A/B over work items per CTA slot (MEDHA_DEC_ITEMS builds in build/)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in dec_it1 dec_it2 dec_it4 dec_it1 dec_it2 dec_it4; do
  MEDHA_LIB_PATH=$PWD/build/$v.so timeout -s KILL 200 python tools/decode_ab.py $v 2>&1 | grep -v Warn
done
