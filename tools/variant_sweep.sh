#!/bin/bash
# time the C2 intersection pass under each built variant (tools/build_variant.sh)
cfg=${CFG:-C2}
for d in variants/*/; do
  n=$(basename $d)
  echo -n "$n "
  PRE=none TG_LIB_PATH=$PWD/$d/libtrigraph_b200.so python tools/l2_sweep.py $cfg 0 2>&1 | tail -1
done
