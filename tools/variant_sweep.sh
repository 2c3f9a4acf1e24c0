#!/bin/bash
# time configs under each built variant (tools/build_variant.sh):
#   CFGS="C2 C3" tools/variant_sweep.sh
for d in variants/*/; do
  n=$(basename $d)
  echo "== $n"
  TG_LIB_PATH=$PWD/$d/libtrigraph_b200.so python tools/run_configs.py ${CFGS:-C2} --steps 3 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['config'], 'orient %.3f'%r['orient_ms'], 'isect %.3f'%r['intersect_ms'], 'T', r['triangles'])"
done
