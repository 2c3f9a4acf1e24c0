# group-kernel unroll sweep: g* variants on C4 (scalar groups), q* on C3 (quad groups)
for d in variants/g*/; do n=$(basename $d); echo "== $n"; TG_LIB_PATH=$PWD/$d/libtrigraph_b200.so timeout 300 python tools/run_configs.py C4 --steps 3 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['config'], 'isect %.2f'%r['intersect_ms'], 'T', r['triangles'])"; done
for d in variants/q*/; do n=$(basename $d); echo "== $n"; TG_LIB_PATH=$PWD/$d/libtrigraph_b200.so timeout 300 python tools/run_configs.py C3 --steps 2 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['config'], 'isect %.2f'%r['intersect_ms'], 'T', r['triangles'])"; done
