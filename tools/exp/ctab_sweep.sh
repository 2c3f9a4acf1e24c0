for d in base minb3; do for cap in 0 262144; do echo "== $d cap $cap"; TG_RANK_CAP=$cap TG_LIB_PATH=$PWD/variants/$d/libtrigraph_b200.so timeout 300 python tools/run_configs.py C3 --steps 2 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['config'], 'isect %.2f'%r['intersect_ms'], 'T', r['triangles'])"; done; done
