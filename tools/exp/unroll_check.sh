# counts with window-non-dividing unrolls must equal the defaults' (C3: 10289641450, C2: 612261)
for d in q3 g6; do echo "== $d"; TG_LIB_PATH=$PWD/variants/$d/libtrigraph_b200.so timeout 300 python tools/run_configs.py C3 C2 --steps 1 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['config'], 'isect %.2f'%r['intersect_ms'], 'T', r['triangles'])"; done
