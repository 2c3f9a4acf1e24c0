"""Would orientation and intersection overlap on one GPU?  Two handles of the
same graph, two streams: orient(g1) on one stream while count(g2) runs on the
other, against the two run back to back.  Library variants with smaller
resident grids (TG_OBLOCKS / TG_SLAB_BLOCKS) so that the two kernels can be
co-resident.  usage: TG_LIB_PATH=... python tools/exp/co_run.py C5"""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from run_configs import CONFIGS, gen  # noqa: E402
from paper_1706_05151_b200 import trigraph as T  # noqa: E402
from paper_1706_05151_b200._lib import check, lib  # noqa: E402

name = sys.argv[1]
L = lib()
kind, p = CONFIGS[name]
pairs, n = gen(kind, dict(p))
g1 = T.build_graph(pairs, n)
g2 = T.build_graph(pairs, n)
del pairs
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
check(L.tg_set_stream(g1._h, C.c_void_p(s1.cuda_stream)))
check(L.tg_set_stream(g2._h, C.c_void_p(s2.cuda_stream)))
d1 = torch.zeros(1, dtype=torch.int64, device="cuda")
d2 = torch.zeros(1, dtype=torch.int64, device="cuda")
for g, d in ((g1, d1), (g2, d2)):
    for _ in range(2):
        check(L.tg_orient_device(g._h))
        check(L.tg_count_device(g._h, C.c_void_p(d.data_ptr())))
torch.cuda.synchronize()


def timed(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e2 = torch.cuda.Event(enable_timing=True)
    e0.record(s1)
    s2.wait_event(e0)
    for _ in range(reps):
        fn()
    e1.record(s1)
    e2.record(s2)
    torch.cuda.synchronize()
    return max(e0.elapsed_time(e1), e0.elapsed_time(e2)) / reps


t_o = timed(lambda: check(L.tg_orient_device(g1._h)))
t_c = timed(lambda: check(L.tg_count_device(g2._h, C.c_void_p(d2.data_ptr()))))


def both():
    check(L.tg_orient_device(g1._h))
    check(L.tg_count_device(g2._h, C.c_void_p(d2.data_ptr())))


t_b = timed(both)
print(json.dumps({"config": name, "lib": os.environ.get("TG_LIB_PATH", "default"), "orient_ms": t_o,
                  "count_ms": t_c, "concurrent_ms": t_b, "serial_sum_ms": t_o + t_c,
                  "triangles": int(d2.item())}), flush=True)
