"""cudaLimitMaxL2FetchGranularity sweep of the intersection pass, one process
per config (the graph is generated once).  usage: l2_fetch.py C5 [steps]"""
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
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
L = lib()
torch.cuda.init()
rt = C.CDLL("libcudart.so.12")
kind, p = CONFIGS[name]
pairs, n = gen(kind, dict(p))
g = T.build_graph(pairs, n)
del pairs
m = g.num_edges()
W = T.ordering_cost(g)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
check(L.tg_set_stream(g._h, C.c_void_p(s.cuda_stream)))
d = torch.zeros(1, dtype=torch.int64, device="cuda")
dp = C.c_void_p(d.data_ptr())
for f in (0, 32, 64, 128):
    if f:
        assert rt.cudaDeviceSetLimit(5, C.c_size_t(f)) == 0
    got = C.c_size_t()
    rt.cudaDeviceGetLimit(C.byref(got), 5)
    check(L.tg_orient_device(g._h))
    check(L.tg_count_device(g._h, dp))
    torch.cuda.synchronize()
    es = [torch.cuda.Event(enable_timing=True) for _ in range(3 * steps)]
    for i in range(steps):
        es[3 * i].record(s)
        check(L.tg_orient_device(g._h))
        es[3 * i + 1].record(s)
        check(L.tg_count_device(g._h, dp))
        es[3 * i + 2].record(s)
    torch.cuda.synchronize()
    o = sum(es[3 * i].elapsed_time(es[3 * i + 1]) for i in range(steps)) / steps
    t = sum(es[3 * i + 1].elapsed_time(es[3 * i + 2]) for i in range(steps)) / steps
    print(json.dumps({"config": name, "fetch_set": f, "fetch_got": got.value, "orient_ms": o,
                      "intersect_ms": t, "triangles": int(d.item()),
                      "hbm_frac_4W": 4 * W / (t / 1e3) / 6549e9}), flush=True)
