#!/usr/bin/env python
"""Run BASELINE.json's configs on one GPU: generate, build, orient + count,
time (CUDA events), cross-check engines.  Usage:
    python tools/run_configs.py C1 C3 C4 [--small]
Prints one JSON line per config."""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1706_05151_b200 import trigraph as T  # noqa: E402
from paper_1706_05151_b200._lib import check, lib  # noqa: E402

CONFIGS = {
    "C1": ("gnm", dict(n=100_000, m=1_000_000, seed=1)),
    "C2": ("pa", dict(n=10_000_000, d=40, seed=7)),
    "C3": ("rmat", dict(scale=24, ef=16, seed=1)),
    "C4": ("ws", dict(n=50_000_000, k=20, beta=0.1, seed=1)),
    "C5": ("pa", dict(n=100_000_000, d=40, seed=7)),
}
SMALL = {"C1": dict(n=100_000, m=1_000_000), "C2": dict(n=200_000), "C3": dict(scale=18),
         "C4": dict(n=1_000_000), "C5": dict(n=1_000_000)}


def gen(kind, p):
    if kind == "gnm":
        return T.gen_gnm(p["n"], p["m"], p["seed"]), p["n"]
    if kind == "pa":
        return T.gen_pa(p["n"], p["d"], p["seed"]), p["n"]
    if kind == "rmat":
        return T.gen_rmat(p["scale"], p["ef"], 0.57, 0.19, 0.19, p["seed"]), 1 << p["scale"]
    if kind == "ws":
        return T.gen_ws(p["n"], p["k"], p["beta"], p["seed"]), p["n"]
    raise ValueError(kind)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--engines", action="store_true")
    a = ap.parse_args()
    L = lib()
    if os.environ.get("TG_L2_PERSIST"):  # experiment: cudaLimitPersistingL2CacheSize (bytes)
        torch.cuda.init()
        rt = C.CDLL("libcudart.so.12")
        mx = C.c_int()
        rt.cudaDeviceGetAttribute(C.byref(mx), 108, 0)  # cudaDevAttrMaxPersistingL2CacheSize
        win = C.c_int()
        rt.cudaDeviceGetAttribute(C.byref(win), 109, 0)  # cudaDevAttrMaxAccessPolicyWindowSize
        want = min(int(os.environ["TG_L2_PERSIST"]), mx.value)
        assert rt.cudaDeviceSetLimit(6, C.c_size_t(want)) == 0
        got = C.c_size_t()
        rt.cudaDeviceGetLimit(C.byref(got), 6)
        print("persisting L2 max", mx.value, "window max", win.value, "set", got.value,
              file=sys.stderr)
    if os.environ.get("TG_L2_FETCH"):  # experiment: cudaLimitMaxL2FetchGranularity (bytes)
        torch.cuda.init()
        rt = C.CDLL("libcudart.so.12")
        v = C.c_size_t(int(os.environ["TG_L2_FETCH"]))
        assert rt.cudaDeviceSetLimit(5, v) == 0
        got = C.c_size_t()
        rt.cudaDeviceGetLimit(C.byref(got), 5)
        print("L2 fetch granularity", got.value, file=sys.stderr)
    if os.environ.get("TG_WARP_VARIANT"):
        L.tg_debug_set_warp_variant(int(os.environ["TG_WARP_VARIANT"]))
    if os.environ.get("TG_RANK_BITMAP") or os.environ.get("TG_RANK_CAP"):
        L.tg_debug_set_rank_bitmap(int(os.environ.get("TG_RANK_BITMAP", "0")),
                                   int(os.environ.get("TG_RANK_CAP", "0")))
    for name in a.configs:
        kind, p = CONFIGS[name]
        p = dict(p)
        if a.small:
            p.update(SMALL[name])
        t0 = time.time()
        if os.environ.get("TG_DEVICE_GEN") and kind in ("rmat", "ws"):
            # generated and built on the device (bit-identical pair streams)
            g = (T.graph_rmat(p["scale"], p["ef"], 0.57, 0.19, 0.19, p["seed"]) if kind == "rmat"
                 else T.graph_ws(p["n"], p["k"], p["beta"], p["seed"]))
            n = g.num_nodes()
            torch.cuda.synchronize()
            t1 = t2 = time.time()
        else:
            pairs, n = gen(kind, p)
            t1 = time.time()
            g = T.build_graph(pairs, n)
            del pairs
            torch.cuda.synchronize()
            t2 = time.time()
        m = g.num_edges()
        W = T.ordering_cost(g)
        s = torch.cuda.Stream()
        torch.cuda.set_stream(s)
        check(L.tg_set_stream(g._h, C.c_void_p(s.cuda_stream)))
        d = torch.zeros(1, dtype=torch.int64, device="cuda")
        dp = C.c_void_p(d.data_ptr())
        for _ in range(2):
            check(L.tg_orient_device(g._h))
            check(L.tg_count_device(g._h, dp))
        torch.cuda.synchronize()
        es = [torch.cuda.Event(enable_timing=True) for _ in range(3 * a.steps)]
        for i in range(a.steps):
            es[3 * i].record(s)
            check(L.tg_orient_device(g._h))
            es[3 * i + 1].record(s)
            check(L.tg_count_device(g._h, dp))
            es[3 * i + 2].record(s)
        torch.cuda.synchronize()
        orient = sum(es[3 * i].elapsed_time(es[3 * i + 1]) for i in range(a.steps)) / a.steps
        isect = sum(es[3 * i + 1].elapsed_time(es[3 * i + 2]) for i in range(a.steps)) / a.steps
        tri = int(d.item())
        rec = {"config": name, "params": p, "n": n, "m": m, "W": W, "triangles": tri,
               "gen_s": round(t1 - t0, 2), "build_s": round(t2 - t1, 2),
               "orient_ms": orient, "intersect_ms": isect,
               "edges_per_s": m / ((orient + isect) / 1e3),
               "hbm_frac_4W": 4 * W / (isect / 1e3) / 6534.5e9}
        if a.engines:
            for eng, pr in ((T.EngineKind.Aop, 8), (T.EngineKind.AnopSurrogate, 8)):
                torch.cuda.synchronize()
                t = time.time()
                rep = T.run_engine(g, T.EngineConfig(engine=eng, ranks=pr))
                rec[f"{T.to_string(eng)}_total"] = rep.total
                rec[f"{T.to_string(eng)}_s"] = round(time.time() - t, 3)
                assert rep.total == tri, (eng, rep.total, tri)
        print(json.dumps(rec), flush=True)
        g.close()
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
