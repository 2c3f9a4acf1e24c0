#!/usr/bin/env python
"""The bench's end-to-end leg decomposed on one B200 (C2 by default): pinned
host CSR -> count through (a) tg_graph_from_csr + tg_count + tg_graph_free
and (b) the streamed tg_count_from_csr, next to the bare H2D copy of the same
bytes (the PCIe floor).  Host clock around synchronised calls.

    python tools/e2e_probe.py [C2] [--chunk ENTRIES ...]
"""
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
sys.path.insert(0, os.path.join(ROOT, "tools"))
from run_configs import CONFIGS, gen  # noqa: E402
from paper_1706_05151_b200 import trigraph as T  # noqa: E402
from paper_1706_05151_b200._lib import check, lib  # noqa: E402


def best(f, reps=4):
    f()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return min(ts), sum(ts) / len(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C2")
    ap.add_argument("--chunk", type=int, nargs="*", default=[0, 1 << 24, 1 << 25, 1 << 27])
    a = ap.parse_args()
    L = lib()
    kind, p = CONFIGS[a.config]
    pairs, n = gen(kind, dict(p))
    g = T.build_graph(pairs, n)
    del pairs
    off_h, adj_h = g.csr()
    want = T.count_node_iterator_n(g)
    g.close()
    off_p = torch.from_numpy(off_h.view(np.int64)).pin_memory()
    adj_p = torch.from_numpy(adj_h.view(np.int32)).pin_memory()
    po, pa = C.c_void_p(off_p.data_ptr()), C.c_void_p(adj_p.data_ptr())
    rec = {"config": a.config, "n": n, "bytes": off_p.numel() * 8 + adj_p.numel() * 4}
    d_off = torch.empty_like(off_p, device="cuda")
    d_adj = torch.empty_like(adj_p, device="cuda")

    def h2d():
        d_off.copy_(off_p, non_blocking=True)
        d_adj.copy_(adj_p, non_blocking=True)
    rec["h2d_s"] = best(h2d)
    rec["h2d_GBps"] = rec["bytes"] / rec["h2d_s"][0] / 1e9
    del d_off, d_adj
    torch.cuda.empty_cache()

    def separate():
        h = C.c_void_p()
        check(L.tg_graph_from_csr(0, n, po, pa, C.byref(h)))
        c = C.c_uint64()
        check(L.tg_count(h, C.byref(c)))
        check(L.tg_graph_free(h))
        assert c.value == want
    rec["graph_from_csr+count_s"] = best(separate)
    for ch in a.chunk:
        L.tg_debug_set_chunk_entries(ch)

        def streamed():
            c = C.c_uint64()
            check(L.tg_count_from_csr(0, n, po, pa, C.byref(c)))
            assert c.value == want
        rec[f"count_from_csr_chunk{ch}_s"] = best(streamed)
    L.tg_debug_set_chunk_entries(0)
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
