#!/usr/bin/env python
"""Per-rank cost model of the ANOP-surrogate engine on one B200 (the ranks run
one after another on the same device): orientation of the core rows + pack,
exchange volume, local + surrogate counting.  Predicts the N-GPU step time
(max over ranks, + all-to-allv volume / NVLink bandwidth).
    python tools/surrogate_model.py C2 8"""
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


def main():
    name, p = sys.argv[1], int(sys.argv[2])
    kind, prm = CONFIGS[name]
    pairs, n = gen(kind, dict(prm))
    g = T.build_graph(pairs, n)
    del pairs
    L = lib()
    b = T.compute_boundaries(g, T.CostKind.Dpd, p).boundaries
    bp = C.c_void_p(b.ctypes.data)
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    ranks = []
    packs = []
    for i in range(p):
        msgs = np.zeros(p, np.uint64)
        words = np.zeros(p, np.uint64)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        check(L.tg_surrogate_pack_sizes(g._h, bp, p, i, C.c_void_p(msgs.ctypes.data),
                                        C.c_void_p(words.ctypes.data)))
        hdr = torch.zeros(int(2 * msgs.sum()) + 1, dtype=torch.int32, device="cuda")
        dat = torch.zeros(int(words.sum()) + 1, dtype=torch.int32, device="cuda")
        check(L.tg_surrogate_pack_device(g._h, bp, p, i, C.c_void_p(hdr.data_ptr()),
                                         C.c_void_p(dat.data_ptr())))
        torch.cuda.synchronize()
        ranks.append({"rank": i, "orient_pack_ms": 1e3 * (time.perf_counter() - t0),
                      "msgs": int(msgs.sum()), "words": int(words.sum())})
        packs.append((msgs, words, hdr, dat))
    total = 0
    for j in range(p):
        hs, ds = [], []
        for i in range(p):
            msgs, words, hdr, dat = packs[i]
            m0, w0 = int(msgs[:j].sum()), int(words[:j].sum())
            hs.append(hdr[2 * m0: 2 * (m0 + int(msgs[j]))])
            ds.append(dat[w0: w0 + int(words[j])])
        rh = torch.cat(hs)
        rd = torch.cat(ds)
        nm = rh.numel() // 2
        rh = rh if rh.numel() else torch.zeros(2, dtype=torch.int32, device="cuda")
        rd = rd if rd.numel() else torch.zeros(1, dtype=torch.int32, device="cuda")
        d.zero_()
        # warm (orients the core again when the cache was replaced), then time
        check(L.tg_surrogate_count_device(g._h, bp, p, j, C.c_void_p(rh.data_ptr()), nm,
                                          C.c_void_p(rd.data_ptr()), C.c_void_p(d.data_ptr())))
        torch.cuda.synchronize()
        d.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        check(L.tg_surrogate_count_device(g._h, bp, p, j, C.c_void_p(rh.data_ptr()), nm,
                                          C.c_void_p(rd.data_ptr()), C.c_void_p(d.data_ptr())))
        e.record()
        torch.cuda.synchronize()
        ranks[j]["count_ms"] = s.elapsed_time(e)
        ranks[j]["recv_words"] = int(rd.numel())
        total += int(d.item())
    out = {"config": name, "p": p, "total": total, "ranks": ranks,
           "sum_words": sum(r["words"] for r in ranks), "m": g.num_edges()}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
