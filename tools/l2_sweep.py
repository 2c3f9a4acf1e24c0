#!/usr/bin/env python
"""Intersection-pass timing under L2 eviction-hint settings (experiment).
    TG_PERSIST_MB=96 python tools/l2_sweep.py C2 "0" "1" "1,0.05" ...
Each setting is TG_HINT[,TG_HOT_FRAC]; one graph, one JSON line per setting."""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from run_configs import CONFIGS, gen  # noqa: E402
from paper_1706_05151_b200 import trigraph as T  # noqa: E402
from paper_1706_05151_b200._lib import check, lib  # noqa: E402


def main():
    name = sys.argv[1]
    kind, p = CONFIGS[name]
    pairs, n = gen(kind, dict(p))
    g = T.build_graph(pairs, n)
    del pairs
    W = T.ordering_cost(g)
    L = lib()
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    check(L.tg_set_stream(g._h, C.c_void_p(s.cuda_stream)))
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    dp = C.c_void_p(d.data_ptr())
    check(L.tg_orient_device(g._h))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for setting in sys.argv[2:]:
        parts = setting.split(",")
        os.environ["TG_HINT"] = parts[0]
        if len(parts) > 1:
            os.environ["TG_HOT_FRAC"] = parts[1]
        else:
            os.environ.pop("TG_HOT_FRAC", None)
        ts = []
        pre = os.environ.get("PRE", "flush")
        for it in range(6):
            if pre != "none":
                flush.fill_(it)
            if pre == "orient":
                check(L.tg_orient_device(g._h))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            check(L.tg_count_device(g._h, dp))
            b.record(s)
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(a.elapsed_time(b))
        print(json.dumps({"config": name, "setting": setting,
                          "persist_mb": os.environ.get("TG_PERSIST_MB"), "pre": pre,
                          "count_ms": round(min(ts), 3), "mean_ms": round(sum(ts) / len(ts), 3),
                          "frac_4W": round(4 * W / (min(ts) / 1e3) / 6534.5e9, 3),
                          "T": int(d.item())}), flush=True)


if __name__ == "__main__":
    main()
