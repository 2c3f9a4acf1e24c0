#!/usr/bin/env python
"""Time the 8(f) rows at full size on one B200: approx_count (sparsified
engines), per-edge triangle counts, variance report.
    python tools/next_rows.py C2 C4"""
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


def timed(f):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t


def main():
    for name in sys.argv[1:]:
        kind, p = CONFIGS[name]
        pairs, n = gen(kind, dict(p))
        g = T.build_graph(pairs, n)
        del pairs
        rec = {"config": name, "m": g.num_edges()}
        exact, rec["count_s"] = timed(lambda: T.count_node_iterator_n(g))
        rec["T"] = exact
        for eng, q in ((T.EngineKind.Sequential, 0.5), (T.EngineKind.Aop, 0.5),
                       (T.EngineKind.AnopSurrogate, 0.5)):
            T.approx_count(g, 8, eng, q, 1)  # warm
            est, dt = timed(lambda: T.approx_count(g, 8, eng, q, 1))
            rec[f"approx_{T.to_string(eng)}8_q{q}"] = {"estimate": est,
                                                       "rel_err": est / max(exact, 1) - 1,
                                                       "s": round(dt, 4)}
        te, dt = timed(lambda: T.per_edge_triangle_counts(g))
        rec["per_edge_s"] = round(dt, 4)
        rec["per_edge_sum_is_3T"] = int(te.sum()) == 3 * exact
        rec["k"] = int((te.astype(np.float64) * (te.astype(np.float64) - 1) / 2).sum())
        plan = T.compute_boundaries(g, T.CostKind.Dpd, 8)
        vr, dt = timed(lambda: T.variance_report(g, plan, 0.5))
        rec["variance_p8"] = {"T": vr.triangles, "k": vr.k, "k_prime": vr.k_prime,
                              "var": vr.var, "var_prime": vr.var_prime, "s": round(dt, 4)}
        print(json.dumps(rec), flush=True)
        del g


if __name__ == "__main__":
    main()
