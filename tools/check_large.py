#!/usr/bin/env python
"""Full-size check of a large config (default C5 = gen_pa(1e8, 40, seed 7),
~2e9 edges) on one B200: count, engine agreement, timing, and an oracle
spot-check of per-rank AOP counts (apex ranges of a 4096-part DPD plan,
counted on the host by the C restatement over the oracle's own graph and
orientation, built from the same pairs).  The full-size goldens are in
tests/golden/reference_full.json (tests/test_gpu_full.py).

    python tools/check_large.py [--n 100000000] [--parts 4096] [--spot 6]
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
from oracle import binding as O  # noqa: E402  (checker only)
from paper_1706_05151_b200 import trigraph as T  # noqa: E402
from paper_1706_05151_b200._lib import check, lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--d", type=int, default=40)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--parts", type=int, default=4096)
    ap.add_argument("--spot", type=int, default=6)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--quick", action="store_true", help="timing only (no engines / oracle)")
    a = ap.parse_args()
    rec = {"config": f"gen_pa({a.n},{a.d},{a.seed})"}
    t0 = time.time()
    pairs = T.gen_pa(a.n, a.d, a.seed)
    rec["gen_s"] = round(time.time() - t0, 1)
    t0 = time.time()
    g = T.build_graph(pairs, a.n)
    # the oracle's own graph + orientation from the same pairs (never from
    # device arrays) for the spot check below
    og = None if a.quick else O.FullGraph(O.HostBuf.from_array(pairs), pairs.shape[0], a.n)
    del pairs
    torch.cuda.synchronize()
    rec["build_s"] = round(time.time() - t0, 2)
    rec["n"], rec["m"] = g.num_nodes(), g.num_edges()
    rec["W"] = T.ordering_cost(g)
    L = lib()
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    check(L.tg_set_stream(g._h, C.c_void_p(s.cuda_stream)))
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    dp = C.c_void_p(d.data_ptr())
    check(L.tg_orient_device(g._h))
    check(L.tg_count_device(g._h, dp))
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3 * a.steps)]
    for i in range(a.steps):
        ev[3 * i].record(s)
        check(L.tg_orient_device(g._h))
        ev[3 * i + 1].record(s)
        check(L.tg_count_device(g._h, dp))
        ev[3 * i + 2].record(s)
    torch.cuda.synchronize()
    rec["orient_ms"] = sum(ev[3 * i].elapsed_time(ev[3 * i + 1]) for i in range(a.steps)) / a.steps
    rec["intersect_ms"] = sum(ev[3 * i + 1].elapsed_time(ev[3 * i + 2])
                              for i in range(a.steps)) / a.steps
    rec["edges_per_s"] = rec["m"] / ((rec["orient_ms"] + rec["intersect_ms"]) / 1e3)
    rec["hbm_frac_4W"] = 4 * rec["W"] / (rec["intersect_ms"] / 1e3) / 6534.5e9
    T_ = int(d.item())
    rec["triangles"] = T_
    torch.cuda.set_stream(torch.cuda.default_stream())
    if a.quick:
        print(json.dumps(rec), flush=True)
        return
    for eng in (T.EngineKind.Aop, T.EngineKind.AnopSurrogate):
        rep = T.run_engine(g, T.EngineConfig(engine=eng, ranks=8))
        rec[f"{T.to_string(eng)}8_total"] = rep.total
        assert rep.total == T_
        assert sum(r.triangles for r in rep.per_rank) == T_
    # oracle spot-check: per-rank AOP counts of a fine plan
    rep = T.run_engine(g, T.EngineConfig(engine=T.EngineKind.Aop, ranks=a.parts))
    rng = np.random.default_rng(1)
    spots = []
    for i in sorted(rng.choice(a.parts, a.spot, replace=False)):
        lo, hi = int(rep.boundaries[i]), int(rep.boundaries[i + 1])
        want = O.lib().orc_count_range(og.n, C.c_void_p(og.eoff.ctypes.data),
                                       C.c_void_p(og.eff.ctypes.data), lo, hi)
        spots.append([int(i), lo, hi, int(rep.per_rank[i].triangles), int(want)])
        assert rep.per_rank[i].triangles == want, spots[-1]
    rec["oracle_spots"] = spots
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
