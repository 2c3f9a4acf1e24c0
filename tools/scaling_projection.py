#!/usr/bin/env python
"""Measured per-rank work of the N-GPU AOP bench step, on ONE B200.

For N in (1, 2, 4, 8) each rank's step -- the full orientation plus the
intersection of its DPD core (engines.hpp:38-54, partition.hpp:116-141) --
is run ALONE on the device and timed with CUDA events (ranks never wait on
each other here; nothing is co-scheduled).  The projected N-GPU step is the
slowest rank plus one 8-byte NCCL all-reduce (taken as 30 us, not measured:
one GPU per call in this environment).  Also reported: the bytes per rank an
all-gather of the oriented lists would move (the alternative of orienting
1/N of the rows per rank).

    python tools/scaling_projection.py C2 [C5]
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from run_configs import CONFIGS, gen  # noqa: E402
from paper_1706_05151_b200 import trigraph as T  # noqa: E402
from paper_1706_05151_b200._lib import check, lib  # noqa: E402

ALLREDUCE_MS = 0.03


def main():
    L = lib()
    for name in sys.argv[1:]:
        kind, p = CONFIGS[name]
        pairs, n = gen(kind, dict(p))
        g = T.build_graph(pairs, n)
        del pairs
        m = g.num_edges()
        s = torch.cuda.Stream()
        torch.cuda.set_stream(s)
        check(L.tg_set_stream(g._h, C.c_void_p(s.cuda_stream)))
        d = torch.zeros(1, dtype=torch.int64, device="cuda")
        dp = C.c_void_p(d.data_ptr())

        def ev():
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            return e

        reps = 3
        check(L.tg_orient_device(g._h))
        torch.cuda.synchronize()
        a = ev()
        for _ in range(reps):
            check(L.tg_orient_device(g._h))
        b = ev()
        torch.cuda.synchronize()
        orient = a.elapsed_time(b) / reps
        rec = {"config": name, "m": m, "orient_ms": orient, "ranks": {}}
        base = None
        for N in (1, 2, 4, 8):
            plan = T.compute_boundaries(g, T.CostKind.Dpd, N).boundaries
            bp = C.c_void_p(plan.ctypes.data)
            per = []
            for r in range(N):
                check(L.tg_aop_rank_device(g._h, bp, N, r, dp))  # warm
                torch.cuda.synchronize()
                a = ev()
                for _ in range(reps):
                    check(L.tg_aop_rank_device(g._h, bp, N, r, dp))
                b = ev()
                torch.cuda.synchronize()
                per.append(a.elapsed_time(b) / reps)
            step = orient + max(per) + (ALLREDUCE_MS if N > 1 else 0.0)
            if base is None:
                base = step
            rec["ranks"][N] = {"count_ms_per_rank": [round(x, 3) for x in per],
                               "count_max_over_mean": max(per) / (sum(per) / N),
                               "projected_step_ms": step,
                               "projected_speedup": base / step,
                               "allgather_bytes_per_rank": int(4 * m * (N - 1) / N)}
        print(json.dumps(rec), flush=True)
        g.close()


if __name__ == "__main__":
    main()
