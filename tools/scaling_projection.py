#!/usr/bin/env python
"""Per-rank work of the N-GPU AOP step (csrc/comm.cu tg_aop_step_comm),
measured rank by rank on ONE B200, and the projected N-GPU step.

The step at N GPUs: rank r orients ONLY its rows (an equal-orientation-cost
split, effective.hpp:37-52), the oriented rows of all ranks are broadcast in
rank order over NVLink (list lengths first: 4 B per vertex), and the rank
counts the apexes of its DPD core (engines.hpp:38-54, partition.hpp:116-141)
as their lists arrive.  Measured here with CUDA events, each piece ALONE on
the device (nothing co-scheduled; ranks never wait on each other):
  orient_r  -- tg_orient_rows_device over rank r's rows;
  count_r   -- tg_aop_rank_device over rank r's core (full orientation);
Modelled (one GPU per call in this environment):
  xfer_r    -- bytes rank r receives (others' oriented entries + lengths)
               at NVLINK_GBS (an assumption, stated in the output);
  + one 8-byte all-reduce (30 us).
  slab_r    -- on PA-like graphs (mean list > 16) every rank fills the n
               slabs from the gathered lists as the slices arrive (slab_rows:
               4 m + 128 n bytes streamed) at SLAB_GBS (an assumption too);
  + one 8-byte all-reduce (30 us).
Projected step = max_r(orient_r + xfer_r + slab_r + count_r) (serial) and
max_r(orient_r + max(xfer_r, slab_r + count_r)) (slab fill and count
overlapped with the broadcasts, as tg_aop_step_comm schedules them -- an
upper bound on overlap).

    python tools/scaling_projection.py C2 [C5] [--nvlink-gbs 700]
"""
import argparse
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
from paper_1706_05151_b200 import comm as M  # noqa: E402
from paper_1706_05151_b200 import trigraph as T  # noqa: E402
from paper_1706_05151_b200._lib import check, lib  # noqa: E402

ALLREDUCE_MS = 0.03


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--nvlink-gbs", type=float, default=700.0,
                    help="assumed NCCL broadcast bandwidth per receiving GPU (GB/s)")
    ap.add_argument("--slab-gbs", type=float, default=5000.0,
                    help="assumed streaming rate of slab_rows (GB/s)")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    L = lib()
    for name in a.configs:
        kind, p = CONFIGS[name]
        pairs, n = gen(kind, dict(p))
        g = T.build_graph(pairs, n)
        del pairs
        m = g.num_edges()
        off, _ = g.csr()
        s = torch.cuda.Stream()
        torch.cuda.set_stream(s)
        check(L.tg_set_stream(g._h, C.c_void_p(s.cuda_stream)))
        d = torch.zeros(1, dtype=torch.int64, device="cuda")
        dp = C.c_void_p(d.data_ptr())

        def timed(fn):
            fn()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(a.reps):
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / a.reps

        t_orient1 = timed(lambda: check(L.tg_orient_device(g._h)))
        t_count1 = timed(lambda: check(L.tg_count_device(g._h, dp)))
        rec = {"config": name, "n": n, "m": m, "nvlink_gbs_assumed": a.nvlink_gbs,
               "one_gpu_ms": {"orient": t_orient1, "count": t_count1,
                              "step": t_orient1 + t_count1}, "N": {}}
        for N in (2, 4, 8):
            rows = M.split_rows(off, N)
            plan = T.compute_boundaries(g, T.CostKind.Dpd, N).boundaries
            bptr = C.c_void_p(np.ascontiguousarray(plan, dtype=np.uint32).ctypes.data)
            ranks = []
            ent = C.c_uint64()
            cnts = []
            for r in range(N):
                lo, hi = int(rows[r]), int(rows[r + 1])
                t_or = timed(lambda: check(L.tg_orient_rows_device(g._h, lo, hi, C.byref(ent))))
                cnts.append(ent.value)
                check(L.tg_orient_device(g._h))  # the full orientation for the core count
                t_ct = timed(lambda: (d.zero_(), check(L.tg_aop_rank_device(g._h, bptr, N, r,
                                                                           dp))))
                ranks.append([lo, hi, t_or, t_ct])
            tot = sum(cnts)
            slab_ms = ((4 * m + 128 * n) / (a.slab_gbs * 1e9) * 1e3) if m > 16 * n else 0.0
            out = []
            for r, (lo, hi, t_or, t_ct) in enumerate(ranks):
                rx = (tot - cnts[r]) * 4 + (n - (hi - lo)) * 4
                t_x = rx / (a.nvlink_gbs * 1e9) * 1e3
                out.append({"rows": [lo, hi], "orient_ms": t_or, "count_ms": t_ct,
                            "recv_bytes": rx, "xfer_ms": t_x, "slab_ms": slab_ms,
                            "serial_ms": t_or + t_x + slab_ms + t_ct + ALLREDUCE_MS,
                            "overlap_ms": t_or + max(t_x, slab_ms + t_ct) + ALLREDUCE_MS})
            ser = max(x["serial_ms"] for x in out)
            ovl = max(x["overlap_ms"] for x in out)
            rec["N"][N] = {"ranks": out, "step_serial_ms": ser, "step_overlap_ms": ovl,
                           "speedup_serial": (t_orient1 + t_count1) / ser,
                           "speedup_overlap": (t_orient1 + t_count1) / ovl}
        print(json.dumps(rec), flush=True)
        torch.cuda.set_stream(torch.cuda.default_stream())
        g.close()


if __name__ == "__main__":
    main()
