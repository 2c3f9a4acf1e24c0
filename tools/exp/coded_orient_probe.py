#!/usr/bin/env python
"""Experiment: C2 one-pass orientation with the 4-byte degree key (default
below TG_CODED_MIN_N) vs the 1-byte monotone degree code forced on
(tg_debug_set_paths(4, 0)); checks the triangle count is unchanged.  Not part
of the library."""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1706_05151_b200._lib import check, lib  # noqa: E402


def main():
    torch.cuda.set_device(0)
    L = lib()
    g, _ = bench.make_graph(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    check(L.tg_set_stream(g._h, C.c_void_p(stream.cuda_stream)))
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = {}
    for mode in (0, 4, 0, 4):
        L.tg_debug_set_paths(mode, 0)
        for _ in range(3):
            check(L.tg_orient_device(g._h))
        torch.cuda.synchronize()
        reps = 20
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(reps):
            check(L.tg_orient_device(g._h))
        e.record(stream)
        torch.cuda.synchronize()
        orient_ms = s.elapsed_time(e) / reps
        s.record(stream)
        for _ in range(reps):
            check(L.tg_count_device(g._h, C.c_void_p(d.data_ptr())))
        e.record(stream)
        torch.cuda.synchronize()
        out.setdefault(f"mode{mode}", []).append(
            {"orient_ms": orient_ms, "count_ms": s.elapsed_time(e) / reps, "T": int(d.item())})
    L.tg_debug_set_paths(0, 0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
