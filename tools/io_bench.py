#!/usr/bin/env python
"""Edge-list text on one B200 (io.hpp:24-64): write_edge_list and
parse_edge_list of a full config's graph, device-resident (CUDA events) and
end to end from host text, next to the reference's own parse_edge_list on a
bounded sample of the same text on the host (oracle/_ref, 1 thread -- the
reference parser is sequential).  Prints one JSON line per config.

    python tools/io_bench.py C2 [C4 ...]
"""
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


def ev_time(f, reps=3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3


def main():
    L = lib()
    for name in sys.argv[1:]:
        kind, p = CONFIGS[name]
        pairs, n = gen(kind, dict(p))
        g = T.build_graph(pairs, n)
        del pairs
        rec = {"config": name, "n": g.num_nodes(), "m": g.num_edges()}
        ln = C.c_uint64()
        check(L.tg_write_edge_list(g._h, None, 0, C.byref(ln)))
        text_d = torch.empty(ln.value, dtype=torch.uint8, device="cuda")
        tp = C.c_void_p(text_d.data_ptr())
        t_w = ev_time(lambda: check(L.tg_write_edge_list(g._h, tp, ln.value, C.byref(ln))))
        rec["text_bytes"] = ln.value
        rec["write_device_s"] = t_w
        rec["write_GBps"] = ln.value / t_w / 1e9
        m = g.num_edges()
        pairs_d = torch.empty(2 * m, dtype=torch.int32, device="cuda")
        cnt, line = C.c_uint64(), C.c_uint64()
        pp = C.c_void_p(pairs_d.data_ptr())
        t_p = ev_time(lambda: check(L.tg_parse_edge_list(0, tp, ln.value, pp, m, C.byref(cnt),
                                                         C.byref(line))))
        assert cnt.value == m
        rec["parse_device_s"] = t_p
        rec["parse_GBps"] = ln.value / t_p / 1e9
        rec["parse_lines_per_s"] = m / t_p
        # end to end: host text -> Graph on the device
        text_h = text_d.cpu().pin_memory()
        del text_d
        torch.cuda.empty_cache()
        t0 = time.perf_counter()
        h = C.c_void_p()
        check(L.tg_graph_from_text(0, C.c_void_p(text_h.data_ptr()), ln.value, 0, C.byref(h),
                                   C.byref(line)))
        torch.cuda.synchronize()
        rec["graph_from_text_e2e_s"] = time.perf_counter() - t0
        g2 = T.Graph(h, 0)
        rec["round_trip_same_m"] = g2.num_edges() == m
        g2.close()
        # the reference's parser on a bounded host sample (~64 MB of the text)
        try:
            from oracle import binding as O  # CPU baseline only
            if O.ref_available():
                sample = bytes(text_h[: min(ln.value, 64 << 20)].numpy())
                sample = sample[: sample.rfind(b"\n") + 1]
                cap = sample.count(b"\n")
                out = np.zeros(2 * cap, dtype=np.uint32)
                line_o = np.zeros(1, dtype=np.uint64)
                msg = C.create_string_buffer(256)
                t0 = time.perf_counter()
                k = O.ref().ref_parse_edge_list(sample, len(sample), out.ctypes.data, cap,
                                                line_o.ctypes.data, C.cast(msg, C.c_void_p), 256)
                dt = time.perf_counter() - t0
                rec["cpu_reference_parse"] = {"bytes": len(sample), "s": dt,
                                              "GBps": len(sample) / dt / 1e9,
                                              "lines": int(k), "threads": 1}
        except Exception as e:  # noqa: BLE001
            rec["cpu_reference_parse"] = f"unavailable: {e}"
        print(json.dumps(rec), flush=True)
        g.close()


if __name__ == "__main__":
    main()
