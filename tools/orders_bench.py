#!/usr/bin/env python
"""Time every OrderKind (order.hpp:17-128) on a full config on one B200:
order construction (rank array / coreness), the orientation + count under
that order, the ordering cost W it induces (sequential.hpp:95-104, the
algorithmic work of the intersection) and NodeIterator++ (sequential.hpp:48-70)
under the degree order.  Prints one JSON line per config.

    python tools/orders_bench.py C2 [C3 ...]
"""
import json
import os
import sys
import time

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
        core, rec["coreness_s"] = timed(lambda: T.coreness(g))
        rec["max_core"] = int(core.max()) if core.size else 0
        for k in (T.OrderKind.by_degree(), T.OrderKind.by_coreness(), T.OrderKind.by_random(1),
                  T.OrderKind.by_id()):
            nm = k.tag.name
            _, rec[f"{nm}_order_s"] = timed(lambda: T.compute_order(g, k))
            W, _ = timed(lambda: T.ordering_cost(g, k))
            t, dt = timed(lambda: T.count_node_iterator_n(g, k))
            t, dt = timed(lambda: T.count_node_iterator_n(g, k))  # cached orientation
            rec[nm] = {"W": W, "count_s": round(dt, 4), "T": t}
        t, dt = timed(lambda: T.count_node_iterator_pp(g))
        rec["node_iterator_pp_degree_s"] = round(dt, 4)
        rec["node_iterator_pp_T"] = t
        print(json.dumps(rec), flush=True)
        g.close()


if __name__ == "__main__":
    main()
