"""compute-sanitizer target: the round-2 kernels on small graphs (slab layout
forced on, 4-bit keys, lists longer than a slab, hubs, the comm step and
ANOP-direct with 3 in-process ranks).  usage:
    compute-sanitizer --tool memcheck python tools/exp/memcheck_slab.py"""
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import binding as O  # noqa: E402
from paper_1706_05151_b200 import comm as M  # noqa: E402
from paper_1706_05151_b200 import trigraph as T  # noqa: E402
from paper_1706_05151_b200._lib import lib  # noqa: E402

L = lib()
graphs = {"pa": T.gen_pa(3000, 40, 5), "pa_dense": T.gen_pa(1500, 90, 2),
          "rmat": T.gen_rmat(11, 16, 0.57, 0.19, 0.19, 3), "random": O.random_graph_pairs(200, 0.3, 9)}
for name, pairs in graphs.items():
    ref = O.build_graph(pairs)
    want, want_tv, _ = O.count(ref, tally=True)
    for paths in (0, 8):
        L.tg_debug_set_paths(paths, 0)
        L.tg_debug_set_slab(1)
        g = T.build_graph(pairs, ref.n)
        assert T.count_node_iterator_n(g) == want
        rep = T.run_engine(g, T.EngineConfig(engine=T.EngineKind.Sequential, track_nodes=True,
                                             collect_triangles=True))
        assert rep.total == want and np.array_equal(rep.node_counts, want_tv)
        g.close()
    L.tg_debug_set_paths(0, 0)
    # 3 in-process ranks: the AOP step on slabs, ANOP-direct
    rows = M.split_rows(ref.off, 3)
    comms = M.Comm.local([0, 0, 0])
    res = [None] * 3

    def work(r):
        torch.cuda.set_device(0)
        lo, hi = int(rows[r]), int(rows[r + 1])
        g = M.graph_from_rows(ref.n, lo, hi, ref.off[lo:hi + 1], ref.adj[ref.off[lo]:ref.off[hi]],
                              np.diff(ref.off).astype(np.uint32))
        a = M.run_engine_comm(g, comms[r], T.EngineConfig(engine=T.EngineKind.Aop))
        d = torch.zeros(1, dtype=torch.int64, device="cuda")
        M.aop_step_comm(g, comms[r], a.boundaries, d.data_ptr())
        torch.cuda.synchronize()
        dr = M.run_engine_comm(g, comms[r], T.EngineConfig(engine=T.EngineKind.AnopDirect))
        res[r] = (int(d.item()), dr.total)
        g.close()

    th = [threading.Thread(target=work, args=(r,)) for r in range(3)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert all(x == (want, want) for x in res), (name, res, want)
    for c in comms:
        c.close()
    L.tg_debug_set_slab(0)
    print(name, "ok", want, flush=True)
