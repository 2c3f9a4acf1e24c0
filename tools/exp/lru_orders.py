#!/usr/bin/env python
"""Experiment: does the apex processing order change the cache behaviour of
the N_u reads?  LRU simulation (tools/exp/lru_sim.cpp, 32-byte sectors) of
NodeIteratorN on gen_pa(n, 40, 7) under several apex orders, cache scaled
with the graph (n = 1e6 -> 12.6 MB, i.e. 126 MB at C2's n = 1e7).
    g++ -O2 -o /tmp/lru_sim tools/exp/lru_sim.cpp && python tools/exp/lru_orders.py 1000000
Measured (n = 1e6): miss rate id 0.445, reverse 0.445, random 0.481,
by smallest neighbour 0.473, by degree 0.437 -- the order barely matters."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import binding as O  # noqa: E402
from paper_1706_05151_b200 import trigraph as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cap = int(126e6 * n / 1e7 / 32)
g = O.build_graph(T.gen_pa(n, 40, 7), n)
eoff, eff = O.effective(g)
with open("/tmp/lru_g.bin", "wb") as f:
    np.array([n], np.uint64).tofile(f)
    eoff.astype(np.uint64).tofile(f)
    np.array([len(eff)], np.uint64).tofile(f)
    eff.astype(np.uint32).tofile(f)
deg = np.diff(g.off.astype(np.int64))
h = np.diff(eoff.astype(np.int64))
mins = np.array([eff[eoff[v]:eoff[v + 1]].min() if h[v] else n for v in range(n)])
orders = {"id": np.arange(n), "rev": np.arange(n)[::-1],
          "random": np.random.default_rng(0).permutation(n),
          "by_min_nbr": np.argsort(mins, kind="stable"), "by_deg": np.argsort(deg, kind="stable")}
for k, o in orders.items():
    o.astype(np.uint32).tofile("/tmp/lru_o.bin")
    r = subprocess.run(["/tmp/lru_sim", "/tmp/lru_g.bin", "/tmp/lru_o.bin", str(cap)],
                       capture_output=True, text=True)
    print(k, r.stdout.strip(), flush=True)
