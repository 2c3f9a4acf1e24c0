"""Reuse structure of the N_u reads of the intersection pass on a PA graph.

Analysis only (oracle-built oriented CSR; never on the product path). Prints
W, the N_v / N_u split, 32-byte sectors touched by the N_u reads with lists
in ID order, and how much of the N_u read volume falls on the hottest lists
(lists ranked by reuse = in-degree in the oriented graph) for a given budget
of list bytes -- the case for a contiguous, L2-pinned hot region.

usage: python tools/exp/pa_reuse.py N [d]
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import binding as O  # noqa: E402

n = int(float(sys.argv[1]))
d = int(sys.argv[2]) if len(sys.argv) > 2 else 40
pairs = O.lib()
from paper_1706_05151_b200 import trigraph as T  # noqa: E402  (generator only)

p = T.gen_pa(n, d, 7)
g = O.build_graph(p)
del p
eoff, eff = O.effective(g)
eoff = eoff.astype(np.int64)
h = np.diff(eoff)
deg = np.diff(g.off.astype(np.int64))
indeg = np.bincount(eff, minlength=g.n).astype(np.int64)  # reads of N_u
W = int((deg * h).sum())
nv = int((h * h).sum())
nu = int((indeg * h).sum())
print(f"n={g.n} m={g.m} W={W} sum h_v^2={nv} ({nv / W:.2f}) sum_(v->u) h_u={nu} ({nu / W:.2f})")
# sectors touched by each N_u read in the compact CSR (lists in ID order)
s0 = (eoff[:-1] * 4) // 32
s1 = (eoff[1:] * 4 + 31) // 32
sec = np.where(h > 0, s1 - s0, 0)
nu_sec_bytes = int((indeg * sec).sum()) * 32
print(f"N_u bytes algorithmic {4 * nu / 1e9:.3f} GB, sector-rounded {nu_sec_bytes / 1e9:.3f} GB "
      f"({nu_sec_bytes / (4 * nu):.2f}x); descriptors {8 * g.m / 1e9:.3f} GB")
# hot-list curve: lists by reuse (in-degree) descending
order = np.argsort(-indeg, kind="stable")
cb = np.cumsum(4 * h[order])
cr = np.cumsum(indeg[order] * h[order])
for frac in (0.005, 0.01, 0.02, 0.05, 0.1, 0.2):
    k = np.searchsorted(cb, frac * cb[-1])
    print(f"  hottest lists holding {frac:5.1%} of the bytes ({cb[k] / 1e6:8.1f} MB): "
          f"{cr[k] / cr[-1]:.3f} of N_u reads; degree >= {deg[order[k]]}")
# by degree threshold (what a degree-keyed layout can do without a sort)
for D in (64, 128, 256, 512, 1024):
    sel = deg >= D
    print(f"  degree >= {D:5d}: {sel.mean():.4f} of vertices, {4 * h[sel].sum() / 1e6:8.1f} MB of "
          f"lists, {(indeg[sel] * h[sel]).sum() / cr[-1]:.3f} of N_u reads")
