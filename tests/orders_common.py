"""Shared helpers for the OrderKind parity tests (oracle and device)."""
import hashlib

import numpy as np

from oracle import binding as O

ENGINE_NAMES = ("seq", "aop", "anop-direct", "anop-surrogate")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sorted_triples(t):
    t = np.asarray(t, dtype=np.uint32).reshape(-1, 3)
    return t[np.lexsort((t[:, 2], t[:, 1], t[:, 0]))]


def fixture_graphs(fx):
    """(name, pairs, n_override, record) for every graph in reference_orders.json."""
    from paper_1706_05151_b200 import trigraph as T  # host generators only

    g5 = np.array([[0, 1], [0, 2], [1, 2], [1, 3], [2, 3], [3, 4]], dtype=np.uint32)
    out = [("g5", g5, 0, fx["g5"])]
    for rec in fx["random"]:
        n, dens, seed = rec["gen"]
        out.append((f"random{n}", O.random_graph_pairs(n, dens, seed), n, rec))
    out.append(("pa20000", T.gen_pa(20000, 20, 3), 0, fx["pa20000"]))
    pairs = T.gen_rmat(12, 8, 0.57, 0.19, 0.19, 5)
    assert sha(np.ascontiguousarray(pairs, dtype=np.uint32)) == fx["rmat12"]["pairs_sha256"]
    out.append(("rmat12", pairs, 0, fx["rmat12"]))
    return out
