"""Pin the C restatement of the SURVEY 8(f) rows against the reference's own
outputs (tests/golden/reference_next.json, made by make_golden.py --next from
the unmodified headers): keep_entry / sparsified run_engine / approx_count
(sparsify.hpp, engines.hpp:335-457), per_edge_triangle_counts
(sequential.hpp:108-122) and variance_report (sparsify.hpp:113-155)."""
import hashlib

import numpy as np
import pytest

from oracle import binding as O

ENGINES = ["seq", "aop", "anop-direct", "anop-surrogate"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def graph(name):
    if name == "pa20000":
        from paper_1706_05151_b200 import trigraph as T
        return O.build_graph(T.gen_pa(20000, 20, 3))
    n, dens, seed = {"random0": (60, 0.3, 11), "random1": (90, 0.5, 12),
                     "random2": (40, 0.8, 13)}[name]
    return O.random_graph(n, dens, seed)


def test_keep_entry_table(next_golden):
    for q, seed, mode, rank, v, u, want in next_golden["keep_entry"]:
        key = 0 if mode == 1 else rank + 1
        assert O.keep_entry(q, seed, key, v, u) == bool(want)


@pytest.mark.parametrize("name", ["random0", "random1", "random2", "pa20000"])
def test_next_rows_golden(next_golden, name):
    rec = next_golden["graphs"][name]
    g = graph(name)
    assert sha(g.adj) == rec["adj_sha256"]
    te = O.per_edge_counts(g)
    assert sha(te) == rec["per_edge_sha256"]
    assert int(te.sum()) == rec["per_edge_sum"] == 3 * O.count(g)[0]
    if "per_edge" in rec:
        assert te.tolist() == rec["per_edge"]
    for r in rec["sparse"]:
        rep = O.run_engine(g, r["engine"], r["ranks"], "DPD", sparsify=r["sparsify"], q=r["q"],
                           seed=r["seed"], track_nodes=True, collect_triangles=True)
        pp = len(r["triangles"])
        assert rep.total == r["total"], r
        assert rep.triangles[:pp].tolist() == r["triangles"]
        assert rep.data_sent[:pp].tolist() == r["data_sent"]
        assert rep.data_recv[:pp].tolist() == r["data_recv"]
        assert sha(rep.node_counts) == r["node_counts_sha256"]
        assert sha(rep.triangles_list) == r["triangles_sha256"]
    for r in rec["approx"]:
        assert O.approx_count(g, r["ranks"], r["engine"], r["q"], r["seed"]) == \
            float.fromhex(r["value"])
    for r in rec["variance"]:
        T, k, kp, var, varp = O.variance_report(g, r["boundaries"], r["q"])
        assert (T, k, kp) == (r["T"], r["k"], r["k_prime"])
        assert var == float.fromhex(r["var"]) and varp == float.fromhex(r["var_prime"])
