"""Pin the oracle's OrderKind restatement (oracle.c orc_compute_order /
orc_coreness / orc_run_engine_ord) against the reference: the golden
fixtures of tests/golden/reference_orders.json, and the unmodified reference
(oracle/_ref) on fresh seeded graphs when it is built."""
import numpy as np
import pytest

from oracle import binding as O
from orders_common import fixture_graphs, sha, sorted_triples


def test_coreness_small_fixtures(orders_golden):
    # test_graph.cpp:51-55
    assert O.coreness(O.build_graph([[0, 1], [0, 2], [1, 2]])).tolist() == orders_golden["k3_coreness"]
    assert O.coreness(O.build_graph([[0, 1], [1, 2]])).tolist() == orders_golden["path_coreness"]
    assert orders_golden["g5"]["coreness"] == [2, 2, 2, 2, 1]


def test_g5_orders_explicit(orders_golden):
    g = O.build_graph([[0, 1], [0, 2], [1, 2], [1, 3], [2, 3], [3, 4]])
    for o in orders_golden["g5"]["orders"]:
        assert O.compute_order(g, o["order"], o["seed"]).tolist() == o["rank"]
        eoff, eff = O.effective(g, o["order"], o["seed"])
        assert eoff.tolist() == o["eff_offsets"] and eff.tolist() == o["eff"]
        assert O.ordering_cost(g, o["order"], o["seed"]) == o["ordering_cost"]
    by = {(o["order"], o["seed"]): o for o in orders_golden["g5"]["orders"]}
    assert by[("id", 0)]["ordering_cost"] == 16  # test_sequential.cpp:86
    assert by[("degree", 0)]["ordering_cost"] == 14  # test_sequential.cpp:85


def test_orders_against_golden(orders_golden):
    for name, pairs, n_over, rec in fixture_graphs(orders_golden):
        g = O.build_graph(pairs, n_over)
        assert sha(g.adj) == rec["adj_sha256"], name
        assert sha(O.coreness(g)) == rec["coreness_sha256"], name
        for o in rec["orders"]:
            order, seed = o["order"], o["seed"]
            assert sha(O.compute_order(g, order, seed)) == o["rank_sha256"], (name, order)
            eoff, eff = O.effective(g, order, seed)
            assert sha(eoff) == o["eff_offsets_sha256"] and sha(eff) == o["eff_sha256"]
            assert O.ordering_cost(g, order, seed) == o["ordering_cost"]
            if name in ("pa20000", "rmat12"):
                continue  # engines on the big fixtures: checked on the device
            for e in o["engines"]:
                r = O.run_engine(g, e["engine"], e["ranks"], order=order, order_seed=seed,
                                 track_nodes=True, collect_triangles=True)
                assert r.total == e["total"] == o["count"]
                assert r.boundaries.tolist() == e["boundaries"]
                assert r.triangles.tolist() == e["triangles"]
                assert r.data_sent.tolist() == e["data_sent"]
                assert r.data_recv.tolist() == e["data_recv"]
                assert sha(r.node_counts) == e["node_counts_sha256"]
                assert sha(sorted_triples(r.triangles_list)) == e["triangles_sha256"]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_orders_against_reference_fresh():
    for seed in range(20):
        n = 30 + 11 * seed
        R = O.ref_random_graph(n, 0.08 + 0.02 * (seed % 9), 9000 + seed)
        g = R.csr()
        assert np.array_equal(O.coreness(g), R.coreness())
        for order in ("id", "degree", "random", "coreness"):
            s = 3 * seed + 1
            assert np.array_equal(O.compute_order(g, order, s), R.compute_order(order, s))
            eoff, eff, cnt, cost = R.effective_order(order, s)
            e2, f2 = O.effective(g, order, s)
            assert np.array_equal(eoff, e2) and np.array_equal(eff, f2)
            assert O.ordering_cost(g, order, s) == cost
            for eng in ("aop", "anop-direct", "anop-surrogate"):
                a = O.run_engine(g, eng, 4, order=order, order_seed=s)
                b = R.run_engine_order(eng, 4, order, s)
                assert a.total == b.total == cnt
                assert a.triangles.tolist() == b.triangles.tolist()
                assert a.data_sent.tolist() == b.data_sent.tolist()
                assert a.boundaries.tolist() == b.boundaries.tolist()
