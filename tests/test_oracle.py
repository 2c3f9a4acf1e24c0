"""CPU tests: pin the oracle (oracle/oracle.c) to the reference's golden
vectors and known-answer tests, and -- where oracle/_ref is built -- to the
reference itself on fresh seeded graphs."""
import hashlib

import numpy as np
import pytest

from oracle import binding as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_g5_golden(small_golden):
    fx = small_golden["g5"]
    g = O.build_graph(fx["pairs"])
    assert g.off.tolist() == fx["offsets"] and g.adj.tolist() == fx["adj"]
    # test_graph.cpp:57-64, :93-119
    assert O.degree_rank(g).tolist() == fx["rank"] == [1, 2, 3, 4, 0]
    eoff, eff = O.effective(g)
    assert eoff.tolist() == fx["eff_offsets"] and eff.tolist() == fx["eff"]
    T, tv, tri = O.count(g, tally=True, listing=True)
    assert T == fx["count"] == 2
    assert tri.tolist() == [[0, 1, 2], [1, 2, 3]]
    assert O.ordering_cost(g) == fx["ordering_cost"] == 14  # test_sequential.cpp:83-87
    for k, v in fx["costs"].items():  # test_partition.cpp:30-44
        assert O.node_costs(g, k)[0].tolist() == v, k
    assert fx["costs"]["DPD"] == [7, 5, 1, 0, 1] and fx["costs"]["NOV"] == [0, 4, 6, 4, 0]
    for rec in fx["plan_025"]:  # test_engines.cpp:28-64
        rep = O.run_engine(g, rec["engine"], 2, "DPD", boundaries=[0, 2, 5],
                           collect_triangles=True)
        assert rep.total == rec["total"] == 2
        assert rep.triangles.tolist() == rec["triangles"]
        assert rep.data_sent.tolist() == rec["data_sent"]
        assert rep.data_recv.tolist() == rec["data_recv"]
        assert rep.triangles_list.tolist() == rec["triangles_list"]
        if rec["engine"] == "aop":
            assert rep.stored.tolist() == fx["overlap_stored_025"]
    by = {r["engine"]: r for r in fx["plan_025"]}
    assert by["aop"]["triangles"] == [2, 0] and by["aop"]["data_sent"] == [0, 0]
    assert by["anop-direct"]["data_sent"] == [3, 3]
    assert by["anop-surrogate"]["triangles"] == [1, 1]
    assert by["anop-surrogate"]["data_sent"] == [2, 0]
    assert O.clustering(g, tv).tolist() == fx["cc"]
    assert fx["node_counts"] == [1, 2, 2, 1, 0]


def test_known_answers(small_golden):
    fx = small_golden
    for n, want in fx["complete"].items():
        n = int(n)
        g = O.build_graph([(u, v) for u in range(n) for v in range(u + 1, n)], n)
        assert O.count(g)[0] == want == n * (n - 1) * (n - 2) // 6
    for rim, want in fx["wheel"].items():
        rim = int(rim)
        pairs = [(0, i) for i in range(1, rim + 1)] + \
                [(i, 1 if i == rim else i + 1) for i in range(1, rim + 1)]
        assert O.run_engine(O.build_graph(pairs), "aop", 2).total == want == rim
    for ab, want in fx["bipartite"].items():
        a, b = map(int, ab.split("x"))
        g = O.build_graph([(u, a + v) for u in range(a) for v in range(b)], a + b)
        assert O.run_engine(g, "anop-direct", 2).total == want == 0
    k8 = O.build_graph([(u, v) for u in range(8) for v in range(u + 1, 8)], 8)
    assert O.run_engine(k8, "anop-surrogate", 3, "NOV").total == fx["k8_nov_surrogate_p3"] == 56


def test_acceptance_suite_golden(small_golden):
    for rec in small_golden["acceptance_suite"]["graphs"]:
        g = O.random_graph(rec["n"], rec["density"], rec["seed"])
        assert sha(g.adj) == rec["adj_sha256"]
        assert O.count(g)[0] == rec["count"]
        for e in rec.get("engines", []):
            rep = O.run_engine(g, e["engine"], e["ranks"], e["cost"], track_nodes=True,
                               collect_triangles=True)
            assert rep.total == e["total"]
            assert rep.boundaries.tolist() == e["boundaries"]
            assert rep.triangles.tolist() == e["triangles"]
            assert rep.data_sent.tolist() == e["data_sent"]
            assert rep.data_recv.tolist() == e["data_recv"]
            assert sha(rep.node_counts) == e["node_counts_sha256"]
            assert sha(rep.triangles_list) == e["triangles_sha256"]


def test_criterion9_golden(small_golden):
    for rec in small_golden["criterion9"]:
        g = O.random_graph(rec["n"], rec["density"], rec["seed"])
        rep = O.run_engine(g, "anop-surrogate", 3, track_nodes=True)
        assert rep.node_counts.tolist() == rec["node_counts"]
        assert [float(x).hex() for x in O.clustering(g, rep.node_counts)] == rec["cc"]


def test_pa20000_golden(small_golden):
    from paper_1706_05151_b200 import trigraph as T  # host generator only

    rec = small_golden["pa20000"]
    g = O.build_graph(T.gen_pa(20000, 20, 3))
    assert sha(g.off) == rec["offsets_sha256"] and sha(g.adj) == rec["adj_sha256"]
    assert sha(O.degree_rank(g)) == rec["rank_sha256"]
    eoff, eff = O.effective(g)
    assert sha(eoff) == rec["eff_offsets_sha256"] and sha(eff) == rec["eff_sha256"]
    T_, tv, _ = O.count(g, tally=True)
    assert T_ == rec["count"] and O.ordering_cost(g) == rec["ordering_cost"]
    assert sha(tv) == rec["node_counts_sha256"]
    assert sha(O.clustering(g, tv)) == rec["cc_sha256"]
    for k, d in rec["costs_sha256"].items():
        assert sha(O.node_costs(g, k)[0]) == d
    for e in rec["engines"][::3]:
        rep = O.run_engine(g, e["engine"], e["ranks"], e["cost"], track_nodes=True,
                           collect_triangles=True)
        assert rep.total == e["total"] and rep.boundaries.tolist() == e["boundaries"]
        assert rep.triangles.tolist() == e["triangles"]
        assert rep.data_sent.tolist() == e["data_sent"]
        assert rep.data_recv.tolist() == e["data_recv"]
        assert sha(rep.triangles_list) == e["triangles_sha256"]


def test_generator_streams_golden(small_golden):
    """The product's host generators reproduce the reference's gen_pa /
    gen_gnp edge streams bit for bit (io.hpp:85-162)."""
    from paper_1706_05151_b200 import trigraph as T

    for rec in small_golden["gen_pa"][:2]:
        g = O.build_graph(T.gen_pa(rec["n"], rec["d"], rec["seed"]), rec["n"])
        assert sha(g.adj) == rec["adj_sha256"] and sha(g.off) == rec["offsets_sha256"]
        assert O.count(g)[0] == rec["count"]
    for rec in small_golden["gen_gnp"][:1]:
        g = O.build_graph(T.gen_gnp(rec["n"], rec["d"], rec["seed"]), rec["n"])
        assert sha(g.adj) == rec["adj_sha256"] and O.count(g)[0] == rec["count"]


def test_boundary_invariant():
    """test_partition.cpp:73-95 / acceptance criterion 6."""
    rng = np.random.default_rng(17)
    for _ in range(200):
        n = int(rng.integers(1, 61))
        f = rng.integers(0, 20, n).astype(np.uint64)
        total = int(f.sum())
        pre = np.concatenate([[0], np.cumsum(f)]).astype(object)
        for p in (1, 2, 3, 4, 8, 16):
            b = O.compute_boundaries(f, p)
            assert b[0] == 0 and b[-1] == n and all(np.diff(b.astype(np.int64)) >= 0)
            for j in range(1, p):
                x = int(b[j])
                assert p * pre[x] >= j * total
                if x > 0:
                    assert p * pre[x - 1] < j * total
    assert O.compute_boundaries([1, 1, 1, 1], 2).tolist() == [0, 2, 4]
    assert O.compute_boundaries([10, 1, 1], 2).tolist() == [0, 1, 3]
    with pytest.raises(ValueError):
        O.compute_boundaries([1], 0)


def test_full_size_goldens_shape(full_golden):
    assert full_golden["C2"]["m"] == 199_999_790  # SURVEY App. A.2, gen_pa(1e7,40,7)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_oracle_matches_reference_fresh():
    rng = np.random.default_rng(2024)
    for _ in range(12):
        n = int(rng.integers(5, 70))
        g = O.random_graph(n, float(rng.uniform(0.05, 0.9)), int(rng.integers(1 << 62)))
        R = O.RefGraph.from_csr(g)
        assert O.count(g)[0] == R.count()
        for eng in ("seq", "aop", "anop-direct", "anop-surrogate"):
            for p in (1, 3, 8):
                for cost in ("N", "D", "DH", "DDH", "DH2", "DPD", "NOV"):
                    a = O.run_engine(g, eng, p, cost, track_nodes=True, collect_triangles=True)
                    b = R.run_engine(eng, p, cost, track_nodes=True, collect_triangles=True)
                    pp = len(a.triangles)
                    assert a.total == b.total
                    assert np.array_equal(a.boundaries, b.boundaries)
                    assert np.array_equal(a.triangles, b.triangles[:pp])
                    assert np.array_equal(a.data_sent, b.data_sent[:pp])
                    assert np.array_equal(a.data_recv, b.data_recv[:pp])
                    assert np.array_equal(a.node_counts, b.node_counts)
                    assert np.array_equal(a.triangles_list, b.triangles_list)
