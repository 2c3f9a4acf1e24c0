"""GPU parity of the SURVEY 8(f) rows through the C ABI: sparsified
run_engine / approx_count (sparsify.hpp, engines.hpp:335-457), per-edge
triangle counts (sequential.hpp:108-122) and variance_report
(sparsify.hpp:113-155) -- bit-exact against the reference's goldens
(tests/golden/reference_next.json) and the C restatement on fresh graphs."""
import hashlib

import numpy as np
import pytest

from oracle import binding as O
from paper_1706_05151_b200 import trigraph as T

pytestmark = pytest.mark.gpu

ENG = {"seq": T.EngineKind.Sequential, "aop": T.EngineKind.Aop,
       "anop-direct": T.EngineKind.AnopDirect, "anop-surrogate": T.EngineKind.AnopSurrogate}
MODE = {"global": T.SparsifyMode.Global, "per-partition": T.SparsifyMode.PerPartition}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sorted_triples(t):
    t = np.asarray(t, dtype=np.uint32).reshape(-1, 3)
    return t[np.lexsort((t[:, 2], t[:, 1], t[:, 0]))]


def graphs():
    yield "pa20000", T.gen_pa(20000, 20, 3), 0
    for name, (n, dens, seed) in (("random0", (60, 0.3, 11)), ("random1", (90, 0.5, 12)),
                                  ("random2", (40, 0.8, 13))):
        yield name, O.random_graph_pairs(n, dens, seed), n


def sparse_cfg(r):
    return T.EngineConfig(engine=ENG[r["engine"]], ranks=r["ranks"], track_nodes=True,
                          collect_triangles=True,
                          sparsify=T.SparsifyConfig(r["q"], r["seed"], MODE[r["sparsify"]]))


def test_next_rows_golden(next_golden):
    for name, pairs, n in graphs():
        rec = next_golden["graphs"][name]
        g = T.build_graph(pairs, n)
        _, adj = g.csr()
        assert sha(adj) == rec["adj_sha256"]
        te = T.per_edge_triangle_counts(g)
        assert sha(te) == rec["per_edge_sha256"], name
        assert int(te.sum()) == rec["per_edge_sum"]
        for r in rec["sparse"]:
            rep = T.run_engine(g, sparse_cfg(r))
            pp = len(r["triangles"])
            assert rep.total == r["total"], (name, r)
            assert [x.triangles for x in rep.per_rank] == r["triangles"]
            assert [x.data_sent for x in rep.per_rank] == r["data_sent"]
            assert [x.data_recv for x in rep.per_rank] == r["data_recv"]
            assert len(rep.per_rank) == pp
            assert sha(rep.node_counts) == r["node_counts_sha256"]
            assert sha(sorted_triples(rep.triangles_list)) == r["triangles_sha256"]
        for r in rec["approx"]:
            assert T.approx_count(g, r["ranks"], ENG[r["engine"]], r["q"], r["seed"]) == \
                float.fromhex(r["value"])
        for r in rec["variance"]:
            vr = T.variance_report(g, T.PartitionPlan(np.array(r["boundaries"], np.uint32)),
                                   r["q"])
            assert (vr.triangles, vr.k, vr.k_prime) == (r["T"], r["k"], r["k_prime"])
            assert vr.var == float.fromhex(r["var"])
            assert vr.var_prime == float.fromhex(r["var_prime"])


@pytest.mark.parametrize("seed", [5, 6])
def test_sparsify_fresh_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    for _ in range(3):
        n = int(rng.integers(30, 150))
        pairs = O.random_graph_pairs(n, float(rng.uniform(0.1, 0.6)), int(rng.integers(1 << 62)))
        ref = O.build_graph(pairs, n)
        g = T.build_graph(pairs, n)
        q = float(rng.choice([0.2, 0.5, 0.9]))
        s = int(rng.integers(1 << 63))
        for eng in ENG:
            for mode in MODE:
                for p in (1, 3, 7):
                    if eng == "seq" and p > 1:
                        continue
                    want = O.run_engine(ref, eng, p, "DPD", sparsify=mode, q=q, seed=s,
                                        track_nodes=True, collect_triangles=True)
                    got = T.run_engine(g, T.EngineConfig(
                        engine=ENG[eng], ranks=p, track_nodes=True, collect_triangles=True,
                        sparsify=T.SparsifyConfig(q, s, MODE[mode])))
                    assert got.total == want.total
                    assert [r.triangles for r in got.per_rank] == want.triangles.tolist()
                    assert [r.data_sent for r in got.per_rank] == want.data_sent.tolist()
                    assert [r.data_recv for r in got.per_rank] == want.data_recv.tolist()
                    assert [r.stored_entries for r in got.per_rank] == want.stored.tolist()
                    assert np.array_equal(got.node_counts, want.node_counts)
                    assert np.array_equal(sorted_triples(got.triangles_list), want.triangles_list)
        assert np.array_equal(T.per_edge_triangle_counts(g), O.per_edge_counts(ref))


def test_next_rows_edge_cases():
    g = T.build_graph(np.zeros((0, 2), np.uint32), 4)
    assert T.per_edge_triangle_counts(g).size == 0
    assert T.approx_count(g, 2, T.EngineKind.Aop, 0.5, 1) == 0.0
    k4 = T.build_graph([(u, v) for u in range(4) for v in range(u + 1, 4)])
    assert T.per_edge_triangle_counts(k4).tolist() == [2] * 6  # each K4 edge is in 2 triangles
    with pytest.raises(ValueError):
        T.approx_count(k4, 2, T.EngineKind.Aop, 0.0, 1)  # sparsify.hpp:28-31
    with pytest.raises(ValueError):
        T.run_engine(k4, T.EngineConfig(sparsify=T.SparsifyConfig(q=1.5)))
    # q = 1 keeps everything: the estimate is the exact count
    assert T.approx_count(k4, 3, T.EngineKind.AnopSurrogate, 1.0, 9) == 4.0
