"""Parity of the CUDA path (through the C ABI) against the reference.

Goldens: tests/golden/reference_*.json, produced by the unmodified reference
(tests/golden/make_golden.py).  Fresh cases are checked against the C
restatement in oracle/ (itself pinned to the reference in
tests/test_oracle.py).  Integer results must be bit-exact; clustering
coefficients are compared bit-exactly too (tolerance 0), which is stricter
than the 1e-12 of acceptance.cpp:418.
"""
import hashlib

import numpy as np
import pytest

from oracle import binding as O
from paper_1706_05151_b200 import trigraph as T
from paper_1706_05151_b200._lib import lib

pytestmark = pytest.mark.gpu

ENG = {"seq": T.EngineKind.Sequential, "aop": T.EngineKind.Aop,
       "anop-direct": T.EngineKind.AnopDirect, "anop-surrogate": T.EngineKind.AnopSurrogate}
COST = {"N": T.CostKind.N, "D": T.CostKind.D, "DH": T.CostKind.Dh, "DDH": T.CostKind.Ddh,
        "DH2": T.CostKind.Dh2, "DPD": T.CostKind.Dpd, "NOV": T.CostKind.Nov}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sorted_triples(t):
    t = np.asarray(t, dtype=np.uint32).reshape(-1, 3)
    return t[np.lexsort((t[:, 2], t[:, 1], t[:, 0]))]


def check_against_oracle(g: T.Graph, ref: O.CSR, engine: str, p: int, cost: str,
                         boundaries=None, lists=True):
    want = O.run_engine(ref, engine, p, cost, boundaries=boundaries, track_nodes=True,
                        collect_triangles=lists)
    cfg = T.EngineConfig(engine=ENG[engine], ranks=p, cost=COST[cost], track_nodes=True,
                         collect_triangles=lists, boundaries=boundaries)
    got = T.run_engine(g, cfg)
    pp = len(want.triangles)
    assert got.total == want.total
    assert got.boundaries.tolist() == want.boundaries.tolist()
    assert [r.triangles for r in got.per_rank] == want.triangles.tolist()
    assert [r.data_sent for r in got.per_rank] == want.data_sent.tolist()
    assert [r.data_recv for r in got.per_rank] == want.data_recv.tolist()
    assert [r.stored_entries for r in got.per_rank] == want.stored.tolist()
    assert np.array_equal(got.node_counts, want.node_counts)
    if lists:
        assert np.array_equal(sorted_triples(got.triangles_list), want.triangles_list)
    assert len(got.per_rank) == pp


# ------------------------------------------------------------------ G5


def test_g5_fixture(small_golden):
    fx = small_golden["g5"]
    g = T.build_graph(fx["pairs"])
    off, adj = g.csr()
    assert off.tolist() == fx["offsets"] and adj.tolist() == fx["adj"]
    assert T.compute_order(g).rank.tolist() == fx["rank"] == [1, 2, 3, 4, 0]
    eff = T.effective_adjacency(g)
    assert eff.offsets.tolist() == fx["eff_offsets"] and eff.entries.tolist() == fx["eff"]
    assert T.count_node_iterator_n(g) == fx["count"] == 2
    assert T.ordering_cost(g) == fx["ordering_cost"] == 14
    for k, v in fx["costs"].items():
        assert T.node_costs(g, COST[k]).f.tolist() == v, k
    for rec in fx["plan_025"]:
        rep = T.run_engine(g, T.EngineConfig(engine=ENG[rec["engine"]], ranks=2,
                                             boundaries=[0, 2, 5], collect_triangles=True,
                                             track_nodes=True))
        assert rep.total == rec["total"]
        assert [r.triangles for r in rep.per_rank] == rec["triangles"]
        assert [r.data_sent for r in rep.per_rank] == rec["data_sent"]
        assert [r.data_recv for r in rep.per_rank] == rec["data_recv"]
        assert sorted_triples(rep.triangles_list).tolist() == rec["triangles_list"]
        if rec["engine"] == "aop":
            assert [r.stored_entries for r in rep.per_rank] == fx["overlap_stored_025"]
    for e in ENG:
        cc = T.clustering_coefficients(g, T.EngineConfig(engine=ENG[e], ranks=2))
        assert cc.triangles_per_node.tolist() == fx["node_counts"] == [1, 2, 2, 1, 0]
        assert cc.coefficient.tolist() == fx["cc"]


def test_known_answers(small_golden):
    fx = small_golden
    for n, want in fx["complete"].items():
        n = int(n)
        pairs = [(u, v) for u in range(n) for v in range(u + 1, n)]
        g = T.build_graph(pairs, n)
        assert T.count_node_iterator_n(g) == want == n * (n - 1) * (n - 2) // 6
        rep = T.run_engine(g, T.EngineConfig(engine=T.EngineKind.AnopSurrogate, ranks=3))
        assert rep.total == want
    for rim, want in fx["wheel"].items():
        rim = int(rim)
        pairs = [(0, i) for i in range(1, rim + 1)] + \
                [(i, 1 if i == rim else i + 1) for i in range(1, rim + 1)]
        g = T.build_graph(pairs)
        assert T.run_engine(g, T.EngineConfig(engine=T.EngineKind.Aop, ranks=2)).total == want == rim
    for ab, want in fx["bipartite"].items():
        a, b = map(int, ab.split("x"))
        g = T.build_graph([(u, a + v) for u in range(a) for v in range(b)], a + b)
        assert T.run_engine(g, T.EngineConfig(engine=T.EngineKind.AnopDirect, ranks=2)).total == want == 0
    k8 = T.build_graph([(u, v) for u in range(8) for v in range(u + 1, 8)], 8)
    rep = T.run_engine(k8, T.EngineConfig(engine=T.EngineKind.AnopSurrogate, ranks=3,
                                          cost=T.CostKind.Nov))
    assert rep.total == fx["k8_nov_surrogate_p3"] == 56


# ------------------------------------------------------- acceptance suite


def test_acceptance_suite(small_golden):
    suite = small_golden["acceptance_suite"]["graphs"]
    for i, rec in enumerate(suite):
        pairs = O.random_graph_pairs(rec["n"], rec["density"], rec["seed"])
        g = T.build_graph(pairs, rec["n"])
        _, adj = g.csr()
        assert sha(adj) == rec["adj_sha256"], i
        assert T.count_node_iterator_n(g) == rec["count"], i
        for e in rec.get("engines", []):
            rep = T.run_engine(g, T.EngineConfig(engine=ENG[e["engine"]], ranks=e["ranks"],
                                                 cost=COST[e["cost"]], track_nodes=True,
                                                 collect_triangles=True))
            assert rep.total == e["total"]
            assert rep.boundaries.tolist() == e["boundaries"]
            assert [r.triangles for r in rep.per_rank] == e["triangles"]
            assert [r.data_sent for r in rep.per_rank] == e["data_sent"]
            assert [r.data_recv for r in rep.per_rank] == e["data_recv"]
            assert sha(rep.node_counts) == e["node_counts_sha256"]
            assert sha(sorted_triples(rep.triangles_list)) == e["triangles_sha256"]
        g.close()


def test_criterion9_clustering(small_golden):
    for rec in small_golden["criterion9"]:
        pairs = O.random_graph_pairs(rec["n"], rec["density"], rec["seed"])
        g = T.build_graph(pairs, rec["n"])
        for e in ENG:
            cc = T.clustering_coefficients(g, T.EngineConfig(engine=ENG[e], ranks=3))
            assert cc.triangles_per_node.tolist() == rec["node_counts"]
            assert [float(x).hex() for x in cc.coefficient] == rec["cc"]


def test_pa20000_all_engines(small_golden, warp_variant):
    rec = small_golden["pa20000"]
    g = T.build_graph(T.gen_pa(20000, 20, 3))
    off, adj = g.csr()
    assert sha(off) == rec["offsets_sha256"] and sha(adj) == rec["adj_sha256"]
    assert sha(T.compute_order(g).rank) == rec["rank_sha256"]
    eff = T.effective_adjacency(g)
    assert sha(eff.offsets) == rec["eff_offsets_sha256"] and sha(eff.entries) == rec["eff_sha256"]
    assert T.count_node_iterator_n(g) == rec["count"]
    assert T.ordering_cost(g) == rec["ordering_cost"]
    for k, d in rec["costs_sha256"].items():
        assert sha(T.node_costs(g, COST[k]).f) == d, k
    cc = T.clustering_coefficients(g, T.EngineConfig(engine=T.EngineKind.Sequential))
    assert sha(cc.triangles_per_node) == rec["node_counts_sha256"]
    assert sha(cc.coefficient) == rec["cc_sha256"]
    for e in rec["engines"]:
        rep = T.run_engine(g, T.EngineConfig(engine=ENG[e["engine"]], ranks=e["ranks"],
                                             cost=COST[e["cost"]], track_nodes=True,
                                             collect_triangles=True))
        assert rep.total == e["total"]
        assert rep.boundaries.tolist() == e["boundaries"]
        assert [r.triangles for r in rep.per_rank] == e["triangles"], e
        assert [r.data_sent for r in rep.per_rank] == e["data_sent"], e
        assert [r.data_recv for r in rep.per_rank] == e["data_recv"], e
        assert sha(rep.node_counts) == e["node_counts_sha256"]
        assert sha(sorted_triples(rep.triangles_list)) == e["triangles_sha256"]


def test_generators_match_reference_streams(small_golden):
    for rec in small_golden["gen_pa"]:
        g = T.build_graph(T.gen_pa(rec["n"], rec["d"], rec["seed"]), rec["n"])
        off, adj = g.csr()
        assert sha(adj) == rec["adj_sha256"] and sha(off) == rec["offsets_sha256"]
        assert T.count_node_iterator_n(g) == rec["count"]
    for rec in small_golden["gen_gnp"]:
        g = T.build_graph(T.gen_gnp(rec["n"], rec["d"], rec["seed"]), rec["n"])
        _, adj = g.csr()
        assert sha(adj) == rec["adj_sha256"]
        assert T.count_node_iterator_n(g) == rec["count"]


# ------------------------------------------------ fresh cases vs the oracle


@pytest.fixture(params=[1, 2, 3, 4], ids=["scalar", "quad-groups", "quads", "scalar-groups"])
def warp_variant(request):
    lib().tg_debug_set_warp_variant(request.param)
    yield request.param
    lib().tg_debug_set_warp_variant(0)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_graphs_all_engines_costs(seed, warp_variant):
    rng = np.random.default_rng(seed)
    for _ in range(4):
        n = int(rng.integers(20, 120))
        dens = float(rng.uniform(0.05, 0.6))
        pairs = O.random_graph_pairs(n, dens, int(rng.integers(1 << 62)))
        ref = O.build_graph(pairs, n)
        g = T.build_graph(pairs, n)
        for engine in ENG:
            for p in (1, 2, 3, 4, 8, 16):
                if engine == "seq" and p > 1:
                    continue
                for cost in ("N", "D", "DH", "DDH", "DH2", "DPD", "NOV"):
                    check_against_oracle(g, ref, engine, p, cost)


def test_edge_cases():
    # empty graph (test_graph.cpp:31-35)
    g = T.build_graph(np.zeros((0, 2), np.uint32))
    assert g.num_nodes() == 0 and g.num_edges() == 0
    assert T.count_node_iterator_n(g) == 0
    rep = T.run_engine(g, T.EngineConfig(engine=T.EngineKind.AnopSurrogate, ranks=4,
                                         track_nodes=True, collect_triangles=True))
    assert rep.total == 0 and rep.boundaries.tolist() == [0, 0, 0, 0, 0]
    # self-loops and duplicates (test_graph.cpp:10-17)
    g = T.build_graph([(0, 1), (1, 0), (2, 2)])
    assert g.num_nodes() == 3 and g.num_edges() == 1
    off, adj = g.csr()
    assert off.tolist() == [0, 1, 2, 2] and adj.tolist() == [1, 0]
    # n_override keeps trailing isolated nodes (test_graph.cpp:46-50)
    g = T.build_graph([(0, 1)], 5)
    assert g.num_nodes() == 5 and g.degree(4) == 0
    # isolated-only graph
    g = T.build_graph(np.zeros((0, 2), np.uint32), 7)
    assert g.num_nodes() == 7 and T.count_node_iterator_n(g) == 0
    # star: hub last in degree order, no triangles (test_graph.cpp:75-79)
    g = T.build_graph([(0, i) for i in range(1, 5)])
    assert T.compute_order(g).rank[0] == 4
    cc = T.clustering_coefficients(g, T.EngineConfig(engine=T.EngineKind.AnopSurrogate, ranks=2))
    assert cc.coefficient.tolist() == [0.0] * 5
    # rank validation (test_engines.cpp:172-175)
    g = T.build_graph([(0, 1), (1, 2), (0, 2)])
    with pytest.raises(ValueError):
        T.run_engine(g, T.EngineConfig(engine=T.EngineKind.Aop, ranks=0))
    with pytest.raises(ValueError):
        T.compute_boundaries(g, T.CostKind.Dpd, 0)
    # empty cores are legal (test_partition.cpp:57-69)
    rep = T.run_engine(g, T.EngineConfig(engine=T.EngineKind.AnopSurrogate, ranks=16))
    assert rep.total == 1


def test_long_lists_block_and_global_paths(warp_variant):
    """Apex lists longer than the warp path (64) go to the CTA path; lists
    longer than the CTA's shared-memory capacity are searched in global
    memory.  Lower the capacity to exercise the global path on a small graph."""
    n = 160
    pairs = [(u, v) for u in range(n) for v in range(u + 1, n) if (u * 7 + v * 13) % 5 != 0]
    pairs += [(0, v) for v in range(n, n + 300)]
    ref = O.build_graph(pairs)
    g = T.build_graph(pairs)
    for cap in (0, 16):
        lib().tg_debug_set_block_cap(cap)
        try:
            for engine in ENG:
                check_against_oracle(g, ref, engine, 1 if engine == "seq" else 3, "DPD")
        finally:
            lib().tg_debug_set_block_cap(0)


def test_orientation_hubs():
    """The one-pass orientation's three routes: tile vertices (degree <= 256),
    warp-per-vertex big vertices (<= 4096) and CTA-per-hub segments of 8192
    entries (a hub of 20000 spans three), against the oracle's oriented CSR,
    count and per-node tallies."""
    rng = np.random.default_rng(5)
    n = 30000
    pairs = [(0, v) for v in range(1, 20001)]            # hub, 3 segments
    pairs += [(1, v) for v in range(2, 5002)]            # hub, 1 segment
    pairs += [(2, v) for v in range(3, 303)]             # big (warp path)
    pairs += [(3, v) for v in range(4, 262)]             # just above the tile limit
    e = rng.integers(0, n, size=(120000, 2))
    pairs = np.concatenate([np.asarray(pairs, np.int64), e]).astype(np.uint32)
    ref = O.build_graph(pairs, n)
    g = T.build_graph(pairs, n)
    eff = T.effective_adjacency(g)
    want_off, want_eff = O.effective(ref)
    assert np.array_equal(eff.offsets, want_off)
    assert np.array_equal(eff.entries, want_eff)
    total, tally = O.count(ref, tally=True)[:2]
    assert T.count_node_iterator_n(g) == total
    check_against_oracle(g, ref, "seq", 1, "DPD", lists=False)
    check_against_oracle(g, ref, "aop", 4, "DPD", lists=False)


def test_device_step_and_rank_entries():
    import ctypes as C
    import torch

    pairs = T.gen_pa(50000, 20, 11)
    ref = O.build_graph(pairs)
    want = O.count(ref)[0]
    g = T.build_graph(pairs)
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    L = lib()
    assert L.tg_step_device(g._h, C.c_void_p(d.data_ptr())) == 0
    torch.cuda.synchronize()
    assert int(d.item()) == want
    assert L.tg_count_device(g._h, C.c_void_p(d.data_ptr())) == 0
    torch.cuda.synchronize()
    assert int(d.item()) == want
    assert L.tg_last_intersect_ms(g._h) > 0
    # the rank-local AOP / surrogate entries, p=3 ranks run one after another
    p = 3
    b = T.compute_boundaries(g, T.CostKind.Dpd, p).boundaries
    bp = C.c_void_p(b.ctypes.data)
    want_rep = O.run_engine(ref, "aop", p, "DPD")
    for i in range(p):
        d.zero_()
        assert L.tg_aop_rank_device(g._h, bp, p, i, C.c_void_p(d.data_ptr())) == 0
        torch.cuda.synchronize()
        assert int(d.item()) == int(want_rep.triangles[i])
    want_s = O.run_engine(ref, "anop-surrogate", p, "DPD")
    send = []
    for i in range(p):
        msgs = np.zeros(p, np.uint64)
        words = np.zeros(p, np.uint64)
        assert L.tg_surrogate_pack_sizes(g._h, bp, p, i, C.c_void_p(msgs.ctypes.data),
                                         C.c_void_p(words.ctypes.data)) == 0
        hdr = torch.zeros(int(2 * msgs.sum()) + 1, dtype=torch.int32, device="cuda")
        dat = torch.zeros(int(words.sum()) + 1, dtype=torch.int32, device="cuda")
        assert L.tg_surrogate_pack_device(g._h, bp, p, i, C.c_void_p(hdr.data_ptr()),
                                          C.c_void_p(dat.data_ptr())) == 0
        torch.cuda.synchronize()
        assert int(msgs.sum()) == int(want_s.data_sent[i])
        send.append((msgs, words, hdr, dat))
    for j in range(p):
        hs, ds = [], []
        for i in range(p):
            msgs, words, hdr, dat = send[i]
            m0, w0 = int(msgs[:j].sum()), int(words[:j].sum())
            hs.append(hdr[2 * m0: 2 * (m0 + int(msgs[j]))])
            ds.append(dat[w0: w0 + int(words[j])])
        rh = torch.cat(hs) if hs else torch.zeros(0, dtype=torch.int32, device="cuda")
        rd = torch.cat(ds)
        nm = rh.numel() // 2
        assert nm == int(want_s.data_recv[j])
        d.zero_()
        rh = rh if rh.numel() else torch.zeros(2, dtype=torch.int32, device="cuda")
        rd = rd if rd.numel() else torch.zeros(1, dtype=torch.int32, device="cuda")
        assert L.tg_surrogate_count_device(g._h, bp, p, j, C.c_void_p(rh.data_ptr()), nm,
                                           C.c_void_p(rd.data_ptr()), C.c_void_p(d.data_ptr())) == 0
        torch.cuda.synchronize()
        assert int(d.item()) == int(want_s.triangles[j])


# ------------------------------------------------------ full-size configs


def test_config1_full(full_golden):
    rec = full_golden["C1"]
    pairs = T.gen_gnm(100_000, 1_000_000, 1)
    assert sha(pairs) == rec["pairs_sha256"]
    g = T.build_graph(pairs, 100_000)
    _, adj = g.csr()
    assert sha(adj) == rec["adj_sha256"]
    assert T.count_node_iterator_n(g) == rec["count"]
    assert T.ordering_cost(g) == rec["ordering_cost"]
    cc = T.clustering_coefficients(g, T.EngineConfig(engine=T.EngineKind.Aop, ranks=8))
    assert sha(cc.triangles_per_node) == rec["node_counts_sha256"]
    assert sha(cc.coefficient) == rec["cc_sha256"]
    for e in rec["engines"]:
        rep = T.run_engine(g, T.EngineConfig(engine=ENG[e["engine"]], ranks=e["ranks"],
                                             cost=COST[e["cost"]], track_nodes=True,
                                             collect_triangles=True))
        assert rep.total == e["total"]
        assert [r.triangles for r in rep.per_rank] == e["triangles"]
        assert [r.data_sent for r in rep.per_rank] == e["data_sent"]
        assert sha(sorted_triples(rep.triangles_list)) == e["triangles_sha256"]


def test_config2_full(full_golden):
    rec = full_golden["C2"]
    pairs = T.gen_pa(10_000_000, 40, 7)
    g = T.build_graph(pairs, 10_000_000)
    del pairs
    assert g.num_edges() == rec["m"]
    _, adj = g.csr()
    assert sha(adj) == rec["adj_sha256"]
    del adj
    assert T.count_node_iterator_n(g) == rec["count"]
    assert T.ordering_cost(g) == rec["ordering_cost"]
    for engine, p in (("aop", 8), ("anop-surrogate", 8)):
        rep = T.run_engine(g, T.EngineConfig(engine=ENG[engine], ranks=p))
        assert rep.total == rec["count"]
