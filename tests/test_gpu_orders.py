"""Every OrderKind of the reference (order.hpp:17-128) on the device, through
the C ABI: compute_order, coreness, effective_adjacency, ordering_cost, the
count and run_engine (EngineConfig::order, engines.hpp:274), bit-exact
against tests/golden/reference_orders.json (made by the unmodified reference)
and against the oracle on fresh graphs."""
import numpy as np
import pytest

from oracle import binding as O
from orders_common import fixture_graphs, sha, sorted_triples
from paper_1706_05151_b200 import trigraph as T
from paper_1706_05151_b200._lib import check, lib

pytestmark = pytest.mark.gpu

ENG = {"seq": T.EngineKind.Sequential, "aop": T.EngineKind.Aop,
       "anop-direct": T.EngineKind.AnopDirect, "anop-surrogate": T.EngineKind.AnopSurrogate}


def kind(order, seed):
    return {"id": T.OrderKind.by_id(), "degree": T.OrderKind.by_degree(),
            "random": T.OrderKind.by_random(seed), "coreness": T.OrderKind.by_coreness()}[order]


def test_coreness_fixtures(orders_golden):
    # test_graph.cpp:51-55
    with T.build_graph([[0, 1], [0, 2], [1, 2]]) as g:
        assert T.coreness(g).tolist() == orders_golden["k3_coreness"]
    with T.build_graph([[0, 1], [1, 2]]) as g:
        assert T.coreness(g).tolist() == orders_golden["path_coreness"]


def test_g5_orders_explicit(orders_golden):
    fx = orders_golden["g5"]
    with T.build_graph([[0, 1], [0, 2], [1, 2], [1, 3], [2, 3], [3, 4]]) as g:
        assert T.coreness(g).tolist() == fx["coreness"]
        for o in fx["orders"]:
            k = kind(o["order"], o["seed"])
            assert T.compute_order(g, k).rank.tolist() == o["rank"]
            e = T.effective_adjacency(g, k)
            assert e.offsets.tolist() == o["eff_offsets"] and e.entries.tolist() == o["eff"]
            assert T.ordering_cost(g, k) == o["ordering_cost"]
            assert T.count_node_iterator_n(g, k) == o["count"] == 2


@pytest.mark.parametrize("which", ["g5", "random", "pa20000", "rmat12"])
def test_orders_against_golden(orders_golden, which):
    for name, pairs, n_over, rec in fixture_graphs(orders_golden):
        if not name.startswith(which):
            continue
        with T.build_graph(pairs, n_over) as g:
            off, adj = g.csr()
            assert sha(adj) == rec["adj_sha256"], name
            assert sha(T.coreness(g)) == rec["coreness_sha256"], name
            for o in rec["orders"]:
                k = kind(o["order"], o["seed"])
                assert sha(T.compute_order(g, k).rank) == o["rank_sha256"], (name, k)
                e = T.effective_adjacency(g, k)
                assert sha(e.offsets) == o["eff_offsets_sha256"], (name, k)
                assert sha(e.entries) == o["eff_sha256"], (name, k)
                assert T.ordering_cost(g, k) == o["ordering_cost"]
                assert T.count_node_iterator_n(g, k) == o["count"]
                for rec_e in o["engines"]:
                    cfg = T.EngineConfig(engine=ENG[rec_e["engine"]], ranks=rec_e["ranks"],
                                         order=k, track_nodes=True, collect_triangles=True)
                    r = T.run_engine(g, cfg)
                    assert r.total == rec_e["total"], (name, k, rec_e["engine"])
                    assert r.boundaries.tolist() == rec_e["boundaries"]
                    assert [x.triangles for x in r.per_rank] == rec_e["triangles"]
                    assert [x.data_sent for x in r.per_rank] == rec_e["data_sent"]
                    assert [x.data_recv for x in r.per_rank] == rec_e["data_recv"]
                    assert sha(r.node_counts) == rec_e["node_counts_sha256"]
                    assert sha(sorted_triples(r.triangles_list)) == rec_e["triangles_sha256"]


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 5, 6])
def test_long_lists_under_id_order(variant):
    """ById orients every edge toward the larger id, so PA's oldest vertices
    carry lists of thousands of entries (the CTA path, and with a lowered
    block cap the global-memory search); every kernel variant must agree with
    the oracle, tallies and listing included."""
    pairs = T.gen_pa(30000, 20, 11)
    ref = O.build_graph(pairs)
    want_T, want_tv, want_tri = O.count(ref, tally=True, listing=True, order="id")
    L = lib()
    try:
        L.tg_debug_set_warp_variant(variant)
        with T.build_graph(pairs) as g:
            for cap in (0, 256):
                L.tg_debug_set_block_cap(cap)
                cfg = T.EngineConfig(engine=T.EngineKind.Sequential, order=T.OrderKind.by_id(),
                                     track_nodes=True, collect_triangles=True)
                r = T.run_engine(g, cfg)
                assert r.total == want_T
                assert np.array_equal(r.node_counts, want_tv)
                assert np.array_equal(sorted_triples(r.triangles_list), want_tri)
    finally:
        L.tg_debug_set_block_cap(0)
        L.tg_debug_set_warp_variant(0)


def test_fresh_graphs_against_oracle():
    for i, (scale, ef, seed) in enumerate(((13, 16, 1), (14, 8, 2))):
        pairs = T.gen_rmat(scale, ef, 0.57, 0.19, 0.19, seed)
        ref = O.build_graph(pairs)
        with T.build_graph(pairs) as g:
            assert np.array_equal(T.coreness(g), O.coreness(ref))
            for order in ("id", "random", "coreness"):
                s = 17 + i
                k = kind(order, s)
                assert np.array_equal(T.compute_order(g, k).rank, O.compute_order(ref, order, s))
                want = O.run_engine(ref, "anop-surrogate", 5, order=order, order_seed=s,
                                    track_nodes=True)
                got = T.run_engine(g, T.EngineConfig(engine=T.EngineKind.AnopSurrogate, ranks=5,
                                                     order=k, track_nodes=True))
                assert got.total == want.total
                assert [x.triangles for x in got.per_rank] == want.triangles.tolist()
                assert [x.data_sent for x in got.per_rank] == want.data_sent.tolist()
                assert np.array_equal(got.node_counts, want.node_counts)
                f, _ = O.node_costs(ref, "NOV", order, s)
                assert np.array_equal(T.node_costs(g, T.CostKind.Nov, k).f, f)


def test_order_switching_and_errors():
    pairs = T.gen_pa(5000, 10, 2)
    ref = O.build_graph(pairs)
    want = O.count(ref)[0]
    with T.build_graph(pairs) as g:
        w_deg = T.ordering_cost(g)
        assert T.count_node_iterator_n(g, "id") == want
        assert T.ordering_cost(g, "id") == O.ordering_cost(ref, "id")
        # back to the default order: the cached orientation must be rebuilt
        assert T.ordering_cost(g) == w_deg == O.ordering_cost(ref)
        assert T.count_node_iterator_n(g) == want
        # the degree-order-only entry points ignore the graph's current order
        T.compute_order(g, T.OrderKind.by_random(3))
        plan = T.compute_boundaries(g, T.CostKind.Dpd, 4)
        vr = T.variance_report(g, plan, 0.5)
        o3 = np.zeros(3, dtype=np.uint64)
        v2 = np.zeros(2, dtype=np.float64)
        O.lib().orc_variance_report(ref.n, O._ptr(ref.off), O._ptr(ref.adj),
                                    O._ptr(plan.boundaries), 4, 0.5, O._ptr(o3), O._ptr(v2))
        assert (vr.triangles, vr.k, vr.k_prime) == tuple(int(x) for x in o3)
        with pytest.raises(ValueError):
            T.compute_order(g, "alphabetical")
        with pytest.raises(ValueError):
            check(lib().tg_set_order(g._h, 9, 0))  # unknown OrderKind::Tag


def test_listing_into_device_buffer():
    """collect_triangles straight into a caller's device buffer (north_star:
    listing to device buffers), per-node tallies alongside; exact vs oracle."""
    import torch

    pairs = T.gen_ws(20000, 20, 0.1, 4)
    ref = O.build_graph(pairs)
    want_T, want_tv, want_tri = O.count(ref, tally=True, listing=True)
    with T.build_graph(pairs) as g:
        out = torch.empty((want_T + 5, 3), dtype=torch.int32, device="cuda")
        cfg = T.EngineConfig(engine=T.EngineKind.Sequential, track_nodes=True,
                             collect_triangles=True)
        r = T.run_engine(g, cfg, triangles_out=out)
        assert r.total == want_T
        assert r.triangles_list.data_ptr() == out.data_ptr()
        got = r.triangles_list.cpu().numpy().view(np.uint32)
        assert np.array_equal(sorted_triples(got), want_tri)
        assert np.array_equal(r.node_counts, want_tv)
        # too small a device buffer: staged listing, TG_ERR_CAPACITY like a host buffer
        small = torch.empty((want_T // 2, 3), dtype=torch.int32, device="cuda")
        with pytest.raises(Exception):
            T.run_engine(g, cfg, triangles_out=small)


def test_node_iterator_pp_all_orders(orders_golden):
    """sequential.hpp:48-70 NodeIterator++ (both variants) under every order
    equals the reference's count (test_sequential.cpp:53-68 shape)."""
    for name, pairs, n_over, rec in fixture_graphs(orders_golden):
        if name == "rmat12":
            continue
        with T.build_graph(pairs, n_over) as g:
            for o in rec["orders"]:
                k = kind(o["order"], o["seed"])
                assert T.count_node_iterator_pp(g, k) == o["count"], (name, k)
                assert T.count_node_iterator_pp(g, k, use_intersection=True) == o["count"]


@pytest.mark.parametrize("chunk", [0, 64, 1000, 4096])
def test_count_from_csr_streamed(chunk):
    """tg_count_from_csr: the streamed host-CSR count (chunked orientation,
    apexes counted once all their lists arrived) equals the oracle for any
    chunking, including chunks smaller than one hub's adjacency."""
    import torch

    L = lib()
    try:
        L.tg_debug_set_chunk_entries(chunk)
        for pairs, n_over in ((T.gen_pa(20000, 20, 3), 0), (T.gen_rmat(12, 8, 0.57, 0.19, 0.19, 5), 0),
                              (T.gen_ws(5000, 10, 0.2, 1), 5003),
                              (np.zeros((0, 2), np.uint32), 7)):
            ref = O.build_graph(pairs, n_over)
            want = O.count(ref)[0]
            assert T.count_from_csr(ref.n, ref.off, ref.adj) == want
            off_p = torch.from_numpy(ref.off.view(np.int64)).pin_memory()
            adj_p = torch.from_numpy(ref.adj.view(np.int32)).pin_memory()
            assert T.count_from_csr(ref.n, off_p, adj_p) == want
    finally:
        L.tg_debug_set_chunk_entries(0)


def test_count_from_csr_range_is_the_aop_rank_body():
    """tg_count_from_csr_range over core i of a DPD plan equals the
    reference's per-rank AOP count (engines.hpp:38-54), streamed from host
    buffers and from device buffers (no-overlap fallback)."""
    import ctypes as C

    import torch

    L = lib()
    pairs = T.gen_pa(20000, 20, 3)
    ref = O.build_graph(pairs)
    want = O.run_engine(ref, "aop", 5)
    d_off = torch.from_numpy(ref.off.view(np.int64)).cuda()
    d_adj = torch.from_numpy(ref.adj.view(np.int32)).cuda()
    try:
        L.tg_debug_set_chunk_entries(4096)
        for i in range(5):
            lo, hi = int(want.boundaries[i]), int(want.boundaries[i + 1])
            t = C.c_uint64()
            check(L.tg_count_from_csr_range(0, ref.n, C.c_void_p(ref.off.ctypes.data),
                                            C.c_void_p(ref.adj.ctypes.data), lo, hi, C.byref(t)))
            assert t.value == int(want.triangles[i])
            check(L.tg_count_from_csr_range(0, ref.n, C.c_void_p(d_off.data_ptr()),
                                            C.c_void_p(d_adj.data_ptr()), lo, hi, C.byref(t)))
            assert t.value == int(want.triangles[i])
        with pytest.raises(ValueError):
            check(L.tg_count_from_csr_range(0, ref.n, C.c_void_p(ref.off.ctypes.data),
                                            C.c_void_p(ref.adj.ctypes.data), 5, 2, C.byref(t)))
    finally:
        L.tg_debug_set_chunk_entries(0)
