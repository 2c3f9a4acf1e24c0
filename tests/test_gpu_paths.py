"""The code paths large graphs take, forced on small ones (tg_debug_set_paths):
compact count/scan/fill orientation (above 2^34 list slots, effective.hpp:37-52),
1-byte degree codes as orientation keys (above 32M vertices, order.hpp:95-104),
4-bit endpoint-quantile degree codes (+8, above 64M vertices)
and 64-bit element indices in the scalar intersection kernels (above 2^32
slots, sequential.hpp:74-91) -- each bit-exact against the oracle for counts,
per-node tallies, listings and per-rank engine results."""
import numpy as np
import pytest

from oracle import binding as O
from paper_1706_05151_b200 import trigraph as T
from paper_1706_05151_b200._lib import lib

pytestmark = pytest.mark.gpu


def sorted_triples(t):
    t = np.asarray(t, dtype=np.uint32).reshape(-1, 3)
    return t[np.lexsort((t[:, 2], t[:, 1], t[:, 0]))]


GRAPHS = {
    "pa": lambda: T.gen_pa(20000, 20, 5),
    "rmat": lambda: T.gen_rmat(14, 16, 0.57, 0.19, 0.19, 3),  # hubs above 4096
    "ws": lambda: T.gen_ws(30000, 10, 0.1, 2),
}


@pytest.mark.parametrize("graph", sorted(GRAPHS))
@pytest.mark.parametrize("orient_mode,force_wide,variant", [
    (1, 0, 0), (5, 0, 0), (6, 0, 0), (1, 1, 1), (1, 1, 4), (6, 1, 1), (2, 1, 4),
    (8, 0, 0), (10, 0, 0)])
def test_forced_large_graph_paths(graph, orient_mode, force_wide, variant):
    pairs = GRAPHS[graph]()
    ref = O.build_graph(pairs)
    want_T, want_tv, want_tri = O.count(ref, tally=True, listing=True)
    want_aop = O.run_engine(ref, "aop", 4)
    want_sur = O.run_engine(ref, "anop-surrogate", 4)
    eoff, eff = O.effective(ref)
    L = lib()
    try:
        L.tg_debug_set_paths(orient_mode, force_wide)
        L.tg_debug_set_warp_variant(variant)
        with T.build_graph(pairs) as g:
            e = T.effective_adjacency(g)
            assert np.array_equal(e.offsets, eoff) and np.array_equal(e.entries, eff)
            r = T.run_engine(g, T.EngineConfig(engine=T.EngineKind.Sequential, track_nodes=True,
                                               collect_triangles=True))
            assert r.total == want_T
            assert np.array_equal(r.node_counts, want_tv)
            assert np.array_equal(sorted_triples(r.triangles_list), want_tri)
            a = T.run_engine(g, T.EngineConfig(engine=T.EngineKind.Aop, ranks=4))
            assert [x.triangles for x in a.per_rank] == want_aop.triangles.tolist()
            s = T.run_engine(g, T.EngineConfig(engine=T.EngineKind.AnopSurrogate, ranks=4))
            assert [x.triangles for x in s.per_rank] == want_sur.triangles.tolist()
            assert [x.data_sent for x in s.per_rank] == want_sur.data_sent.tolist()
            off, adj = g.csr()
            assert T.count_from_csr(len(off) - 1, off, adj) == want_T
    finally:
        L.tg_debug_set_paths(0, 0)
        L.tg_debug_set_warp_variant(0)


@pytest.mark.parametrize("graph", sorted(GRAPHS))
@pytest.mark.parametrize("cap", [0, 1024, 65536])
@pytest.mark.parametrize("order", ["degree", "id", "coreness"])
def test_rank_bitmap_cta_path(graph, cap, order):
    """The bitmap CTA path (ctab.cuh), forced on with several window
    capacities so apexes split between it and the hash CTA path: counts,
    tallies, listings, AOP per-rank counts and per-edge counts exact."""
    pairs = GRAPHS[graph]()
    ref = O.build_graph(pairs)
    want_T, want_tv, want_tri = O.count(ref, tally=True, listing=True, order=order)
    want_aop = O.run_engine(ref, "aop", 3, order=order)
    L = lib()
    kinds = {"degree": T.OrderKind.by_degree(), "id": T.OrderKind.by_id(),
             "coreness": T.OrderKind.by_coreness()}
    try:
        L.tg_debug_set_rank_bitmap(1, cap)
        with T.build_graph(pairs) as g:
            cfg = T.EngineConfig(engine=T.EngineKind.Sequential, order=kinds[order],
                                 track_nodes=True, collect_triangles=True)
            r = T.run_engine(g, cfg)
            assert r.total == want_T
            assert np.array_equal(r.node_counts, want_tv)
            assert np.array_equal(sorted_triples(r.triangles_list), want_tri)
            a = T.run_engine(g, T.EngineConfig(engine=T.EngineKind.Aop, ranks=3, order=kinds[order]))
            assert [x.triangles for x in a.per_rank] == want_aop.triangles.tolist()
            if order == "degree":
                assert np.array_equal(T.per_edge_triangle_counts(g), O.per_edge_counts(ref))
                assert T.count_node_iterator_n(g) == want_T
    finally:
        L.tg_debug_set_rank_bitmap(0, 0)
