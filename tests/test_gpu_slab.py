"""The slab layout of the oriented lists (csrc/slab.cuh, prep.cu orient_slab):
each list's first 32 entries in its own 128-byte-aligned slab, lists longer
than a slab stored whole above the slabs.  effective_adjacency
(effective.hpp:37-52), count_node_iterator_n with every sink
(sequential.hpp:17-46,74-91), the AOP rank bodies (engines.hpp:38-54) and the
clustering coefficients (engines.hpp:422-435) through it must equal the oracle
bit for bit -- on the graphs it is chosen for (PA) and, forced on, on graphs
with lists longer than a slab, hubs, heavy apexes and empty rows."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import binding as O
from paper_1706_05151_b200 import trigraph as T
from paper_1706_05151_b200._lib import check, lib

pytestmark = pytest.mark.gpu


def hub_clique(n, k):
    """a k-clique (lists up to k-1 long) + a hub of degree n-1 + a sparse tail"""
    e = [[a, b] for a in range(k) for b in range(a + 1, k)]
    e += [[n - 1, v] for v in range(n - 1)]
    e += [[v, v + 1] for v in range(k, n - 2)]
    return np.array(e, np.uint32)


GRAPHS = {
    "pa": lambda: T.gen_pa(30000, 40, 5),            # the automatic case (h ~ 20)
    "pa_dense": lambda: T.gen_pa(6000, 90, 2),       # h ~ 45: most lists longer than a slab
    "pa_33": lambda: T.gen_pa(8000, 64, 9),          # h ~ 32: lists right at the slab size
    "rmat": lambda: T.gen_rmat(13, 16, 0.57, 0.19, 0.19, 3),  # hubs, apexes with h > 64
    "random": lambda: O.random_graph_pairs(400, 0.3, 9),      # h up to ~70
    "ws": lambda: T.gen_ws(20000, 20, 0.1, 3),
    "hub_clique": lambda: hub_clique(6000, 80),      # a hub above the CTA threshold (4096)
    "tiny": lambda: np.array([[0, 1], [1, 2], [0, 2], [5, 6]], np.uint32),
}


@pytest.fixture
def slab():
    L = lib()
    yield L
    L.tg_debug_set_slab(0)
    L.tg_debug_set_warp_variant(0)


@pytest.mark.parametrize("graph", sorted(GRAPHS))
@pytest.mark.parametrize("mode", [1, 0, 2])
def test_slab_matches_oracle(slab, graph, mode):
    pairs = GRAPHS[graph]()
    ref = O.build_graph(pairs)
    want, want_tv, want_tri = O.count(ref, tally=True, listing=True)
    slab.tg_debug_set_slab(mode)
    g = T.build_graph(pairs, ref.n)
    assert T.count_node_iterator_n(g) == want
    # the exported EffectiveAdjacency is the compact one whatever the layout
    eoff, eadj = O.effective(ref)
    e = T.effective_adjacency(g)
    assert np.array_equal(e.offsets, eoff) and np.array_equal(e.entries, eadj)
    # the device-resident step (bench path): orientation + count, twice
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(2):
        check(slab.tg_orient_device(g._h))
        check(slab.tg_count_device(g._h, C.c_void_p(d.data_ptr())))
        torch.cuda.synchronize()
        assert int(d.item()) == want
    # sinks: per-node tallies, listing, clustering coefficients
    rep = T.run_engine(g, T.EngineConfig(engine=T.EngineKind.Sequential, track_nodes=True,
                                         collect_triangles=True))
    assert rep.total == want
    assert np.array_equal(rep.node_counts, want_tv)
    tri = rep.triangles_list
    tri = tri[np.lexsort((tri[:, 2], tri[:, 1], tri[:, 0]))] if len(tri) else tri.reshape(0, 3)
    assert np.array_equal(tri, want_tri.reshape(-1, 3))
    cc = T.clustering_coefficients(g, T.EngineConfig(engine=T.EngineKind.Aop, ranks=3))
    assert np.array_equal(cc.coefficient, O.clustering(ref, want_tv))
    # AOP rank bodies over apex ranges, surrogate ranks (partition-local lists)
    if ref.n >= 8:
        r5 = O.run_engine(ref, "aop", 5, "DPD")
        b = np.ascontiguousarray(r5.boundaries[:6], dtype=np.uint32)
        for r in range(5):
            d.zero_()
            check(slab.tg_aop_rank_device(g._h, C.c_void_p(b.ctypes.data), 5, r,
                                          C.c_void_p(d.data_ptr())))
            torch.cuda.synchronize()
            assert int(d.item()) == int(r5.triangles[r]), r
        s3 = O.run_engine(ref, "anop-surrogate", 3, "DPD")
        got = T.run_engine(g, T.EngineConfig(engine=T.EngineKind.AnopSurrogate, ranks=3))
        assert [x.triangles for x in got.per_rank] == list(s3.triangles)
    # other orders re-decide the layout
    for order in ("id", "random"):
        assert T.count_node_iterator_n(g, order) == O.count(ref, order=order, seed=0)[0]
    assert T.count_node_iterator_n(g, "degree") == want
    g.close()


@pytest.mark.parametrize("graph", ["pa", "rmat", "hub_clique", "random"])
def test_slab_with_nibble_codes(slab, graph):
    """the slab orientation keyed by the 4-bit degree codes (n > 64M path)"""
    pairs = GRAPHS[graph]()
    ref = O.build_graph(pairs)
    want = O.count(ref)[0]
    eoff, eadj = O.effective(ref)
    try:
        slab.tg_debug_set_paths(8, 0)
        slab.tg_debug_set_slab(1)
        g = T.build_graph(pairs, ref.n)
        e = T.effective_adjacency(g)
        assert np.array_equal(e.offsets, eoff) and np.array_equal(e.entries, eadj)
        assert T.count_node_iterator_n(g) == want
        g.close()
    finally:
        slab.tg_debug_set_paths(0, 0)


def test_slab_next_rows(slab):
    """SURVEY 8(f) rows over the slab layout: sparsified engines
    (sparsify.hpp, engines.hpp:335-457: they read the oriented lists through
    their descriptors), per-edge counts (sequential.hpp:108-122, the LIST sink
    of the slab kernel) and the non-degree orders"""
    pairs = T.gen_pa(4000, 44, 8)
    ref = O.build_graph(pairs)
    slab.tg_debug_set_slab(1)
    g = T.build_graph(pairs, ref.n)
    assert T.count_node_iterator_n(g) == O.count(ref)[0]
    assert np.array_equal(T.per_edge_triangle_counts(g), O.per_edge_counts(ref))
    modes = {"global": T.SparsifyMode.Global, "per-partition": T.SparsifyMode.PerPartition}
    engines = {"seq": T.EngineKind.Sequential, "aop": T.EngineKind.Aop,
               "anop-direct": T.EngineKind.AnopDirect, "anop-surrogate": T.EngineKind.AnopSurrogate}
    for eng, kind in engines.items():
        for mode, mk in modes.items():
            p = 1 if eng == "seq" else 4
            want = O.run_engine(ref, eng, p, "DPD", sparsify=mode, q=0.6, seed=77,
                                track_nodes=True, collect_triangles=True)
            got = T.run_engine(g, T.EngineConfig(engine=kind, ranks=p, track_nodes=True,
                                                 collect_triangles=True,
                                                 sparsify=T.SparsifyConfig(0.6, 77, mk)))
            assert got.total == want.total, (eng, mode)
            assert [r.triangles for r in got.per_rank] == want.triangles.tolist()
            assert [r.data_sent for r in got.per_rank] == want.data_sent.tolist()
            assert np.array_equal(got.node_counts, want.node_counts)
    for eng in ("aop", "anop-direct", "anop-surrogate"):
        want = O.run_engine(ref, eng, 5, "DPD")
        got = T.run_engine(g, T.EngineConfig(engine=engines[eng], ranks=5))
        assert [r.triangles for r in got.per_rank] == want.triangles.tolist(), eng
        assert [r.data_sent for r in got.per_rank] == want.data_sent.tolist(), eng
        assert [r.stored_entries for r in got.per_rank] == want.stored.tolist(), eng
    g.close()


def test_slab_quad_kernel_on_slab_layout(slab):
    """the descriptor-driven kernels read the slab layout too (variant sweep)"""
    pairs = T.gen_pa(20000, 50, 11)
    ref = O.build_graph(pairs)
    want = O.count(ref)[0]
    slab.tg_debug_set_slab(1)
    for variant in (1, 2, 3, 4):
        slab.tg_debug_set_warp_variant(variant)
        g = T.build_graph(pairs, ref.n)
        assert T.count_node_iterator_n(g) == want, variant
        g.close()
