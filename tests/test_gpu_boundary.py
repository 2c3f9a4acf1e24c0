"""The reference's own hot-path signatures through the C ABI (VERDICT r1
item 3): effective_adjacency(g, OrderRank) (effective.hpp:37-52 with
order.hpp:31-35) and count_node_iterator_n(eff, sink) (sequential.hpp:17-46,
74-91) with NullSink / NodeTallySink / ListSink / any callable, against the
oracle and the reference's goldens."""
import numpy as np
import pytest

from oracle import binding as O
from paper_1706_05151_b200 import trigraph as T

pytestmark = pytest.mark.gpu


def test_g5_apex_first_emission_order():
    """test_sequential.cpp:33-43: two triangles, emitted (0,1,2), (1,2,3)."""
    g = T.build_graph([[0, 1], [0, 2], [1, 2], [1, 3], [2, 3], [3, 4]])
    eff = T.effective_adjacency(g, T.compute_order(g, T.OrderKind.by_degree()))
    raw = []
    total = T.count_node_iterator_n(eff, lambda v, u, w: raw.append((v, u, w)))
    assert total == 2
    assert raw == [(0, 1, 2), (1, 2, 3)]
    assert T.count_node_iterator_n(eff) == 2
    assert T.count_node_iterator_n(eff, T.NullSink()) == 2
    tally = T.NodeTallySink(5)
    T.count_node_iterator_n(eff, tally)
    assert tally.counts.tolist() == [1, 2, 2, 1, 0]
    ls = T.ListSink()
    T.count_node_iterator_n(eff, ls)
    assert sorted(map(tuple, ls.triangles.tolist())) == [(0, 1, 2), (1, 2, 3)]


@pytest.mark.parametrize("seed", [3, 11, 29])
def test_callable_sink_replays_reference_order(seed):
    """The raw device listing, replayed, equals the oracle's emission
    sequence (v ascending, u along N_v, w ascending) exactly."""
    pairs = O.random_graph_pairs(70, 0.3, seed)
    ref = O.build_graph(pairs, 70)
    eoff, eff = O.effective(ref)
    want = []
    for v in range(ref.n):
        nv = eff[eoff[v]:eoff[v + 1]]
        for u in nv:
            for w in np.intersect1d(nv, eff[eoff[u]:eoff[u + 1]]):
                want.append((v, int(u), int(w)))
    g = T.build_graph(pairs, 70)
    e = T.effective_adjacency(g, T.compute_order(g))
    assert np.array_equal(e.offsets, eoff) and np.array_equal(e.entries, eff)
    got = []
    assert T.count_node_iterator_n(e, lambda v, u, w: got.append((v, u, w))) == len(want)
    assert got == want
    # and the adopted-EffectiveAdjacency value path from host arrays
    e2 = T.EffectiveAdjacency(eoff, eff)
    tally = T.NodeTallySink(ref.n)
    T.count_node_iterator_n(e2, tally)
    _, tv, _ = O.count(ref, tally=True)
    assert np.array_equal(tally.counts, tv)


@pytest.mark.parametrize("order", ["id", "random", "coreness"])
def test_effective_adjacency_under_an_order_rank(orders_golden, order):
    """effective_adjacency(g, OrderRank) for the OrderRank of every
    OrderKind equals the reference's (reference_orders.json, G5 explicit)."""
    fx = orders_golden["g5"]
    g = T.build_graph([[0, 1], [0, 2], [1, 2], [1, 3], [2, 3], [3, 4]])
    for o in fx["orders"]:
        if o["order"] != order:
            continue
        rank = T.OrderRank(np.array(o["rank"], dtype=np.uint32))
        e = T.effective_adjacency(g, rank)
        assert e.offsets.tolist() == o["eff_offsets"]
        assert e.entries.tolist() == o["eff"]
        assert T.count_node_iterator_n(e) == o["count"]
        assert T.ordering_cost(g, rank) == o["ordering_cost"]


def test_order_rank_arbitrary_permutation_and_validation():
    pairs = O.random_graph_pairs(60, 0.25, 5)
    ref = O.build_graph(pairs, 60)
    g = T.build_graph(pairs, 60)
    rng = np.random.default_rng(7)
    for _ in range(4):
        perm = rng.permutation(60).astype(np.uint32)
        e = T.effective_adjacency(g, T.OrderRank(perm))
        want_off = np.zeros(61, np.uint64)
        lists = []
        for v in range(60):
            nb = ref.adj[ref.off[v]:ref.off[v + 1]]
            keep = nb[perm[nb] > perm[v]]
            lists.append(keep)
            want_off[v + 1] = want_off[v] + len(keep)
        assert np.array_equal(e.offsets, want_off)
        assert np.array_equal(e.entries, np.concatenate(lists).astype(np.uint32))
        assert T.count_node_iterator_n(e) == O.count(ref)[0]
    with pytest.raises(ValueError):
        T.effective_adjacency(g, T.OrderRank(np.zeros(60, np.uint32)))  # not a permutation
    with pytest.raises(ValueError):
        T.EffectiveAdjacency(np.array([0, 2], np.uint64), np.array([3, 1], np.uint32))._handle()
