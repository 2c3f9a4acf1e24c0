"""The id-window encoding of the count (csrc/window.cu): oriented lists split
into a 64-bit mask of the entries within 32 ids of their row plus a short
far list; count_node_iterator_n (sequential.hpp:74-91) and the AOP rank body
(engines.hpp:38-54) through it must equal the oracle bit for bit -- on the
graphs it is chosen for (Watts-Strogatz, rings, bands) and, forced on, on
graphs where most apexes are deferred to the generic kernels (PA, random,
R-MAT), with id-window edge cases (ids < 32, the last ids, empty lists)."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import binding as O
from paper_1706_05151_b200 import trigraph as T
from paper_1706_05151_b200._lib import check, lib

pytestmark = pytest.mark.gpu


def ring(n, k):
    return np.array([[v, (v + j) % n] for v in range(n) for j in range(1, k + 1)], np.uint32)


def band_plus_far(n, k, seed):
    rng = np.random.default_rng(seed)
    e = [[v, v + j] for v in range(n) for j in range(1, k + 1) if v + j < n]
    e += rng.integers(0, n, size=(n // 3, 2)).tolist()
    return np.array(e, np.uint32)


GRAPHS = {
    "ws": lambda: T.gen_ws(40000, 20, 0.1, 3),
    "ws_beta0": lambda: T.gen_ws(5000, 10, 0.0, 1),
    "ring40": lambda: ring(2000, 20),  # wrap-around entries at both ends
    "band": lambda: band_plus_far(3000, 31, 4),
    "pa": lambda: T.gen_pa(20000, 20, 5),
    "rmat": lambda: T.gen_rmat(12, 16, 0.57, 0.19, 0.19, 3),
    "random": lambda: O.random_graph_pairs(300, 0.2, 9),
}


@pytest.fixture
def window_mode():
    L = lib()
    yield L
    L.tg_debug_set_window(0)


@pytest.mark.parametrize("graph", sorted(GRAPHS))
@pytest.mark.parametrize("mode", [1, 0])
def test_window_count_matches_oracle(window_mode, graph, mode):
    pairs = GRAPHS[graph]()
    ref = O.build_graph(pairs)
    want = O.count(ref)[0]
    window_mode.tg_debug_set_window(mode)
    g = T.build_graph(pairs, ref.n)
    assert T.count_node_iterator_n(g) == want
    # the device-resident step (bench path): orientation + count
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(2):
        check(window_mode.tg_orient_device(g._h))
        check(window_mode.tg_count_device(g._h, C.c_void_p(d.data_ptr())))
        torch.cuda.synchronize()
        assert int(d.item()) == want
    # AOP rank bodies over apex ranges (per-rank = triangles by apex owner)
    rep = O.run_engine(ref, "aop", 5, "DPD")
    b = np.ascontiguousarray(rep.boundaries[:6], dtype=np.uint32)
    for r in range(5):
        d.zero_()
        check(window_mode.tg_aop_rank_device(g._h, C.c_void_p(b.ctypes.data), 5, r,
                                              C.c_void_p(d.data_ptr())))
        torch.cuda.synchronize()
        assert int(d.item()) == int(rep.triangles[r]), r
    # other orders key the same encoding
    for order in ("id", "random"):
        assert T.count_node_iterator_n(g, order) == O.count(ref, order=order, seed=0)[0]
    g.close()
