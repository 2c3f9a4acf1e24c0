"""The engines across ranks (csrc/comm.cu, paper_1706_05151_b200/comm.py):
AOP (engines.hpp:38-54), ANOP-surrogate (engines.hpp:146-198, partition.hpp:
210-239) and clustering at the owner (engines.hpp:211-268) with N = 1..4
ranks, each on its own host thread, exchanging through the in-process
transport (N ranks on the one B200 of this box; the exchange is
host-orchestrated device copies, no kernel waits on another rank), and NCCL
with one rank.  Checked against the oracle (pinned to the reference):
boundaries, per-rank triangles, data_sent / data_recv, stored entries
(Σ = m for the surrogate's non-overlapping partitions), T_v / C_v of each
owner's core -- with the whole graph on every rank and with rank-local rows."""
import threading

import numpy as np
import pytest
import torch

from oracle import binding as O
from paper_1706_05151_b200 import comm as M
from paper_1706_05151_b200 import trigraph as T

pytestmark = pytest.mark.gpu

GRAPHS = {
    "pa": lambda: T.gen_pa(20000, 20, 3),
    "rmat": lambda: T.gen_rmat(12, 8, 0.57, 0.19, 0.19, 5),
    "ws": lambda: T.gen_ws(20000, 10, 0.1, 2),
    "random": lambda: O.random_graph_pairs(150, 0.2, 7),
}


def run_ranks(n, fn):
    """fn(rank, comm) on n threads over one in-process group; results by rank."""
    comms = M.Comm.local([0] * n)
    out, err = [None] * n, [None] * n

    def work(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r, comms[r])
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    for c in comms:
        c.close()
    return out


def rank_graph(ref, pairs, rows, r, local_rows):
    if not local_rows:
        return T.build_graph(pairs, ref.n)
    lo, hi = int(rows[r]), int(rows[r + 1])
    deg = np.diff(ref.off).astype(np.uint32)
    return M.graph_from_rows(ref.n, lo, hi, ref.off[lo:hi + 1], ref.adj[ref.off[lo]:ref.off[hi]],
                             deg)


@pytest.mark.parametrize("graph", sorted(GRAPHS))
@pytest.mark.parametrize("nranks", [1, 2, 3, 4])
@pytest.mark.parametrize("local_rows", [False, True])
def test_engines_across_ranks(graph, nranks, local_rows):
    pairs = GRAPHS[graph]()
    ref = O.build_graph(pairs)
    rows = M.split_rows(ref.off, nranks)
    want_aop = O.run_engine(ref, "aop", nranks, "DPD")
    want_sur = O.run_engine(ref, "anop-surrogate", nranks, "DPD")
    want_dir = O.run_engine(ref, "anop-direct", nranks, "DPD")
    want_T, want_tv, _ = O.count(ref, tally=True)
    want_cc = O.clustering(ref, want_tv)

    def body(r, comm):
        g = rank_graph(ref, pairs, rows, r, local_rows)
        a = M.run_engine_comm(g, comm, T.EngineConfig(engine=T.EngineKind.Aop))
        s = M.run_engine_comm(g, comm, T.EngineConfig(engine=T.EngineKind.AnopSurrogate))
        dr = M.run_engine_comm(g, comm, T.EngineConfig(engine=T.EngineKind.AnopDirect))
        b, tv, cc = M.clustering_comm(g, comm)
        d = torch.zeros(1, dtype=torch.int64, device="cuda")
        M.aop_step_comm(g, comm, a.boundaries, d.data_ptr())
        torch.cuda.synchronize()
        step = int(d.item())
        g.close()
        return a, s, (b, tv, cc), step, dr

    res = run_ranks(nranks, body)
    for r, (a, s, (b, tv, cc), step, dr) in enumerate(res):
        assert a.total == want_T == s.total == step == dr.total
        # ANOP-direct (engines.hpp:80-141): request / reply data path
        assert dr.boundaries.tolist() == want_dir.boundaries[:nranks + 1].tolist()
        assert [x.triangles for x in dr.per_rank] == want_dir.triangles[:nranks].tolist()
        assert [x.data_sent for x in dr.per_rank] == want_dir.data_sent[:nranks].tolist()
        assert [x.data_recv for x in dr.per_rank] == want_dir.data_recv[:nranks].tolist()
        assert sum(x.stored_entries for x in dr.per_rank) == ref.m
        assert a.boundaries.tolist() == want_aop.boundaries[:nranks + 1].tolist()
        assert [x.triangles for x in a.per_rank] == want_aop.triangles[:nranks].tolist()
        assert [x.stored_entries for x in a.per_rank] == want_aop.stored[:nranks].tolist()
        assert [x.data_sent for x in a.per_rank] == [0] * nranks
        assert s.boundaries.tolist() == want_sur.boundaries[:nranks + 1].tolist()
        assert [x.triangles for x in s.per_rank] == want_sur.triangles[:nranks].tolist()
        assert [x.data_sent for x in s.per_rank] == want_sur.data_sent[:nranks].tolist()
        assert [x.data_recv for x in s.per_rank] == want_sur.data_recv[:nranks].tolist()
        assert [x.stored_entries for x in s.per_rank] == want_sur.stored[:nranks].tolist()
        assert sum(x.stored_entries for x in s.per_rank) == ref.m  # non-overlapping
        lo, hi = int(b[r]), int(b[r + 1])
        assert np.array_equal(tv, want_tv[lo:hi])
        assert np.array_equal(cc, want_cc[lo:hi])


@pytest.mark.parametrize("graph", ["pa", "rmat", "random"])
@pytest.mark.parametrize("nranks", [1, 3])
@pytest.mark.parametrize("slab_mode", [1, 2])
def test_aop_step_slab_layout(graph, nranks, slab_mode):
    """tg_aop_step_comm with the gathered lists in the slab layout (slab.cuh;
    automatic on PA-like graphs, forced here) and without it"""
    from paper_1706_05151_b200._lib import lib

    pairs = GRAPHS[graph]() if graph != "pa" else T.gen_pa(20000, 44, 3)
    ref = O.build_graph(pairs)
    rows = M.split_rows(ref.off, nranks)
    want = O.run_engine(ref, "aop", nranks, "DPD")

    def body(r, comm):
        g = rank_graph(ref, pairs, rows, r, True)
        plan = M.run_engine_comm(g, comm, T.EngineConfig(engine=T.EngineKind.Aop)).boundaries
        d = torch.zeros(1, dtype=torch.int64, device="cuda")
        out = []
        for _ in range(2):
            M.aop_step_comm(g, comm, plan, d.data_ptr())
            torch.cuda.synchronize()
            out.append(int(d.item()))
        g.close()
        return out

    try:
        lib().tg_debug_set_slab(slab_mode)
        for out in run_ranks(nranks, body):
            assert out == [want.total, want.total]
    finally:
        lib().tg_debug_set_slab(0)


def test_boundary_override_and_other_costs():
    pairs = GRAPHS["pa"]()
    ref = O.build_graph(pairs)
    rows = M.split_rows(ref.off, 3)
    plan = [0, 2000, 2000, ref.n]  # an empty core included
    want = O.run_engine(ref, "anop-surrogate", 3, "DPD", boundaries=plan)
    want_nov = O.run_engine(ref, "aop", 3, "NOV")

    def body(r, comm):
        g = rank_graph(ref, pairs, rows, r, True)
        s = M.run_engine_comm(g, comm, T.EngineConfig(engine=T.EngineKind.AnopSurrogate,
                                                      ranks=3, boundaries=plan))
        a = M.run_engine_comm(g, comm, T.EngineConfig(engine=T.EngineKind.Aop, ranks=3,
                                                      cost=T.CostKind.Nov))
        return s, a

    for s, a in run_ranks(3, body):
        assert s.boundaries.tolist() == plan
        assert [x.triangles for x in s.per_rank] == want.triangles[:3].tolist()
        assert [x.data_sent for x in s.per_rank] == want.data_sent[:3].tolist()
        assert a.boundaries.tolist() == want_nov.boundaries[:4].tolist()
        assert [x.triangles for x in a.per_rank] == want_nov.triangles[:3].tolist()


def test_nccl_single_rank():
    pairs = GRAPHS["rmat"]()
    ref = O.build_graph(pairs)
    comm = M.Comm.init(0, 1, 0, M.Comm.unique_id())
    g = T.build_graph(pairs, ref.n)
    for eng, name in ((T.EngineKind.Aop, "aop"), (T.EngineKind.AnopSurrogate, "anop-surrogate")):
        rep = M.run_engine_comm(g, comm, T.EngineConfig(engine=eng))
        want = O.run_engine(ref, name, 1, "DPD")
        assert rep.total == want.total
        assert rep.per_rank[0].stored_entries == want.stored[0]
    g.close()
    comm.close()


def test_rank_local_graph_refuses_single_device_paths():
    pairs = GRAPHS["random"]()
    ref = O.build_graph(pairs)
    deg = np.diff(ref.off).astype(np.uint32)
    g = M.graph_from_rows(ref.n, 0, 40, ref.off[:41], ref.adj[:ref.off[40]], deg)
    with pytest.raises(ValueError):
        T.count_node_iterator_n(g)
    g.close()
