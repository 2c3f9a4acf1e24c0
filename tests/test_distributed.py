"""The multi-process path (paper_1706_05151_b200/distributed.py) on CPU:
world_size 2 and 3 over gloo, with an oracle-backed RankBackend, checked
against the reference semantics (per-rank T, data_sent, data_recv, plan,
total) of the oracle's run_engine.  The GPU backend runs the same driver on
the B200 box (tests/test_gpu_distributed.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import binding as O
from paper_1706_05151_b200 import distributed as D
from paper_1706_05151_b200.trigraph import CostKind, EngineKind

COSTNAME = {CostKind.N: "N", CostKind.Dpd: "DPD", CostKind.Nov: "NOV"}


class OracleRankBackend(D.RankBackend):
    """Per-rank compute restated on the oracle's CSR (test infrastructure)."""

    def __init__(self, g: O.CSR):
        self.g = g
        self.device = torch.device("cpu")
        self.eoff, self.eff = O.effective(g)

    def lst(self, v):
        return self.eff[self.eoff[v]:self.eoff[v + 1]]

    def plan(self, cost, p):
        f, _ = O.node_costs(self.g, COSTNAME[cost])
        return O.compute_boundaries(f, p)

    def aop_count(self, b, rank):
        t = 0
        for v in range(int(b[rank]), int(b[rank + 1])):
            nv = self.lst(v)
            for u in nv:
                t += len(np.intersect1d(nv, self.lst(u), assume_unique=True))
        return t

    def pack(self, b, rank):
        p = len(b) - 1
        inner = b[1:-1]
        per = [[] for _ in range(p)]
        for v in range(int(b[rank]), int(b[rank + 1])):
            nv = self.lst(v)
            owners = np.searchsorted(inner, nv, side="right")
            for j in sorted(set(int(o) for o in owners) - {rank}):
                per[j].append(v)
        msgs = np.array([len(x) for x in per], np.uint64)
        words = np.array([sum(len(self.lst(v)) for v in x) for x in per], np.uint64)
        hdr, dat = [], []
        for j in range(p):
            for v in per[j]:
                hdr += [v, len(self.lst(v))]
                dat += list(self.lst(v))
        return (msgs, words, torch.tensor(hdr, dtype=torch.int32),
                torch.tensor(dat, dtype=torch.int32))

    def _core_triangles(self, b, rank):
        for v in range(int(b[rank]), int(b[rank + 1])):
            nv = self.lst(v)
            for u in nv:
                for w in np.intersect1d(nv, self.lst(u), assume_unique=True):
                    yield v, int(u), int(w)

    def aop_tally(self, b, rank):
        tv = torch.zeros(self.g.n, dtype=torch.int64)
        for t in self._core_triangles(b, rank):
            for x in t:
                tv[x] += 1
        return tv

    def cc(self, tally):
        return torch.from_numpy(O.clustering(self.g, tally.numpy().astype(np.uint64)))

    def aop_list(self, b, rank):
        rows = [sorted(t) for t in self._core_triangles(b, rank)]
        return torch.tensor(rows, dtype=torch.int32).reshape(-1, 3)

    def surrogate_count(self, b, rank, hdr, nmsgs, data):
        cb, ce = int(b[rank]), int(b[rank + 1])
        t = 0
        for v in range(cb, ce):  # local intersections (u in core)
            nv = self.lst(v)
            for u in nv[(nv >= cb) & (nv < ce)]:
                t += len(np.intersect1d(nv, self.lst(u), assume_unique=True))
        h = hdr.numpy().reshape(-1, 2)
        d = data.numpy().astype(np.uint32)
        o = 0
        for k in range(nmsgs):  # SurrogateCount on received lists
            x = d[o:o + h[k, 1]]
            o += h[k, 1]
            for u in x[(x >= cb) & (x < ce)]:
                t += len(np.intersect1d(self.lst(u), x, assume_unique=True))
        return t


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for (n, dens, seed, engine, cost) in cases:
            g = O.random_graph(n, dens, seed)
            rep = D.run_engine_distributed(OracleRankBackend(g), engine, cost)
            out.append((rep.total, rep.boundaries.tolist(),
                        [(r.triangles, r.data_sent, r.data_recv) for r in rep.per_rank]))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_engines_match_reference_semantics(world):
    cases = []
    rng = np.random.default_rng(world)
    for i in range(3):
        n = int(rng.integers(25, 60))
        dens = float(rng.uniform(0.15, 0.5))
        seed = int(rng.integers(1 << 60))
        for engine in (EngineKind.Aop, EngineKind.AnopSurrogate):
            for cost in (CostKind.N, CostKind.Dpd, CostKind.Nov):
                cases.append((n, dens, seed, engine, cost))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k, (n, dens, seed, engine, cost) in enumerate(cases):
        g = O.random_graph(n, dens, seed)
        name = "aop" if engine == EngineKind.Aop else "anop-surrogate"
        want = O.run_engine(g, name, world, COSTNAME[cost])
        for r in range(world):  # every rank returns the same report
            total, b, per = results[r][k]
            assert total == want.total
            assert b == want.boundaries.tolist()
            assert [x[0] for x in per] == want.triangles.tolist()
            assert [x[1] for x in per] == want.data_sent.tolist()
            assert [x[2] for x in per] == want.data_recv.tolist()


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        g = O.random_graph(97, 0.2, 5)
        off = torch.from_numpy(g.off.view(np.int64))
        adj = torch.from_numpy(g.adj.view(np.int32))
        d_off, d_adj = D.gather_host_csr(g.n, off, adj, torch.device("cpu"))
        q.put((rank, bool(torch.equal(d_off, off) and torch.equal(d_adj, adj))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sliced_upload_gather_reassembles_the_csr(world):
    """distributed.gather_host_csr (the N > 1 e2e path): each rank ships
    1/world of the arrays; after the all-gather every rank holds them whole
    (slices padded to equal sizes for the collective)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(results.values())


def _sinks_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = O.random_graph(60, 0.3, 17)
        be = OracleRankBackend(g)
        total, tv, cc = D.clustering_distributed(be, CostKind.Dpd)
        tri, off, tot2 = D.list_triangles_distributed(be, CostKind.Dpd)
        q.put((rank, total, tv.tolist(), cc.tolist(), tri.numpy().tolist(), off, tot2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_tallies_cc_and_listing(world):
    """clustering_distributed / list_triangles_distributed:
    every rank returns the reference's T_v and C_v; the per-rank listings,
    placed at their all-gathered offsets, are exactly the triangle list."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sinks_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=240)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = O.random_graph(60, 0.3, 17)
    T, want_tv, want_tri = O.count(g, tally=True, listing=True)
    want_cc = O.clustering(g, want_tv)
    parts = [None] * world
    for r in range(world):
        total, tv, cc, tri, off, tot2 = res[r]
        assert total == T == tot2
        assert tv == want_tv.tolist()
        assert np.array_equal(np.array(cc), want_cc)
        parts[r] = (off, tri)
    allt = []
    for off, tri in sorted(parts, key=lambda x: x[0]):
        assert off == len(allt)
        allt += tri
    got = np.array(allt, dtype=np.uint32).reshape(-1, 3)
    got = got[np.lexsort((got[:, 2], got[:, 1], got[:, 0]))]
    assert np.array_equal(got, want_tri)
