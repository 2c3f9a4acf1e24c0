"""The engines across GPUs through the C ABI (csrc/comm.cu): one rank per
GPU, each holding rows of the graph, NCCL for the exchange.

Reference semantics (engines.hpp): AOP (:38-54) -- rank i counts the
triangles whose apex lies in core i of the cost plan (partition.hpp:116-141);
ANOP-surrogate (:146-198) -- rank i stores only its core lists
(partition.hpp:210-239) and ships (v, N_v) once per distinct remote owner;
aggregate_clustering (:211-268) -- tallies summed at their owner.

    comm = Comm.from_process_group(device)        # torchrun, NCCL under it
    g = graph_from_rows(n, lo, hi, off_rows, adj_rows, degrees, device)
    rep = run_engine_comm(g, comm, EngineConfig(engine=EngineKind.AnopSurrogate))

``Comm.local(devices)`` builds in-process ranks (one host thread each) whose
exchange is host-orchestrated device copies -- the tests run N ranks on one
GPU with it.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from ._lib import TgConfig, TgRankStats, check, lib
from .trigraph import (CostKind, EngineConfig, EngineKind, Graph, RankStats, RunReport, _cfg,
                       _p)


class Comm:
    """A tg_comm: NCCL (tg_comm_init) or an in-process group (tg_comm_init_local)."""

    def __init__(self, handle: C.c_void_p, device: int):
        self._h = handle
        self.device = device

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().tg_comm_unique_id(C.cast(buf, C.c_void_p)))
        return bytes(buf)

    @classmethod
    def init(cls, device: int, nranks: int, rank: int, uid: bytes) -> "Comm":
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        check(lib().tg_comm_init(device, nranks, rank, C.cast(buf, C.c_void_p), C.byref(h)))
        return cls(h, device)

    @classmethod
    def local(cls, devices: List[int]) -> List["Comm"]:
        n = len(devices)
        devs = (C.c_int * n)(*devices)
        hs = (C.c_void_p * n)()
        check(lib().tg_comm_init_local(n, C.cast(devs, C.c_void_p), C.cast(hs, C.c_void_p)))
        return [cls(C.c_void_p(hs[i]), devices[i]) for i in range(n)]

    @classmethod
    def from_process_group(cls, device: int, group=None) -> "Comm":
        """One NCCL communicator over a torch.distributed process group: rank
        0 makes the unique id, the group's backend carries it to the others."""
        import torch.distributed as dist

        obj = [cls.unique_id() if dist.get_rank(group) == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls.init(device, dist.get_world_size(group), dist.get_rank(group), obj[0])

    def info(self):
        n, r = C.c_int32(), C.c_int32()
        check(lib().tg_comm_info(self._h, C.byref(n), C.byref(r)))
        return n.value, r.value

    @property
    def size(self) -> int:
        return self.info()[0]

    @property
    def rank(self) -> int:
        return self.info()[1]

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().tg_comm_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def graph_from_rows(n: int, row_lo: int, row_hi: int, offsets, adj, degrees,
                    device: int = 0) -> Graph:
    """Rows [row_lo, row_hi) of an n-vertex symmetric CSR (offsets: rows+1
    entries, any base; adj: the rows' entries) plus every vertex's degree --
    one rank's share of the input (tg_graph_from_rows)."""
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    a = np.ascontiguousarray(adj, dtype=np.uint32)
    deg = np.ascontiguousarray(degrees, dtype=np.uint32)
    if off.shape[0] != row_hi - row_lo + 1 or deg.shape[0] != n:
        raise ValueError("offsets must have row_hi-row_lo+1 entries, degrees n")
    h = C.c_void_p()
    check(lib().tg_graph_from_rows(device, n, row_lo, row_hi, _p(off), _p(a) if a.size else None,
                                   _p(deg), C.byref(h)))
    return Graph(h, device)


def split_rows(off: np.ndarray, parts: int) -> np.ndarray:
    """parts+1 row boundaries splitting a CSR into equal orientation cost
    (adjacency entries + 32 per row, the library's own split: csrc/comm.cu
    k_volume_split), rounded to whole 32-vertex tiles (the default input
    distribution; tile-aligned rows orient with the one-pass tile kernel)."""
    n = off.shape[0] - 1
    cost = off.astype(np.float64) + 32.0 * np.arange(n + 1, dtype=np.float64)
    tgt = (np.arange(parts + 1, dtype=np.float64) * float(cost[-1]) / parts)
    b = np.searchsorted(cost, tgt, side="left").astype(np.uint64) & ~np.uint64(31)
    b[0], b[-1] = 0, n
    return np.maximum.accumulate(np.minimum(b, n)).astype(np.uint32)


def run_engine_comm(g: Graph, comm: Comm, cfg: Optional[EngineConfig] = None) -> RunReport:
    """run_engine across the communicator (tg_run_engine_comm): Aop,
    AnopDirect or AnopSurrogate counts; every rank returns the same report."""
    p = comm.size
    cfg = cfg or EngineConfig(engine=EngineKind.Aop, ranks=p)
    c, keep = _cfg(EngineConfig(engine=cfg.engine, ranks=p, cost=cfg.cost, order=cfg.order,
                                boundaries=cfg.boundaries))
    stats = (TgRankStats * p)()
    b = np.zeros(p + 1, dtype=np.uint32)
    total = C.c_uint64()
    check(lib().tg_run_engine_comm(g._h, comm._h, C.byref(c), C.byref(total),
                                   C.cast(stats, C.c_void_p), _p(b)))
    del keep
    rep = RunReport(engine=EngineKind(cfg.engine), ranks=p, cost=CostKind(cfg.cost),
                    total=total.value, boundaries=b)
    rep.per_rank = [RankStats(s.triangles, s.data_sent, s.data_recv, s.realized_cost,
                              s.stored_entries) for s in stats]
    return rep


def aop_step_comm(g: Graph, comm: Comm, boundaries, d_total_ptr: int) -> None:
    """One AOP step on this rank (tg_aop_step_comm): T lands in the device
    u64 at d_total_ptr on every rank; stream-ordered on the graph's stream."""
    b = np.ascontiguousarray(boundaries, dtype=np.uint32)
    check(lib().tg_aop_step_comm(g._h, comm._h, _p(b), C.c_void_p(d_total_ptr)))


def clustering_comm(g: Graph, comm: Comm, cost: CostKind = CostKind.Dpd, boundaries=None):
    """clustering_coefficients across the communicator: (boundaries, T_v and
    C_v of this rank's core range [b_r, b_r+1))."""
    p = comm.size
    c, keep = _cfg(EngineConfig(engine=EngineKind.Aop, ranks=p, cost=cost,
                                boundaries=boundaries))
    r = comm.rank
    b = np.zeros(p + 1, dtype=np.uint32)
    # (outputs sized n: the core range is known only once the plan is made)
    n = g.num_nodes()
    tv = np.zeros(max(n, 1), dtype=np.uint64)
    cc = np.zeros(max(n, 1), dtype=np.float64)
    check(lib().tg_clustering_comm(g._h, comm._h, C.byref(c), _p(b), _p(tv), _p(cc)))
    del keep
    k = int(b[r + 1] - b[r])
    return b, tv[:k].copy(), cc[:k].copy()
