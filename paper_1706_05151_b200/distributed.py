"""One process per GPU: the paper's AOP and ANOP-surrogate engines over
torch.distributed (NCCL over NVLink on B200; gloo for CPU tests).

Reference semantics (engines.hpp):
  * AOP (:38-54, run_engine :367-381): rank i counts the triangles whose apex
    lies in core i = [b_i, b_{i+1}) of the cost-function plan
    (partition.hpp:116-141).  Each GPU holds the oriented lists its core
    touches (here: the full oriented CSR, replicated; the trimmed halo size is
    what the reference would store).  No data-path communication.
  * ANOP-surrogate (:146-198): rank i holds only its core lists, ships (v, N_v)
    once per distinct remote owner of N_v's entries (LastProc), and every
    owner runs SurrogateCount (:60-76) on what it receives.  The one exchange
    step is an all-to-allv of message headers (v, len) and list payloads.
  * The global count is one all-reduce of a single int64 (engines.hpp:407);
    per-rank stats (triangles, data_sent, data_recv) are all-gathered so every
    rank returns the same RunReport.

The compute side is a RankBackend; CudaRankBackend drives
libtrigraph_b200.so on this rank's GPU.  tests/test_distributed.py plugs an
oracle backend into the same driver to test the exchange logic with gloo.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np
import torch
import torch.distributed as dist

from ._lib import check, lib
from .trigraph import CostKind, EngineKind, Graph, RankStats, RunReport, compute_boundaries


class RankBackend:
    """Per-rank compute used by run_engine_distributed."""

    device: torch.device

    def plan(self, cost: CostKind, p: int) -> np.ndarray:  # p+1 boundaries
        raise NotImplementedError

    def aop_count(self, b: np.ndarray, rank: int) -> int:
        raise NotImplementedError

    def pack(self, b: np.ndarray, rank: int) -> Tuple[np.ndarray, np.ndarray, torch.Tensor,
                                                       torch.Tensor]:
        """(msgs_per_dest, words_per_dest, headers int32[2*M], data int32[W]),
        destination-major."""
        raise NotImplementedError

    def surrogate_count(self, b: np.ndarray, rank: int, hdr: torch.Tensor, nmsgs: int,
                        data: torch.Tensor) -> int:
        raise NotImplementedError

    def aop_tally(self, b: np.ndarray, rank: int) -> torch.Tensor:
        """int64[n]: T_v over the triangles whose apex is in core `rank`,
        counted at all three corners (RankSink tallies, engines.hpp:303-321)."""
        raise NotImplementedError

    def cc(self, tally: torch.Tensor) -> torch.Tensor:
        """float64[n]: C_v = 2 T_v / (d (d - 1)), 0 for d < 2 (engines.hpp:258-267)."""
        raise NotImplementedError

    def aop_list(self, b: np.ndarray, rank: int) -> torch.Tensor:
        """int32[k, 3]: the triangles whose apex is in core `rank`, ascending ids
        per triple (ListSink normalisation, sequential.hpp:39-44)."""
        raise NotImplementedError


class CudaRankBackend(RankBackend):
    """This rank's GPU through the C ABI (Graph resident on `device`)."""

    def __init__(self, g: Graph):
        # The library launches on its own stream; every entry point below
        # synchronises the device before handing buffers to torch / NCCL.
        self.g = g
        self.device = torch.device("cuda", g.device)
        self._acc = torch.zeros(1, dtype=torch.int64, device=self.device)

    def _sync(self):
        torch.cuda.synchronize(self.device)

    def plan(self, cost, p):
        return compute_boundaries(self.g, cost, p).boundaries

    def aop_count(self, b, rank):
        b = np.ascontiguousarray(b, dtype=np.uint32)
        self._acc.zero_()
        self._sync()
        check(lib().tg_aop_rank_device(self.g._h, C.c_void_p(b.ctypes.data), len(b) - 1, rank,
                                       C.c_void_p(self._acc.data_ptr())))
        self._sync()
        return int(self._acc.item())

    def pack(self, b, rank):
        b = np.ascontiguousarray(b, dtype=np.uint32)
        p = len(b) - 1
        msgs = np.zeros(p, np.uint64)
        words = np.zeros(p, np.uint64)
        check(lib().tg_surrogate_pack_sizes(self.g._h, C.c_void_p(b.ctypes.data), p, rank,
                                            C.c_void_p(msgs.ctypes.data),
                                            C.c_void_p(words.ctypes.data)))
        hdr = torch.empty(int(2 * msgs.sum()), dtype=torch.int32, device=self.device)
        dat = torch.empty(int(words.sum()), dtype=torch.int32, device=self.device)
        if hdr.numel():
            check(lib().tg_surrogate_pack_device(self.g._h, C.c_void_p(b.ctypes.data), p, rank,
                                                 C.c_void_p(hdr.data_ptr()),
                                                 C.c_void_p(dat.data_ptr() if dat.numel() else 0)))
        self._sync()
        return msgs, words, hdr, dat

    def surrogate_count(self, b, rank, hdr, nmsgs, data):
        b = np.ascontiguousarray(b, dtype=np.uint32)
        self._acc.zero_()
        self._sync()
        hp = hdr.data_ptr() if hdr.numel() else 0
        dp = data.data_ptr() if data.numel() else 0
        check(lib().tg_surrogate_count_device(self.g._h, C.c_void_p(b.ctypes.data), len(b) - 1,
                                              rank, C.c_void_p(hp), nmsgs, C.c_void_p(dp),
                                              C.c_void_p(self._acc.data_ptr())))
        self._sync()
        return int(self._acc.item())


    def aop_tally(self, b, rank):
        b = np.ascontiguousarray(b, dtype=np.uint32)
        n = self.g.num_nodes()
        tv = torch.zeros(max(n, 1), dtype=torch.int64, device=self.device)
        self._acc.zero_()
        self._sync()
        check(lib().tg_aop_rank_sinks_device(self.g._h, C.c_void_p(b.ctypes.data), len(b) - 1,
                                             rank, C.c_void_p(self._acc.data_ptr()),
                                             C.c_void_p(tv.data_ptr()), None, 0, None))
        self._sync()
        return tv[:n]

    def cc(self, tally):
        n = self.g.num_nodes()
        out = torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)
        if n:
            check(lib().tg_cc_from_tally_device(self.g._h, C.c_void_p(tally.data_ptr()),
                                                C.c_void_p(out.data_ptr())))
        self._sync()
        return out[:n]

    def aop_list(self, b, rank):
        k = self.aop_count(b, rank)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        tri = torch.empty((max(k, 1), 3), dtype=torch.int32, device=self.device)
        cur = torch.zeros(1, dtype=torch.int64, device=self.device)
        self._acc.zero_()
        self._sync()
        check(lib().tg_aop_rank_sinks_device(self.g._h, C.c_void_p(b.ctypes.data), len(b) - 1,
                                             rank, C.c_void_p(self._acc.data_ptr()), None,
                                             C.c_void_p(tri.data_ptr()), k,
                                             C.c_void_p(cur.data_ptr())))
        self._sync()
        return tri[:k]


def _all_to_allv(t: torch.Tensor, send_counts: List[int], recv_counts: List[int],
                 group=None) -> torch.Tensor:
    # always entered: all_to_all_single is a collective, and a rank with no
    # traffic of its own must still pair with its peers (zero splits are legal)
    out = torch.empty(sum(recv_counts), dtype=t.dtype, device=t.device)
    dist.all_to_all_single(out, t, output_split_sizes=recv_counts,
                           input_split_sizes=send_counts, group=group)
    return out


def gather_host_csr(n: int, offsets: torch.Tensor, adj: torch.Tensor, device,
                    group=None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Every rank ends with the full CSR (Graph, graph.hpp:19-53) in its HBM,
    having copied only 1/p of it over its own host link: rank r uploads slice
    r of the offsets and of the adjacency (pinned host tensors -> HBM), then
    one all-gather per array assembles the rest over NVLink (NCCL) -- the
    CSR is replicated for AOP (engines.hpp:38-54), and the host link, not
    NVLink, is the narrow one.  Returns (offsets int64[n+1], adj int32[2m])
    views on `device`."""
    p = dist.get_world_size(group)
    rank = dist.get_rank(group)
    out = []
    for src, count in ((offsets, n + 1), (adj, adj.numel())):
        chunk = max(1, -(-count // p))  # equal slices (NCCL all-gather), last one padded
        full = torch.empty(p * chunk, dtype=src.dtype, device=device)
        mine = torch.zeros(chunk, dtype=src.dtype, device=device)
        a0 = min(count, rank * chunk)
        a1 = min(count, a0 + chunk)
        if a1 > a0:
            mine[: a1 - a0].copy_(src[a0:a1], non_blocking=True)
        dist.all_gather_into_tensor(full, mine, group=group)
        out.append(full[:count])
    return out[0], out[1]


def count_aop_from_host_csr(n: int, offsets: torch.Tensor, adj: torch.Tensor, b: np.ndarray,
                            device, group=None) -> int:
    """AOP (engines.hpp:38-54) end to end from host buffers on every rank:
    gather_host_csr, then this rank's core [b_r, b_r+1) counted on its GPU
    (tg_count_from_csr_range), then the one all-reduce of T."""
    rank = dist.get_rank(group)
    d_off, d_adj = gather_host_csr(n, offsets, adj, device, group)
    torch.cuda.current_stream(device).synchronize()
    t = C.c_uint64()
    check(lib().tg_count_from_csr_range(torch.device(device).index or 0, n,
                                        C.c_void_p(d_off.data_ptr()),
                                        C.c_void_p(d_adj.data_ptr()) if d_adj.numel() else None,
                                        int(b[rank]), int(b[rank + 1]), C.byref(t)))
    total = torch.tensor([t.value], dtype=torch.int64, device=device)
    dist.all_reduce(total, group=group)
    return int(total.item())


def _shared_plan(backend: RankBackend, cost: CostKind, group) -> np.ndarray:
    """The cost-function plan (partition.hpp:116-141); every rank derives the
    same one, rank 0's copy is authoritative."""
    p = dist.get_world_size(group)
    b = np.ascontiguousarray(backend.plan(cost, p), dtype=np.uint32)
    bt = torch.from_numpy(b.astype(np.int64)).to(backend.device)
    dist.broadcast(bt, 0, group=group)
    return bt.cpu().numpy().astype(np.uint32)


def clustering_distributed(backend: RankBackend, cost: CostKind = CostKind.Dpd, group=None):
    """clustering_coefficients (engines.hpp:422-435) with ranks = the process
    group, AOP: each rank tallies the triangles of its core apexes at all
    three corners into a full n-vector on its GPU, one all-reduce sums them
    (the owner-side aggregation of engines.hpp:229-254, done for every vertex
    at once), and C_v is computed on the device.  Every rank returns the same
    (total, T_v uint64[n], C_v float64[n])."""
    rank = dist.get_rank(group)
    b = _shared_plan(backend, cost, group)
    tv = backend.aop_tally(b, rank)
    dist.all_reduce(tv, group=group)
    cc = backend.cc(tv)
    tvh = tv.cpu().numpy().astype(np.uint64)
    return int(tvh.sum()) // 3, tvh, cc.cpu().numpy()


def list_triangles_distributed(backend: RankBackend, cost: CostKind = CostKind.Dpd, group=None):
    """Triangle listing (collect_triangles, engines.hpp:313-319) with ranks =
    the process group, AOP: each rank lists the triangles of its core apexes
    into a buffer on its own GPU; an all-gather of the per-rank counts gives
    each rank its offset in the global list.  Returns (local int32[k, 3] on
    this rank's device, offset, total)."""
    p = dist.get_world_size(group)
    rank = dist.get_rank(group)
    b = _shared_plan(backend, cost, group)
    tri = backend.aop_list(b, rank)
    k = torch.tensor([tri.shape[0]], dtype=torch.int64, device=backend.device)
    ks = [torch.empty_like(k) for _ in range(p)]
    dist.all_gather(ks, k, group=group)
    counts = [int(x.item()) for x in ks]
    return tri, sum(counts[:rank]), sum(counts)


def run_engine_distributed(backend: RankBackend, engine: EngineKind = EngineKind.Aop,
                           cost: CostKind = CostKind.Dpd, group=None) -> RunReport:
    """run_engine (engines.hpp:335-418) with ranks = the process group."""
    p = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = backend.device
    if engine not in (EngineKind.Aop, EngineKind.AnopSurrogate):
        raise ValueError("distributed engines: Aop and AnopSurrogate")
    b = _shared_plan(backend, cost, group)
    sent = recv = 0
    if engine == EngineKind.Aop:
        tri = backend.aop_count(b, rank)
    else:
        msgs, words, hdr, dat = backend.pack(b, rank)
        counts = torch.tensor(np.stack([msgs, words], 1).astype(np.int64), device=dev)
        rcounts = torch.empty_like(counts)
        dist.all_to_all_single(rcounts, counts, group=group)  # one (msgs, words) row per peer
        rc = rcounts.cpu().numpy()
        rmsgs = [int(x) for x in rc[:, 0]]
        rwords = [int(x) for x in rc[:, 1]]
        rhdr = _all_to_allv(hdr, [2 * int(x) for x in msgs], [2 * x for x in rmsgs], group)
        rdat = _all_to_allv(dat, [int(x) for x in words], rwords, group)
        tri = backend.surrogate_count(b, rank, rhdr, sum(rmsgs), rdat)
        sent, recv = int(msgs.sum()), sum(rmsgs)
    mine = torch.tensor([tri, sent, recv], dtype=torch.int64, device=dev)
    allst = [torch.empty_like(mine) for _ in range(p)]
    dist.all_gather(allst, mine, group=group)
    total = torch.tensor([tri], dtype=torch.int64, device=dev)
    dist.all_reduce(total, group=group)  # the one tiny all-reduce of T
    rep = RunReport(engine=engine, ranks=p, cost=cost, total=int(total.item()), boundaries=b)
    rep.per_rank = [RankStats(int(s[0]), int(s[1]), int(s[2])) for s in
                    (t.cpu().numpy() for t in allst)]
    return rep
