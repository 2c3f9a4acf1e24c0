"""Python mirror of the reference `trigraph` API over the B200 C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/trigraph/ (cited per symbol); the work runs in
libtrigraph_b200.so on the GPU.  Deviations, all documented in DESIGN.md:

* ``Graph`` is device-resident (one CUDA device per Graph).
* Every OrderKind is supported (ByDegree, the north_star path, is the
  default; order.hpp:85-128), and so is a caller-supplied ``OrderRank``.
* ``ExecMode`` is accepted for signature parity and ignored: device results
  are mode-independent (acceptance.cpp:438-468).
* ``RankStats.realized_cost`` is algorithmic work (sum of h_v + h_u over the
  rank's oriented edges), not merge comparisons.
* ``std::invalid_argument`` maps to ``ValueError``.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._lib import ParseError, TgConfig, TgRankStats, check, lib  # noqa: F401 (ParseError re-exported)

NodeId = np.uint32


def _p(a: Optional[np.ndarray]):
    return None if a is None else C.c_void_p(a.ctypes.data)


class EngineKind(enum.IntEnum):  # engines.hpp:24
    Sequential = 0
    Aop = 1
    AnopDirect = 2
    AnopSurrogate = 3


ENGINE_NAMES = {EngineKind.Sequential: "seq", EngineKind.Aop: "aop",
                EngineKind.AnopDirect: "anop-direct", EngineKind.AnopSurrogate: "anop-surrogate"}


def to_string(x) -> str:  # engines.hpp:26-34, partition.hpp:24-35
    if isinstance(x, EngineKind):
        return ENGINE_NAMES[x]
    if isinstance(x, CostKind):
        return {CostKind.Dh: "DH", CostKind.Ddh: "DDH", CostKind.Dh2: "DH2",
                CostKind.Dpd: "DPD", CostKind.Nov: "NOV"}.get(x, x.name)
    raise TypeError(x)


class CostKind(enum.IntEnum):  # partition.hpp:18
    N = 0
    D = 1
    Dh = 2
    Ddh = 3
    Dh2 = 4
    Dpd = 5
    Nov = 6


class ExecMode(enum.IntEnum):  # runtime.hpp:27 (accepted, no effect on the device)
    Interleaved = 0
    Concurrent = 1


class Graph:
    """Immutable undirected simple graph in CSR form, resident on one GPU
    (graph.hpp:19-53).  Build with :func:`build_graph` or :meth:`from_csr`."""

    def __init__(self, handle: C.c_void_p, device: int):
        self._h = handle
        self.device = device

    @classmethod
    def from_csr(cls, n: int, offsets, adj, device: int = 0) -> "Graph":
        """Adopt an already-built CSR (Graph ctor, graph.hpp:22-23)."""
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        a = np.ascontiguousarray(adj, dtype=np.uint32)
        if off.shape[0] != n + 1:
            raise ValueError("offsets must have n+1 entries")
        h = C.c_void_p()
        check(lib().tg_graph_from_csr(device, n, _p(off), _p(a) if a.size else None, C.byref(h)))
        return cls(h, device)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().tg_graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _info(self):
        n, m = C.c_uint64(), C.c_uint64()
        check(lib().tg_graph_info(self._h, C.byref(n), C.byref(m)))
        return n.value, m.value

    def num_nodes(self) -> int:  # graph.hpp:25
        return self._info()[0]

    def num_edges(self) -> int:  # graph.hpp:26
        return self._info()[1]

    def csr(self):
        """(offsets uint64[n+1], adj uint32[2m]) copied back to the host."""
        n, m = self._info()
        off = np.zeros(n + 1, dtype=np.uint64)
        adj = np.zeros(max(2 * m, 1), dtype=np.uint32)
        check(lib().tg_graph_csr(self._h, _p(off), _p(adj)))
        return off, adj[: 2 * m]

    def degree(self, v: int) -> int:  # graph.hpp:28
        off, _ = self.csr()
        return int(off[v + 1] - off[v])

    def neighbors(self, v: int) -> np.ndarray:  # graph.hpp:30-32
        off, adj = self.csr()
        return adj[off[v]:off[v + 1]]

    def edges(self) -> np.ndarray:  # graph.hpp:40-46: (u, v), u < v, u then v ascending
        off, adj = self.csr()
        src = np.repeat(np.arange(len(off) - 1, dtype=np.uint32), np.diff(off).astype(np.int64))
        keep = src < adj
        return np.stack([src[keep], adj[keep]], axis=1)


def build_graph(edge_pairs, n_override: int = 0, device: int = 0) -> Graph:
    """graph.hpp:58-85 -- drops self-loops, symmetrises, sorts and uniques on
    the device.  ``edge_pairs``: (E, 2) uint32 array-like (host or a
    device pointer-backed torch tensor via ``build_graph_device``)."""
    pairs = np.ascontiguousarray(np.asarray(edge_pairs, dtype=np.uint32).reshape(-1, 2))
    h = C.c_void_p()
    check(lib().tg_graph_from_edges(device, _p(pairs) if pairs.size else None, pairs.shape[0],
                                    n_override, C.byref(h)))
    return Graph(h, device)


def count_from_csr(n: int, offsets, adj, device: int = 0) -> int:
    """count_node_iterator_n(effective_adjacency(Graph(n, offsets, adj))) in
    one call from a host CSR (graph.hpp:22, sequential.hpp:74-91): the
    upload is streamed in vertex chunks and overlapped with orientation and
    counting (pass page-locked buffers, e.g. ``torch.Tensor.pin_memory()``
    views, for the overlap).  ``offsets``/``adj``: numpy arrays or objects
    with ``data_ptr()``."""
    def ptr(a, dt):
        if hasattr(a, "data_ptr"):
            return C.c_void_p(a.data_ptr()), a
        a = np.ascontiguousarray(a, dtype=dt)
        return (_p(a) if a.size else None), a
    po, ko = ptr(offsets, np.uint64)
    pa, ka = ptr(adj, np.uint32)
    t = C.c_uint64()
    check(lib().tg_count_from_csr(device, int(n), po, pa, C.byref(t)))
    del ko, ka
    return t.value


def build_graph_from_pointer(ptr: int, num_pairs: int, n_override: int = 0,
                             device: int = 0) -> Graph:
    """build_graph from a raw (host or device) pointer to interleaved pairs."""
    h = C.c_void_p()
    check(lib().tg_graph_from_edges(device, C.c_void_p(ptr), num_pairs, n_override, C.byref(h)))
    return Graph(h, device)


class OrderTag(enum.IntEnum):  # order.hpp:19 OrderKind::Tag
    ById = 0
    ByDegree = 1
    ByRandom = 2
    ByCoreness = 3


@dataclass(frozen=True)
class OrderKind:  # order.hpp:17-28
    tag: OrderTag = OrderTag.ByDegree
    seed: int = 0

    @staticmethod
    def by_id() -> "OrderKind":
        return OrderKind(OrderTag.ById, 0)

    @staticmethod
    def by_degree() -> "OrderKind":
        return OrderKind(OrderTag.ByDegree, 0)

    @staticmethod
    def by_random(seed: int) -> "OrderKind":
        return OrderKind(OrderTag.ByRandom, int(seed))

    @staticmethod
    def by_coreness() -> "OrderKind":
        return OrderKind(OrderTag.ByCoreness, 0)


_ORDER_NAMES = {"by_id": OrderTag.ById, "id": OrderTag.ById, "ById": OrderTag.ById,
                "by_degree": OrderTag.ByDegree, "degree": OrderTag.ByDegree,
                "ByDegree": OrderTag.ByDegree, "by_random": OrderTag.ByRandom,
                "random": OrderTag.ByRandom, "ByRandom": OrderTag.ByRandom,
                "by_coreness": OrderTag.ByCoreness, "coreness": OrderTag.ByCoreness,
                "ByCoreness": OrderTag.ByCoreness}


def _order(kind, seed: int = 0) -> OrderKind:
    """OrderKind from an OrderKind, an OrderTag or a name (cli.hpp:67-72
    spellings: id, degree, random, coreness)."""
    if kind is None:
        return OrderKind.by_degree()
    if isinstance(kind, OrderKind):
        return kind
    if isinstance(kind, str):
        if kind not in _ORDER_NAMES:
            raise ValueError(f"unknown ordering '{kind}'")
        kind = _ORDER_NAMES[kind]
    return OrderKind(OrderTag(int(kind)), int(seed) if int(kind) == OrderTag.ByRandom else 0)


def _use_order(g: "Graph", kind) -> None:
    if isinstance(kind, OrderRank):  # order.hpp:31-35, a caller's permutation
        r = np.ascontiguousarray(kind.rank, dtype=np.uint32)
        if r.shape[0] != g.num_nodes():
            raise ValueError("OrderRank: rank must have num_nodes() entries")
        check(lib().tg_set_order_rank(g._h, _p(r) if r.size else None))
        return
    o = _order(kind)
    check(lib().tg_set_order(g._h, int(o.tag), int(o.seed)))


# ---------------------------------------------------------------- edge lists


def _text_ptr(text):
    """(pointer, length, keep-alive) of bytes / str / a CUDA uint8 tensor."""
    if hasattr(text, "data_ptr"):
        return C.c_void_p(text.data_ptr()), int(text.numel() * text.element_size()), text
    if isinstance(text, str):
        text = text.encode("latin-1")
    buf = np.frombuffer(bytes(text), dtype=np.uint8)
    return (_p(buf) if buf.size else None), int(buf.size), buf


def parse_edge_list(text, device: int = 0) -> np.ndarray:
    """io.hpp:24-50 on the device: (E, 2) uint32 pairs in file order.  Raises
    ParseError (with ``.line``) like the reference."""
    ptr, n, keep = _text_ptr(text)
    cnt, line = C.c_uint64(), C.c_uint64()
    if isinstance(keep, np.ndarray):  # host text: at most one edge per line
        cap = int(np.count_nonzero(keep == 10)) + 1
    else:  # device text: ask for the count first
        check(lib().tg_parse_edge_list(device, ptr, n, None, 0, C.byref(cnt), C.byref(line)),
              line.value)
        cap = cnt.value
    out = np.zeros((max(cap, 1), 2), dtype=np.uint32)
    check(lib().tg_parse_edge_list(device, ptr, n, _p(out), cap, C.byref(cnt), C.byref(line)),
          line.value)
    del keep
    return out[: cnt.value]


def build_graph_from_text(text, n_override: int = 0, device: int = 0) -> "Graph":
    """build_graph(parse_edge_list(text), n_override) with both on the device
    (cli.hpp:81-88 --input)."""
    ptr, n, keep = _text_ptr(text)
    h, line = C.c_void_p(), C.c_uint64()
    check(lib().tg_graph_from_text(device, ptr, n, n_override, C.byref(h), C.byref(line)),
          line.value)
    del keep
    return Graph(h, device)


def write_edge_list(g: "Graph") -> bytes:
    """io.hpp:52-64 on the device: "u v\n" for every edge u < v."""
    n = C.c_uint64()
    check(lib().tg_write_edge_list(g._h, None, 0, C.byref(n)))
    buf = np.zeros(max(n.value, 1), dtype=np.uint8)
    check(lib().tg_write_edge_list(g._h, _p(buf), n.value, C.byref(n)))
    return buf[: n.value].tobytes()


@dataclass
class OrderRank:  # order.hpp:31-35
    rank: np.ndarray

    def precedes(self, u: int, v: int) -> bool:
        return bool(self.rank[u] < self.rank[v])


def coreness(g: Graph) -> np.ndarray:
    """order.hpp:39-83 core numbers (device peeling), uint64[n]."""
    n = g.num_nodes()
    c = np.zeros(max(n, 1), dtype=np.uint64)
    check(lib().tg_coreness(g._h, _p(c)))
    return c[:n]


def compute_order(g: Graph, kind=None) -> OrderRank:
    """order.hpp:85-128 compute_order(g, kind) for every OrderKind (default
    by_degree, the hot path).  ``kind``: OrderKind, OrderTag or a name."""
    _use_order(g, kind)
    n = g.num_nodes()
    r = np.zeros(max(n, 1), dtype=np.uint32)
    check(lib().tg_compute_order(g._h, _p(r)))
    return OrderRank(r[:n])


class EffectiveAdjacency:  # effective.hpp:17-35
    """N_v lists (ID-sorted) as host arrays, EffectiveAdjacency(offsets, eff)
    (effective.hpp:18-20).  Counting it (count_node_iterator_n) adopts a copy
    on ``device`` once (tg_eff_from_csr) and runs there."""

    def __init__(self, offsets, entries, device: int = 0):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.entries = np.ascontiguousarray(entries, dtype=np.uint32)
        self.device = device
        self._h = None

    def num_nodes(self) -> int:
        return self.offsets.shape[0] - 1

    def total_entries(self) -> int:
        return int(self.entries.shape[0])

    def eff(self, v: int) -> np.ndarray:
        return self.entries[self.offsets[v]:self.offsets[v + 1]]

    def effdeg(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])

    def _handle(self):
        if self._h is None:
            h = C.c_void_p()
            check(lib().tg_eff_from_csr(self.device, self.num_nodes(), _p(self.offsets),
                                        _p(self.entries) if self.entries.size else None,
                                        C.byref(h)))
            self._h = h
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().tg_eff_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def effective_adjacency(g: Graph, order=None) -> EffectiveAdjacency:
    """effective.hpp:37-52 under ``order`` -- an OrderKind / name (default
    by_degree) or an OrderRank from compute_order (the reference's
    effective_adjacency(g, order)) -- oriented on the device."""
    _use_order(g, order)
    n, m = g._info()
    off = np.zeros(n + 1, dtype=np.uint64)
    eff = np.zeros(max(m, 1), dtype=np.uint32)
    check(lib().tg_effective_adjacency(g._h, _p(off), _p(eff)))
    return EffectiveAdjacency(off, eff[:m], g.device)


class NullSink:  # sequential.hpp:19-21
    def __call__(self, v, u, w):
        pass


class NodeTallySink:  # sequential.hpp:24-33
    def __init__(self, n: int):
        self.counts = np.zeros(n, dtype=np.uint64)

    def __call__(self, v, u, w):
        self.counts[v] += 1
        self.counts[u] += 1
        self.counts[w] += 1


class ListSink:  # sequential.hpp:36-46
    def __init__(self):
        self.triangles = np.zeros((0, 3), dtype=np.uint32)

    def __call__(self, v, u, w):
        t = np.sort(np.array([[v, u, w]], dtype=np.uint32), axis=1)
        self.triangles = np.concatenate([self.triangles, t])


def _eff_count(e: EffectiveAdjacency, sink):
    h = e._handle()
    n = e.num_nodes()
    t, nt = C.c_uint64(), C.c_uint64()
    if sink is None or isinstance(sink, NullSink):
        check(lib().tg_eff_count(h, C.byref(t), None, None, 0, 0, C.byref(nt)))
        return t.value
    if isinstance(sink, NodeTallySink):  # device TALLY path
        tv = np.zeros(max(n, 1), dtype=np.uint64)
        check(lib().tg_eff_count(h, C.byref(t), _p(tv), None, 0, 0, C.byref(nt)))
        sink.counts[:n] += tv[:n]
        return t.value
    check(lib().tg_eff_count(h, C.byref(t), None, None, 0, 0, C.byref(nt)))
    T = t.value
    tri = np.zeros((max(T, 1), 3), dtype=np.uint32)
    raw = 0 if isinstance(sink, ListSink) else 1
    check(lib().tg_eff_count(h, C.byref(t), None, _p(tri), T, raw, C.byref(nt)))
    tri = tri[:T]
    if isinstance(sink, ListSink):  # device LIST path (normalised triples)
        sink.triangles = np.concatenate([sink.triangles, tri])
        return T
    # any callable sink(v, u, w): raw device listing, replayed on the host in
    # the reference's emission order -- v ascending, u along the ID-sorted
    # N_v, w ascending (sequential.hpp:78-86)
    tri = tri[np.lexsort((tri[:, 2], tri[:, 1], tri[:, 0]))]
    for v, u, w in tri.tolist():
        sink(v, u, w)
    return T


def count_node_iterator_n(g, sink=None, order=None) -> int:
    """sequential.hpp:74-91.  ``g``: an EffectiveAdjacency (the reference's
    count_node_iterator_n(eff, sink)) -- ``sink`` None / NullSink (count),
    NodeTallySink / ListSink (the device sinks) or any callable (v, u, w),
    called once per triangle in the reference's order -- or a Graph
    (counted over effective_adjacency(g, order), default by_degree)."""
    if isinstance(g, EffectiveAdjacency):
        return _eff_count(g, sink)
    if isinstance(sink, (OrderKind, OrderTag, OrderRank, str, int)):
        sink, order = None, sink  # count_node_iterator_n(g, order)
    if sink is not None and not isinstance(sink, NullSink):
        return _eff_count(effective_adjacency(g, order), sink)
    _use_order(g, order)
    t = C.c_uint64()
    check(lib().tg_count(g._h, C.byref(t)))
    return t.value


def count_node_iterator_pp(g: Graph, order=None, use_intersection: bool = False) -> int:
    """sequential.hpp:48-70 NodeIterator++ (the paper's baseline) under
    ``order`` (default by_degree), on the device."""
    _use_order(g, order)
    t = C.c_uint64()
    check(lib().tg_count_node_iterator_pp(g._h, int(bool(use_intersection)), C.byref(t)))
    return t.value


def ordering_cost(g: Graph, order=None) -> int:
    """sequential.hpp:95-104: W = sum_v d_v * h_v under ``order`` (default
    by_degree)."""
    _use_order(g, order)
    t = C.c_uint64()
    check(lib().tg_ordering_cost(g._h, C.byref(t)))
    return t.value


@dataclass
class CostVector:  # partition.hpp:38-43
    f: np.ndarray
    prefix: np.ndarray

    def total(self) -> int:
        return int(self.prefix[-1]) if self.prefix.size else 0


def node_costs(g: Graph, kind: CostKind, order=None) -> CostVector:
    """partition.hpp:45-91 (DpdVariant::EffectiveOnly) over
    effective_adjacency(g, order) (default by_degree)."""
    _use_order(g, order)
    n = g.num_nodes()
    f = np.zeros(max(n, 1), dtype=np.uint64)
    pre = np.zeros(max(n, 1), dtype=np.uint64)
    check(lib().tg_node_costs(g._h, int(kind), _p(f), _p(pre)))
    return CostVector(f[:n], pre[:n])


@dataclass
class PartitionPlan:  # partition.hpp:95-110
    boundaries: np.ndarray

    def ranks(self) -> int:
        return len(self.boundaries) - 1

    def core_begin(self, i: int) -> int:
        return int(self.boundaries[i])

    def core_end(self, i: int) -> int:
        return int(self.boundaries[i + 1])

    def in_core(self, i: int, v: int) -> bool:
        return self.core_begin(i) <= v < self.core_end(i)

    def owner(self, v: int) -> int:
        inner = self.boundaries[1:-1]
        return int(np.searchsorted(inner, v, side="right"))


def compute_boundaries(g: Graph, kind: CostKind, p: int, order=None) -> PartitionPlan:
    """partition.hpp:116-141 over node_costs(g, kind, order): exact 128-bit
    search."""
    if p < 1:
        raise ValueError("compute_boundaries: p must be >= 1")
    _use_order(g, order)
    b = np.zeros(p + 1, dtype=np.uint32)
    check(lib().tg_compute_boundaries(g._h, int(kind), p, _p(b)))
    return PartitionPlan(b)


class SparsifyMode(enum.IntEnum):  # sparsify.hpp:22-24 SparsifyConfig::Mode
    PerPartition = 2
    Global = 1


@dataclass
class SparsifyConfig:  # sparsify.hpp:22-33
    q: float = 1.0
    seed: int = 0
    mode: SparsifyMode = SparsifyMode.Global

    def validate(self):
        if not (0.0 < self.q <= 1.0):
            raise ValueError("sparsify: q must be in (0, 1]")


@dataclass
class EngineConfig:  # engines.hpp:270-280
    engine: EngineKind = EngineKind.Aop
    ranks: int = 1
    cost: CostKind = CostKind.Dpd
    order: object = field(default_factory=OrderKind.by_degree)  # OrderKind (or a name)
    mode: ExecMode = ExecMode.Interleaved
    track_nodes: bool = False
    collect_triangles: bool = False
    sparsify: Optional[SparsifyConfig] = None
    boundaries: Optional[Sequence[int]] = None


@dataclass
class RankStats:  # engines.hpp:282-287 (+ stored_entries)
    triangles: int = 0
    data_sent: int = 0
    data_recv: int = 0
    realized_cost: int = 0
    stored_entries: int = 0


@dataclass
class RunReport:  # engines.hpp:289-298
    engine: EngineKind = EngineKind.Sequential
    ranks: int = 1
    cost: CostKind = CostKind.Dpd
    total: int = 0
    per_rank: list = field(default_factory=list)
    boundaries: np.ndarray = None
    node_counts: Optional[np.ndarray] = None
    triangles_list: Optional[np.ndarray] = None


def _cfg(cfg: EngineConfig):
    o = _order(cfg.order)
    c = TgConfig()
    c.order_set = 1
    c.order = int(o.tag)
    c.order_seed = int(o.seed)
    c.engine = int(cfg.engine)
    c.cost = int(cfg.cost)
    c.ranks = int(cfg.ranks)
    keep = None
    if cfg.boundaries is not None:
        keep = np.ascontiguousarray(cfg.boundaries, dtype=np.uint32)
        p = 1 if cfg.engine == EngineKind.Sequential else int(cfg.ranks)
        if keep.shape[0] != p + 1:
            raise ValueError("boundaries must have ranks+1 entries")
        c.boundaries = keep.ctypes.data
    c.track_nodes = int(bool(cfg.track_nodes))
    c.collect_triangles = int(bool(cfg.collect_triangles))
    if cfg.sparsify is not None:
        cfg.sparsify.validate()  # engines.hpp:336
        c.sparsify = int(cfg.sparsify.mode)
        c.sparsify_q = float(cfg.sparsify.q)
        c.sparsify_seed = int(cfg.sparsify.seed)
    return c, keep


def run_engine(g: Graph, cfg: EngineConfig, triangles_out=None) -> RunReport:
    """engines.hpp:335-418.  ``triangles_list`` rows are normalised to
    ascending ids (engines.hpp:313-319); row order is unspecified, as in the
    reference (compare sorted).  ``triangles_out``: optional device buffer
    (a CUDA tensor of >= 3*T int32/uint32 words, e.g. shape (T, 3)) that the
    listing kernels write in place; ``triangles_list`` is then a view of it."""
    if cfg.engine != EngineKind.Sequential and int(cfg.ranks) < 1:
        raise ValueError("run_engine: ranks must be >= 1")
    c, keep = _cfg(cfg)
    p = 1 if cfg.engine == EngineKind.Sequential else int(cfg.ranks)
    n = g.num_nodes()
    stats = (TgRankStats * p)()
    b = np.zeros(p + 1, dtype=np.uint32)
    total = C.c_uint64()
    tv = np.zeros(max(n, 1), dtype=np.uint64) if cfg.track_nodes else None
    if triangles_out is not None and cfg.collect_triangles:
        if triangles_out.element_size() != 4 or not triangles_out.is_contiguous():
            raise ValueError("triangles_out must be a contiguous 32-bit device buffer")
        tri = None
        cap = triangles_out.numel() // 3
        tri_ptr = C.c_void_p(triangles_out.data_ptr())
    else:
        cap = count_node_iterator_n(g, cfg.order) if cfg.collect_triangles else 0
        tri = np.zeros((max(cap, 1), 3), dtype=np.uint32) if cfg.collect_triangles else None
        tri_ptr = _p(tri)
    ntri = C.c_uint64()
    check(lib().tg_run_engine(g._h, C.byref(c), C.byref(total), C.cast(stats, C.c_void_p), _p(b),
                              _p(tv), tri_ptr, cap, C.byref(ntri)))
    del keep
    rep = RunReport(engine=EngineKind(cfg.engine), ranks=p, cost=CostKind(cfg.cost),
                    total=total.value, boundaries=b)
    rep.per_rank = [RankStats(s.triangles, s.data_sent, s.data_recv, s.realized_cost,
                              s.stored_entries) for s in stats]
    if cfg.track_nodes:
        rep.node_counts = tv[:n]
    if cfg.collect_triangles:
        if tri is None:
            rep.triangles_list = triangles_out.view(-1)[: 3 * ntri.value].view(-1, 3)
        else:
            rep.triangles_list = tri[: ntri.value]
    return rep


@dataclass
class ClusteringResult:  # engines.hpp:203-206
    triangles_per_node: np.ndarray
    coefficient: np.ndarray


def clustering_coefficients(g: Graph, cfg: EngineConfig) -> ClusteringResult:
    """engines.hpp:422-435: per-node T_v and C_v = 2 T_v / (d (d-1)) (fp64,
    IEEE-rounded on the device; 0 when d < 2)."""
    if cfg.engine != EngineKind.Sequential and int(cfg.ranks) < 1:
        raise ValueError("run_engine: ranks must be >= 1")
    c, keep = _cfg(cfg)
    n = g.num_nodes()
    tv = np.zeros(max(n, 1), dtype=np.uint64)
    cc = np.zeros(max(n, 1), dtype=np.float64)
    check(lib().tg_clustering_coefficients(g._h, C.byref(c), _p(tv), _p(cc)))
    del keep
    return ClusteringResult(tv[:n], cc[:n])


def approx_count(g: Graph, p: int, engine: EngineKind, q: float, seed: int,
                 mode: ExecMode = ExecMode.Interleaved, boundaries=None,
                 cost: CostKind = CostKind.Dpd) -> float:
    """engines.hpp:440-457: sparsify-then-count estimate T' / q^3 (AOP draws
    per partition, the other engines one draw per edge)."""
    keep = None if boundaries is None else np.ascontiguousarray(boundaries, dtype=np.uint32)
    out = C.c_double()
    check(lib().tg_approx_count(g._h, int(p), int(engine), float(q), int(seed), _p(keep),
                                int(cost), C.byref(out)))
    return out.value


def per_edge_triangle_counts(g: Graph) -> np.ndarray:
    """sequential.hpp:108-122: t_e for every edge, in Graph::edges() order
    (u < v; graph.hpp:40-46).  The reference returns a map keyed by (u, v);
    pair it with ``Graph.edges()``.  t_e does not depend on the order; the
    degree order (as cli.hpp:312-313) keeps the listing short."""
    _use_order(g, None)
    m = g.num_edges()
    te = np.zeros(max(m, 1), dtype=np.uint64)
    check(lib().tg_per_edge_triangle_counts(g._h, _p(te)))
    return te[:m]


@dataclass
class VarianceReport:  # sparsify.hpp:113-121
    triangles: int = 0
    k: int = 0
    k_prime: int = 0
    q: float = 1.0
    var: float = 0.0
    var_prime: float = 0.0


def variance_report(g: Graph, plan: PartitionPlan, q: float) -> VarianceReport:
    """sparsify.hpp:113-155: k = pairs of triangles sharing an edge, k' =
    those whose apexes have the same owner; variances of the 1/q^3 estimator."""
    b = np.ascontiguousarray(plan.boundaries, dtype=np.uint32)
    o3 = np.zeros(3, dtype=np.uint64)
    v2 = np.zeros(2, dtype=np.float64)
    check(lib().tg_variance_report(g._h, _p(b), b.shape[0] - 1, float(q), _p(o3), _p(v2)))
    return VarianceReport(int(o3[0]), int(o3[1]), int(o3[2]), float(q), float(v2[0]),
                          float(v2[1]))


# ---------------------------------------------------------------- generators


def graph_rmat(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int,
               device: int = 0) -> Graph:
    """gen_rmat generated on the device (the same pairs as ``gen_rmat``) and
    built into a Graph there, n = 2^scale."""
    h = C.c_void_p()
    check(lib().tg_graph_from_rmat(device, scale, edge_factor, a, b, c, seed, C.byref(h)))
    return Graph(h, device)


def graph_ws(n: int, k: int, beta: float, seed: int, device: int = 0) -> Graph:
    """gen_ws generated on the device (the same pairs as ``gen_ws``) and built
    into a Graph there."""
    h = C.c_void_p()
    check(lib().tg_graph_from_ws(device, n, k, beta, seed, C.byref(h)))
    return Graph(h, device)


def normalized_triangle_count(triangles: int, n: int) -> float:
    """stats.hpp:21-23: mean triangles per node."""
    return 0.0 if n == 0 else float(triangles) / float(n)


def estimate_p_opt(n: float, dbar: float, base_n: float, base_dbar: float,
                   base_p_opt: float) -> int:
    """stats.hpp:11-19: p_opt extrapolated linearly in average degree and in
    sqrt(n) from a calibrated base network (llround, as std::llround)."""
    import math
    if n <= 0 or dbar <= 0 or base_n <= 0 or base_dbar <= 0 or base_p_opt <= 0:
        raise ValueError("estimate_p_opt: all inputs must be positive")
    est = base_p_opt * (dbar / base_dbar) * math.sqrt(n / base_n)
    return int(math.floor(est + 0.5)) if est >= 0 else int(math.ceil(est - 0.5))


def _pairs_from(fn, *args) -> np.ndarray:
    ptr = C.c_void_p()
    cnt = C.c_uint64()
    check(fn(*args, C.byref(ptr), C.byref(cnt)))
    E = cnt.value
    try:
        if E == 0:
            return np.zeros((0, 2), dtype=np.uint32)
        buf = (C.c_uint32 * (2 * E)).from_address(ptr.value)
        return np.frombuffer(buf, dtype=np.uint32).reshape(E, 2).copy()
    finally:
        lib().tg_free_host(ptr)


def gen_pa(n: int, d: int, seed: int) -> np.ndarray:
    """io.hpp:129-162 gen_pa edge stream (d = average degree, d/2 attachments)."""
    return _pairs_from(lib().tg_gen_pa, n, d, seed)


def gen_gnp(n: int, d: float, seed: int) -> np.ndarray:
    """io.hpp:85-123 gen_gnp edge stream."""
    return _pairs_from(lib().tg_gen_gnp, n, d, seed)


def gen_gnm(n: int, m: int, seed: int) -> np.ndarray:
    return _pairs_from(lib().tg_gen_gnm, n, m, seed)


def gen_rmat(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int) -> np.ndarray:
    return _pairs_from(lib().tg_gen_rmat, scale, edge_factor, a, b, c, seed)


def gen_ws(n: int, k: int, beta: float, seed: int) -> np.ndarray:
    return _pairs_from(lib().tg_gen_ws, n, k, beta, seed)
