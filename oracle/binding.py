"""ctypes bindings for the oracle -- TEST INFRASTRUCTURE ONLY.

Loaded only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
``--impl reference`` legs.  Two libraries:

* ``liboracle.so``   -- plain-C restatement of the reference (oracle.c).
* ``_ref/libtrigraph_ref.so`` -- the unmodified reference headers behind a
  C shim (ref_shim.cpp); present wherever `make -C oracle` ran with
  /root/reference mounted (it then travels to the GPU box as a built file).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
U64, U32, F64 = np.uint64, np.uint32, np.float64
P = C.c_void_p

ENGINES = {"seq": 0, "aop": 1, "anop-direct": 2, "anop-surrogate": 3}
COSTS = {"N": 0, "D": 1, "DH": 2, "DDH": 3, "DH2": 4, "DPD": 5, "NOV": 6}
ORDERS = {"id": 0, "degree": 1, "random": 2, "coreness": 3}  # order.hpp:19 OrderKind::Tag

_orc = None
_ref = None


def _ptr(a):
    return None if a is None else a.ctypes.data_as(P)


def lib():
    global _orc
    if _orc is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle not built: {path} (run make -C oracle)")
        L = C.CDLL(path)
        u64, vp, i32, dbl = C.c_uint64, C.c_void_p, C.c_int, C.c_double
        sig = {
            "orc_build_graph": (u64, [vp, u64, u64, C.POINTER(vp), C.POINTER(vp)]),
            "orc_free": (None, [vp]),
            "orc_degree_rank": (None, [u64, vp, vp]),
            "orc_effective": (u64, [u64, vp, vp, vp, vp, C.POINTER(vp)]),
            "orc_count": (u64, [u64, vp, vp, vp, vp, u64]),
            "orc_count_range": (u64, [u64, vp, vp, u64, u64]),
            "orc_ordering_cost": (u64, [u64, vp, vp, vp]),
            "orc_node_costs": (None, [u64, vp, vp, vp, vp, i32, vp, vp]),
            "orc_compute_boundaries": (i32, [vp, u64, u64, vp]),
            "orc_owner": (u64, [vp, u64, C.c_uint32]),
            "orc_run_engine": (u64, [u64, vp, vp, i32, u64, i32, vp, vp, vp, vp, vp,
                                     vp, vp, vp, u64]),
            "orc_run_engine_ex": (u64, [u64, vp, vp, i32, u64, i32, vp, vp, vp, vp, vp,
                                        vp, vp, vp, u64, i32, dbl, u64]),
            "orc_keep_entry": (i32, [dbl, u64, u64, C.c_uint32, C.c_uint32]),
            "orc_approx_count": (dbl, [u64, vp, vp, u64, i32, dbl, u64, vp, i32]),
            "orc_per_edge_counts": (None, [u64, vp, vp, vp]),
            "orc_variance_report": (None, [u64, vp, vp, vp, u64, dbl, vp, vp]),
            "orc_cc": (None, [u64, vp, vp, vp]),
            "orc_random_graph_pairs": (u64, [u64, dbl, u64, vp, u64]),
            "orc_coreness": (None, [u64, vp, vp, vp]),
            "orc_parse_edge_list": (u64, [C.c_char_p, u64, vp, u64, vp, vp, vp, vp]),
            "orc_write_edge_list": (u64, [u64, vp, vp, vp, u64]),
            "orc_compute_order": (i32, [u64, vp, vp, i32, u64, vp]),
            "orc_run_engine_ord": (u64, [u64, vp, vp, i32, u64, i32, vp, vp, vp, vp, vp,
                                         vp, vp, vp, u64, i32, dbl, u64, i32, u64]),
            # fullsize.c
            "orc_gen_pa": (u64, [u64, u64, u64, C.POINTER(vp)]),
            "orc_gen_gnm": (u64, [u64, u64, u64, C.POINTER(vp)]),
            "orc_gen_rmat": (u64, [C.c_uint32, u64, dbl, dbl, dbl, u64, i32, C.POINTER(vp)]),
            "orc_gen_ws": (u64, [u64, u64, dbl, u64, i32, C.POINTER(vp)]),
            "orc_build_graph_lean": (u64, [vp, u64, u64, i32, C.POINTER(vp), C.POINTER(vp)]),
            "orc_effective_mt": (u64, [u64, vp, vp, vp, i32, vp, C.POINTER(vp)]),
            "orc_tri_hash": (u64, [C.c_uint32, C.c_uint32, C.c_uint32]),
            "orc_count_full": (u64, [u64, vp, vp, vp, u64, i32, vp, vp, vp, vp]),
            "orc_surrogate_messages": (None, [u64, vp, vp, vp, u64, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libtrigraph_ref.so"))


def ref():
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libtrigraph_ref.so")
        if not os.path.exists(path):
            raise RuntimeError(f"reference shim not built: {path}")
        L = C.CDLL(path)
        u64, vp, i32, dbl = C.c_uint64, C.c_void_p, C.c_int, C.c_double
        sig = {
            "ref_graph_from_pairs": (vp, [vp, u64, u64]),
            "ref_graph_from_csr": (vp, [u64, vp, vp]),
            "ref_random_graph": (vp, [u64, dbl, u64]),
            "ref_complete": (vp, [u64]),
            "ref_wheel": (vp, [u64]),
            "ref_complete_bipartite": (vp, [u64, u64]),
            "ref_g5": (vp, []),
            "ref_gen_pa": (vp, [u64, u64, u64]),
            "ref_gen_gnp": (vp, [u64, dbl, u64]),
            "ref_graph_free": (None, [vp]),
            "ref_num_nodes": (u64, [vp]),
            "ref_num_edges": (u64, [vp]),
            "ref_graph_csr": (None, [vp, vp, vp]),
            "ref_degree_rank": (None, [vp, vp]),
            "ref_effective": (u64, [vp, vp, vp]),
            "ref_count": (u64, [vp]),
            "ref_ordering_cost": (u64, [vp]),
            "ref_node_costs": (None, [vp, i32, vp, vp]),
            "ref_compute_boundaries": (i32, [vp, u64, u64, vp]),
            "ref_overlap_stored": (u64, [vp, vp, u64, u64]),
            "ref_run_engine": (u64, [vp, i32, u64, i32, vp, vp, vp, vp, vp, vp, vp, u64,
                                     vp, i32]),
            "ref_clustering": (i32, [vp, i32, u64, i32, vp, vp]),
            "ref_run_engine_sparse": (u64, [vp, i32, u64, i32, vp, i32, dbl, u64, vp, vp, vp,
                                            vp, vp, vp, u64, vp]),
            "ref_approx_count": (dbl, [vp, u64, i32, dbl, u64, vp, i32]),
            "ref_keep_entry": (i32, [dbl, u64, i32, u64, C.c_uint32, C.c_uint32]),
            "ref_per_edge_counts": (u64, [vp, vp]),
            "ref_variance_report": (None, [vp, vp, u64, dbl, vp, vp]),
            "ref_eff_from_arrays": (vp, [u64, vp, vp]),
            "ref_eff_free": (None, [vp]),
            "ref_seq_sample": (dbl, [vp, vp, u64, vp, vp]),
            "ref_aop_threads": (dbl, [vp, vp, u64, vp, vp, vp, vp]),
            "ref_compute_order": (None, [vp, i32, u64, vp]),
            "ref_coreness": (None, [vp, vp]),
            "ref_parse_edge_list": (u64, [C.c_char_p, u64, vp, u64, vp, vp, u64]),
            "ref_write_edge_list": (u64, [vp, vp, u64]),
            "ref_effective_order": (u64, [vp, i32, u64, vp, vp, vp, vp]),
            "ref_run_engine_order": (u64, [vp, i32, u64, i32, i32, u64, vp, vp, vp, vp, vp,
                                           vp, u64, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _ref = L
    return _ref


# ---------------------------------------------------------------- oracle API


@dataclass
class CSR:
    n: int
    off: np.ndarray  # uint64[n+1]
    adj: np.ndarray  # uint32[2m]

    @property
    def m(self) -> int:
        return int(self.off[-1]) // 2


def build_graph(pairs, n_override: int = 0) -> CSR:
    """graph.hpp:58-85 via the C restatement."""
    pairs = np.ascontiguousarray(np.asarray(pairs, dtype=U32).reshape(-1, 2))
    L = lib()
    po, pa = C.c_void_p(), C.c_void_p()
    n = L.orc_build_graph(_ptr(pairs), pairs.shape[0], n_override, C.byref(po), C.byref(pa))
    off = np.ctypeslib.as_array(C.cast(po, C.POINTER(C.c_uint64)), (n + 1,)).copy()
    m2 = int(off[-1])
    adj = (np.ctypeslib.as_array(C.cast(pa, C.POINTER(C.c_uint32)), (max(m2, 1),))[:m2].copy())
    L.orc_free(po)
    L.orc_free(pa)
    return CSR(int(n), off, adj)


def degree_rank(g: CSR) -> np.ndarray:
    r = np.zeros(g.n, dtype=U32)
    lib().orc_degree_rank(g.n, _ptr(g.off), _ptr(r))
    return r


def compute_order(g: CSR, order="degree", seed: int = 0) -> np.ndarray:
    """order.hpp:85-128 compute_order(g, OrderKind{order, seed}).rank."""
    r = np.zeros(max(g.n, 1), dtype=U32)
    if lib().orc_compute_order(g.n, _ptr(g.off), _ptr(g.adj), ORDERS[order], int(seed),
                               _ptr(r)) != 0:
        raise ValueError(f"unknown order {order!r}")
    return r[: g.n]


def coreness(g: CSR) -> np.ndarray:
    """order.hpp:39-83 core numbers."""
    c = np.zeros(max(g.n, 1), dtype=U64)
    lib().orc_coreness(g.n, _ptr(g.off), _ptr(g.adj), _ptr(c))
    return c[: g.n]


def effective(g: CSR, order="degree", seed: int = 0):
    rank = compute_order(g, order, seed)
    eoff = np.zeros(g.n + 1, dtype=U64)
    pe = C.c_void_p()
    m = lib().orc_effective(g.n, _ptr(g.off), _ptr(g.adj), _ptr(rank), _ptr(eoff), C.byref(pe))
    eff = np.ctypeslib.as_array(C.cast(pe, C.POINTER(C.c_uint32)), (max(m, 1),))[:m].copy()
    lib().orc_free(pe)
    return eoff, eff


def count(g: CSR, tally=False, listing=False, order="degree", seed: int = 0):
    eoff, eff = effective(g, order, seed)
    L = lib()
    T = L.orc_count(g.n, _ptr(eoff), _ptr(eff), None, None, 0)
    tv = np.zeros(g.n, dtype=U64) if tally else None
    tri = np.zeros((max(T, 1), 3), dtype=U32) if listing else None
    if tally or listing:
        L.orc_count(g.n, _ptr(eoff), _ptr(eff), _ptr(tv), _ptr(tri), T)
    if listing:
        tri = tri[:T]
        tri = tri[np.lexsort((tri[:, 2], tri[:, 1], tri[:, 0]))]
    return int(T), tv, tri


def ordering_cost(g: CSR, order="degree", seed: int = 0) -> int:
    return int(lib().orc_ordering_cost(g.n, _ptr(g.off), _ptr(g.adj),
                                       _ptr(compute_order(g, order, seed))))


def node_costs(g: CSR, kind: str, order="degree", seed: int = 0):
    eoff, eff = effective(g, order, seed)
    f = np.zeros(g.n, dtype=U64)
    pre = np.zeros(g.n, dtype=U64)
    lib().orc_node_costs(g.n, _ptr(g.off), _ptr(g.adj), _ptr(eoff), _ptr(eff), COSTS[kind],
                         _ptr(f), _ptr(pre))
    return f, pre


def compute_boundaries(f, p: int):
    f = np.asarray(f, dtype=U64)
    pre = np.cumsum(f, dtype=U64) if len(f) else np.zeros(0, dtype=U64)
    b = np.zeros(p + 1, dtype=U32)
    if lib().orc_compute_boundaries(_ptr(pre), len(f), p, _ptr(b)) != 0:
        raise ValueError("compute_boundaries: p must be >= 1")
    return b


@dataclass
class Report:
    total: int
    boundaries: np.ndarray
    triangles: np.ndarray
    data_sent: np.ndarray
    data_recv: np.ndarray
    stored: np.ndarray
    node_counts: np.ndarray | None = None
    triangles_list: np.ndarray | None = None


SPARSIFY = {None: 0, "global": 1, "per-partition": 2}


def run_engine(g: CSR, engine="aop", ranks=1, cost="DPD", boundaries=None,
               track_nodes=False, collect_triangles=False, sparsify=None, q=1.0,
               seed=0, order="degree", order_seed=0) -> Report:
    """engines.hpp:335-418 run_engine via the C restatement; sparsify =
    None | "global" | "per-partition" (SparsifyConfig, sparsify.hpp:22-33);
    order = EngineConfig::order (engines.hpp:274)."""
    e = ENGINES[engine]
    p = 1 if engine == "seq" else int(ranks)
    if p == 0:
        raise ValueError("run_engine: ranks must be >= 1")
    L = lib()
    bo = np.zeros(p + 1, dtype=U32)
    bi = None if boundaries is None else np.ascontiguousarray(boundaries, dtype=U32)
    tri, sent, recv, st = (np.zeros(p, dtype=U64) for _ in range(4))
    tv = np.zeros(g.n, dtype=U64) if track_nodes else None
    T, _, _ = count(g) if collect_triangles else (0, None, None)
    lst = np.zeros((max(T, 1), 3), dtype=U32) if collect_triangles else None
    total = L.orc_run_engine_ord(g.n, _ptr(g.off), _ptr(g.adj), e, p, COSTS[cost], _ptr(bi),
                                 _ptr(bo), _ptr(tri), _ptr(sent), _ptr(recv), _ptr(st),
                                 _ptr(tv), _ptr(lst), T, SPARSIFY[sparsify], float(q), int(seed),
                                 ORDERS[order], int(order_seed))
    if collect_triangles:
        T = min(T, int(total))  # sparsified runs list only the kept triangles
        lst = lst[:T]
        lst = lst[np.lexsort((lst[:, 2], lst[:, 1], lst[:, 0]))]
    return Report(int(total), bo, tri, sent, recv, st, tv, lst)


def keep_entry(q, seed, rank_key, v, u) -> bool:
    """sparsify.hpp:58-62 keep_entry (rank key resolved: 0 Global, rank+1
    PerPartition)."""
    return bool(lib().orc_keep_entry(float(q), int(seed), int(rank_key), int(v), int(u)))


def approx_count(g: CSR, p, engine, q, seed, boundaries=None, cost="DPD") -> float:
    """engines.hpp:440-457 approx_count."""
    bi = None if boundaries is None else np.ascontiguousarray(boundaries, dtype=U32)
    return float(lib().orc_approx_count(g.n, _ptr(g.off), _ptr(g.adj), int(p), ENGINES[engine],
                                        float(q), int(seed), _ptr(bi), COSTS[cost]))


def per_edge_counts(g: CSR) -> np.ndarray:
    """sequential.hpp:108-122 per_edge_triangle_counts, Graph::edges() order."""
    te = np.zeros(max(len(g.adj) // 2, 1), dtype=U64)
    lib().orc_per_edge_counts(g.n, _ptr(g.off), _ptr(g.adj), _ptr(te))
    return te[: len(g.adj) // 2]


def variance_report(g: CSR, boundaries, q):
    """sparsify.hpp:113-155 variance_report -> (T, k, k', var, var')."""
    b = np.ascontiguousarray(boundaries, dtype=U32)
    o3 = np.zeros(3, dtype=U64)
    v2 = np.zeros(2, dtype=F64)
    lib().orc_variance_report(g.n, _ptr(g.off), _ptr(g.adj), _ptr(b), len(b) - 1, float(q),
                              _ptr(o3), _ptr(v2))
    return int(o3[0]), int(o3[1]), int(o3[2]), float(v2[0]), float(v2[1])


class ParseError(RuntimeError):
    """io.hpp:18-22: ParseError(line, what) -> "line N: what"."""

    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self.line = line


def parse_edge_list(text: bytes) -> np.ndarray:
    """io.hpp:24-50 via the C restatement: (E, 2) uint32 pairs in file order."""
    L = lib()
    line = np.zeros(1, dtype=U64)
    kind = np.zeros(1, dtype=np.int32)
    tb = np.zeros(1, dtype=U64)
    te = np.zeros(1, dtype=U64)
    cnt = L.orc_parse_edge_list(text, len(text), None, 0, _ptr(line), _ptr(kind), _ptr(tb),
                                _ptr(te))
    if cnt == 2**64 - 1:
        if int(kind[0]) == 1:
            raise ParseError(int(line[0]), "expected two integer tokens")
        tok = text[int(tb[0]):int(te[0])].decode("latin-1")
        raise ParseError(int(line[0]), f"trailing token '{tok}'")
    out = np.zeros((max(cnt, 1), 2), dtype=U32)
    L.orc_parse_edge_list(text, len(text), _ptr(out), cnt, _ptr(line), _ptr(kind), _ptr(tb),
                          _ptr(te))
    return out[:cnt]


def write_edge_list(g: CSR) -> bytes:
    """io.hpp:52-64 via the C restatement."""
    L = lib()
    n = L.orc_write_edge_list(g.n, _ptr(g.off), _ptr(g.adj), None, 0)
    buf = C.create_string_buffer(max(n, 1))
    L.orc_write_edge_list(g.n, _ptr(g.off), _ptr(g.adj), C.cast(buf, vp_t), n)
    return buf.raw[:n]


vp_t = C.c_void_p


def ref_parse_edge_list(text: bytes):
    """The unmodified reference's parse_edge_list: pairs, or (line, message)."""
    R = ref()
    line = np.zeros(1, dtype=U64)
    msg = C.create_string_buffer(512)
    cnt = R.ref_parse_edge_list(text, len(text), None, 0, _ptr(line), C.cast(msg, vp_t), 512)
    if cnt == 2**64 - 1:
        return int(line[0]), msg.value.decode("latin-1")
    out = np.zeros((max(cnt, 1), 2), dtype=U32)
    R.ref_parse_edge_list(text, len(text), _ptr(out), cnt, _ptr(line), C.cast(msg, vp_t), 512)
    return out[:cnt]


def clustering(g: CSR, tv) -> np.ndarray:
    c = np.zeros(g.n, dtype=F64)
    lib().orc_cc(g.n, _ptr(g.off), _ptr(np.ascontiguousarray(tv, dtype=U64)), _ptr(c))
    return c


def random_graph_pairs(n: int, density: float, seed: int) -> np.ndarray:
    """proj/tests/oracles.hpp:49-57 random_graph's accepted pairs."""
    cap = n * (n - 1) // 2
    out = np.zeros((max(cap, 1), 2), dtype=U32)
    c = lib().orc_random_graph_pairs(n, density, seed, _ptr(out), cap)
    return out[:c]


def random_graph(n: int, density: float, seed: int) -> CSR:
    return build_graph(random_graph_pairs(n, density, seed), n)


# --------------------------------------------------- reference (oracle/_ref)


class RefGraph:
    """Owns a reference trigraph::Graph built by the unmodified headers."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_graph_free(self.h)
            self.h = None

    @property
    def n(self) -> int:
        return int(ref().ref_num_nodes(self.h))

    @property
    def m(self) -> int:
        return int(ref().ref_num_edges(self.h))

    def csr(self) -> CSR:
        n, m = self.n, self.m
        off = np.zeros(n + 1, dtype=U64)
        adj = np.zeros(max(2 * m, 1), dtype=U32)
        ref().ref_graph_csr(self.h, _ptr(off), _ptr(adj))
        return CSR(n, off, adj[: 2 * m])

    @classmethod
    def from_pairs(cls, pairs, n_override=0):
        pairs = np.ascontiguousarray(np.asarray(pairs, dtype=U32).reshape(-1, 2))
        return cls(ref().ref_graph_from_pairs(_ptr(pairs), pairs.shape[0], n_override))

    @classmethod
    def from_csr(cls, g: CSR):
        return cls(ref().ref_graph_from_csr(g.n, _ptr(g.off), _ptr(g.adj)))

    def degree_rank(self):
        r = np.zeros(self.n, dtype=U32)
        ref().ref_degree_rank(self.h, _ptr(r))
        return r

    def write_edge_list(self) -> bytes:
        n = int(ref().ref_write_edge_list(self.h, None, 0))
        buf = C.create_string_buffer(max(n, 1))
        ref().ref_write_edge_list(self.h, C.cast(buf, vp_t), n)
        return buf.raw[:n]

    def compute_order(self, order="degree", seed=0):
        r = np.zeros(max(self.n, 1), dtype=U32)
        ref().ref_compute_order(self.h, ORDERS[order], int(seed), _ptr(r))
        return r[: self.n]

    def coreness(self):
        c = np.zeros(max(self.n, 1), dtype=U64)
        ref().ref_coreness(self.h, _ptr(c))
        return c[: self.n]

    def effective_order(self, order="degree", seed=0):
        """(eoff, eff, count, ordering_cost) under compute_order(g, order)."""
        o, sd = ORDERS[order], int(seed)
        m = int(ref().ref_effective_order(self.h, o, sd, None, None, None, None))
        eoff = np.zeros(self.n + 1, dtype=U64)
        eff = np.zeros(max(m, 1), dtype=U32)
        cnt = np.zeros(1, dtype=U64)
        cost = np.zeros(1, dtype=U64)
        ref().ref_effective_order(self.h, o, sd, _ptr(eoff), _ptr(eff), _ptr(cnt), _ptr(cost))
        return eoff, eff[:m], int(cnt[0]), int(cost[0])

    def run_engine_order(self, engine, ranks, order, order_seed=0, cost="DPD",
                         track_nodes=False, collect_triangles=False):
        e = ENGINES[engine]
        p = 1 if engine == "seq" else int(ranks)
        bo = np.zeros(max(p, 1) + 1, dtype=U32)
        tri, sent, recv = (np.zeros(max(p, 1), dtype=U64) for _ in range(3))
        tv = np.zeros(self.n, dtype=U64) if track_nodes else None
        cap = self.count() if collect_triangles else 0
        lst = np.zeros((max(cap, 1), 3), dtype=U32) if collect_triangles else None
        nl = np.zeros(1, dtype=U64)
        total = ref().ref_run_engine_order(self.h, e, int(ranks), COSTS[cost], ORDERS[order],
                                           int(order_seed), _ptr(bo), _ptr(tri), _ptr(sent),
                                           _ptr(recv), _ptr(tv), _ptr(lst), cap, _ptr(nl))
        if total == 2**64 - 1:
            raise ValueError("run_engine: ranks must be >= 1")
        return Report(int(total), bo, tri, sent, recv, np.zeros(p, dtype=U64), tv,
                      None if lst is None else lst[: int(nl[0])])

    def effective(self):
        m = int(ref().ref_effective(self.h, None, None))
        eoff = np.zeros(self.n + 1, dtype=U64)
        eff = np.zeros(max(m, 1), dtype=U32)
        ref().ref_effective(self.h, _ptr(eoff), _ptr(eff))
        return eoff, eff[:m]

    def count(self) -> int:
        return int(ref().ref_count(self.h))

    def ordering_cost(self) -> int:
        return int(ref().ref_ordering_cost(self.h))

    def node_costs(self, kind: str):
        f = np.zeros(self.n, dtype=U64)
        pre = np.zeros(self.n, dtype=U64)
        ref().ref_node_costs(self.h, COSTS[kind], _ptr(f), _ptr(pre))
        return f, pre

    def overlap_stored(self, b, i):
        b = np.ascontiguousarray(b, dtype=U32)
        return int(ref().ref_overlap_stored(self.h, _ptr(b), len(b) - 1, i))

    def run_engine(self, engine="aop", ranks=1, cost="DPD", boundaries=None,
                   track_nodes=False, collect_triangles=False, concurrent=False):
        e = ENGINES[engine]
        p = 1 if engine == "seq" else int(ranks)
        bo = np.zeros(max(p, 1) + 1, dtype=U32)
        bi = None if boundaries is None else np.ascontiguousarray(boundaries, dtype=U32)
        tri, sent, recv = (np.zeros(max(p, 1), dtype=U64) for _ in range(3))
        tv = np.zeros(self.n, dtype=U64) if track_nodes else None
        cap = self.count() if collect_triangles else 0
        lst = np.zeros((max(cap, 1), 3), dtype=U32) if collect_triangles else None
        nl = np.zeros(1, dtype=U64)
        total = ref().ref_run_engine(self.h, e, int(ranks), COSTS[cost], _ptr(bi), _ptr(bo),
                                     _ptr(tri), _ptr(sent), _ptr(recv), _ptr(tv), _ptr(lst),
                                     cap, _ptr(nl), 1 if concurrent else 0)
        if total == 2**64 - 1:
            raise ValueError("run_engine: ranks must be >= 1")
        return Report(int(total), bo, tri, sent, recv, np.zeros(p, dtype=U64), tv,
                      None if lst is None else lst[: int(nl[0])])

    def run_engine_sparse(self, engine, ranks, sparsify, q, seed, cost="DPD",
                          boundaries=None, track_nodes=False, collect_triangles=False):
        e = ENGINES[engine]
        p = 1 if engine == "seq" else int(ranks)
        bo = np.zeros(max(p, 1) + 1, dtype=U32)
        bi = None if boundaries is None else np.ascontiguousarray(boundaries, dtype=U32)
        tri, sent, recv = (np.zeros(max(p, 1), dtype=U64) for _ in range(3))
        tv = np.zeros(self.n, dtype=U64) if track_nodes else None
        cap = self.count() if collect_triangles else 0
        lst = np.zeros((max(cap, 1), 3), dtype=U32) if collect_triangles else None
        nl = np.zeros(1, dtype=U64)
        total = ref().ref_run_engine_sparse(self.h, e, int(ranks), COSTS[cost], _ptr(bi),
                                            SPARSIFY[sparsify], float(q), int(seed), _ptr(bo),
                                            _ptr(tri), _ptr(sent), _ptr(recv), _ptr(tv),
                                            _ptr(lst), cap, _ptr(nl))
        if total == 2**64 - 1:
            raise ValueError("run_engine: invalid arguments")
        return Report(int(total), bo, tri, sent, recv, np.zeros(p, dtype=U64), tv,
                      None if lst is None else lst[: int(nl[0])])

    def approx_count(self, p, engine, q, seed, boundaries=None, cost="DPD"):
        bi = None if boundaries is None else np.ascontiguousarray(boundaries, dtype=U32)
        return float(ref().ref_approx_count(self.h, int(p), ENGINES[engine], float(q), int(seed),
                                            _ptr(bi), COSTS[cost]))

    def per_edge_counts(self):
        te = np.zeros(max(self.m, 1), dtype=U64)
        k = ref().ref_per_edge_counts(self.h, _ptr(te))
        return te[:k]

    def variance_report(self, boundaries, q):
        b = np.ascontiguousarray(boundaries, dtype=U32)
        o3 = np.zeros(3, dtype=U64)
        v2 = np.zeros(2, dtype=F64)
        ref().ref_variance_report(self.h, _ptr(b), len(b) - 1, float(q), _ptr(o3), _ptr(v2))
        return int(o3[0]), int(o3[1]), int(o3[2]), float(v2[0]), float(v2[1])

    def clustering(self, engine="aop", ranks=1, cost="DPD"):
        tv = np.zeros(self.n, dtype=U64)
        c = np.zeros(self.n, dtype=F64)
        if ref().ref_clustering(self.h, ENGINES[engine], ranks, COSTS[cost], _ptr(tv),
                                _ptr(c)) != 0:
            raise ValueError("clustering_coefficients: ranks must be >= 1")
        return tv, c


def ref_random_graph(n, density, seed) -> RefGraph:
    return RefGraph(ref().ref_random_graph(n, density, seed))


def ref_fixture(name: str, *args) -> RefGraph:
    return RefGraph(getattr(ref(), "ref_" + name)(*args))


# ---------------------------------------------------------------- full size
# fullsize.c: the configs' generators and the memory-lean multi-threaded
# pipeline behind the C3/C4/C5 goldens (tests/golden/make_golden_full.py).

import weakref  # noqa: E402


class HostBuf:
    """A malloc'ed oracle buffer; freed with orc_free when dropped.  `.array`
    is a zero-copy numpy view (keep the HostBuf alive while it is used)."""

    def __init__(self, ptr: C.c_void_p, ctype, count: int):
        self.ptr = ptr
        self.count = count
        self.array = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), (max(count, 1),))[:count]
        self._fin = weakref.finalize(self, lib().orc_free, ptr)

    @classmethod
    def from_array(cls, a: np.ndarray, ctype=C.c_uint32) -> "HostBuf":
        """malloc'ed copy of a numpy array (for the consuming C calls)."""
        a = np.ascontiguousarray(a)
        libc = C.CDLL(None)
        libc.malloc.restype = C.c_void_p
        libc.malloc.argtypes = [C.c_size_t]
        ptr = C.c_void_p(libc.malloc(max(a.nbytes, 1)))
        if not ptr.value:
            raise MemoryError("malloc failed")
        C.memmove(ptr, a.ctypes.data, a.nbytes)
        return cls(ptr, ctype, a.nbytes // C.sizeof(ctype))

    def release(self) -> C.c_void_p:
        """Hand the pointer to a consuming C call (no free here)."""
        self._fin.detach()
        self.array = None
        return self.ptr


CONFIGS = {  # BASELINE.json configs (seeds recorded with the goldens)
    "C1": ("gnm", dict(n=100_000, m=1_000_000, seed=1)),
    "C2": ("pa", dict(n=10_000_000, d=40, seed=7)),
    "C3": ("rmat", dict(scale=24, ef=16, a=0.57, b=0.19, c=0.19, seed=1)),
    "C4": ("ws", dict(n=50_000_000, k=20, beta=0.1, seed=1)),
    "C5": ("pa", dict(n=100_000_000, d=40, seed=7)),
}


def threads_default() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def gen_pairs(kind: str, p: dict, threads: int = 0):
    """The config generators (fullsize.c).  Returns (HostBuf of 2E uint32, E, n)."""
    L, t = lib(), threads or threads_default()
    pp = C.c_void_p()
    if kind == "pa":
        E, n = L.orc_gen_pa(p["n"], p["d"], p["seed"], C.byref(pp)), p["n"]
    elif kind == "gnm":
        E, n = L.orc_gen_gnm(p["n"], p["m"], p["seed"], C.byref(pp)), p["n"]
    elif kind == "rmat":
        E = L.orc_gen_rmat(p["scale"], p["ef"], p.get("a", 0.57), p.get("b", 0.19),
                           p.get("c", 0.19), p["seed"], t, C.byref(pp))
        n = 1 << p["scale"]
    elif kind == "ws":
        E, n = L.orc_gen_ws(p["n"], p["k"], p["beta"], p["seed"], t, C.byref(pp)), p["n"]
    else:
        raise ValueError(kind)
    if E == 2**64 - 1:
        raise ValueError(f"bad generator arguments {kind} {p}")
    return HostBuf(pp, C.c_uint32, 2 * E), int(E), int(n)


class FullGraph:
    """Graph + ByDegree EffectiveAdjacency built by the full-size oracle."""

    def __init__(self, pairs: HostBuf, E: int, n_override: int, threads: int = 0):
        L, t = lib(), threads or threads_default()
        self.threads = t
        po, pa = C.c_void_p(), C.c_void_p()
        n = L.orc_build_graph_lean(pairs.release(), E, n_override, t, C.byref(po), C.byref(pa))
        self.n = int(n)
        self._off = HostBuf(po, C.c_uint64, self.n + 1)
        self.off = self._off.array
        self._adj = HostBuf(pa, C.c_uint32, int(self.off[-1]))
        self.adj = self._adj.array
        self.rank = np.zeros(max(self.n, 1), dtype=U32)
        L.orc_degree_rank(self.n, _ptr(self.off), _ptr(self.rank))
        self.eoff = np.zeros(self.n + 1, dtype=U64)
        pe = C.c_void_p()
        m = L.orc_effective_mt(self.n, _ptr(self.off), _ptr(self.adj), _ptr(self.rank), t,
                               _ptr(self.eoff), C.byref(pe))
        self._eff = HostBuf(pe, C.c_uint32, int(m))
        self.eff = self._eff.array

    @property
    def m(self) -> int:
        return int(self.off[-1]) // 2

    def csr(self) -> CSR:
        return CSR(self.n, self.off, self.adj)

    def ordering_cost(self) -> int:
        """sequential.hpp:95-104: sum_v d_v * h_v."""
        d = np.diff(self.off)
        h = np.diff(self.eoff)
        return int((d * h).sum(dtype=U64))

    def dpd_boundaries(self, p: int) -> np.ndarray:
        """compute_boundaries(node_costs(DPD), p) (partition.hpp:60-69, 116-141)."""
        f = np.zeros(max(self.n, 1), dtype=U64)
        pre = np.zeros(max(self.n, 1), dtype=U64)
        lib().orc_node_costs(self.n, _ptr(self.off), _ptr(self.adj), _ptr(self.eoff),
                             _ptr(self.eff), COSTS["DPD"], _ptr(f), _ptr(pre))
        b = np.zeros(p + 1, dtype=U32)
        lib().orc_compute_boundaries(_ptr(pre), self.n, p, _ptr(b))
        return b

    def count(self, boundaries=None, tally=False, digest=False):
        """count_node_iterator_n on all threads.  Returns dict(total, tally,
        apex (AOP per-rank T), mid (surrogate per-rank T), digest)."""
        p = 0 if boundaries is None else len(boundaries) - 1
        b = None if boundaries is None else np.ascontiguousarray(boundaries, dtype=U32)
        tv = np.zeros(max(self.n, 1), dtype=U64) if tally else None
        apex = np.zeros(max(p, 1), dtype=U64) if p else None
        mid = np.zeros(max(p, 1), dtype=U64) if p else None
        dg = np.zeros(2, dtype=U64) if digest else None
        total = lib().orc_count_full(self.n, _ptr(self.eoff), _ptr(self.eff), _ptr(b), p,
                                     self.threads, _ptr(tv), _ptr(apex), _ptr(mid), _ptr(dg))
        return {"total": int(total), "tally": None if tv is None else tv[: self.n],
                "apex": None if apex is None else apex[:p].tolist(),
                "mid": None if mid is None else mid[:p].tolist(),
                "digest": None if dg is None else [int(x) for x in dg]}

    def surrogate_messages(self, boundaries):
        b = np.ascontiguousarray(boundaries, dtype=U32)
        p = len(b) - 1
        sent = np.zeros(p, dtype=U64)
        recv = np.zeros(p, dtype=U64)
        lib().orc_surrogate_messages(self.n, _ptr(self.eoff), _ptr(self.eff), _ptr(b), p,
                                     _ptr(sent), _ptr(recv))
        return sent.tolist(), recv.tolist()

    def clustering(self, tally) -> np.ndarray:
        c = np.zeros(max(self.n, 1), dtype=F64)
        lib().orc_cc(self.n, _ptr(self.off), _ptr(tally), _ptr(c))
        return c[: self.n]


def tri_digest_np(tri) -> list:
    """The listing digest of oracle.h orc_tri_hash over an (T, 3) array of
    normalised triples (ascending within each row), numpy (wrapping uint64)."""
    t = np.asarray(tri, dtype=U64).reshape(-1, 3)

    def mix(x):
        x = x + U64(0x9E3779B97F4A7C15)
        x ^= x >> U64(30)
        x *= U64(0xBF58476D1CE4E5B9)
        x ^= x >> U64(27)
        x *= U64(0x94D049BB133111EB)
        x ^= x >> U64(31)
        return x

    with np.errstate(over="ignore"):
        h = mix(mix(mix(t[:, 0]) ^ t[:, 1]) ^ t[:, 2])
        return [int(h.sum(dtype=U64)), int(mix(h).sum(dtype=U64))]
