"""Generate tests/golden/*.json from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference is mounted and `make -C oracle` built
oracle/_ref/libtrigraph_ref.so):

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --next     # only the 8(f) rows (sparsify, t_e)
    python tests/golden/make_golden.py --orders   # only the OrderKind fixtures
    python tests/golden/make_golden.py --io       # only the edge-list text fixtures
    python tests/golden/make_golden.py --full     # + full-size C1/C2 goldens

Every number in the fixtures comes from the reference's own functions
(build_graph, compute_order, effective_adjacency, count_node_iterator_n,
node_costs, compute_boundaries, run_engine, clustering_coefficients,
gen_pa, gen_gnp, oracles::random_graph ...) called through ref_shim.cpp.
Large arrays are stored as sha256 digests of their little-endian bytes.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import binding as B  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
ENGINES = ["seq", "aop", "anop-direct", "anop-surrogate"]
COSTS = list(B.COSTS)


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def engine_record(R: B.RefGraph, engine, p, cost, boundaries=None):
    rep = R.run_engine(engine, p, cost, boundaries=boundaries, track_nodes=True,
                       collect_triangles=True)
    pp = 1 if engine == "seq" else p
    return {
        "engine": engine, "ranks": p, "cost": cost,
        "boundaries_in": None if boundaries is None else [int(x) for x in boundaries],
        "total": rep.total,
        "boundaries": rep.boundaries[: pp + 1].tolist(),
        "triangles": rep.triangles[:pp].tolist(),
        "data_sent": rep.data_sent[:pp].tolist(),
        "data_recv": rep.data_recv[:pp].tolist(),
        "node_counts_sha256": digest(rep.node_counts),
        "triangles_sha256": digest(rep.triangles_list),
    }


def graph_record(R: B.RefGraph, name: str, pairs=None, n_override=0, engines=True):
    g = R.csr()
    eoff, eff = R.effective()
    tv, cc = R.clustering("seq", 1)
    rec = {
        "name": name, "n": g.n, "m": g.m,
        "offsets_sha256": digest(g.off), "adj_sha256": digest(g.adj),
        "rank_sha256": digest(R.degree_rank()),
        "eff_offsets_sha256": digest(eoff), "eff_sha256": digest(eff),
        "count": R.count(), "ordering_cost": R.ordering_cost(),
        "node_counts_sha256": digest(tv), "cc_sha256": digest(cc),
        "costs_sha256": {k: digest(R.node_costs(k)[0]) for k in COSTS},
    }
    if pairs is not None:
        rec["pairs_sha256"] = digest(np.ascontiguousarray(pairs, dtype=np.uint32))
        rec["n_override"] = n_override
    if engines:
        rec["engines"] = [engine_record(R, e, p, c) for e in ENGINES for p in (1, 2, 3, 4, 8)
                          for c in ("N", "DPD", "NOV") if not (e == "seq" and (p > 1 or c != "DPD"))]
    return rec


def small():
    fx = {}
    # G5 (proj/tests/oracles.hpp:20-22) -- explicit values, tests read them directly
    R = B.ref_fixture("g5")
    g = R.csr()
    eoff, eff = R.effective()
    tv, cc = R.clustering("aop", 2)
    fx["g5"] = {
        "pairs": [[0, 1], [0, 2], [1, 2], [1, 3], [2, 3], [3, 4]],
        "offsets": g.off.tolist(), "adj": g.adj.tolist(),
        "rank": R.degree_rank().tolist(),
        "eff_offsets": eoff.tolist(), "eff": eff.tolist(),
        "count": R.count(), "ordering_cost": R.ordering_cost(),
        "costs": {k: R.node_costs(k)[0].tolist() for k in COSTS},
        "node_counts": tv.tolist(), "cc": cc.tolist(),
        "plan_025": [engine_record(R, e, 2, "DPD", [0, 2, 5]) for e in ENGINES[1:]],
        "overlap_stored_025": [R.overlap_stored([0, 2, 5], i) for i in range(2)],
    }
    for e in fx["g5"]["plan_025"]:
        rr = R.run_engine(e["engine"], 2, "DPD", boundaries=[0, 2, 5], collect_triangles=True)
        e["triangles_list"] = rr.triangles_list.tolist()
    # complete graphs, wheels, bipartite (acceptance.cpp:239-264)
    fx["complete"] = {n: B.ref_fixture("complete", n).count() for n in range(3, 11)}
    fx["wheel"] = {r: B.ref_fixture("wheel", r).count() for r in range(4, 13)}
    fx["bipartite"] = {f"{a}x{b}": B.ref_fixture("complete_bipartite", a, b).count()
                       for a, b in ((3, 4), (5, 5), (1, 6))}
    # K8 / NOV / surrogate / p=3 (test_engines.cpp:90-94)
    fx["k8_nov_surrogate_p3"] = B.ref_fixture("complete", 8).run_engine(
        "anop-surrogate", 3, "NOV").total
    # the acceptance suite: 200 seeded graphs (acceptance.cpp:76-88)
    suite = []
    import ctypes as C
    st = B.lib()
    mt = (C.c_uint64 * 313)()
    st.orc_mt64_seed.argtypes = [C.c_void_p, C.c_uint64]
    st.orc_mt64_next.argtypes = [C.c_void_p]
    st.orc_mt64_next.restype = C.c_uint64
    st.orc_mt64_seed(C.addressof(mt), 20240201)
    for i in range(200):
        n = 8 + st.orc_mt64_next(C.addressof(mt)) % 93
        density = 0.02 + 0.93 * (i / 199.0)
        seed = st.orc_mt64_next(C.addressof(mt))
        R = B.ref_random_graph(n, density, seed)
        rec = {"n": int(n), "density": density, "seed": int(seed), "count": R.count(),
               "adj_sha256": digest(R.csr().adj)}
        if i % 10 == 0:  # per-rank records for every 10th graph
            rec["engines"] = [engine_record(R, e, p, c) for e in ENGINES[1:] for p in (2, 3, 8)
                              for c in ("N", "DPD", "NOV")]
        suite.append(rec)
    fx["acceptance_suite"] = {"seed": 20240201, "graphs": suite}
    # per-node tallies / CC (acceptance.cpp:399-426, seed 911)
    st.orc_mt64_seed(C.addressof(mt), 911)
    c9 = []
    for i in range(40):
        n = 10 + st.orc_mt64_next(C.addressof(mt)) % 50
        density = 0.05 + 0.02 * i
        seed = st.orc_mt64_next(C.addressof(mt))
        R = B.ref_random_graph(n, density, seed)
        tv, cc = R.clustering("anop-surrogate", 3)
        c9.append({"n": int(n), "density": density, "seed": int(seed), "node_counts": tv.tolist(),
                   "cc": [float(x).hex() for x in cc]})
    fx["criterion9"] = c9
    # generator streams (io.hpp:85-162) -- digests of the reference graphs
    fx["gen_pa"] = [dict(n=n, d=d, seed=s, **{k: v for k, v in graph_record(
        B.ref_fixture("gen_pa", n, d, s), f"pa{n}", engines=False).items()
        if k in ("m", "adj_sha256", "offsets_sha256", "count", "ordering_cost")})
        for (n, d, s) in ((10000, 20, 1), (2000, 40, 7), (200000, 40, 7))]
    fx["gen_gnp"] = [dict(n=n, d=d, seed=s, **{k: v for k, v in graph_record(
        B.ref_fixture("gen_gnp", n, float(d), s), f"gnp{n}", engines=False).items()
        if k in ("m", "adj_sha256", "offsets_sha256", "count")})
        for (n, d, s) in ((2000, 20, 42), (100000, 20, 7))]
    # a PA graph with full per-engine records at p up to 8
    R = B.ref_fixture("gen_pa", 20000, 20, 3)
    fx["pa20000"] = graph_record(R, "gen_pa(20000,20,3)")
    return fx


def sparse_record(R: B.RefGraph, engine, p, mode, q, seed):
    rep = R.run_engine_sparse(engine, p, mode, q, seed, track_nodes=True, collect_triangles=True)
    pp = 1 if engine == "seq" else p
    return {
        "engine": engine, "ranks": p, "sparsify": mode, "q": q, "seed": seed,
        "total": rep.total,
        "triangles": rep.triangles[:pp].tolist(),
        "data_sent": rep.data_sent[:pp].tolist(),
        "data_recv": rep.data_recv[:pp].tolist(),
        "node_counts_sha256": digest(rep.node_counts),
        "triangles_sha256": digest(rep.triangles_list),
    }


def next_rows():
    """sparsification (sparsify.hpp, engines.hpp:440-457),
    per-edge triangle counts (sequential.hpp:108-122), variance_report."""
    fx = {}
    rng = np.random.default_rng(1706)
    keep = []
    for _ in range(256):
        q = float(rng.choice([0.1, 0.25, 0.5, 0.9, 1.0]))
        seed = int(rng.integers(1 << 63))
        mode = int(rng.integers(1, 3))
        rank = int(rng.integers(0, 16))
        v, u = (int(x) for x in rng.integers(0, 1 << 32, size=2))
        keep.append([q, seed, mode, rank, v, u, int(B.ref().ref_keep_entry(q, seed, mode, rank, v,
                                                                          u))])
    fx["keep_entry"] = keep
    graphs = [("pa20000", B.ref_fixture("gen_pa", 20000, 20, 3))]
    for i, (n, dens, seed) in enumerate(((60, 0.3, 11), (90, 0.5, 12), (40, 0.8, 13))):
        graphs.append((f"random{i}", B.ref_random_graph(n, dens, seed)))
    recs = {}
    for name, R in graphs:
        g = R.csr()
        te = R.per_edge_counts()
        rec = {"n": g.n, "m": g.m, "adj_sha256": digest(g.adj),
               "per_edge_sha256": digest(te), "per_edge_sum": int(te.sum()),
               "k": int(sum(int(c) * (int(c) - 1) // 2 for c in te))}
        if name != "pa20000":
            rec["per_edge"] = te.tolist()
        rec["sparse"] = [sparse_record(R, e, p, mode, q, 77 + p)
                         for e in ENGINES for mode in ("global", "per-partition")
                         for (p, q) in ((1, 0.5), (3, 0.5), (4, 0.25), (8, 0.7))
                         if not (e == "seq" and p > 1)]
        rec["approx"] = [{"engine": e, "ranks": p, "q": q, "seed": 5,
                          "value": float(R.approx_count(p, e, q, 5)).hex()}
                         for e in ENGINES for (p, q) in ((1, 0.5), (4, 0.3))]
        pre = R.node_costs("DPD")[1]
        f = R.node_costs("DPD")[0]
        rec["variance"] = []
        for p in (2, 4, 8):
            b = np.zeros(p + 1, dtype=np.uint32)
            B.ref().ref_compute_boundaries(f.ctypes.data, len(f), p, b.ctypes.data)
            T, k, kp, var, varp = R.variance_report(b, 0.5)
            rec["variance"].append({"boundaries": b.tolist(), "q": 0.5, "T": T, "k": k,
                                    "k_prime": kp, "var": var.hex(), "var_prime": varp.hex()})
        recs[name] = rec
    fx["graphs"] = recs
    return fx


ORDERS = [("id", 0), ("degree", 0), ("random", 42), ("random", 43), ("coreness", 0)]


def order_record(R: B.RefGraph, engines=(("aop", 3), ("anop-direct", 2), ("anop-surrogate", 4)),
                 explicit=False):
    """compute_order / coreness / effective_adjacency / count / ordering_cost
    and run_engine under every OrderKind (order.hpp:85-128, engines.hpp:274)."""
    g = R.csr()
    core = R.coreness()
    rec = {"n": g.n, "m": g.m, "adj_sha256": digest(g.adj), "coreness_sha256": digest(core),
           "orders": []}
    if explicit:
        rec["coreness"] = core.tolist()
    for order, seed in ORDERS:
        rank = R.compute_order(order, seed)
        eoff, eff, cnt, cost = R.effective_order(order, seed)
        o = {"order": order, "seed": seed, "rank_sha256": digest(rank),
             "eff_offsets_sha256": digest(eoff), "eff_sha256": digest(eff),
             "count": cnt, "ordering_cost": cost, "engines": []}
        if explicit:
            o["rank"] = rank.tolist()
            o["eff_offsets"] = eoff.tolist()
            o["eff"] = eff.tolist()
        for e, p in engines:
            rep = R.run_engine_order(e, p, order, seed, track_nodes=True, collect_triangles=True)
            o["engines"].append({
                "engine": e, "ranks": p, "total": rep.total,
                "boundaries": rep.boundaries[: p + 1].tolist(),
                "triangles": rep.triangles[:p].tolist(),
                "data_sent": rep.data_sent[:p].tolist(),
                "data_recv": rep.data_recv[:p].tolist(),
                "node_counts_sha256": digest(rep.node_counts),
                "triangles_sha256": digest(rep.triangles_list)})
        rec["orders"].append(o)
    return rec


def orders():
    """Every OrderKind of the reference (order.hpp:17-128): the order-dependent
    results on G5 (explicit), small fixtures and seeded graphs."""
    from paper_1706_05151_b200 import trigraph as T  # generators only (host harness)
    fx = {"g5": order_record(B.ref_fixture("g5"), explicit=True),
          "k3_coreness": B.ref_fixture("complete", 3).coreness().tolist(),
          "path_coreness": B.RefGraph.from_pairs([[0, 1], [1, 2]]).coreness().tolist()}
    fx["random"] = []
    for i in range(12):
        n, dens, seed = 20 + 9 * i, 0.05 + 0.07 * i, 500 + i
        rec = order_record(B.ref_random_graph(n, dens, seed))
        rec.update({"gen": [n, dens, seed]})
        fx["random"].append(rec)
    fx["pa20000"] = order_record(B.ref_fixture("gen_pa", 20000, 20, 3),
                                 engines=(("aop", 8), ("anop-surrogate", 8)))
    pairs = T.gen_rmat(12, 8, 0.57, 0.19, 0.19, 5)
    rec = order_record(B.RefGraph.from_pairs(pairs), engines=(("aop", 4), ("anop-surrogate", 4)))
    rec["pairs_sha256"] = digest(np.ascontiguousarray(pairs, dtype=np.uint32))
    fx["rmat12"] = rec
    return fx


def io_texts():
    """Edge-list texts for parse_edge_list (io.hpp:24-50): the reference tests'
    cases, the istream corner cases (signs, overflow, \\v/\\f, CRLF, NUL,
    trailing tokens) and seeded random texts."""
    import random
    rng = random.Random(1706)
    texts = [b"", b"0 1\n1 2\n", b"# comment\n3 4\n", b"\n  \n# only comments\n", b"0 x\n",
             b"0 1\n\n2 y\n", b"1 2 3\n", b"12+3\n", b"12-3", b"-1 -2\n", b"+5 +6\r\n",
             b" \t# x\n1 2", b"1\n2\n", b"\v1 2\n", b"1 2\v\n", b"1 2 #c\n",
             b"4294967296 4294967297\n", b"18446744073709551615 0\n",
             b"18446744073709551616 0\n", b"-18446744073709551615 1\n",
             b"-18446744073709551616 1\n", b"00012 0003\n", b"1 2\x00\n", b"\r\n\r\n1\t2\r\n",
             b"1 2\n3 4\n5 6\n7 8 x\n9 10\n", b"#\n#\n 3  4 \n\f5 6\n", b"- 1\n", b"+\n", b"1 +\n"]
    ws = [b"", b" ", b"\t", b"  ", b"\r", b" \v", b"\f"]
    nums = [b"0", b"1", b"42", b"+7", b"-3", b"4294967295", b"4294967296",
            b"18446744073709551615", b"007", b"123456"]
    for _ in range(300):
        lines = []
        for _ in range(rng.randint(0, 12)):
            r = rng.random()
            if r < 0.1:
                lines.append(rng.choice(ws) + b"# c " + rng.choice(nums))
            elif r < 0.15:
                lines.append(rng.choice(ws))
            else:
                lines.append(rng.choice(ws) + rng.choice(nums) + rng.choice(ws[1:]) +
                             rng.choice(nums) + rng.choice(ws) +
                             (b" x" if rng.random() < 0.02 else b""))
        texts.append(b"\n".join(lines) + (b"\n" if rng.random() < 0.5 else b""))
    return texts


def io_rows():
    """parse_edge_list / write_edge_list (io.hpp:18-64) through the reference."""
    from paper_1706_05151_b200 import trigraph as T  # generators only (host harness)
    cases = []
    for t in io_texts():
        r = B.ref_parse_edge_list(t)
        if isinstance(r, tuple):
            cases.append({"text": t.decode("latin-1"), "error_line": r[0], "error": r[1]})
        else:
            cases.append({"text": t.decode("latin-1"), "pairs": r.reshape(-1).tolist()})
    fx = {"parse": cases}
    for name, R in (("g5", B.ref_fixture("g5")), ("pa20000", B.ref_fixture("gen_pa", 20000, 20, 3)),
                    ("rmat12", B.RefGraph.from_pairs(T.gen_rmat(12, 8, 0.57, 0.19, 0.19, 5)))):
        txt = R.write_edge_list()
        rec = {"len": len(txt), "sha256": hashlib.sha256(txt).hexdigest(), "m": R.m, "n": R.n}
        if name == "g5":
            rec["text"] = txt.decode("latin-1")
        fx["write_" + name] = rec
    return fx


def full():
    sys.path.insert(0, ROOT)
    from paper_1706_05151_b200 import trigraph as T  # generators only (host harness)
    fx = {}
    t = time.time()
    pairs = T.gen_gnm(100_000, 1_000_000, 1)
    R = B.RefGraph.from_pairs(pairs, 100_000)
    rec = graph_record(R, "C1 gnm(1e5,1e6,seed=1)", pairs, 100_000, engines=False)
    rec["engines"] = [engine_record(R, e, p, "DPD") for e in ENGINES for p in (1, 8)
                      if not (e == "seq" and p > 1)]
    fx["C1"] = rec
    print("C1", time.time() - t, flush=True)
    t = time.time()
    R = B.ref_fixture("gen_pa", 10_000_000, 40, 7)
    g = R.csr()
    print("C2 gen", time.time() - t, flush=True)
    t0 = time.time()
    cnt = R.count()
    fx["C2"] = {"name": "C2 gen_pa(1e7,40,seed=7)", "n": g.n, "m": g.m, "count": cnt,
                "ordering_cost": R.ordering_cost(), "count_seconds_1thread": time.time() - t0,
                "adj_sha256": digest(g.adj), "offsets_sha256": digest(g.off)}
    print("C2", fx["C2"], flush=True)
    return fx


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--next", action="store_true", help="only reference_next.json")
    ap.add_argument("--orders", action="store_true", help="only reference_orders.json")
    ap.add_argument("--io", action="store_true", help="only reference_io.json")
    a = ap.parse_args()
    if not B.ref_available():
        sys.exit("oracle/_ref not built (make -C oracle with /root/reference mounted)")
    sys.path.insert(0, ROOT)
    fx = io_rows()
    with open(os.path.join(OUT, "reference_io.json"), "w") as f:
        json.dump(fx, f, indent=0, sort_keys=True)
    print("wrote reference_io.json")
    if a.io:
        sys.exit(0)
    fx = orders()
    with open(os.path.join(OUT, "reference_orders.json"), "w") as f:
        json.dump(fx, f, indent=0, sort_keys=True)
    print("wrote reference_orders.json")
    if a.orders:
        sys.exit(0)
    fx = next_rows()
    with open(os.path.join(OUT, "reference_next.json"), "w") as f:
        json.dump(fx, f, indent=0, sort_keys=True)
    print("wrote reference_next.json")
    if a.next:
        sys.exit(0)
    fx = small()
    with open(os.path.join(OUT, "reference_small.json"), "w") as f:
        json.dump(fx, f, indent=0, sort_keys=True)
    print("wrote reference_small.json")
    if a.full:
        fx = full()
        with open(os.path.join(OUT, "reference_full.json"), "w") as f:
            json.dump(fx, f, indent=1, sort_keys=True)
        print("wrote reference_full.json")
