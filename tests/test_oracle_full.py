"""The full-size oracle (oracle/fullsize.c) pinned on sizes the reference
finishes in seconds (CPU): its generators against the library's host
generators and the reference's gen_pa; its build / orientation / counting /
per-rank / messaging / tally / listing-digest outputs against oracle.c and
against the unmodified reference (oracle/_ref).  This is what licenses the
C3/C4/C5 goldens in tests/golden/reference_full.json."""
import ctypes as C
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import binding as B

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("kind,p", [
    ("pa", dict(n=30_000, d=40, seed=7)),
    ("pa", dict(n=5_000, d=6, seed=3)),
    ("gnm", dict(n=20_000, m=100_000, seed=1)),
    ("rmat", dict(scale=13, ef=16, a=0.57, b=0.19, c=0.19, seed=1)),
    ("ws", dict(n=200_000, k=20, beta=0.1, seed=1)),
])
def test_generators_match_library(kind, p):
    from paper_1706_05151_b200 import trigraph as T  # host generators only

    buf, E, _ = B.gen_pairs(kind, p, threads=3)
    if kind == "pa":
        want = T.gen_pa(p["n"], p["d"], p["seed"])
    elif kind == "gnm":
        want = T.gen_gnm(p["n"], p["m"], p["seed"])
    elif kind == "rmat":
        want = T.gen_rmat(p["scale"], p["ef"], p["a"], p["b"], p["c"], p["seed"])
    else:
        want = T.gen_ws(p["n"], p["k"], p["beta"], p["seed"])
    assert np.array_equal(buf.array.reshape(-1, 2), want)


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")
def test_gen_pa_matches_reference():
    """io.hpp:129-162 through the reference itself (CSR digest)."""
    buf, E, n = B.gen_pairs("pa", dict(n=20_000, d=20, seed=3))
    g = B.FullGraph(buf, E, n, threads=2)
    R = B.ref_fixture("gen_pa", 20_000, 20, 3)
    rc = R.csr()
    assert np.array_equal(g.off, rc.off) and np.array_equal(g.adj, rc.adj)


def _cases():
    yield "pa", dict(n=20_000, d=20, seed=3)
    yield "rmat", dict(scale=12, ef=8, a=0.57, b=0.19, c=0.19, seed=5)
    yield "ws", dict(n=30_000, k=10, beta=0.3, seed=2)
    yield "gnm", dict(n=3_000, m=30_000, seed=9)


@pytest.mark.parametrize("kind,p", list(_cases()))
@pytest.mark.parametrize("threads", [1, 5])
def test_pipeline_matches_oracle_and_reference(kind, p, threads):
    buf, E, n = B.gen_pairs(kind, p, threads)
    pairs = buf.array.copy().reshape(-1, 2)
    g = B.FullGraph(buf, E, n, threads)
    ref = B.build_graph(pairs, n)  # oracle.c
    assert np.array_equal(g.off, ref.off) and np.array_equal(g.adj, ref.adj)
    eoff, eff = B.effective(ref)
    assert np.array_equal(g.eoff, eoff) and np.array_equal(g.eff, eff)
    assert g.ordering_cost() == B.ordering_cost(ref)
    b = g.dpd_boundaries(8)
    want_b = B.compute_boundaries(B.node_costs(ref, "DPD")[0], 8)
    assert b.tolist() == want_b.tolist()
    r = g.count(b, tally=True, digest=True)
    T_, tv, tri = B.count(ref, tally=True, listing=True)
    assert r["total"] == T_
    assert np.array_equal(r["tally"], tv)
    assert r["digest"] == B.tri_digest_np(tri)
    aop = B.run_engine(ref, "aop", 8, "DPD")
    assert r["apex"] == aop.triangles.tolist()
    sur = B.run_engine(ref, "anop-surrogate", 8, "DPD")
    assert r["mid"] == sur.triangles.tolist()
    sent, recv = g.surrogate_messages(b)
    assert sent == sur.data_sent.tolist() and recv == sur.data_recv.tolist()
    assert np.array_equal(g.clustering(r["tally"]), B.clustering(ref, tv))
    if B.ref_available():  # and the unmodified reference
        R = B.RefGraph.from_pairs(pairs, n)
        assert R.count() == T_
        ra = R.run_engine("aop", 8, "DPD")
        rs = R.run_engine("anop-surrogate", 8, "DPD")
        assert ra.triangles[:8].tolist() == r["apex"]
        assert rs.triangles[:8].tolist() == r["mid"]
        assert rs.data_sent[:8].tolist() == sent and rs.data_recv[:8].tolist() == recv
        rtv, rcc = R.clustering("seq", 1)
        assert np.array_equal(rtv, r["tally"])
        assert np.array_equal(rcc, g.clustering(r["tally"]))


def test_empty_and_loops():
    """Loops dropped, duplicates merged, n from n_override (graph.hpp:58-85)."""
    pairs = np.array([[3, 3], [0, 1], [1, 0], [1, 2], [2, 0], [0, 1]], dtype=np.uint32)
    g = B.FullGraph(B.HostBuf.from_array(pairs), 6, 10, threads=2)
    ref = B.build_graph(pairs, 10)
    assert g.n == 10 and np.array_equal(g.off, ref.off) and np.array_equal(g.adj, ref.adj)
    assert g.count()["total"] == 1
    e = B.FullGraph(B.HostBuf.from_array(np.zeros((0, 2), np.uint32)), 0, 0, threads=2)
    assert e.n == 0 and e.count()["total"] == 0


def test_full_records_are_consistent():
    """The committed full-size records: C1/C2 oracle records equal the
    reference-made ones; per-rank sums equal the totals; T_v sums to 3T."""
    with open(os.path.join(GOLDEN, "reference_full.json")) as f:
        fx = json.load(f)
    for c in ("C1", "C2"):
        o = fx.get(c + "_oracle")
        if o is None:
            continue
        for k in ("n", "m", "count", "ordering_cost", "adj_sha256", "offsets_sha256"):
            assert o[k] == fx[c][k], (c, k)
    if "node_counts_sha256" in fx.get("C2", {}) and "C2_oracle" in fx:
        assert fx["C2"]["node_counts_sha256"] == fx["C2_oracle"]["node_counts_sha256"]
        assert fx["C2"]["cc_sha256"] == fx["C2_oracle"]["cc_sha256"]
    for c in ("C2", "C3", "C4", "C5"):
        o = fx.get(c + "_oracle")
        if o is None:
            continue
        assert sum(o["aop8_triangles"]) == o["count"]
        assert sum(o["surrogate8_triangles"]) == o["count"]
        assert sum(o["surrogate8_data_sent"]) == sum(o["surrogate8_data_recv"])
        assert len(o["dpd8_boundaries"]) == 9 and o["dpd8_boundaries"][-1] == o["n"]


def test_bench_cpu_baseline_c1():
    """bench.py's CPU legs on C1: the reference AOP sample counts exactly the
    sampled cores' triangles; the 1-thread leg runs."""
    import bench

    buf, E, n = B.gen_pairs("gnm", dict(n=100_000, m=1_000_000, seed=1))
    cb = bench.CpuBaseline(buf, E, n, threads=4)
    try:
        cb.R = 1
        dt, tb, e, t, st = cb.aop(0)
        assert t == 1269 and e == 1_000_000 and st >= e
        cb.R = 7
        tot = sum(cb.aop(r)[3] for r in range(7))
        assert tot == 1269
        s, e1, t1 = cb.seq(3, 1)
        assert s >= 0 and e1 > 0
    finally:
        cb.close()
