"""Full-size goldens for BASELINE.json's configs (SURVEY §8(c) "full-scale
goldens") -- TEST INFRASTRUCTURE ONLY.

    python tests/golden/make_golden_full.py C3 C4 C5      # oracle records
    python tests/golden/make_golden_full.py C2 --pin-ref  # + the reference's own C2 T_v / C_v

Every number comes from the oracle (oracle/fullsize.c + oracle.c), run on the
config's seeded pairs made by the oracle's generators -- never from device
arrays: build_graph (graph.hpp:58-85) -> compute_order(ByDegree)
(order.hpp:95-104) -> effective_adjacency (effective.hpp:37-52) ->
count_node_iterator_n with NodeTallySink / ListSink (sequential.hpp:24-46,
74-91) on all host threads, plus the p=8 DPD plan (partition.hpp:60-69,
116-141) with the AOP / ANOP-surrogate per-rank counts and surrogate
messages (engines.hpp:38-76, 146-198) and C_v (engines.hpp:258-267).

The full-size oracle is itself pinned: against oracle/_ref (the unmodified
reference) on small graphs (tests/test_oracle_full.py) and, here, at C1/C2
against the reference-made records already in reference_full.json (CSR
digests, count, W) and -- with --pin-ref -- the reference's own C2
clustering_coefficients (T_v / C_v digests).

Records are merged into tests/golden/reference_full.json under
"<config>_oracle" (C1/C2 keep their reference-made records).
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

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_full.json")
P = 8


def sha(a) -> str:
    h = hashlib.sha256()
    mv = memoryview(np.ascontiguousarray(a)).cast("B")
    step = 1 << 30
    for i in range(0, len(mv), step):
        h.update(mv[i:i + step])
    return h.hexdigest()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def record(name: str, threads: int) -> dict:
    kind, p = B.CONFIGS[name]
    t0 = time.time()
    pairs, E, n0 = B.gen_pairs(kind, p, threads)
    rec = {"config": name, "generator": kind, "params": p, "pairs": E,
           "pairs_sha256": sha(pairs.array)}
    log(name, "gen", round(time.time() - t0, 1), "s")
    t = time.time()
    g = B.FullGraph(pairs, E, n0, threads)
    rec.update(n=g.n, m=g.m, offsets_sha256=sha(g.off), adj_sha256=sha(g.adj),
               eff_offsets_sha256=sha(g.eoff), eff_sha256=sha(g.eff),
               ordering_cost=g.ordering_cost(), h_max=int(np.diff(g.eoff).max()),
               d_max=int(np.diff(g.off).max()))
    log(name, "build+orient", round(time.time() - t, 1), "s", "n", g.n, "m", g.m)
    t = time.time()
    b = g.dpd_boundaries(P)
    r = g.count(b, tally=True, digest=True)
    rec["count_seconds"] = round(time.time() - t, 1)
    log(name, "count", rec["count_seconds"], "s", "T", r["total"])
    sent, recv = g.surrogate_messages(b)
    cc = g.clustering(r["tally"])
    rec.update(count=r["total"], node_counts_sha256=sha(r["tally"]), cc_sha256=sha(cc),
               listing_digest=r["digest"], dpd8_boundaries=b.tolist(), aop8_triangles=r["apex"],
               surrogate8_triangles=r["mid"], surrogate8_data_sent=sent,
               surrogate8_data_recv=recv, threads=threads,
               wall_seconds=round(time.time() - t0, 1))
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--pin-ref", action="store_true",
                    help="C2: also record the reference's own T_v / C_v digests")
    a = ap.parse_args()
    threads = a.threads or B.threads_default()
    with open(OUT) as f:
        fx = json.load(f)
    for name in a.configs:
        rec = record(name, threads)
        ref = fx.get(name)
        if ref:  # pinned by the reference's own full-size record
            for k in ("n", "m", "count", "ordering_cost", "offsets_sha256", "adj_sha256"):
                if k in ref:
                    assert ref[k] == rec[k], (name, k, ref[k], rec[k])
            log(name, "matches the reference record")
        if name == "C2" and a.pin_ref and B.ref_available():
            t = time.time()
            R = B.ref_fixture("gen_pa", 10_000_000, 40, 7)
            tv, cc = R.clustering("seq", 1)
            fx["C2"]["node_counts_sha256"] = sha(tv)
            fx["C2"]["cc_sha256"] = sha(cc)
            assert fx["C2"]["node_counts_sha256"] == rec["node_counts_sha256"]
            assert fx["C2"]["cc_sha256"] == rec["cc_sha256"]
            log("C2 reference clustering_coefficients", round(time.time() - t, 1), "s: match")
        fx[name + "_oracle"] = rec
        with open(OUT, "w") as f:
            json.dump(fx, f, indent=1, sort_keys=True)
        log("wrote", name)


if __name__ == "__main__":
    main()
