#!/usr/bin/env python
"""bench.py -- exact triangle counting on B200: oriented edges/s + HBM roofline.

Workload (BASELINE.json configs[1], the config the metric is quoted on):
C2 = preferential attachment PA(n=1e7, 20 attachments/vertex), i.e. the
reference's gen_pa(1e7, 40, seed=7) edge stream (io.hpp:129-162), ~2e8
undirected edges, generated bit-identically on the host (synthetic data).

A step = one pass of the hot path over the graph resident in HBM:
degree-ordered orientation (effective_adjacency, effective.hpp:37-52) +
NodeIteratorN intersection over every oriented edge (sequential.hpp:74-91).
value = oriented edges (m) processed per second by the whole job.
At N GPUs (torchrun), rank i runs the AOP rank body for core i of the
DPD cost-balanced plan (partition.hpp:116-141, engines.hpp:38-54) and the
count is summed with one NCCL all-reduce; total work is fixed (strong scaling).

e2e = the same metric through the reference-facing C ABI with HOST buffers:
tg_count_from_csr (pinned host CSR -> HBM in vertex chunks, each chunk
oriented on arrival and every apex counted as soon as all its lists are
resident; 8-byte result back) per step, timed with the host clock around
synchronised calls.

--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified trigraph headers) on all host cores: the AOP rank bodies
build_overlap_partition + aop_count on std::threads over a rotating sample
of a 256-part DPD plan of the same graph.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "exact triangle count: oriented edges/sec + achieved HBM GB/s at 1/2/4/8 B200"
UNIT = "oriented edges/s"
WORKLOAD = "C2: PA(n=1e7, d=20 attachments) = gen_pa(1e7, 40, seed=7), ~2e8 edges"
N_NODES, PA_D, SEED = 10_000_000, 40, 7


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ inputs


def make_graph(device: int):
    from paper_1706_05151_b200 import trigraph as T

    t0 = time.time()
    pairs = T.gen_pa(N_NODES, PA_D, SEED)
    t1 = time.time()
    g = T.build_graph(pairs, N_NODES, device=device)
    t2 = time.time()
    log(f"[bench] gen_pa {t1 - t0:.1f}s, device build_graph {t2 - t1:.2f}s, "
        f"n={g.num_nodes()} m={g.num_edges()}")
    return g, pairs


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def profile_traffic():
    """Per-launch DRAM bytes of the intersection pass from the committed
    ncu --set full capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_intersect.json")
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_pass")
    except Exception:
        return None


# ------------------------------------------------------------------ CPU legs


def ref_setup(pairs):
    """Reference Graph from the oracle's CSR build (input prep, untimed),
    then the reference's compute_order + effective_adjacency (untimed)."""
    from oracle import binding as O

    t0 = time.time()
    csr = O.build_graph(pairs, N_NODES)
    if O.ref_available():
        R = O.RefGraph.from_csr(csr)
        O.ref().ref_prepare(R.h)
        kind = "reference"
    else:
        R, kind = None, "port"
    log(f"[bench] CPU baseline setup ({kind}) {time.time() - t0:.1f}s")
    return O, csr, R, kind


def ref_sample(O, R, csr, parts, which, threads):
    import numpy as np

    if R is not None:
        w = np.ascontiguousarray(which, dtype=np.uint64)
        e = np.zeros(1, np.uint64)
        t = np.zeros(1, np.uint64)
        dt = O.ref().ref_aop_sample(R.h, parts, C.c_void_p(w.ctypes.data), len(w), threads,
                                    C.c_void_p(e.ctypes.data), C.c_void_p(t.ctypes.data))
        return float(dt), int(e[0]), int(t[0])
    # oracle port (only when oracle/_ref is absent): NodeIteratorN over the
    # apexes of the sampled DPD parts, one thread
    eoff, eff, b = _port_state(O, csr, parts)
    t0 = time.time()
    edges = tris = 0
    for i in which:
        lo, hi = int(b[i]), int(b[i + 1])
        tris += int(O.lib().orc_count_range(csr.n, C.c_void_p(eoff.ctypes.data),
                                            C.c_void_p(eff.ctypes.data), lo, hi))
        edges += int(eoff[hi] - eoff[lo])
    return time.time() - t0, edges, tris


_PORT = {}


def _port_state(O, csr, parts):
    if "eoff" not in _PORT:
        _PORT["eoff"], _PORT["eff"] = O.effective(csr)
        f, _ = O.node_costs(csr, "DPD")
        _PORT["b"] = O.compute_boundaries(f, parts)
    return _PORT["eoff"], _PORT["eff"], _PORT["b"]


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU arm
    from paper_1706_05151_b200 import trigraph as T

    pairs = T.gen_pa(N_NODES, PA_D, SEED)
    O, csr, R, kind = ref_setup(pairs)
    del pairs
    threads = cpu_threads()
    parts = 256
    budget = float(os.environ.get("TG_REF_BUDGET_S", "150"))
    # calibrate: one batch of `threads` parts
    order = [(k * 97) % parts for k in range(parts)]  # rotating strided sample
    pos = 0

    def take(k):
        nonlocal pos
        w = [order[(pos + i) % parts] for i in range(k)]
        pos = (pos + k) % parts
        return w

    if R is None:
        threads = 1
    dt, e, t = ref_sample(O, R, csr, parts, take(threads), threads)  # one batch
    steps_total = args.steps + args.warmup
    per_step = max(1, int((budget / steps_total) / max(dt, 1e-3))) * threads
    per_step = min(per_step, parts)
    for _ in range(args.warmup):
        ref_sample(O, R, csr, parts, take(per_step), threads)
    tt = ee = 0
    for _ in range(args.steps):
        dt, e, t = ref_sample(O, R, csr, parts, take(per_step), threads)
        tt += dt
        ee += e
    value = ee / tt if tt > 0 else 0.0
    sample = (f"{per_step} of 256 DPD parts per step (rotating), build_overlap_partition + "
              f"aop_count on {threads} std::threads; order+orientation precomputed untimed")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1000 * tt / max(args.steps, 1),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
           "data": "synthetic (seeded gen_pa stream)", "impl": "reference",
           "config": {"workload": WORKLOAD, "parallelism": f"cpu{threads}"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ GPU arm


def run_ours(args):
    import numpy as np
    import torch

    from paper_1706_05151_b200 import trigraph as T
    from paper_1706_05151_b200._lib import check, lib

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = lib()
    g, pairs = make_graph(local)
    n, m = g.num_nodes(), g.num_edges()
    W = T.ordering_cost(g)
    # a dedicated (non-default) stream shared by the library and torch, so the
    # CUDA events below bracket exactly the library's launches
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    check(L.tg_set_stream(g._h, C.c_void_p(stream.cuda_stream)))
    d_total = torch.zeros(1, dtype=torch.int64, device="cuda")
    dptr = C.c_void_p(d_total.data_ptr())
    want = None

    if ws > 1:
        plan = T.compute_boundaries(g, T.CostKind.Dpd, ws).boundaries
        bptr = C.c_void_p(plan.ctypes.data)

        def step():
            check(L.tg_orient_device(g._h))
            ev_mid.append(torch.cuda.Event(enable_timing=True))
            ev_mid[-1].record(stream)
            d_total.zero_()
            check(L.tg_aop_rank_device(g._h, bptr, ws, rank, dptr))
            dist.all_reduce(d_total)
    else:
        def step():
            check(L.tg_orient_device(g._h))
            ev_mid.append(torch.cuda.Event(enable_timing=True))
            ev_mid[-1].record(stream)
            check(L.tg_count_device(g._h, dptr))

    ev_mid = []
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    T_total = int(d_total.item())
    ev_mid.clear()
    # timed region: inputs (1.7 GB CSR + 0.8 GB oriented CSR) exceed the
    # 126 MB L2, so no explicit flush between steps
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    launches0 = L.tg_kernel_launches()
    starts, ends = [], []
    for _ in range(args.steps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        step()
        e.record(stream)
        starts.append(s)
        ends.append(e)
    torch.cuda.synchronize()
    launches = L.tg_kernel_launches() - launches0
    clk = clocks.stop()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    isect_ms = [mid.elapsed_time(e) for mid, e in zip(ev_mid, ends)]
    tot_ms = starts[0].elapsed_time(ends[-1])
    if dist:
        t = torch.tensor([tot_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        dist.barrier()
    ms_per_step = tot_ms / args.steps
    value = m / (ms_per_step / 1e3)
    isect_avg = sum(isect_ms) / len(isect_ms)
    orient_avg = sum(a - b for a, b in zip(step_ms, isect_ms)) / len(step_ms)
    isect_max = isect_avg  # slowest rank's intersection pass (kernel-only metric)
    if dist:
        t = torch.tensor([isect_avg], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        isect_max = float(t.item())

    # ---- e2e through the public API with host buffers (N = 1: the streamed
    # tg_count_from_csr; N > 1: distributed.count_aop_from_host_csr)
    off_h, adj_h = g.csr()
    off_p = torch.from_numpy(off_h.view(np.int64)).pin_memory()
    adj_p = torch.from_numpy(adj_h.view(np.int32)).pin_memory()
    del off_h, adj_h
    h2d = off_p.numel() * 8 + adj_p.numel() * 4
    e2e_t = []
    for i in range(args.e2e_warmup + args.e2e_steps):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if dist:
            # each rank uploads 1/N of the host CSR, NCCL all-gathers the rest
            # over NVLink, counts its AOP core; one all-reduce of T (8 bytes
            # back to the host)
            from paper_1706_05151_b200.distributed import count_aop_from_host_csr
            cnt = count_aop_from_host_csr(n, off_p, adj_p, plan, torch.device("cuda", local))
        else:
            # one reference-facing call: Graph(n, offsets, adj) + by_degree
            # orientation + count, the upload streamed under the compute
            c64 = C.c_uint64()
            check(L.tg_count_from_csr(local, n, C.c_void_p(off_p.data_ptr()),
                                      C.c_void_p(adj_p.data_ptr()), C.byref(c64)))
            cnt = c64.value
        t1 = time.perf_counter()
        assert cnt == T_total
        dt = t1 - t0
        if dist:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        if i >= args.e2e_warmup:
            e2e_t.append(dt)
    e2e_s = sum(e2e_t) / len(e2e_t)
    # the PCIe floor on this box: the bare pinned H2D of the same bytes
    d_off = torch.empty_like(off_p, device="cuda")
    d_adj = torch.empty_like(adj_p, device="cuda")
    h2d_t = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d_off.copy_(off_p, non_blocking=True)
        d_adj.copy_(adj_p, non_blocking=True)
        torch.cuda.synchronize()
        h2d_t.append(time.perf_counter() - t0)
    del d_off, d_adj
    h2d_floor = min(h2d_t)

    if rank != 0:
        return
    # ---- roofline of the intersection pass: 4 bytes x W algorithmic elements
    peak, peak_kind = measured_peak()
    if ws > 1:
        w_rank = W / ws  # DPD balances W across ranks (max/mean ~1.0 at p=8)
    else:
        w_rank = W
    achieved = 4.0 * w_rank / (isect_avg / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": profile_traffic(),
                "kernel": "intersect pass (k_intersect_quad + k_intersect_ctaq)",
                "algorithmic_bytes_per_pass": 4 * w_rank, "W": W,
                "pass_ms": isect_avg, "orient_ms": orient_avg, "peak_source": peak_kind}

    # ---- CPU baseline (reference on the host cores), bounded sample
    cpu = None
    if ws == 1 and not args.no_cpu:
        O, csr, R, kind = ref_setup(pairs)
        threads = cpu_threads() if R is not None else 1
        parts = 256
        which = [(k * 97) % parts for k in range(min(parts, max(threads, args.cpu_parts)))]
        dt, e, t = ref_sample(O, R, csr, parts, which, threads)
        cpu = {"value": e / dt if dt > 0 else None, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": f"{len(which)} of 256 DPD-plan AOP parts of the same graph "
                         f"({e} oriented edges): build_overlap_partition + aop_count on "
                         f"{threads} std::threads, {dt:.1f}s"}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded gen_pa stream, bit-identical to the reference generator)",
        "config": {"workload": WORKLOAD, "n": n, "m": m, "triangles": T_total,
                   "parallelism": f"aop{ws}" if ws > 1 else "single",
                   "step": "orientation + intersection over the HBM-resident graph",
                   "l2": "inputs (1.7 GB CSR, 0.8 GB oriented CSR) > 126 MB L2; no flush"},
        "intersections_per_s": value,
        # oriented edges / intersection time (kernel only, the
        # orientation excluded), slowest rank at N > 1
        "kernel_only": {"edges_per_s": m / (isect_max / 1e3), "intersect_ms": isect_max,
                        "orient_ms": orient_avg},
        "elements_per_s": W / (ms_per_step / 1e3) / ws * ws,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": m / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 8 * ws, "ms_per_step": 1e3 * e2e_s,
                "step_ms": [round(1e3 * x, 3) for x in e2e_t],
                "h2d_only_ms": 1e3 * h2d_floor,  # bare copy of the same bytes (not the metric)
                "path": ("tg_count_from_csr(pinned host CSR): chunked H2D overlapped with "
                         "orientation and the count of every apex whose lists arrived"
                         if ws == 1 else
                         "per rank: 1/N of the pinned host CSR uploaded, NCCL all-gather of "
                         "the rest over NVLink, tg_count_from_csr_range (its DPD core), "
                         "NCCL all-reduce of the 8-byte counts; max over ranks")},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-warmup", type=int, default=2)
    ap.add_argument("--cpu-parts", type=int, default=32)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
