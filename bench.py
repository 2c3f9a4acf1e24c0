#!/usr/bin/env python
"""bench.py -- exact triangle counting on B200: oriented edges/s + HBM roofline.

Workload (--config, default C5): BASELINE.json's largest configuration that
fits one B200, C5 = preferential attachment PA(n=1e8, 20 attachments/vertex),
the reference generator's own edge stream gen_pa(1e8, 40, seed=7)
(io.hpp:129-162), ~2e9 undirected edges, generated bit-identically on the
host (synthetic data; the other configs C1-C4 are selectable and are parity
cases in tests/).

A step = one pass of the hot path over the graph resident in HBM:
degree-ordered orientation (effective_adjacency, effective.hpp:37-52) +
NodeIteratorN intersection over every oriented edge (sequential.hpp:74-91).
value = oriented edges (m) processed per second by the whole job.
At N GPUs (torchrun), the step is csrc/comm.cu's AOP step: rank i orients
its 1/N of the rows, the oriented rows are broadcast in rank order over
NVLink (NCCL) while rank i counts the apexes of core i of the DPD
cost-balanced plan (partition.hpp:116-141, engines.hpp:38-54) whose lists
arrived, and T is summed with one all-reduce; total work is fixed (strong
scaling).

e2e = the same metric through the reference-facing C ABI with HOST buffers:
tg_count_from_csr (pinned host CSR -> HBM in vertex chunks, each chunk
oriented on arrival and every apex counted as soon as all its lists are
resident; 8-byte result back) per step, timed with the host clock around
synchronised calls.

cpu_baseline / --impl reference: the reference's own code
(oracle/_ref: the unmodified trigraph headers) on the host cores, on the
oracle-built EffectiveAdjacency of the same graph (setup, untimed):
  * all cores: the reference AOP through its public API with p = nproc --
    each std::thread runs build_overlap_partition (partition.hpp:171-206,
    timed separately) then aop_count (engines.hpp:38-54, the counting phase,
    the value) on a rotating cost-balanced sub-range of its DPD core;
  * one thread: count_node_iterator_n's loop (sequential.hpp:74-91, the
    reference's intersect_visit) over the same sub-ranges.
The reference arm never loads libtrigraph_b200.so: its input is made by the
oracle's generators (oracle/fullsize.c).
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
CONFIGS = {  # BASELINE.json configs[0..4]
    "C1": ("gnm", dict(n=100_000, m=1_000_000, seed=1),
           "C1: Erdos-Renyi G(n=1e5, m=1e6), seed 1"),
    "C2": ("pa", dict(n=10_000_000, d=40, seed=7),
           "C2: PA(n=1e7, d=20 attachments) = gen_pa(1e7, 40, seed=7), ~2e8 edges"),
    "C3": ("rmat", dict(scale=24, ef=16, a=0.57, b=0.19, c=0.19, seed=1),
           "C3: R-MAT scale 24, edge factor 16, (0.57,0.19,0.19,0.05), seed 1, ~2.6e8 edges"),
    "C4": ("ws", dict(n=50_000_000, k=20, beta=0.1, seed=1),
           "C4: Watts-Strogatz n=5e7, k=20, beta=0.1, seed 1, ~5e8 edges"),
    "C5": ("pa", dict(n=100_000_000, d=40, seed=7),
           "C5: PA(n=1e8, d=20 attachments) = gen_pa(1e8, 40, seed=7), ~2e9 edges "
           "(largest BASELINE config; fits one B200)"),
}
DEFAULT_CONFIG = "C5"
TRAFFIC_PROFILES = {  # ncu --set full captures of the intersection pass (profiles/)
    "C2": "profiles/ncu_intersect.json",
    "C5": "profiles/ncu_intersect_C5.json",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


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


def product_pairs(cfg: str):
    """The config's pairs from the library's host generators (the GPU arm)."""
    from paper_1706_05151_b200 import trigraph as T

    kind, p, _ = CONFIGS[cfg]
    if kind == "pa":
        return T.gen_pa(p["n"], p["d"], p["seed"]), p["n"]
    if kind == "gnm":
        return T.gen_gnm(p["n"], p["m"], p["seed"]), p["n"]
    if kind == "rmat":
        return T.gen_rmat(p["scale"], p["ef"], p["a"], p["b"], p["c"], p["seed"]), 1 << p["scale"]
    if kind == "ws":
        return T.gen_ws(p["n"], p["k"], p["beta"], p["seed"]), p["n"]
    raise ValueError(kind)


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def profile_traffic(cfg: str):
    """(bytes per intersection pass, source) from the committed ncu --set
    full capture of this config (dram__bytes_read.sum + write.sum), or
    (None, reason)."""
    rel = TRAFFIC_PROFILES.get(cfg)
    if not rel:
        return None, f"no ncu capture committed for {cfg}"
    try:
        with open(os.path.join(ROOT, rel)) as f:
            return json.load(f).get("dram_bytes_per_pass"), rel + " (ncu --set full, per pass)"
    except Exception:
        return None, f"{rel} missing"


# ------------------------------------------------------------------ CPU legs


class CpuBaseline:
    """The reference's own counting code on the host cores (oracle/_ref),
    over the oracle-built EffectiveAdjacency of the config's graph."""

    def __init__(self, pairs_buf, E: int, n: int, threads: int):
        import numpy as np

        from oracle import binding as O

        self.O, self.np = O, np
        if not O.ref_available():
            raise RuntimeError("oracle/_ref not built (make -C oracle with /root/reference)")
        t0 = time.time()
        self.threads = threads
        g = O.FullGraph(pairs_buf, E, n, threads)  # consumes pairs_buf
        self.n, self.m = g.n, g.m
        self.h = O.ref().ref_eff_from_arrays(g.n, C.c_void_p(g.eoff.ctypes.data),
                                             C.c_void_p(g.eff.ctypes.data))
        # DPD plan with p = nproc: node_costs (oracle, pinned) -> the
        # reference's compute_boundaries (partition.hpp:116-141)
        f = np.zeros(max(g.n, 1), dtype=np.uint64)
        pre = np.zeros(max(g.n, 1), dtype=np.uint64)
        O.lib().orc_node_costs(g.n, C.c_void_p(g.off.ctypes.data), C.c_void_p(g.adj.ctypes.data),
                               C.c_void_p(g.eoff.ctypes.data), C.c_void_p(g.eff.ctypes.data),
                               O.COSTS["DPD"], C.c_void_p(f.ctypes.data),
                               C.c_void_p(pre.ctypes.data))
        self.b = np.zeros(threads + 1, dtype=np.uint32)
        O.ref().ref_compute_boundaries(C.c_void_p(f.ctypes.data), g.n, threads,
                                       C.c_void_p(self.b.ctypes.data))
        self.prefix = pre[: g.n]
        del g, f
        self.R = 256
        self.setup_s = time.time() - t0
        log(f"[cpu] setup {self.setup_s:.1f}s (oracle build + orientation, DPD plan p={threads})")

    def close(self):
        if self.h:
            self.O.ref().ref_eff_free(self.h)
            self.h = None

    def ranges(self, r: int):
        """Sub-range r of R of every core, equal DPD cost: 2p uint32."""
        np, pre, b = self.np, self.prefix, self.b
        out = np.zeros(2 * self.threads, dtype=np.uint32)
        for i in range(self.threads):
            lo, hi = int(b[i]), int(b[i + 1])
            if hi <= lo:
                out[2 * i] = out[2 * i + 1] = lo
                continue
            c0 = int(pre[lo - 1]) if lo else 0
            c1 = int(pre[hi - 1])
            a = c0 + (c1 - c0) * r // self.R
            z = c0 + (c1 - c0) * (r + 1) // self.R
            s = int(np.searchsorted(pre[lo:hi], a, side="right")) + lo if r else lo
            e = int(np.searchsorted(pre[lo:hi], z, side="right")) + lo if r + 1 < self.R else hi
            out[2 * i], out[2 * i + 1] = s, max(s, e)
        return out

    def aop(self, r: int):
        """One all-core sample: (count_s, build_s, edges, triangles, stored)."""
        s = self.ranges(r % self.R)
        tb = C.c_double()
        e, t, st = C.c_uint64(), C.c_uint64(), C.c_uint64()
        dt = self.O.ref().ref_aop_threads(self.h, C.c_void_p(s.ctypes.data), self.threads,
                                          C.byref(tb), C.byref(e), C.byref(t), C.byref(st))
        return float(dt), tb.value, e.value, t.value, st.value

    def seq(self, r: int, core: int):
        """One 1-thread sample, sub-range r of one core: (seconds, edges,
        triangles)."""
        s = self.ranges(r % self.R)[2 * core: 2 * core + 2].copy()
        e, t = C.c_uint64(), C.c_uint64()
        dt = self.O.ref().ref_seq_sample(self.h, C.c_void_p(s.ctypes.data), 1,
                                         C.byref(e), C.byref(t))
        return float(dt), e.value, t.value

    def calibrate(self, target_s: float):
        """Pick R (sub-ranges per core) so one all-core sample -- partition
        building plus counting -- takes ~target_s seconds."""
        self.R = 1024
        dt, tb, _, _, _ = self.aop(0)
        full = (dt + tb) * self.R
        self.R = max(1, min(1 << 20, int(round(full / max(target_s, 1e-3)))))
        log(f"[cpu] calibration: full all-core build+count ~{full:.0f}s -> R={self.R}")

    def report(self, samples: int = 3, seq_budget_s: float = 8.0):
        rates = [self.aop(17 * k + 1) for k in range(samples)]
        ct = sum(x[0] for x in rates)
        bt = sum(x[1] for x in rates)
        ed = sum(x[2] for x in rates)
        st = sum(x[4] for x in rates)
        s_t = s_e = 0
        k = 0
        while s_t < seq_budget_s and k < 4 * self.threads:
            dt, e, _ = self.seq(31 * k + 5, k % self.threads)
            s_t += dt
            s_e += e
            k += 1
        return {"value": ed / ct if ct > 0 else None, "unit": UNIT, "cores": self.threads,
                "kind": "reference",
                "sample": (f"{samples} samples x {self.threads} std::threads (p = nproc DPD "
                           f"cores, each thread 1/{self.R} of its core's cost, rotating): "
                           f"reference aop_count over build_overlap_partition, "
                           f"{ed} oriented edges counted in {ct:.2f}s"),
                "counting_s": ct, "partition_build_s": bt,
                "partition_stored_entries": st,
                "one_thread": {"value": s_e / s_t if s_t > 0 else None, "unit": UNIT,
                               "cores": 1,
                               "sample": f"count_node_iterator_n loop over {k} sub-ranges "
                                         f"(1/{self.R} of a core each; {s_e} oriented edges, "
                                         f"{s_t:.2f}s)"},
                "setup_s": self.setup_s}


def oracle_pairs(cfg: str, threads: int):
    from oracle import binding as O

    kind, p, _ = CONFIGS[cfg]
    return O.gen_pairs(kind, p, threads)


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU arm
    threads = cpu_threads()
    t0 = time.time()
    buf, E, n = oracle_pairs(args.config, threads)
    log(f"[ref] oracle generator {time.time() - t0:.1f}s, {E} pairs")
    cb = CpuBaseline(buf, E, n, threads)
    cb.calibrate(args.ref_step_s)
    for k in range(args.warmup):
        cb.aop(k)
    ct = bt = 0.0
    ed = 0
    for k in range(args.steps):
        dt, tb, e, _, _ = cb.aop(args.warmup + k)
        ct += dt
        bt += tb
        ed += e
    value = ed / ct if ct > 0 else 0.0
    one = cb.report(samples=1, seq_budget_s=args.ref_seq_s)["one_thread"]
    cb.close()
    sample = (f"per step: {threads} std::threads, each the reference build_overlap_partition "
              f"(timed apart: {bt:.2f}s over the run) + aop_count (the counting phase, timed) "
              f"on 1/{cb.R} of its p = {threads} DPD core, rotating")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1000 * ct / max(args.steps, 1),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
           "data": "synthetic (seeded generator of the config, oracle/fullsize.c)",
           "impl": "reference",
           "config": {"workload": CONFIGS[args.config][2], "n": cb.n, "m": cb.m,
                      "parallelism": f"cpu{threads}"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                            "sample": sample, "partition_build_s": bt, "counting_s": ct,
                            "one_thread": one, "setup_s": cb.setup_s},
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
    t0 = time.time()
    pairs, n0 = product_pairs(args.config)
    E_pairs = int(pairs.shape[0])
    t1 = time.time()
    # build_graph on the device from device-resident pairs, timed with CUDA
    # events (graph.hpp:58-85: radix sort + unique + offsets)
    d_pairs = torch.from_numpy(pairs.view(np.int32)).to(f"cuda:{local}")
    torch.cuda.synchronize()
    eb0, eb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eb0.record()
    g = T.build_graph_from_pointer(d_pairs.data_ptr(), pairs.shape[0], n0, device=local)
    eb1.record()
    torch.cuda.synchronize()
    build_ms = eb0.elapsed_time(eb1)
    del d_pairs
    torch.cuda.empty_cache()
    n, m = g.num_nodes(), g.num_edges()
    log(f"[bench] {args.config}: host generator {t1 - t0:.1f}s, device build_graph "
        f"{build_ms:.1f} ms, n={n} m={m}")
    W = T.ordering_cost(g)
    # a dedicated (non-default) stream shared by the library and torch, so the
    # CUDA events below bracket exactly the library's launches
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    check(L.tg_set_stream(g._h, C.c_void_p(stream.cuda_stream)))
    d_total = torch.zeros(1, dtype=torch.int64, device="cuda")
    dptr = C.c_void_p(d_total.data_ptr())

    use_comm = ws > 1 or args.force_comm
    if use_comm:
        # one NCCL communicator over the job (csrc/comm.cu): each rank orients
        # its 1/N of the rows, the oriented rows are broadcast in rank order
        # over NVLink while each rank counts the apexes of its DPD core whose
        # lists arrived; one all-reduce of T
        from paper_1706_05151_b200 import comm as M

        comm = (M.Comm.from_process_group(local) if ws > 1
                else M.Comm.init(local, 1, 0, M.Comm.unique_id()))
        plan = M.run_engine_comm(g, comm, T.EngineConfig(engine=T.EngineKind.Aop)).boundaries

        def step():
            M.aop_step_comm(g, comm, plan, d_total.data_ptr())
            ev_mid.append(None)
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
    # timed region: the inputs (CSR + oriented CSR) exceed the 126 MB L2 for
    # C2-C5, so no explicit flush between steps
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
    # (the N-GPU step overlaps its count with the transfers: no separate
    # intersection time -- the step is the figure)
    isect_ms = step_ms if use_comm else [mid.elapsed_time(e) for mid, e in zip(ev_mid, ends)]
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
    # tg_count_from_csr; N > 1: each rank uploads its rows + the degrees,
    # tg_graph_from_rows, then the AOP step across the ranks)
    off_h, adj_h = g.csr()
    if use_comm:
        rows = M.split_rows(off_h, ws)
        lo, hi = int(rows[rank]), int(rows[rank + 1])
        deg_p = torch.from_numpy(np.diff(off_h).astype(np.uint32).view(np.int32)).pin_memory()
        off_p = torch.from_numpy(off_h[lo:hi + 1].view(np.int64)).pin_memory()
        adj_p = torch.from_numpy(adj_h[off_h[lo]:off_h[hi]].view(np.int32)).pin_memory()
        h2d = off_p.numel() * 8 + adj_p.numel() * 4 + deg_p.numel() * 4
    else:
        off_p = torch.from_numpy(off_h.view(np.int64)).pin_memory()
        adj_p = torch.from_numpy(adj_h.view(np.int32)).pin_memory()
        h2d = off_p.numel() * 8 + adj_p.numel() * 4
    del off_h, adj_h
    e2e_t = []
    for i in range(args.e2e_warmup + args.e2e_steps):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if use_comm:
            gr = M.graph_from_rows(n, lo, hi, off_p.numpy().view(np.uint64),
                                   adj_p.numpy().view(np.uint32), deg_p.numpy().view(np.uint32),
                                   device=local)
            check(L.tg_set_stream(gr._h, C.c_void_p(stream.cuda_stream)))
            M.aop_step_comm(gr, comm, plan, d_total.data_ptr())
            cnt = int(d_total.item())
            gr.close()
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
    del d_off, d_adj, off_p, adj_p
    h2d_floor = min(h2d_t)

    if rank != 0:
        return
    # ---- roofline of the intersection pass: 4 bytes x W algorithmic elements
    peak, peak_kind = measured_peak()
    w_rank = W / ws if ws > 1 else W  # DPD balances W across ranks
    achieved = 4.0 * w_rank / (isect_avg / 1e3) / 1e9  # (N > 1: over the whole step)
    traffic, traffic_src = profile_traffic(args.config)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "dram_gbs": (traffic / (isect_avg / 1e3) / 1e9) if traffic else None,
                "kernel": "intersection pass (k_intersect_slab on the PA configs C2 / C5; the quad / "
                          "group / window / CTA kernels otherwise)",
                "algorithmic_bytes_per_pass": 4 * w_rank, "W": W,
                "pass_ms": isect_avg, "orient_ms": orient_avg, "peak_source": peak_kind}

    # ---- CPU baseline (the reference's counting code on the host cores),
    # bounded sample of the same graph
    cpu = None
    if ws == 1 and not args.no_cpu:
        from oracle import binding as O

        threads = cpu_threads()
        buf = O.HostBuf.from_array(pairs)
        del pairs
        cb = CpuBaseline(buf, E_pairs, n0, threads)
        cb.calibrate(args.cpu_step_s)
        cpu = cb.report(samples=args.cpu_samples, seq_budget_s=args.cpu_seq_s)
        cb.close()
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded generator of the config, bit-identical to the reference "
                "gen_pa stream / the oracle's generators)",
        "config": {"workload": CONFIGS[args.config][2], "n": n, "m": m, "triangles": T_total,
                   "parallelism": f"aop{ws}" if use_comm else "single",
                   "step": "orientation + intersection over the HBM-resident graph",
                   "l2": "inputs (CSR + oriented CSR) > 126 MB L2; no flush"},
        "intersections_per_s": value,
        # oriented edges / intersection time (kernel only, the
        # orientation excluded), slowest rank at N > 1
        "kernel_only": ({"edges_per_s": m / (isect_max / 1e3), "intersect_ms": isect_max,
                         "orient_ms": orient_avg} if not use_comm else None),
        "elements_per_s": W / (ms_per_step / 1e3),
        "build_graph": {"ms": build_ms, "pairs": E_pairs,
                        "path": "device pairs -> CSR (CUB radix sort + unique), CUDA events"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": m / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 8 * ws, "ms_per_step": 1e3 * e2e_s,
                "step_ms": [round(1e3 * x, 3) for x in e2e_t],
                "h2d_only_ms": 1e3 * h2d_floor,  # bare copy of the same bytes (not the metric)
                "path": ("tg_count_from_csr(pinned host CSR): chunked H2D overlapped with "
                         "orientation and the count of every apex whose lists arrived"
                         if not use_comm else
                         "per rank: its rows of the pinned host CSR + the degrees uploaded "
                         "(tg_graph_from_rows), tg_aop_step_comm (rows oriented, oriented rows "
                         "broadcast over NVLink, core counted as lists arrive, all-reduce of "
                         "T); max over ranks")},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    # one JSON line on stdout: NCCL's own messages (its version banner) go to stderr
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-warmup", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--force-comm", action="store_true",
                    help="the N-GPU step (csrc/comm.cu) even at N = 1 (tests)")
    ap.add_argument("--cpu-samples", type=int, default=3)
    ap.add_argument("--cpu-step-s", type=float, default=3.0,
                    help="all-core build + count seconds per CPU-baseline sample")
    ap.add_argument("--cpu-seq-s", type=float, default=6.0)
    ap.add_argument("--ref-step-s", type=float, default=2.0,
                    help="--impl reference: all-core build + count seconds per step")
    ap.add_argument("--ref-seq-s", type=float, default=6.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
