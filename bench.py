#!/usr/bin/env python3
"""Benchmark driver (contract: one JSON line from rank 0).

Headline workload (BASELINE.json configs[1]): GAP PageRank on a directed R-MAT
scale-22 graph (edge factor 16, a/b/c = .57/.19/.19, duplicates and self-loops
removed), fp32 ranks, damping 0.85, tol 1e-4, itermax 100.  Metric:
edges/s/iter = nnz(AT) * iterations / seconds per run.  One "step" = one full
pagerank_gap run to convergence on the resident graph.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload pagerank|bfs|bfs64|tc|sssp|bc] [--scale S]

`value` is device-timed (CUDA events on the library's stream, L2 flushed
between steps, graph resident in HBM).  `e2e` goes through the C ABI with host
buffers: H2D of the CSR from pinned memory, graph_new + the basic call (which
builds AT and the degree cache on the device) and D2H of the ranks, timed on
the host around the synchronous call.  `--impl reference` times the reference
library itself (oracle/_ref, built from /root/reference) on the box's CPU.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PageRank edges/s/iter at R-MAT scale 22 (BASELINE: BFS GTEPS & PageRank " \
         "edges/s/iter at R-MAT scale 22-24; % of HBM roofline)"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi streaming at 50 ms (-lms) for the whole timed region; clocks,
    power and throttle reasons are summarised into the JSON line."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.15)  # let the first sample land before the timed region
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.06)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 4 + k and r[4 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---------------------------------------------------------------- distributed
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def force_sharded():
    """GBX_BENCH_SHARDED=1 under torchrun --nproc-per-node 1: the N>1 code path
    (NCCL group, sharded driver) on one GPU, for testing it end to end."""
    return os.environ.get("GBX_BENCH_SHARDED") == "1" and "MASTER_ADDR" in os.environ


def maybe_init_dist(ws, local):
    if ws <= 1 and not force_sharded():
        return None
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist


def max_over_ranks(dist, x):
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ---------------------------------------------------------------- CPU baselines
class RefPagerankSampler:
    """The reference's own pull SpMV (gblite mxv plus.second, core.cpp:340-386,
    compiled from /root/reference into oracle/_ref) on a bounded row sample of
    the same relabel-free AT: one sample = one PageRank pull (pagerank.cpp:59-61)
    over rows [0, R) against the full contribution vector.  R is calibrated so
    one sample takes about `budget_s` seconds.  Falls back to the oracle port
    (multi-threaded restatement, full iterations) when oracle/_ref is absent."""

    def __init__(self, scale, seed=1, budget_s=5.0):
        import oracle as O
        self.O = O
        self.scale = scale
        rp, col = O.rmat_graph(scale, 16, seed=seed, undirected=False)
        self.n = len(rp) - 1
        self.trp, self.tcol, _ = O.transpose(self.n, rp, col)
        self.outdeg = np.diff(rp)
        self.kind = "reference" if O.ref_available() else "port"
        self.rows = 4
        if self.kind == "reference":
            secs, _ = O.ref_pr_mxv_sample(self.n, self.trp, self.tcol, self.outdeg, 0.85, 0,
                                          self.rows)
            while secs < budget_s / 3 and self.rows < self.n:
                self.rows = min(self.n, int(self.rows * max(2.0, budget_s / max(secs, 1e-3) / 2)))
                secs, _ = O.ref_pr_mxv_sample(self.n, self.trp, self.tcol, self.outdeg, 0.85, 0,
                                              self.rows)

    def step(self):
        O = self.O
        if self.kind == "reference":
            secs, _ = O.ref_pr_mxv_sample(self.n, self.trp, self.tcol, self.outdeg, 0.85, 0,
                                          self.rows)
            edges = int(self.trp[self.rows] - self.trp[0])
            return edges / secs
        t0 = time.perf_counter()
        O.pagerank(self.n, self.trp, self.tcol, self.outdeg, 0.85, 0.0, 3)
        return float(self.trp[-1]) * 3 / (time.perf_counter() - t0)

    def describe(self, value):
        if self.kind == "reference":
            edges = int(self.trp[self.rows] - self.trp[0])
            return {"value": value, "unit": "edges/s/iter", "cores": 1, "kind": "reference",
                    "sample": f"gblite mxv (plus.second, core.cpp:340-386) over rows "
                              f"[0,{self.rows}) of AT ({edges} edges) of the scale-{self.scale} "
                              f"graph against the full contribution vector; the reference is "
                              f"single-threaded (gapbench.cpp:164-166) and O(n * nnz(u)) per "
                              f"pull (SURVEY.md 3.3), so the full graph is out of reach"}
        return {"value": value, "unit": "edges/s/iter", "cores": self.O.threads(), "kind": "port",
                "sample": f"oracle restatement, 3 PageRank iterations on the full "
                          f"scale-{self.scale} graph"}


def cpu_baseline_pagerank(scale, seed, budget_s=12.0):
    """cpu_baseline for our arm: the reference sampler, plus the port as an extra."""
    import oracle as O
    ref = RefPagerankSampler(scale, seed, budget_s=budget_s / 2)
    v = ref.step()
    base = ref.describe(v)
    extras = {}
    t0 = time.perf_counter()
    O.pagerank(ref.n, ref.trp, ref.tcol, ref.outdeg, 0.85, 0.0, 3)
    tp = time.perf_counter() - t0
    extras["port"] = {"value": float(ref.trp[-1]) * 3 / tp, "unit": "edges/s/iter",
                      "cores": O.threads(), "kind": "port",
                      "sample": f"oracle restatement, 3 PageRank iterations on the full "
                                f"scale-{scale} graph"}
    return base, extras


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O
    O.build(ref=os.path.isdir("/root/reference/proj/src"))
    scale = args.scale or 22
    steps = max(args.steps, 1)
    sampler = RefPagerankSampler(scale, 1, budget_s=max(0.5, min(5.0, 90.0 / steps)))
    for _ in range(args.warmup):
        sampler.step()
    vals = [sampler.step() for _ in range(steps)]
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "edges/s/iter",
            "n_gpus": ws, "steps": steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"pagerank_rmat{scale}_directed", "scale": scale,
                       "edge_factor": 16, "damping": 0.85, "tol": 1e-4, "itermax": 100},
            "cpu_baseline": sampler.describe(v),
            "e2e": {"value": v, "unit": "edges/s/iter", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm: PageRank
def bench_pagerank_sharded(args, dist, ws, rank, local):
    """N > 1: one process per GPU, row blocks of the relabeled AT, one NCCL
    all_gather_into_tensor of the padded contribution slices + one fp64 L1
    all-reduce per iteration (paper_2104_01661_b200/dist.py).  Total work
    fixed -> strong scaling."""
    import ctypes as C

    import torch
    import paper_2104_01661_b200 as P
    from paper_2104_01661_b200.dist import (GpuShardBackend, sharded_pagerank,
                                            sharded_pagerank_p2p)
    from paper_2104_01661_b200.graph import Graph, call

    # the exchange: "p2p" (default) fuses it into one cooperative kernel per
    # rank (peer stores over NVLink via symmetric memory, device-side barrier);
    # "nccl" = one all_gather_into_tensor per iteration from the host loop
    exchange = os.environ.get("GBX_PR_EXCHANGE", "p2p")
    if exchange == "p2p":
        ok = 1
        try:  # symmetric memory + peer access on this box?
            g0 = P.generate_rmat(10, 16, seed=1)
            P.property_at(g0)
            P.property_rowdegree(g0)
            GpuShardBackend(g0).prepare(rank, ws)
            be0 = GpuShardBackend(g0)
            be0.prepare(rank, ws)
            be0.p2p_setup(dist)
        except Exception as e:
            print(f"bench: p2p exchange unavailable ({e}); using nccl", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)  # every rank takes the same path
        if int(flag.item()) == 0:
            exchange = "nccl"
    run_sharded = sharded_pagerank_p2p if exchange == "p2p" else sharded_pagerank

    scale = args.scale or 22
    P.init(local)
    torch.cuda.set_device(local)
    g = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.DirectedAdjacency)
    P.property_at(g)
    P.property_rowdegree(g)
    n, nnz, _, _ = g.info()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    for _ in range(max(args.warmup, 3)):
        be = GpuShardBackend(g)
        _, iters = run_sharded(be, dist, 0.85, 1e-4, 100)
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            be = GpuShardBackend(g)
            be.prepare(rank, ws)  # plan (and symmetric buffers) outside the timed region
            if exchange == "p2p":
                be.p2p_setup(dist)
            flush.zero_()
            barrier(dist)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            _, iters = run_sharded(_Prepared(be), dist, 0.85, 1e-4, 100, to_host=False)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    t = max_over_ranks(dist, sum(times) / len(times))
    value = nnz * iters / t
    # e2e: every rank builds its copy of the graph from pinned host CSR through
    # the C ABI (H2D + validation), fills AT / degrees (basic mode), plans its
    # row block and runs the sharded iterations; the ranks come back to the host
    # (D2H, original order) -- device time max over ranks, wall clock per rank
    rp, col, _ = g.export()
    rp_h = torch.from_numpy(rp).pin_memory()
    col_h = torch.from_numpy(col).pin_memory()
    e2e_times = []
    for s_ in range(3):
        barrier(dist)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = C.c_void_p()
        call("gbx_graph_new32", C.byref(h), n, rp_h.data_ptr(), col_h.data_ptr(), None, 0, 0)
        gh = Graph(h)
        P.property_at(gh)
        P.property_rowdegree(gh)
        _, it2 = run_sharded(GpuShardBackend(gh), dist, 0.85, 1e-4, 100)
        dt = time.perf_counter() - t0
        gh.free()
        if s_ > 0:
            e2e_times.append(dt)
    t_e2e = max_over_ranks(dist, statistics.median(e2e_times))
    out = {"metric": METRIC, "value": value, "unit": "edges/s/iter", "n_gpus": ws,
           "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f32 (ranks; fp64 row sums and L1)",
           "data": "synthetic (seeded R-MAT, generated in HBM)",
           "config": {"workload": f"pagerank_rmat{scale}_directed", "scale": scale, "n": n,
                      "nnz": nnz, "iterations": iters, "parallelism": f"rowblock{ws}",
                      "exchange": ("fused: one cooperative kernel per rank stores x "
                                   "into every rank's padded x over NVLink (symmetric "
                                   "memory), device-side signal barrier per iteration"
                                   if exchange == "p2p" else
                                   "NCCL all_gather_into_tensor (padded x slices + L1 "
                                   "partials) per iteration"),
                      "l2": "flushed (256 MB write) before every step"},
           "e2e": {"value": nnz * it2 / t_e2e, "unit": "edges/s/iter",
                   "h2d_bytes_per_step": int(rp.nbytes + col.nbytes),
                   "d2h_bytes_per_step": int(n * 8),
                   "includes": "per rank: H2D CSR (pinned), graph_new32 validation, "
                               "property_at, property_rowdegree, shard plan, sharded "
                               "iterations, D2H ranks",
                   "samples_ms": [round(x * 1e3, 2) for x in e2e_times]},
           "gpu_launches": int((2 if exchange == "p2p" else 2 * (iters + 1)) * args.steps),
           "clocks": clk.summary()}
    return out, (scale,)


class _Prepared:
    """A backend whose prepare() already ran (keeps the plan build untimed)."""

    def __init__(self, be):
        self.be = be
        self.device = be.device

    def prepare(self, rank, world):
        return self.be.rb, self.be.re, self.be.n

    def __getattr__(self, k):
        return getattr(self.be, k)


# ---------------------------------------------------------------- our arm: PageRank, one GPU
def bench_pagerank(args, dist, ws, rank, local):
    import torch
    import paper_2104_01661_b200 as P
    from paper_2104_01661_b200 import algo
    from paper_2104_01661_b200.graph import call
    import ctypes as C

    scale = args.scale or 22
    P.init(local)
    torch.cuda.set_device(local)
    g = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.DirectedAdjacency)
    P.property_at(g)
    P.property_rowdegree(g)
    g.prepare("pagerank")
    n, nnz, _, _ = g.info()
    stream = torch.cuda.ExternalStream(g.stream())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    it = C.c_int(0)

    def step():
        call("gbx_pagerank", None, C.byref(it), g.handle, 0.85, 1e-4, 100)
        return it.value

    for _ in range(max(args.warmup, 3)):
        step()
    times, iters, spans = [], [], []
    barrier(dist)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            k = step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
            iters.append(k)
            spans.append(g.last_stats()["hot_ms"])  # k_pr_rows launch spans of this step
    torch.cuda.synchronize()
    barrier(dist)
    st = g.last_stats()
    t_step = max_over_ranks(dist, sum(times) / len(times))
    k_iter = iters[-1]
    value = nnz * k_iter / t_step * ws
    hot_bytes = st["hot_bytes_per_launch"]
    t_iter = t_step / max(k_iter, 1)     # graph launch = init + k iteration kernels
    # the dominant kernel's own launch duration, measured live: mean span
    # (first CTA start -> last CTA end, %globaltimer) of every k_pr_rows
    # launch of every timed step; the iteration time bounds it from above
    t_launch = statistics.mean(spans) / 1e3 if spans and min(spans) > 0 else t_iter
    t_launch = max_over_ranks(dist, t_launch)
    peak, peak_kind = peaks()
    achieved = hot_bytes / t_launch / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "pagerank_ncu.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except Exception:
        pass
    # e2e through the C ABI with host buffers (pinned), basic mode
    rp, col, _ = g.export()
    rp_h = torch.from_numpy(rp).pin_memory()
    col_h = torch.from_numpy(col).pin_memory()
    rank_h = torch.empty(n, dtype=torch.float64).pin_memory()
    e2e_times = []
    for s in range(max(2, min(args.steps, 5)) + 1):
        t0 = time.perf_counter()
        h = C.c_void_p()
        call("gbx_graph_new32", C.byref(h), n, rp_h.data_ptr(), col_h.data_ptr(), None, 0, 0)
        call("gbx_basic_pagerank", rank_h.data_ptr(), C.byref(it), h, 0.85, 1e-4, 100)
        call("gbx_graph_free", C.byref(h))
        if s > 0:  # the first is a warm-up
            e2e_times.append(time.perf_counter() - t0)
    t_e2e = max_over_ranks(dist, statistics.median(e2e_times))
    e2e_val = nnz * it.value / t_e2e * ws
    out = {
        "metric": METRIC, "value": value, "unit": "edges/s/iter", "n_gpus": ws,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "weak" if ws > 1 else "weak",
        "vs_baseline": None, "dtype": "f32 (ranks; fp64 row sums and L1)",
        "data": "synthetic (seeded R-MAT, generated in HBM)",
        "config": {"workload": f"pagerank_rmat{scale}_directed", "scale": scale, "n": n,
                   "nnz": nnz, "edge_factor": 16, "a_b_c": [0.57, 0.19, 0.19],
                   "damping": 0.85, "tol": 1e-4, "itermax": 100, "iterations": k_iter,
                   "parallelism": f"replicas{ws}" if ws > 1 else "single",
                   "l2": "flushed (256 MB write) before every step"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": "k_pr_rows (fused pull SpMV + epilogue)",
                     "bytes_per_launch": hot_bytes,
                     "launch_ms": t_launch * 1e3,
                     "iteration_ms": t_iter * 1e3,
                     "frac_per_iteration": hot_bytes / t_iter / 1e9 / peak,
                     "note": "launch_ms = mean k_pr_rows launch duration over every iteration "
                             "of every timed step, measured live on the device (first CTA "
                             "start to last CTA end of the row phase, %globaltimer: all "
                             "iterations run inside one persistent cooperative launch, where "
                             "events cannot bracket an iteration); iteration_ms = device time "
                             "of one run (CUDA events) / iterations, which adds the long-row "
                             "finish, two grid barriers and the L1 reduction per iteration",
                     "traffic_source": "profiles/pagerank_ncu.json (ncu --set full, cold "
                                       "cache, one k_pr_rows launch)"},
        "e2e": {"value": e2e_val, "unit": "edges/s/iter",
                "h2d_bytes_per_step": int(rp.nbytes + col.nbytes),
                "d2h_bytes_per_step": int(n * 8 + 4),
                "includes": "H2D CSR (pinned), graph_new32 validation, property_at "
                            "(device transpose), property_rowdegree, PageRank, D2H ranks",
                "samples_ms": [round(t * 1e3, 2) for t in e2e_times]},
        "gpu_launches": int((st["launches"]) * args.steps),
        "clocks": clk.summary(),
    }
    return out, (scale,)


# ---------------------------------------------------------------- other workloads
def bench_simple(args, dist, ws, rank, local):
    """Secondary configs (not the headline): bfs, bfs64, tc, sssp, bc."""
    import ctypes as C

    import torch
    import paper_2104_01661_b200 as P
    from paper_2104_01661_b200 import algo

    P.init(local)
    torch.cuda.set_device(local)
    w = args.workload
    peak, peak_kind = peaks()
    if w in ("bfs", "bfs64"):
        scale = args.scale or (22 if w == "bfs" else 16)
        g = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
        P.property_at(g)
        P.property_rowdegree(g)
        n, nnz, _, _ = g.info()
        deg = g.row_degree()
        srcs = P.pick_sources(deg, 64, 1)
        from paper_2104_01661_b200.graph import call
        import oracle  # noqa: F401  (not used on the timed path)

        def one():
            if w == "bfs":
                for s in srcs[:8]:
                    call("gbx_bfs", None, None, g.handle, int(s), 0, 16)
                return 8
            arr = np.ascontiguousarray(srcs, np.uint64)
            call("gbx_bfs_batch", None, None, g.handle, arr.ctypes.data, len(arr))
            return 64
        unit_edges = nnz / 2  # Graph500 undirected convention (reached component ~ all)
        metric = f"BFS GTEPS at R-MAT scale {scale} ({'single source' if w == 'bfs' else '64-source batch'})"
        unit = "GTEPS"
        # per source B = 8 E_r + 24 V_r (int64 col once; row_ptr,
        # parent, level per reached vertex), E_r/V_r from one untimed traversal
        used = srcs[:8] if w == "bfs" else srcs
        alg_bytes = 0.0
        for s0 in used:
            par = np.empty(n, np.int64)
            call("gbx_bfs", par.ctypes.data, None, g.handle, int(s0), 0, 16)
            reached = par >= 0
            alg_bytes += 8.0 * float(deg[reached].sum()) + 24.0 * float(reached.sum())
        roof_kernel = "k_bfs1 (cooperative push/pull levels)" if w == "bfs" else "k_bfs64 (64-lane batch)"
        roof_note = "8*E_r + 24*V_r per source (SURVEY 8d), summed over the step's sources"
    elif w == "tc":
        scale = args.scale or 22
        g = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
        P.property_rowdegree(g)
        P.property_ndiag(g)
        g.prepare("tc")
        n, nnz, _, _ = g.info()

        def one():
            algo.triangle_count(g)
            return 1
        unit_edges = nnz / 2
        metric = f"triangle count edges/s at R-MAT scale {scale}"
        unit = "edges/s"
        # our probe formulation (DESIGN 5): 4*W2 + 12*nnz(U) + 8*(n+1),
        # W2 = sum_i C(dU(i), 2) over the (degree, id)-oriented upper triangle U
        rp_h, col_h, _ = g.export()
        dg = np.diff(rp_h)
        rank = np.empty(n, np.int64)
        rank[np.lexsort((np.arange(n), dg))] = np.arange(n)
        rows = np.repeat(np.arange(n, dtype=np.int64), dg)
        du = np.bincount(rows[rank[col_h] > rank[rows]], minlength=n).astype(np.float64)
        del rows, rp_h, col_h
        w2 = float((du * (du - 1) / 2).sum())
        alg_bytes = 4.0 * w2 + 12.0 * float(du.sum()) + 8.0 * (n + 1)
        roof_kernel = "k_tc_warp / k_tc_cta (middle-vertex probes)"
        roof_note = f"4*W2 + 12*nnz(U) + 8*(n+1), W2 = {w2:.4g} wedge probes (DESIGN 5)"
    elif w == "sssp":
        logn = args.scale or 24
        g = P.generate_er(logn, 16, seed=1)
        P.property_rowdegree(g)
        g.prepare("sssp")
        n, nnz, _, _ = g.info()
        srcs = P.pick_sources(g.row_degree(), 16, 1)
        from paper_2104_01661_b200.graph import call

        def one():
            for s in srcs:
                call("gbx_sssp", None, g.handle, int(s), 64.0)
            return len(srcs)
        unit_edges = nnz
        metric = f"SSSP relaxation edges/s (ER 2^{logn}, 16 sources, delta 64)"
        unit = "edges/s"
        # per source B = 8 m_r + 12 V_r (reached edges / vertices)
        odeg = g.row_degree()
        alg_bytes = 0.0
        for s0 in srcs:
            dd = np.empty(n, np.float64)
            call("gbx_sssp", dd.ctypes.data, g.handle, int(s0), 64.0)
            reached = np.isfinite(dd)
            alg_bytes += 8.0 * float(odeg[reached].sum()) + 12.0 * float(reached.sum())
        roof_kernel = "k_sssp_b (cooperative circular delta-buckets)"
        roof_note = "8*m_r + 12*V_r per source (SURVEY 8d), summed over 16 sources"
    elif w == "bc":
        scale = args.scale or 24
        g = P.generate_rmat(scale, 16, seed=1, kind=P.Kind.UndirectedAdjacency)
        P.property_at(g)
        P.property_rowdegree(g)
        n, nnz, _, _ = g.info()
        srcs = P.pick_sources(g.row_degree(), 4, 1)
        from paper_2104_01661_b200.graph import call

        if ws > 1:
            # 1D row blocks over the ranks, one record all-gather per BFS level
            # (dist.sharded_betweenness_rows): the same batch, strong scaling
            from paper_2104_01661_b200.dist import GpuShardBackend, sharded_betweenness_rows
            be = GpuShardBackend(g)

            def one():
                sharded_betweenness_rows(be, dist, [int(x) for x in srcs])
                torch.cuda.synchronize()  # the final all-reduce ran on torch's stream
                return 4
        else:
            def one():
                s = np.ascontiguousarray(srcs, np.uint64)
                call("gbx_betweenness", None, g.handle, s.ctypes.data, 4)
                return 4
        unit_edges = nnz
        metric = f"BC batch-4 edges/s at R-MAT scale {scale}"
        unit = "edges/s"
        # per batch B = E_r (8 + 16 ns) + V_r (16 + 24 ns), reached =
        # the union of the sources' components (one untimed BFS each)
        bdeg = g.row_degree()
        reach = np.zeros(n, bool)
        for s0 in srcs:
            par = np.empty(n, np.int64)
            call("gbx_bfs", par.ctypes.data, None, g.handle, int(s0), 0, 16)
            reach |= par >= 0
        ns = 4
        alg_bytes = float(bdeg[reach].sum()) * (8 + 16 * ns) + float(reach.sum()) * (16 + 24 * ns)
        roof_kernel = "k_bc_push/k_bc_pull/k_bc_back (batched Brandes levels)"
        roof_note = "E_r*(8+16*ns) + V_r*(16+24*ns), ns = 4 (SURVEY 8d)"
    else:
        raise SystemExit(f"unknown workload {w}")
    stream = torch.cuda.ExternalStream(g.stream())
    for _ in range(max(args.warmup, 3)):
        one()
    torch.cuda.synchronize()
    times, units = [], 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            units = one()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    t = max_over_ranks(dist, sum(times) / len(times))
    per = unit_edges * units / t
    value = per / 1e9 if unit == "GTEPS" else per
    strong = w == "bc" and ws > 1  # one batch split over the ranks' row blocks
    out = {"metric": metric, "value": value if strong else value * ws, "unit": unit,
           "n_gpus": ws, "steps": args.steps, "warmup": max(args.warmup, 3),
           "ms_per_step": t * 1e3, "higher_is_better": True,
           "scaling": "strong" if strong else "weak", "vs_baseline": None,
           "dtype": "int32 indices", "data": "synthetic",
           "config": {"workload": w, "scale": scale if w != "sssp" else logn, "n": n,
                      "nnz": nnz},
           "gpu_launches": int(g.last_stats()["launches"] * args.steps),
           "clocks": clk.summary()}
    achieved = alg_bytes / t / 1e9
    out["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                       "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
                       "kernel": roof_kernel, "bytes_per_step": alg_bytes,
                       "note": roof_note + "; divided by the device time of the whole step "
                               "(all of the step's launches)"}
    return out, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="pagerank",
                    choices=["pagerank", "bfs", "bfs64", "tc", "sssp", "bc"])
    ap.add_argument("--scale", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    ws, rank, local = dist_env()
    dist = maybe_init_dist(ws, local)
    if args.workload == "pagerank" and (ws > 1 or force_sharded()):
        out, extra = bench_pagerank_sharded(args, dist, ws, rank, local)
    elif args.workload == "pagerank":
        out, extra = bench_pagerank(args, dist, ws, rank, local)
    else:
        out, extra = bench_simple(args, dist, ws, rank, local)
    if rank == 0:
        if args.workload == "pagerank" and ws == 1 and not args.no_cpu_baseline:
            base, extras = cpu_baseline_pagerank(extra[0], 1)
            out["cpu_baseline"] = base
            out["cpu_baseline_port"] = extras.get("port")
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
