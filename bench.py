#!/usr/bin/env python
"""Benchmark of the hot path (BASELINE.json metric: random trees/s and
leaf-evals/s on 1 B200; % of the FP64 issue roofline).

A step = one pass of every §8(a) row over the workload: tree walk with
order-binned reduction (rt_sums_dev), [merge across ranks], finalisation
(rt_finalize_dev) and per-node [L/M] Padé (rt_pade_dev).  Default workload:
cfg4 (BASELINE.json configs[3]: 1024 nodes on the planes x=0, y=0, z=0 of
[-2,2]^3, 1e7 trees/node, d = 3, t = 1, K = 16, [7/7]) — the configuration the
north star's roofline target is stated on.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4|cfg2|cfg3|cfg1]
    python bench.py --impl reference ...   # the CPU oracle on the same config

Multi-GPU (torchrun): weak scaling; rank r samples trees [r*N, (r+1)*N) of
every node, the per-node sums are merged with one all-reduce (0.4 MB).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

# FP64 pipe: 64 lanes/clk/SM on B200 (sm_100), 148 SMs, 1965 MHz max clock
# (MEASURED_PEAKS.json sm_max_mhz; /opt/skills/guides/B200_PROFILING.md).
N_SM, FP64_LANES, F_MAX_MHZ = 148, 64, 1965.0

# Algorithmic FP64 work: the FP64 operations the sampling
# CONTRACT itself requires per unit, costed with SURVEY.md §8(d)'s fixed table
# (FP64 ops: log 20, exp 15, sincospi 20 per angle, sqrt 8, div 8, tanh 25;
# fma/mul/add/compare 1), times the units one launch processes (its event
# counters).  The contract is DESIGN.md R29 for Strategy A: per particle ONE
# Gamma(m+1) variate (m multiplies of the uniforms + 1 log), its split into
# the clock and the radii' Exp(1) shares (m+1 multiplies, m subtractions),
# S = e0/λ, the leaf test, 2D·h, τ - S, per radius 2 multiplies + 1 sqrt,
# one angle per normal pair plus the third normal's (d = 3), d FMAs — not the
# textbook draws SURVEY §8(d) listed (a log per exponential variate and per
# Box–Muller radius), which the kernel does not perform.  Strategy B keeps
# the textbook Box–Muller draws (R8).  Per leaf: g (its argument, the
# transcendental or reciprocal, the amplitude) + 1 mul — Gaussian data on
# independent FP64 trees: |x|², one FMA into the tree's exponent sum and the
# amplitude per leaf, the exponential once per tree (the kernel's closed form,
# DESIGN.md §4); per split: 1 mul (Strategy A's shift and variable
# coefficients: their exponents and denominators accumulated per split, the
# exponential and reciprocal once per tree — the same closed form); per
# tree: 1 mul + 2 adds.  The FP32-position variant is credited only its
# FP64 part (clock, weights, product, sums).  basis="survey" gives SURVEY
# §8(d)'s original textbook count (reported beside it).
SV = dict(log=20, exp=15, sqrt=8, div=8, tanh=25, sincospi=20)


def algo_fp64_per_unit(eq: dict, basis: str = "contract") -> dict:
    d = eq["dim"]
    strat = eq.get("strategy", 0)
    f32 = eq.get("precision", 0) == W.PREC_FP32_POS
    pairs = (d + 1) // 2
    if basis == "survey" or strat == 2:
        clock = 2 if strat == 2 else SV["log"]             # B: h = τS, τ_c = τ(1 - S)
        pos = (pairs * (SV["log"] + SV["sqrt"] + SV["sincospi"])
               + SV["sqrt"] + d)                           # σ sqrt(h); y_k + (σ√h) ξ_k
        per_particle = clock + pos + 3                     # τ - S, S > τ, 2D h
    else:
        m = 1 if d <= 2 else 2                             # radii Exp(1) shares
        gamma = m + SV["log"]                              # U1…U_{m+1}, -log
        spacings = (m + 1) + m                             # G·spacing, spacing differences
        clock = 4                                          # e0/λ, S > τ, 2D h, τ - S
        radii = m * (2 + SV["sqrt"])                       # sqrt(2 e · 2Dh)
        angles = (1 if d <= 2 else 2) * SV["sincospi"]
        pos = radii + angles + d
        per_particle = gamma + spacings + clock + (0 if f32 else pos)
    r2 = 2 * d - 1
    g = {W.G_CONST: 0,
         W.G_TANH_STEP: 1 + SV["tanh"] + 2,                # x/s, tanh, amp (1 + ·)/2
         W.G_GAUSS: r2 + 1 + SV["exp"] + 1,                # |x|², /s², exp, amp
         W.G_LORENTZ: r2 + 1 + 1 + SV["div"] + 1}[eq["init_kind"]]   # |x|², /s², 1 +, 1/·, amp
    if f32 and basis != "survey":
        g = 0                                              # g in single precision
    var = any(eq.get("coef_kind", [0] * 9))
    ring = not f32 and not eq.get("shared") and basis != "survey"
    defer_g = ring and eq["init_kind"] == W.G_GAUSS
    defer_w = ring and (strat == 1 or var)
    # the kernel's closed forms (RingVals): exponential and
    # rational factors are carried as an exponent sum X and a denominator
    # product D and evaluated once per tree
    tree_g = 0
    if defer_g:
        g = r2 + 1 + 1                                     # |x|², fma into X, amp
    if defer_g or defer_w:
        tree_g = SV["exp"] + 1                             # e^X, × the tree product
    split = 1                                              # Π *= w_k
    if strat == 1:
        split += 2 if defer_w else SV["exp"] + 2           # e^{(k-1)λτ_c}: (k-1)λ, fma into X
        tree_g += SV["div"] if defer_w else 0              # e^{+X} = 1 / e^{-X}
    if strat == 2:
        split += 1                                         # η(τ) = τ
    if var:
        # e^{-y²/s²}/(τ_c + t0): y², /s², X +=, τ_c + t0, D *= (deferred)
        split += 5 if defer_w else SV["exp"] + SV["div"] + 4
        tree_g += SV["div"] + 1 if defer_w else 0          # 1/D, ×
    return dict(particle=per_particle,
                leaf=g + 1 + (1 if strat == 2 else 0),     # Π *= g (/ q)
                split=split,
                tree=3 + (1 if strat == 1 else 0) + tree_g)   # ΣC += C, ΣC² += C·C (× e^{λt})


def algo_fp64_ops(eq: dict, stats: dict, n_points: int = 1, basis: str = "contract") -> float:
    """Algorithmic FP64 lane-ops of one launch from its event counters.

    Shared trees (f4): the statistics count per (node, tree), but the method
    walks each tree once for all n_points nodes — particles and splits are
    credited once per tree; the g evaluations (leaves) and the per-tree
    accumulation happen per node (Gaussian data: one exponential per (node,
    tree), the leaves' moments once per tree)."""
    u = algo_fp64_per_unit(eq, basis)
    walk = 1.0 / n_points if eq.get("shared") else 1.0
    if eq.get("shared") and eq["init_kind"] == W.G_GAUSS:
        # Gaussian data: the leaf product is W amp^L
        # e^{-(L|x+μ|² + V)/s²} — per leaf, once per tree: Σδ (d), Σ|δ|² (d + 1),
        # Π *= amp (1); per tree once: μ (reciprocal + d), V (d); per (node,
        # tree): x + μ (d), |·|² (d), L·q + V, /s², exp, W × (3)
        d = eq["dim"]
        per_leaf = 2 * d + 2 + (1 if eq.get("strategy", 0) == 2 else 0)
        per_tree_once = SV["div"] + 2 * d
        per_node_tree = 2 * d + 3 + SV["exp"]
        return (stats["particles"] * walk * u["particle"] + stats["leaves"] * walk * per_leaf +
                stats["splits"] * walk * u["split"] + stats["trees"] * walk * per_tree_once +
                stats["trees"] * (per_node_tree + u["tree"]))
    return (stats["particles"] * walk * u["particle"] + stats["leaves"] * u["leaf"] +
            stats["splits"] * walk * u["split"] + stats["trees"] * u["tree"])


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = []          # (sm MHz, reasons bitmask) every ~2 ms through NVML
        self._stop = None

    def _poll_nvml(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            while not self._stop.is_set():
                self.nvml.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                  pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
                self._stop.wait(0.002)
        except Exception:  # noqa: BLE001 — clocks are diagnostics only
            pass

    def __enter__(self):
        import threading
        self._stop = threading.Event()
        self._thread = threading.Thread(target=self._poll_nvml, daemon=True)
        self._thread.start()
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._thread.join(timeout=5)
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()

    def summary(self) -> dict:
        rows = [r.split(",") for r in getattr(self, "out", "").strip().splitlines() if r.strip()]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                s = float(r[1]); mx = max(mx, float(r[2])); p = float(r[3])
            except (ValueError, IndexError):
                continue
            if p > 200.0:                          # under load
                sm.append(s)
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        if not sm and self.nvml:
            # timed region shorter than nvidia-smi's start-up: NVML samples
            # taken every ~2 ms inside it (SM clock, clock-event reasons)
            bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4}
            sm = [float(c) for c, _ in self.nvml]
            for _, r in self.nvml:
                for nm, b in bits.items():
                    if r & b:
                        reasons.add(nm)
            if not mx:
                try:
                    import pynvml
                    mx = float(pynvml.nvmlDeviceGetMaxClockInfo(
                        pynvml.nvmlDeviceGetHandleByIndex(self.index), pynvml.NVML_CLOCK_SM))
                except Exception:  # noqa: BLE001
                    pass
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                    "samples": len(sm), "samples_under_load": len(sm), "source": "nvml (2 ms)"}
        if not sm:   # no usable sample at all: every row
            sm = [float(r[1]) for r in rows if len(r) > 1 and r[1].strip().replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(rows), "samples_under_load": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def oracle_sample(cfg: dict, budget_s: float):
    """Time the oracle as it stands (single-threaded) on a bounded sample of the
    workload: the first nodes x first trees, sized to about budget_s."""
    import oracle
    oracle.build()
    eq, t = cfg["eq"], cfg["t"]
    pts = W.nodes(cfg)
    t0 = time.perf_counter()
    _, st = oracle.sums(eq, pts[:1], t, 2000, seed=cfg["seed"])
    per_tree = (time.perf_counter() - t0) / 2000
    n_nodes = min(len(pts), 16)
    # (a subset of the workload: never more trees per node than it has)
    n_trees = min(cfg["n_trees"], max(64, int(budget_s / per_tree / n_nodes)))
    t0 = time.perf_counter()
    _, st = oracle.sums(eq, pts[:n_nodes], t, n_trees, seed=cfg["seed"])
    dt = time.perf_counter() - t0
    return dict(seconds=dt, trees=st["trees"], leaves=st["leaves"], particles=st["particles"],
                sample=f"{n_nodes} nodes x {n_trees} trees of {cfg['name']} (first nodes, first trees)")


def _oracle_worker(a):
    """One single-threaded oracle instance on its own nodes (all-cores baseline)."""
    import oracle
    eq, pts, t, n_trees, seed = a
    t0 = time.perf_counter()
    _, st = oracle.sums(eq, pts, t, n_trees, seed=seed)
    return time.perf_counter() - t0, st["trees"], st["leaves"]


def oracle_sample_all_cores(cfg: dict, budget_s: float):
    """The oracle as it stands, one single-threaded instance per host core on
    disjoint nodes (no change to the oracle itself), sized to ~budget_s."""
    import multiprocessing as mp
    import oracle
    oracle.build()
    cores = os.cpu_count() or 1
    eq, t = cfg["eq"], cfg["t"]
    pts = W.nodes(cfg)
    t0 = time.perf_counter()
    oracle.sums(eq, pts[:1], t, 2000, seed=cfg["seed"])
    per_tree = (time.perf_counter() - t0) / 2000
    n_trees = min(cfg["n_trees"], max(64, int(budget_s / per_tree)))
    jobs = [(eq, pts[i % len(pts):i % len(pts) + 1], t, n_trees, cfg["seed"]) for i in range(cores)]
    with mp.get_context("spawn").Pool(cores) as pool:
        pool.map(_oracle_worker, [(eq, pts[:1], t, 64, cfg["seed"])] * cores)   # start-up, oracle load
        t0 = time.perf_counter()
        res = pool.map(_oracle_worker, jobs)
        wall = time.perf_counter() - t0
    trees = sum(r[1] for r in res)
    return dict(seconds=wall, trees=trees, leaves=sum(r[2] for r in res), cores=cores,
                sample=f"{cores} processes x (1 node x {n_trees} trees) of {cfg['name']}")


def run_reference(args, cfg):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    budget = float(os.environ.get("RT_REF_STEP_S", "4.0"))
    times, trees, leaves = [], 0, 0
    for s in range(args.warmup + args.steps):
        r = oracle_sample(cfg, budget)
        if s >= args.warmup:
            times.append(r["seconds"]); trees += r["trees"]; leaves += r["leaves"]
            sample = r["sample"]
    tot = sum(times)
    v = trees / tot
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "trees/s", "n_gpus": ws,
            "host_only": True,   # the oracle runs on one host core, no GPU work
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config_json(cfg, ws),
            "leaf_evals_per_s": leaves / tot,
            "cpu_baseline": {"value": v, "unit": "trees/s", "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "trees/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


METRIC = "random trees/sec and leaf-evals/sec on 1 B200; % of FP64 issue roofline"


def _config_json(cfg, ws, graphed=None):
    eq = cfg["eq"]
    d = {"workload": cfg["name"], "nodes": int(len(W.nodes(cfg))), "trees_per_node": cfg["n_trees"],
            "dim": eq["dim"], "t": cfg["t"], "K": eq["K"], "pade": f"[{cfg['L']}/{cfg['M']}]",
            "b": eq["b"][: eq["degree"] + 1], "g": ["const", "tanh_step", "gauss", "lorentz"][eq["init_kind"]],
            "parallelism": f"trees sharded over {ws} GPU(s)" if ws > 1 else "1 GPU",
            "l2": "256 MiB buffer written between timed steps (inputs are KB-sized)"}
    if graphed is not None:
        d["steps_as"] = "CUDA graph replays (one captured graph per step)" if graphed else "eager launches"
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--trees", type=int, default=0, help="override trees per node")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay each timed step as a captured CUDA graph (auto: on at N=1) so "
                         "latency-bound configs are not timed on Python launch overhead")
    args = ap.parse_args()
    cfg = W.get(args.config)
    cfg["name"] = args.config
    if args.trees:
        cfg["n_trees"] = args.trees
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import paper_2402_06491_b200 as P

    ws, rank, local = _dist()
    # (RT_BENCH_DRY_MULTI=1: a dry run of the N > 1 logic with every rank on
    # cuda:0 and gloo collectives — the multi-rank code path exercised on a
    # 1-GPU box; never a measurement)
    dry = os.environ.get("RT_BENCH_DRY_MULTI") == "1"
    if dry:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        if dry:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    eq, t, N, seed = cfg["eq"], cfg["t"], cfg["n_trees"], cfg["seed"]
    K, L, M = eq["K"], cfg["L"], cfg["M"]
    pts = W.nodes(cfg)
    n = len(pts)
    x = torch.as_tensor(pts, device="cuda")
    est = P.Estimator(eq)
    sums = torch.empty((n, K + 2, 3), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    from paper_2402_06491_b200.dist import merge_sums, tree_range
    off, n_rank = tree_range(rank, ws, N)

    def step(walk=None):
        cur = torch.cuda.current_stream()    # (the capture stream inside a graph capture)
        if walk is not None:
            walk[0].record(cur)
        est.sums(x, t, n_rank, seed, tree_offset=off, out=sums)
        if walk is not None:
            walk[1].record(cur)
        merge_sums(sums)                     # one all-reduce of (K+2)x3 doubles per node
        c, se, us, ses = P.finalize(sums, K, N * ws)
        u, fl = P.pade(c, L, M, se_sum=ses)
        return u, ses

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st_one = est.stats()            # counters of one launch (same every step)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    # the tree-walk call of each step (its memset, walk and task reduction;
    # the walk is > 99.9 % of it), events on the launch stream — no host sync
    # inside the timed region, so the steps are enqueued back to back
    def _tev():
        # external: recorded inside a captured graph as a timed external event node
        try:
            return torch.cuda.Event(enable_timing=True, external=True)
        except TypeError:
            return torch.cuda.Event(enable_timing=True)
    walk_ev = [(_tev(), _tev()) for _ in range(args.steps)]
    # one captured graph per timed step (its own walk events), replayed in the
    # timed loop: the same kernels with the same arguments, without the host's
    # per-launch overhead between them (matters only for latency-bound configs)
    graphs = None
    if args.graph == "on" or (args.graph == "auto" and ws == 1):
        try:
            graphs = []
            for s_ in range(args.steps):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    step(walk_ev[s_])
                graphs.append(g)
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001 — timing method only; the kernels are the same
            print(f"[bench] CUDA graph capture unavailable ({e}); timing eager steps", file=sys.stderr)
            graphs = None
            torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            flush.fill_(s)                        # evict L2 between timed steps
            ev[s][0].record(stream)
            if graphs is not None:
                graphs[s].replay()
            else:
                u, ses = step(walk_ev[s])
            ev[s][1].record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    walk_ms = [a.elapsed_time(b) for a, b in walk_ev]
    tot_ms = sum(step_ms)
    walk_avg = sum(walk_ms) / len(walk_ms)
    if dist is not None:
        tt = torch.tensor([tot_ms, walk_avg], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tot_ms, walk_avg = tt.tolist()
    trees_all = n * N * ws * args.steps
    value = trees_all / (tot_ms / 1e3)
    leaves_all = st_one["leaves"] * ws * args.steps
    ops = algo_fp64_ops(eq, st_one, n)
    ops_survey = algo_fp64_ops(eq, st_one, n, basis="survey")
    peak = N_SM * FP64_LANES * F_MAX_MHZ * 1e6 / 1e12       # T lane-ops/s
    achieved = ops / (walk_avg / 1e3) / 1e12
    clocks = clk.summary()
    # measured FP64 FMA throughput (K0) beside the nominal peak
    try:
        k0 = P.rt.fp64_peak()["lane_ops_per_s"] / 1e12
    except Exception:   # noqa: BLE001 — diagnostic only
        k0 = None
    # DRAM traffic and the hardware FP64-pipe share of the tree-walk launch
    # from the committed ncu captures of this same command
    # (profiles/r2/traffic_<workload>.json, the latest round first), else null
    traffic, hw = None, {}
    for rnd in ("r2", "r1"):
        tf = os.path.join(ROOT, "profiles", rnd, f"traffic_{cfg['name']}.json")
        if os.path.exists(tf) and not args.trees:
            tj = json.load(open(tf))
            traffic = tj["dram_bytes_read"] + tj["dram_bytes_write"]
            hw = {k: tj[k] for k in ("fp64_pipe_pct", "issue_active_pct", "inst_per_iteration",
                                     "source") if k in tj}
            break

    # ---- end to end through the public host API (rt_interface_values) -----
    e2e = None
    if ws > 1:
        # N ranks: each rank's host points go up, it samples ITS tree range
        # (rt_sums_dev(tree_offset)), the sums are merged by one all-reduce,
        # every rank finalises + resums the merged series and reads back u and
        # its standard error — the sharded job end to end
        pin = torch.as_tensor(pts).pin_memory()
        out_u = torch.empty(n, dtype=torch.float64).pin_memory()
        out_se = torch.empty_like(out_u).pin_memory()

        def e2e_step():
            xd = pin.to("cuda", non_blocking=True)
            s_ = est.sums(xd, t, n_rank, seed, tree_offset=off)
            merge_sums(s_)
            c_, _, _, ses_ = P.finalize(s_, K, N * ws)
            u_, _ = P.pade(c_, L, M, se_sum=ses_)
            out_u.copy_(u_, non_blocking=True)
            out_se.copy_(ses_, non_blocking=True)
            torch.cuda.synchronize()

        e2e_step()
        dist.barrier()
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 3))
        for _ in range(e2e_steps):
            e2e_step()
        e2e_s = time.perf_counter() - t0
        tt = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = tt.item()
        e2e = {"value": n * N * ws * e2e_steps / e2e_s, "unit": "trees/s",
               "h2d_bytes_per_step": n * eq["dim"] * 8, "d2h_bytes_per_step": 2 * n * 8,
               "api": "per rank: host points -> rt_sums_dev(tree range) -> all-reduce -> "
                      "rt_finalize_dev -> rt_pade_dev -> host (u, se)"}
    elif cfg["nodes"]["kind"] == "planes":
        planes = cfg["nodes"]["planes"]
        est.interface_values(planes, n, t, N, seed, L, M)          # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 3))
        for _ in range(e2e_steps):
            est.interface_values(planes, n, t, N, seed, L, M)
        e2e_s = time.perf_counter() - t0
        e2e = {"value": n * N * e2e_steps / e2e_s, "unit": "trees/s",
               "h2d_bytes_per_step": n * eq["dim"] * 8,
               "d2h_bytes_per_step": n * eq["dim"] * 8 + n * 8 * 2 + n * 4,
               "api": "rt_interface_values (host buffers; node placement, walk, Padé, copies)"}
    else:
        pin = torch.as_tensor(pts).pin_memory()
        oc = torch.empty((n, K + 1), dtype=torch.float64).pin_memory()
        os_ = torch.empty_like(oc).pin_memory()
        est.estimate_host(pin, t, N, seed, oc, os_)
        t0 = time.perf_counter()
        for _ in range(max(1, min(args.steps, 3))):
            est.estimate_host(pin, t, N, seed, oc, os_)
        e2e_s = time.perf_counter() - t0
        e2e = {"value": n * N * max(1, min(args.steps, 3)) / e2e_s, "unit": "trees/s",
               "h2d_bytes_per_step": pin.numel() * 8, "d2h_bytes_per_step": 2 * oc.numel() * 8,
               "api": "rt_estimate (pinned host buffers)"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        r = oracle_sample(cfg, float(os.environ.get("RT_CPU_BASELINE_S", "15")))
        cpu = {"value": r["trees"] / r["seconds"], "unit": "trees/s", "cores": 1, "kind": "oracle",
               "sample": r["sample"], "leaf_evals_per_s": r["leaves"] / r["seconds"]}
        try:   # the same oracle on every host core (one instance per core)
            ra = oracle_sample_all_cores(cfg, float(os.environ.get("RT_CPU_BASELINE_S", "15")) / 2)
            cpu["all_cores"] = {"value": ra["trees"] / ra["seconds"], "cores": ra["cores"],
                                "sample": ra["sample"]}
        except Exception as e:   # noqa: BLE001 — a baseline, never fatal
            cpu["all_cores"] = {"error": str(e)[:200]}
    line = {
        "metric": METRIC, "value": value, "unit": "trees/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_json(cfg, ws, graphs is not None),
        "leaf_evals_per_s": leaves_all / (tot_ms / 1e3),
        "particles_per_s": st_one["particles"] * ws * args.steps / (tot_ms / 1e3),
        "pruned_fraction": st_one["pruned"] / max(1, st_one["trees"]),
        "roofline": {"bound": "alu", "kernel": "tree_walk_kernel", "achieved": achieved,
                     "peak": peak, "unit": "T FP64 lane-ops/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram read + write)",
                     "launch_ms": walk_avg,
                     "algorithmic_fp64_ops_per_launch": ops,
                     "basis": "DESIGN.md R29 contract units (one log per particle), SURVEY 8(d) cost table",
                     "frac_survey_textbook_table": ops_survey / (walk_avg / 1e3) / 1e12 / peak,
                     "ncu_hardware": hw or None,
                     "peak_basis": "148 SM x 64 FP64 lanes/clk x 1965 MHz (B200_PROFILING.md nominal; MEASURED_PEAKS.json has no FP64 entry)",
                     "frac_at_measured_clock": (achieved / (N_SM * FP64_LANES * clocks["sm_mhz"] * 1e6 / 1e12)
                                                if clocks.get("sm_mhz") else None),
                     "peak_measured_dfma": k0,
                     "frac_of_measured_dfma": achieved / k0 if k0 else None},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clocks,
        "gpu_launches": 4 * args.steps,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
