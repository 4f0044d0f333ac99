"""NEXT row f1 measurement: cfg3's probabilistic domain decomposition
(BASELINE.json configs[2]) through rt_pdd_solve — phase times T_MC (tree walk
at every nodal point and time level + Padé), T_INT (tensor splines), T_LOCAL
(four subdomain CN/ADI solves) as in the paper's Tables A-D,
and the field error against the single-domain reference (oracle/pdd_oracle).

    python tools/bench_pdd.py [--trees 1000000] [--out gpurun_out/pdd_bench]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2402_06491_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from oracle import pdd_oracle as PO  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trees", type=int, default=1_000_000)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "pdd_bench"))
    a = ap.parse_args()
    eq = W.get("cfg3")["eq"]
    g = PO.g_fn(eq)
    t0 = time.perf_counter()
    x, u = PO.single_domain(g, eq["b"][: eq["degree"] + 1], 1.0, 6.0, 0.05, 0.5, 500)
    t_ref = time.perf_counter() - t0
    i0 = int(np.argmin(np.abs(x + 2.0)))
    ref = u[i0:i0 + 81, i0:i0 + 81]
    rows = []
    for boundary, shared in ((1, 0), (0, 0), (1, 1)):
        est = P.Estimator(dict(eq, shared=shared))
        cfg = dict(lo=-2.0, hi=2.0, T=0.5, n_cells=80, n_steps=500, n_s=17, n_t=6, boundary=boundary,
                   L=5, M=5, n_trees=a.trees, seed=7)
        est.pdd_solve(cfg)                          # warm-up
        t0 = time.perf_counter()
        F, V, ms = est.pdd_solve(cfg)
        wall = (time.perf_counter() - t0) * 1e3
        d = np.abs(F - ref)
        n_pts = (6 if boundary else 2) * cfg["n_s"] * (cfg["n_t"] - 1)
        r = dict(workload="cfg3 PDD" + (" (shared trees)" if shared else ""),
                 boundary=["zero Dirichlet", "probabilistic"][boundary],
                 nodal_points=n_pts, trees_per_point=a.trees, grid=f"{cfg['n_cells'] + 1}^2",
                 steps=cfg["n_steps"], **ms, wall_ms=wall, max_err=float(d.max()), mean_err=float(d.mean()),
                 reference="single-domain CN/ADI on [-6,6]^2, h=0.05, dt=1e-3 (numpy, %.1f s on the host)" % t_ref)
        rows.append(r)
        print(json.dumps(r), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out + ".jsonl", "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
    md = ["# cfg3 PDD (NEXT row f1) on 1 x B200", "",
          "| workload | outer edges | nodal points x levels | trees/point | T_MC ms | T_INT ms | T_LOCAL ms | wall ms | max err | mean err |",
          "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        md.append(f"| {r['workload']} | {r['boundary']} | {r['nodal_points']} | {r['trees_per_point']:.0e} | {r['T_MC']:.2f} | "
                  f"{r['T_INT']:.3f} | {r['T_LOCAL']:.2f} | {r['wall_ms']:.1f} | {r['max_err']:.2e} | {r['mean_err']:.2e} |")
    md += ["", "Error against " + rows[0]["reference"] + "; grid 81^2 on [-2,2]^2, 500 steps, "
           "nodal lines x = 0, y = 0 (and the four edges) with 17 points x 6 levels."]
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
