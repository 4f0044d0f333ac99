"""Throughput of the NEXT-row paths (f2: Strategy A with the e^{λt} shift and
variable coefficients; f3: Strategy B) on the paper's Examples 1, 3, 5
(workloads ex1A/ex1B/ex3A/ex3B/ex5A/ex5B): tree-walk launch time (CUDA
events on its stream, best of 3 after a warm-up), trees/s, leaf-evals/s and
the algorithmic FP64 roofline fraction (bench.py's cost model).

    python tools/bench_next.py [--out gpurun_out/next_bench]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2402_06491_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

NAMES = ("ex1A", "ex1B", "ex2A", "ex2B", "ex3A", "ex3B", "ex5A", "ex5B", "cfg2", "cfg3", "cfg4",
         "cfg2_sh", "cfg3_sh", "cfg4_sh")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "next_bench"))
    a = ap.parse_args()
    peak = bench.N_SM * bench.FP64_LANES * bench.F_MAX_MHZ * 1e6
    rows = []
    for name in NAMES:
        cfg = W.get(name)
        eq, t, N = cfg["eq"], cfg["t"], cfg["n_trees"]
        x = torch.as_tensor(W.nodes(cfg), device="cuda")
        n = x.shape[0]
        est = P.Estimator(eq)
        est.sums(x, t, N, cfg["seed"])
        ms = []
        for _ in range(3):
            est.sums(x, t, N, cfg["seed"])
            torch.cuda.synchronize()
            st = est.stats()
            ms.append(st["kernel_ms"])
        kms = min(ms)
        st_ops = dict(st)   # (shared trees: the walk is credited once per tree, bench.algo_fp64_ops)
        c, se = est.estimate(x, t, N, cfg["seed"])
        u, fl = P.pade(c, cfg["L"], cfg["M"])
        r = dict(workload=name, strategy=["potential", "A_shift", "B"][eq.get("strategy", 0)]
                 + (" shared" if eq.get("shared") else ""),
                 q=eq.get("q") if eq.get("strategy", 0) == 2 else None, dim=eq["dim"], nodes=n,
                 trees_per_node=N, t=t, kernel_ms=kms, trees_per_s=n * N / (kms / 1e3),
                 leaf_evals_per_s=st["leaves"] / (kms / 1e3),
                 particles_per_tree=st["particles"] / st["trees"],
                 pruned_fraction=st["pruned"] / st["trees"],
                 fp64_roofline_frac=bench.algo_fp64_ops(eq, st_ops, n) / (kms / 1e3) / peak,
                 u_mid=float(u[n // 2].item()))
        rows.append(r)
        print(json.dumps(r), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out + ".jsonl", "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
    md = ["# NEXT-row throughput (1 x B200, tree-walk launch, best of 3)", "",
          "| workload | strategy | d | nodes x trees | t | launch ms | trees/s | leaf-evals/s | particles/tree | pruned | frac |",
          "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        md.append(f"| {r['workload']} | {r['strategy']}{'' if r['q'] is None else ' q=%.3g' % r['q']} | {r['dim']} | "
                  f"{r['nodes']} x {r['trees_per_node']:.0e} | {r['t']} | {r['kernel_ms']:.2f} | {r['trees_per_s']:.3e} | "
                  f"{r['leaf_evals_per_s']:.3e} | {r['particles_per_tree']:.2f} | {r['pruned_fraction']:.3f} | "
                  f"{r['fp64_roofline_frac']:.3f} |")
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
