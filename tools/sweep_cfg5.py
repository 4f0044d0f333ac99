"""cfg5 throughput sweep (BASELINE.json configs[4]): the cfg2 equation on
linspace(-3, 3, n) for n in {64, 1024, 16384} x trees/node {1e4, 1e6, 1e7} x
t in {0.25, 1, 2}, FP64 and the FP32-position variant.  Each point times the
tree-walk launch (CUDA events on its stream, after a warm-up launch) and
reports trees/s, leaf-evals/s, particles/s and the algorithmic FP64 roofline
fraction (bench.py's cost model).

    python tools/sweep_cfg5.py [--out profiles/r1/cfg5_sweep] [--quick]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cfg5_sweep"))
    ap.add_argument("--quick", action="store_true", help="skip the 16384 x 1e7 points")
    a = ap.parse_args()
    peak = bench.N_SM * bench.FP64_LANES * bench.F_MAX_MHZ * 1e6
    rows = []
    for fp32 in (False, True):
        for t in W.CFG5_T:
            for n in W.CFG5_NODES:
                for N in W.CFG5_TREES:
                    if a.quick and n * N > 2e10:
                        continue
                    cfg = W.cfg5(n, N, t, fp32_pos=fp32)
                    x = torch.as_tensor(W.nodes(cfg), device="cuda")
                    est = P.Estimator(cfg["eq"])
                    reps = 3 if n * N <= 1e9 else 1
                    if n * N <= 1e10:
                        est.sums(x, t, N, cfg["seed"])          # warm-up
                    ms = []
                    for _ in range(reps):
                        est.sums(x, t, N, cfg["seed"])
                        torch.cuda.synchronize()
                        st = est.stats()
                        ms.append(st["kernel_ms"])
                    kms = min(ms)
                    ops = bench.algo_fp64_ops(cfg["eq"], st)
                    r = dict(precision="fp32_pos" if fp32 else "fp64", t=t, nodes=n, trees_per_node=N,
                             kernel_ms=kms, trees_per_s=n * N / (kms / 1e3),
                             leaf_evals_per_s=st["leaves"] / (kms / 1e3),
                             particles_per_s=st["particles"] / (kms / 1e3),
                             particles_per_tree=st["particles"] / st["trees"],
                             pruned_fraction=st["pruned"] / st["trees"],
                             fp64_roofline_frac=ops / (kms / 1e3) / peak)
                    rows.append(r)
                    print(json.dumps(r), flush=True)
                    del est, x
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out + ".jsonl", "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
    md = ["# cfg5 throughput sweep (1 x B200, tree-walk launch time)", "",
          "cfg2 equation, d = 1, g = 0.4 exp(-x^2), K = 12; nodes linspace(-3, 3, n).  "
          "frac = algorithmic FP64 lane-ops (bench.py cost model: R29 contract units, DESIGN.md §5) / "
          "(148 x 64 x 1.965 GHz); the FP32-position variant is credited only its FP64 part (clock, "
          "weights, product, sums), so its frac is not comparable with the FP64 rows — compare trees/s.", "",
          "| precision | t | nodes | trees/node | launch ms | trees/s | leaf-evals/s | particles/tree | pruned | frac |",
          "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        md.append(f"| {r['precision']} | {r['t']} | {r['nodes']} | {r['trees_per_node']:.0e} | {r['kernel_ms']:.2f} | "
                  f"{r['trees_per_s']:.3e} | {r['leaf_evals_per_s']:.3e} | {r['particles_per_tree']:.2f} | "
                  f"{r['pruned_fraction']:.3f} | {r['fp64_roofline_frac']:.3f} |")
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
