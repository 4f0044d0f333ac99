"""Load-balance diagnostics: per-warp start/end times of the tree-walk kernel.

    RT_WARP_TIMES=gpurun_out/wt.txt python tools/warp_times.py [cfg] [trees]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_06491_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
path = os.environ["RT_WARP_TIMES"]
if os.path.exists(path):
    os.remove(path)
x = torch.as_tensor(W.nodes(cfg), device="cuda")
est = P.Estimator(cfg["eq"])
for _ in range(2):
    est.sums(x, cfg["t"], N, cfg["seed"])
torch.cuda.synchronize()
line = open(path).read().strip().splitlines()[-1]
t = np.array(line.split(), dtype=np.float64).reshape(-1, 4)
np.save(path + ".npy", t)
t0 = t[:, 0].min()
s, e = (t[:, 0] - t0) / 1e6, (t[:, 1] - t0) / 1e6
T = e.max()
print(f"warps {len(t)}  kernel {T:.2f} ms  start max {s.max():.3f} ms")
print(f"end quantiles (ms): " + " ".join(f"{q}:{np.quantile(e, q):.2f}" for q in (0, .01, .1, .5, .9, .99, 1)))
print(f"mean active fraction {((e - s).sum() / (len(t) * T)):.3f}")
print(f"stats {est.stats()}")
it = t[:, 3]
print(f"iterations per warp: min {it.min():.0f} median {np.median(it):.0f} max {it.max():.0f}")
sm = t[:, 2].astype(int)
wib = np.arange(len(t)) % 4
for k in range(4):
    print(f"warp-in-CTA {k}: mean end {e[wib == k].mean():.2f} ms")
per_sm = np.array([e[sm == q].mean() for q in np.unique(sm)])
print(f"per-SM mean end: min {per_sm.min():.2f} max {per_sm.max():.2f}; CTAs per SM {np.bincount(sm).max() // 4}")
rate = it / (e - s)
print(f"iterations/ms per warp: min {rate.min():.1f} median {np.median(rate):.1f} max {rate.max():.1f}")
# correlation of end time with iterations
print(f"corr(end, iterations) {np.corrcoef(e, it)[0, 1]:.3f}")
