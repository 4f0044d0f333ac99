"""Time a few cfg5 points through rt_sums_dev (CUDA events on the launch
stream, best of 5 after a warm-up): python tools/cfg5_points.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_06491_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

eq = W.get("cfg2")["eq"]
for n, N, t in ((64, 1_000_000, 0.25), (1024, 1_000_000, 0.25), (64, 1_000_000, 2.0), (1024, 1_000_000, 1.0)):
    x = torch.as_tensor(W.linspace(-3, 3, n).reshape(-1, 1), device="cuda")
    est = P.Estimator(eq)
    est.sums(x, t, N, seed=1)
    torch.cuda.synchronize()
    ts = []
    for rep in range(5):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        est.sums(x, t, N, seed=2 + rep)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"cfg5 n={n} N={N} t={t}: {min(ts):.3f} ms, {n * N / (min(ts) * 1e-3):.4e} trees/s", flush=True)
