"""Per-tree relative differences |C_gpu - C_oracle| / |C_oracle| of the
production kernel (rt_trace_dev) against the oracle on the parity cases, split
by |C| (R30).  python tools/tree_rel_err.py"""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2402_06491_b200 as P  # noqa: E402

spec = importlib.util.spec_from_file_location("gp", os.path.join(ROOT, "tests", "test_gpu_parity.py"))
gp = importlib.util.module_from_spec(spec)
spec.loader.exec_module(gp)
worst = 0.0
for name in ["cfg1", "cfg2", "cfg2_t2", "cfg3", "cfg4", "d3_gauss", "d2_lorentz", "heat_d2_tanh",
             "shift_ex1", "B_ex3", "B_cfg2_k1", "B_d3_var", "ex2_shift", "neg_cfg2_t2", "neg_big_d3",
             "pot_var", "sh_cfg2", "sh_d3_shift"]:
    eq, pts, t, N = gp.CASES[name]
    rec, _ = P.Estimator(eq).trace(torch.as_tensor(pts, device="cuda"), t, N, seed=12345)
    ref = oracle.trees(eq, pts, t, N, seed=12345)
    keep = ref["pruned"] == 0
    Cg, Co = rec["C"][keep], ref["C"][keep]
    nz = Co != 0
    rel = np.abs(Cg[nz] - Co[nz]) / np.abs(Co[nz])
    big = np.abs(Co[nz]) >= 1e-20
    w_all = rel.max() if rel.size else 0.0
    w_big = rel[big].max() if big.any() else 0.0
    w_small = rel[~big].max() if (~big).any() else 0.0
    worst = max(worst, w_all)
    print(f"{name:14s} trees {rel.size:7d}  max rel {w_all:.2e}  |C|>=1e-20 {w_big:.2e}  "
          f"|C|<1e-20 {w_small:.2e} (n={int((~big).sum())})  p99.9 {np.quantile(rel, 0.999):.2e}")
print(f"worst {worst:.2e}")
