"""Seeded, synthetic workload definitions shared by the CUDA path's tests/bench
and by the oracle's tests.

This module holds NO arithmetic of the method (no normalisation, no random
trees, no Padé): only the equation coefficients, initial-data choices, horizons,
sample sizes and node coordinates of the BASELINE.json configs, restated in
SURVEY.md §8(d) "Synthetic inputs" and DESIGN.md §3 (input recipe).

Node layouts follow the readings in DESIGN.md:
  * 1-D configs: ``linspace(lo, hi, n)`` with the explicit formula
    ``lo + (hi - lo) * (j / (n - 1))`` (j = 0..n-1).
  * cfg3: the interfaces x = 0 and y = 0 of [-2,2]^2, 128 nodes each,
    plane-major, free coordinate ascending.
  * cfg4: the planes x = 0, y = 0, z = 0 of [-2,2]^3, a 19 x 19 grid on each,
    plane-major, row-major in ascending free axes, exact duplicates of earlier
    points skipped, first 1024 kept.

The paper's experiments use analytic equations only (§3, Examples
1-5, lines 787-1141); no dataset or benchmark suite is involved, so nothing
here stands in for one.
"""
from __future__ import annotations

import copy
from typing import Dict, List

import numpy as np

# Initial-data kinds (mirrors rt_init in include/rt.h; the numbering is part of
# the boundary, not of the method).
G_CONST, G_TANH_STEP, G_GAUSS, G_LORENTZ = 0, 1, 2, 3
OFFSPRING_ABS, OFFSPRING_UNIFORM = 0, 1
PREC_FP64, PREC_FP32_POS = 0, 1


def linspace(lo: float, hi: float, n: int) -> np.ndarray:
    """Explicit linspace: lo + (hi - lo) * (j / (n - 1)); the product's node
    generator (rt_interface_values) is specified with the same formula."""
    if n == 1:
        return np.array([lo], dtype=np.float64)
    j = np.arange(n, dtype=np.float64)
    return lo + (hi - lo) * (j / float(n - 1))


def plane_nodes(dim: int, planes: List[dict], max_points: int) -> np.ndarray:
    """Nodes on axis-aligned planes ``x_axis = value`` (C14).

    Each plane carries a tensor grid of ``n_per_dim`` linspace points over
    [lo, hi] along every free axis (row-major, ascending free-axis order).
    Plane-major emission; points equal (exactly) to an earlier point are
    skipped; at most ``max_points`` are returned.
    """
    out: List[tuple] = []
    seen = set()
    for pl in planes:
        free = [a for a in range(dim) if a != pl["axis"]]
        s = linspace(pl["lo"], pl["hi"], pl["n_per_dim"])
        grids = np.meshgrid(*([s] * len(free)), indexing="ij")
        flat = [g.reshape(-1) for g in grids]
        for q in range(flat[0].size if flat else 1):
            p = [0.0] * dim
            p[pl["axis"]] = float(pl["value"])
            for f, a in enumerate(free):
                p[a] = float(flat[f][q])
            key = tuple(p)
            if key in seen:
                continue
            seen.add(key)
            out.append(key)
            if len(out) >= max_points:
                return np.array(out, dtype=np.float64).reshape(-1, dim)
    return np.array(out, dtype=np.float64).reshape(-1, dim)


STRAT_POTENTIAL, STRAT_A_SHIFT, STRAT_B = 0, 1, 2
COEF_CONST, COEF_GAUSS_RATIONAL = 0, 1


def _eq(dim, b, g_kind, g_amp, g_scale, K, D=1.0, lam=0.0,
        offspring=OFFSPRING_ABS, precision=PREC_FP64, strategy=STRAT_POTENTIAL, q=0.5,
        coef_kind=None, coef_axis=0, coef_scale=1.0, coef_t0=0.1, shared=0) -> dict:
    """Equation parameters (the fields of rt_eq_params / or_params).

    strategy: 0 exponential clock with potential -λu; 1 Strategy A with the
    shift u = v e^{λt}; 2 Strategy B (q = P(leaf)).  coef_kind[k] = 1 makes the
    coefficient of u^k variable: b_k exp(-x_a²/s²)/(t + t0) (Example 5).
    shared = 1: every node sees the same trees (NEXT row f4)."""
    bb = list(b) + [0.0] * (9 - len(b))
    ck = list(coef_kind) + [0] * (9 - len(coef_kind)) if coef_kind else [0] * 9
    return dict(dim=dim, D=D, degree=len(b) - 1, b=bb, lam=lam,
                offspring=offspring, init_kind=g_kind, init_amp=g_amp,
                init_scale=g_scale, K=K, precision=precision, strategy=strategy, q=q,
                coef_kind=ck, coef_axis=coef_axis, coef_scale=coef_scale, coef_t0=coef_t0,
                shared=shared)


# BASELINE.json "configs".  b = (b_0, b_1, ...) with
# f(u) = sum_k b_k u^k.
B_KPP = (0.0, -1.0, 1.0)                       # cfg1: f = u^2 - u
B_CFG2 = (0.0, -1.0, 0.5, 0.8, -0.3)           # cfg2/3/5
B_CFG4 = (0.0, -1.0, 0.3, 0.3, 0.0, 0.2)       # cfg4

_CFG4_PLANES = [dict(axis=a, value=0.0, lo=-2.0, hi=2.0, n_per_dim=19)
                for a in range(3)]
_CFG3_PLANES = [dict(axis=a, value=0.0, lo=-2.0, hi=2.0, n_per_dim=128)
                for a in range(2)]

CONFIGS: Dict[str, dict] = {
    "cfg1": dict(eq=_eq(1, B_KPP, G_TANH_STEP, 1.0, 1.0, K=12), t=0.5,
                 nodes=dict(kind="linspace", lo=-2.0, hi=2.0, n=16),
                 n_trees=10_000, seed=0, L=5, M=5),
    "cfg1_const": dict(eq=_eq(1, B_KPP, G_CONST, 0.3, 1.0, K=12), t=0.5,
                       nodes=dict(kind="linspace", lo=-2.0, hi=2.0, n=16),
                       n_trees=10_000, seed=0, L=5, M=5),
    "cfg2": dict(eq=_eq(1, B_CFG2, G_GAUSS, 0.4, 1.0, K=12), t=1.0,
                 nodes=dict(kind="linspace", lo=-3.0, hi=3.0, n=64),
                 n_trees=1_000_000, seed=0, L=5, M=5),
    "cfg3": dict(eq=_eq(2, B_CFG2, G_GAUSS, 0.5, 1.0, K=12), t=0.5,
                 nodes=dict(kind="planes", planes=_CFG3_PLANES, max_points=256),
                 n_trees=1_000_000, seed=0, L=5, M=5),
    "cfg4": dict(eq=_eq(3, B_CFG4, G_LORENTZ, 0.5, 1.0, K=16), t=1.0,
                 nodes=dict(kind="planes", planes=_CFG4_PLANES, max_points=1024),
                 n_trees=10_000_000, seed=0, L=7, M=7),
}

# NEXT rows f2 / f3: the paper's Examples
# on the same node layouts, Strategy A with the
# e^{λt} shift and Strategy B (q = 2/3, inside the admissible range q >= 1/2
# of a single quadratic term).  Examples 1-2 data read at t = 0
# (SURVEY C16): e^{-x^2/4}/sqrt(4 pi) = Gaussian with amp 1/sqrt(4 pi), scale 2.
_GN = 1.0 / (4.0 * 3.141592653589793) ** 0.5
_EX1 = dict(b=(0.0, 0.0, -1.0), g=(G_GAUSS, _GN, 2.0))
# Example 2: u_t = u_xx + u^2, negative data -6 e^{-x^2/4}/sqrt(4 pi),
# |u0| > 1 at the origin
_EX2 = dict(b=(0.0, 0.0, 1.0), g=(G_GAUSS, -6.0 * _GN, 2.0))
_EX3 = dict(b=(0.0, 0.0, -1.25, -1.0), g=(G_TANH_STEP, 1.0, 2.0 * 2.0 ** 0.5))
_EX5 = dict(coef_kind=[0, 0, 1], coef_axis=0, coef_scale=1.0, coef_t0=0.1)
for _s, _tag in ((STRAT_A_SHIFT, "A"), (STRAT_B, "B")):
    CONFIGS[f"ex1{_tag}"] = dict(eq=_eq(1, _EX1["b"], *_EX1["g"], K=12, strategy=_s, q=2.0 / 3.0),
                                t=0.5, nodes=dict(kind="linspace", lo=-3.0, hi=3.0, n=64),
                                n_trees=1_000_000, seed=0, L=5, M=5)
    CONFIGS[f"ex2{_tag}"] = dict(eq=_eq(1, _EX2["b"], *_EX2["g"], K=12, strategy=_s, q=2.0 / 3.0),
                                t=0.5, nodes=dict(kind="linspace", lo=-3.0, hi=3.0, n=64),
                                n_trees=1_000_000, seed=0, L=5, M=5)
    CONFIGS[f"ex3{_tag}"] = dict(eq=_eq(1, _EX3["b"], *_EX3["g"], K=12, strategy=_s, q=0.75),
                                t=0.5, nodes=dict(kind="linspace", lo=-3.0, hi=3.0, n=64),
                                n_trees=1_000_000, seed=0, L=5, M=5)
    CONFIGS[f"ex5{_tag}"] = dict(eq=_eq(2, _EX1["b"], *_EX1["g"], K=12, strategy=_s, q=2.0 / 3.0, **_EX5),
                                t=0.5, nodes=dict(kind="planes", planes=_CFG3_PLANES, max_points=256),
                                n_trees=1_000_000, seed=0, L=5, M=5)

# NEXT row f4: the BASELINE configs with shared trees (every node sees the
# same trees) — a different sampling contract, same per-node law.
for _n in ("cfg2", "cfg3", "cfg4"):
    _c = copy.deepcopy(CONFIGS[_n])
    _c["eq"]["shared"] = 1
    CONFIGS[_n + "_sh"] = _c

# cfg5: throughput sweep on the cfg2 equation (BASELINE.json configs[4]).
CFG5_NODES = (64, 1024, 16384)
CFG5_TREES = (10_000, 1_000_000, 10_000_000)
CFG5_T = (0.25, 1.0, 2.0)


def cfg5(n_nodes: int, n_trees: int, t: float, fp32_pos: bool = False) -> dict:
    return dict(eq=_eq(1, B_CFG2, G_GAUSS, 0.4, 1.0, K=12,
                       precision=PREC_FP32_POS if fp32_pos else PREC_FP64),
                t=t, nodes=dict(kind="linspace", lo=-3.0, hi=3.0, n=n_nodes),
                n_trees=n_trees, seed=0, L=5, M=5)


def get(name: str, **overrides) -> dict:
    cfg = copy.deepcopy(CONFIGS[name])
    for k, v in overrides.items():
        if k in cfg["eq"]:
            cfg["eq"][k] = v
        else:
            cfg[k] = v
    return cfg


def nodes(cfg: dict) -> np.ndarray:
    """[n, d] float64 node coordinates of a config."""
    spec = cfg["nodes"]
    d = cfg["eq"]["dim"]
    if spec["kind"] == "linspace":
        x = linspace(spec["lo"], spec["hi"], spec["n"])
        return np.ascontiguousarray(x.reshape(-1, 1)) if d == 1 else \
            np.ascontiguousarray(np.column_stack([x] + [np.zeros_like(x)] * (d - 1)))
    if spec["kind"] == "planes":
        return plane_nodes(d, spec["planes"], spec["max_points"])
    if spec["kind"] == "explicit":
        return np.ascontiguousarray(np.asarray(spec["points"], dtype=np.float64).reshape(-1, d))
    raise ValueError(spec["kind"])


def random_nodes(n: int, dim: int, seed: int, lo: float = -3.0, hi: float = 3.0) -> np.ndarray:
    """Seeded uniform nodes (parity cases off the configs' grids)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=(n, dim)).astype(np.float64)
