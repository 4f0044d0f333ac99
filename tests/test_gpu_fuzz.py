"""Randomised GPU parity: seeded random equations through the C ABI against
the CPU oracle, tree by tree (structure bit-exact, C to 1e-12) and per
(node, order bin) sums — the same bar as test_gpu_parity.test_tree_parity.

The hand-picked cases there follow the paper's examples and the
BASELINE.json configs; these draws reach the combinations none of them
picks: degrees up to 8 with up to eight offspring kinds (the kernel's
n_support > 5 threshold path, k = 8 children, label step β = 3), k = 0 and
k = 1 offspring, λ overrides, the uniform offspring rule, every initial-data
shape with negative and |g| > 1 amplitudes, variable coefficients under all
three strategies, shared trees, empty supports, K from 0 to the label-width
limit 1 + Kβ <= 56 (PAPER.md:90-101 normalisation, 197-239 the walk,
259-293 the weights, 304-357 Strategy B, 759-765 pruning).

The generator draws inputs only (coefficients, shapes, sizes); it holds none
of the method's arithmetic.
"""
import numpy as np
import pytest

import workloads as W
from test_gpu_parity import P, abs_sums, assert_nodes_close, assert_sum_c_close, assert_trees_equal, dev  # noqa: F401 (P: fixture)

N_CASES = 48


def fuzz_case(seed: int):
    """One random (equation, nodes, t, N) inside rt_create's contract (rt.h)."""
    r = np.random.default_rng(1000 + seed)
    dim = int(r.integers(1, 4))
    degree = int(r.integers(1, 9))
    b = r.uniform(-1.2, 1.2, degree + 1)
    for k in range(degree + 1):
        if k != 1 and r.random() < 0.35:
            b[k] = 0.0
    if r.random() < 0.5:
        b[degree] = r.choice([-1.0, 1.0]) * r.uniform(0.2, 1.2)   # keep the top degree often
    strategy = int(r.choice([W.STRAT_POTENTIAL, W.STRAT_POTENTIAL, W.STRAT_A_SHIFT, W.STRAT_B]))
    lam = float(r.uniform(0.5, 2.0)) if r.random() < 0.3 else 0.0
    offspring = int(r.integers(0, 2))
    g_kind = int(r.integers(0, 4))
    amp = float(r.choice([-1.0, 1.0]) * r.uniform(0.1, 1.6))
    scale = float(r.uniform(0.6, 2.0))
    shared = int(r.random() < 0.25)
    coef_kind = [0] * 9
    if not shared and r.random() < 0.35:
        for k in range(degree + 1):
            if b[k] != 0.0 and (k >= 2 or (k == 1 and strategy != W.STRAT_POTENTIAL)) and r.random() < 0.6:
                coef_kind[k] = 1
    kmax = max([k for k in range(2, degree + 1) if b[k] != 0.0] + [1])
    beta = max(1, int(np.ceil(np.log2(kmax))))
    K = int(r.integers(0, min(16, 55 // beta) + 1))
    eq = W._eq(dim, tuple(float(v) for v in b), g_kind, amp, scale, K=K, D=float(r.uniform(0.3, 1.5)),
               lam=lam, offspring=offspring, strategy=strategy, q=float(r.uniform(0.45, 0.85)),
               coef_kind=coef_kind, coef_axis=int(r.integers(0, dim)), coef_scale=float(r.uniform(0.8, 2.0)),
               coef_t0=float(r.uniform(0.1, 0.5)), shared=shared)
    n = int(r.integers(2, 9))
    pts = r.uniform(-2.0, 2.0, (n, dim))
    t = float(r.uniform(0.3, 2.0))
    N = int(r.integers(300, 1500))
    return eq, pts, t, N


def test_generator_reaches_the_rare_paths():
    """The draws cover what they are for (checked on the inputs alone)."""
    cases = [fuzz_case(s)[0] for s in range(N_CASES)]
    nsup = [sum(1 for k in range(e["degree"] + 1) if e["b"][k] != 0.0 and k != 1) for e in cases]
    assert max(nsup) >= 6                                    # > 5 offspring kinds (+ maybe k = 1)
    assert any(e["degree"] == 8 and e["b"][8] != 0.0 for e in cases)
    assert any(e["b"][0] != 0.0 for e in cases)              # k = 0 offspring
    assert {e["strategy"] for e in cases} == {0, 1, 2}
    assert any(e["shared"] for e in cases) and any(any(e["coef_kind"]) for e in cases)
    assert any(e["K"] == 0 for e in cases) or any(e["K"] <= 2 for e in cases)
    assert {e["init_kind"] for e in cases} == {0, 1, 2, 3}


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(N_CASES))
def test_fuzz_tree_parity(P, orc, seed):
    eq, pts, t, N = fuzz_case(seed)
    est = P.Estimator(eq)
    rec, sums = est.trace(dev(pts), t, N, seed=4242 + seed)
    ref = orc.trees(eq, pts, t, N, seed=4242 + seed)
    assert_trees_equal(rec, ref, eq["K"])
    s_ref, st_ref = orc.sums(eq, pts, t, N, seed=4242 + seed)
    s_gpu = sums.cpu().numpy()
    assert np.array_equal(s_gpu[:, :, 2], s_ref[:, :, 2]), "bin counts differ"
    assert_sum_c_close(s_gpu[:, :, 0], s_ref[:, :, 0], abs_sums(ref, eq["K"]))
    assert_nodes_close(s_gpu[:, :, 1], s_ref[:, :, 1], what="sum C^2")
    st = est.stats()
    assert st["trees"] == st_ref["trees"] and st["pruned"] == st_ref["pruned"]
    assert st["splits"] == st_ref["splits"]
