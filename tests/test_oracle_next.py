"""Pins of the oracle's NEXT-row extensions (
DESIGN.md §10) against mathematics other than itself:

  Strategy A shift u = v e^{λt}:
     the per-order coefficients of the Duhamel/Picard expansion of
     u' = z f(u) — closed forms for f = b_2 u^2 with constant data;
     Examples 1-3 equations against finite differences.
  Strategy B: the same per-order closed forms (B expands
     the same Duhamel series), the law of the tree structure
     P(Ne = n) = q^{n+1} (1-q)^n Catalan(n) for binary trees (Eq. pk with
     N_D(k, 2) = Catalan; k = 4, Ne = 3 gives the 5 trees
     of Fig. bbm_k4_Ne3), finite differences for Examples 1-3.
  Variable coefficients c(x,t) = b e^{-x_a^2/s^2}/(t + t0) (Example 5,
     PAPER.md:1084-1088): a time-only closed form (s -> large) and a 1-D
     finite-difference solve with the space-time dependent reaction.

A plausible mistake — the e^{(k-1)τ} factor on the parent's instead of the
child's horizon, a missing e^{λt}, η(τ) = τ(1-S) instead of τ, g/q or
c/(1-q) dropped, the coefficient's time argument off — moves an estimate by
many standard errors in at least one of these."""
import math

import numpy as np
import pytest
from scipy import stats

import closed_forms as cf
import workloads as W

Z = 4.0
GAUSS_NORM = 1.0 / math.sqrt(4.0 * math.pi)       # Examples 1-2: e^{-x^2/4}/sqrt(4 pi)


def _eq(b, strategy, g_kind=W.G_CONST, amp=0.3, scale=1.0, K=12, **kw):
    return W._eq(1, b, g_kind, amp, scale, K=K, strategy=strategy, **kw)


@pytest.mark.parametrize("strategy,q", [(W.STRAT_A_SHIFT, 0.5), (W.STRAT_B, 0.6), (W.STRAT_B, 0.75)])
@pytest.mark.parametrize("b2,u0,t", [(-1.0, 0.3, 0.5), (1.0, -0.4, 0.7), (0.8, 0.5, 0.4)])
def test_constant_data_orders(orc, strategy, q, b2, u0, t):
    """u' = z b2 u^2, u(0) = u0: u_z = u0/(1 - z b2 u0 t), c_n = u0 (b2 u0 t)^n.
    Both the shift form and Strategy B sample this Duhamel series."""
    eq = _eq((0.0, 0.0, b2), strategy, amp=u0, q=q)
    c, se, us, ses, _ = orc.estimate(eq, np.array([[0.0], [1.3]]), t, 60_000, seed=11)
    exact = np.array([u0 * (b2 * u0 * t) ** n for n in range(eq["K"] + 1)])
    for i in range(2):
        z = (c[i] - exact) / np.maximum(se[i], 1e-300)
        assert np.all(np.abs(z[:6]) < Z), z[:6]
    tot = u0 / (1.0 - b2 * u0 * t)
    assert abs(us[1] - tot) < Z * ses[1] + 1e-9


def test_shift_matches_potential_form(orc):
    """The shift form and the potential form (λ = 1 with a k = 1 offspring of
    weight 1) estimate the same u for Example 1's equation, at nodes 0 and 1."""
    b = (0.0, 0.0, -1.0)
    pts = np.array([[0.0], [1.0]])
    shift = _eq(b, W.STRAT_A_SHIFT, W.G_GAUSS, GAUSS_NORM, 2.0)
    pot = _eq(b, W.STRAT_POTENTIAL, W.G_GAUSS, GAUSS_NORM, 2.0, lam=1.0)
    _, _, ua, sa, _ = orc.estimate(shift, pts, 0.5, 80_000, seed=3)
    _, _, ub, sb, _ = orc.estimate(pot, pts, 0.5, 80_000, seed=4)
    assert np.all(np.abs(ua - ub) < Z * np.hypot(sa, sb))


def _fd(b, g, t, xs):
    return cf.fd_at(b, g, t, xs, dx=0.02, dt=1e-3)


EXAMPLES = {
    # Example 1: u_t = u_xx - u^2, u0 = e^{-x^2/4}/sqrt(4 pi)
    "ex1": ((0.0, 0.0, -1.0), W.G_GAUSS, GAUSS_NORM, 2.0, 0.5),
    # Example 2: u_t = u_xx + u^2, u0 = -6 e^{-x^2/4}/sqrt(4 pi)
    "ex2": ((0.0, 0.0, 1.0), W.G_GAUSS, -6.0 * GAUSS_NORM, 2.0, 0.25),
    # Example 3: u_t = u_xx - 1.25 u^2 - u^3, u0 = 1/(1 + e^{-x/sqrt 2})
    #            = 0.5 (1 + tanh(x / (2 sqrt 2)))
    "ex3": ((0.0, 0.0, -1.25, -1.0), W.G_TANH_STEP, 1.0, 2.0 * math.sqrt(2.0), 0.2),
}


def _g(kind, amp, scale):
    if kind == W.G_GAUSS:
        return lambda x: amp * np.exp(-x * x / scale ** 2)
    return lambda x: amp * 0.5 * (1.0 + np.tanh(x / scale))


@pytest.mark.parametrize("ex", list(EXAMPLES))
@pytest.mark.parametrize("strategy", [W.STRAT_A_SHIFT, W.STRAT_B])
def test_examples_against_fd(orc, ex, strategy):
    b, kind, amp, scale, t = EXAMPLES[ex]
    xs = np.array([-1.0, 0.0, 1.5])
    eq = _eq(b, strategy, kind, amp, scale, K=14, q=0.6)
    _, _, us, ses, _ = orc.estimate(eq, xs[:, None], t, 40_000, seed=5)
    ref = _fd(b, _g(kind, amp, scale), t, xs)
    z = (us - ref) / ses
    assert np.all(np.abs(z) < Z), (us, ref, z)


def test_strategy_b_tree_law(orc):
    """Binary trees of Strategy B: P(Ne = n) = q̂^{n+1} (1-q̂)^n Catalan(n)
    (Eq. pk with N_D(k, 2) = Catalan; the 5 = Catalan(3)
    trees with k = 4, Ne = 3 of Fig. bbm_k4_Ne3), chi-square at q = 0.6."""
    eq = _eq((0.0, 0.0, 1.0), W.STRAT_B, q=0.6, K=30)
    qh = orc.normalize(eq)["q_hat"]
    rec = orc.trees(eq, np.array([[0.0]]), 1.0, 200_000, seed=21)[0]
    ne = rec["ne"][rec["pruned"] == 0]
    nmax = 12
    obs = np.array([np.sum(ne == n) for n in range(nmax)] + [np.sum(ne >= nmax) + np.sum(rec["pruned"])])
    p = np.array([qh ** (n + 1) * (1 - qh) ** n * cf.catalan(n) for n in range(nmax)])
    p = np.append(p, 1.0 - p.sum())
    e = p * rec.size
    keep = e > 20
    o2, e2 = obs[keep], e[keep]
    if e[~keep].sum() > 0:
        o2 = np.append(o2, obs[~keep].sum())
        e2 = np.append(e2, e[~keep].sum())
    chi2 = float(np.sum((o2 - e2) ** 2 / e2))
    assert stats.chi2.sf(chi2, len(o2) - 1) > 1e-3, chi2
    # leaves = Ne + 1 for binary trees, and P(Ne = 3) carries Catalan(3) = 5
    assert np.all(rec["leaves"][rec["pruned"] == 0] == ne + 1)
    assert abs(obs[3] / rec.size - 5 * qh ** 4 * (1 - qh) ** 3) < Z * math.sqrt(p[3] / rec.size)


@pytest.mark.parametrize("strategy", [W.STRAT_A_SHIFT, W.STRAT_B])
def test_variable_coefficient_time_only(orc, strategy):
    """c(x,t) = -e^{-x^2/s^2}/(t + t0) with s = 1e4 (x-independent to 1e-8)
    and constant data: u' = -z u^2/(t + t0) gives
    c_n = u0 (-u0 ln((t + t0)/t0))^n."""
    u0, t, t0 = 0.4, 0.6, 0.1
    eq = _eq((0.0, 0.0, -1.0), strategy, amp=u0, q=0.6, coef_kind=[0, 0, 1],
             coef_scale=1e4, coef_t0=t0)
    c, se, us, ses, _ = orc.estimate(eq, np.array([[0.5]]), t, 80_000, seed=8)
    L = math.log((t + t0) / t0)
    exact = np.array([u0 * (-u0 * L) ** n for n in range(eq["K"] + 1)])
    z = (c[0] - exact) / np.maximum(se[0], 1e-300)
    assert np.all(np.abs(z[:6]) < Z), z[:6]


@pytest.mark.parametrize("strategy", [W.STRAT_A_SHIFT, W.STRAT_B])
def test_variable_coefficient_fd(orc, strategy):
    """Example 5's coefficient in 1-D:
    u_t = u_xx - e^{-x^2}/(t + 0.1) u^2, u0 = e^{-x^2/4}/sqrt(4 pi), t = 0.5,
    against finite differences with the space-time dependent reaction."""
    t = 0.5
    eq = _eq((0.0, 0.0, -1.0), strategy, W.G_GAUSS, GAUSS_NORM, 2.0, K=14, q=0.6,
             coef_kind=[0, 0, 1], coef_scale=1.0, coef_t0=0.1)
    xs = np.array([-0.7, 0.0, 1.2])
    _, _, us, ses, _ = orc.estimate(eq, xs[:, None], t, 40_000, seed=9)
    x, u = cf.fd_solve_1d_xt(lambda v, xx, tt: -np.exp(-xx * xx) / (tt + 0.1) * v * v,
                             lambda xx: GAUSS_NORM * np.exp(-xx * xx / 4.0), t, dx=0.02, dt=1e-3)
    ref = np.interp(xs, x, u)
    z = (us - ref) / ses
    assert np.all(np.abs(z) < Z), (us, ref, z)


def test_invalid_strategy_parameters(orc):
    for kw in (dict(strategy=3), dict(strategy=W.STRAT_B, q=0.0), dict(strategy=W.STRAT_B, q=1.0),
               dict(strategy=W.STRAT_POTENTIAL, coef_kind=[0, 1]),
               dict(strategy=W.STRAT_A_SHIFT, coef_kind=[0, 0, 1], coef_t0=0.0)):
        with pytest.raises(ValueError):
            orc.normalize(_eq((0.0, 0.0, -1.0), **kw))


# ---------------------------------------------------------------------------
# NEXT row f4: shared trees (common random numbers across nodes)
def test_shared_trees_structure_is_node_independent(orc):
    """Every node sees the same trees: structure records identical across
    nodes, and with constant data identical contributions."""
    eq = W._eq(1, W.B_CFG2, W.G_CONST, 0.4, 1.0, K=12, shared=1)
    pts = np.array([[-2.0], [0.0], [0.3], [2.5]])
    rec = orc.trees(eq, pts, 1.0, 3_000, seed=4)
    for f in ("ne", "leaves", "particles", "pruned"):
        assert np.all(rec[f] == rec[f][0:1]), f
    assert np.all(rec["C"] == rec["C"][0:1])


def test_shared_trees_translation(orc):
    """For a tree with one leaf (Ne = 0) C_i = g(x_i + δ): with Gaussian data
    log C_i = log A - (x_i + δ)^2, so δ recovered from two nodes predicts C at a
    third (the leaves are evaluated at x_i + a common displacement)."""
    eq = W._eq(1, (0.0, -1.0, 0.5), W.G_GAUSS, 1.0, 1.0, K=12, shared=1)
    pts = np.array([[0.0], [1.0], [-0.7]])
    rec = orc.trees(eq, pts, 0.6, 2_000, seed=9)
    one = rec["ne"][0] == 0
    c0, c1, c2 = (rec["C"][i][one] for i in range(3))
    # -(x+δ)^2: log c0 - log c1 = (1+δ)^2 - δ^2 = 1 + 2δ
    delta = (np.log(c0) - np.log(c1) - 1.0) / 2.0
    assert np.allclose(np.log(c2), -(-0.7 + delta) ** 2, rtol=0, atol=1e-9)


@pytest.mark.parametrize("strategy", [W.STRAT_POTENTIAL, W.STRAT_A_SHIFT, W.STRAT_B])
def test_shared_trees_same_law(orc, strategy):
    """Per node the estimator is unchanged in law: shared-tree estimates of the
    Example-1 equation agree with finite differences within 4 s.e."""
    b, kind, amp, scale, t = EXAMPLES["ex1"]
    xs = np.array([-1.0, 0.0, 0.8])
    eq = _eq(b, strategy, kind, amp, scale, K=14, q=0.6, shared=1,
             lam=1.0 if strategy == W.STRAT_POTENTIAL else 0.0)
    _, _, us, ses, _ = orc.estimate(eq, xs[:, None], t, 40_000, seed=6)
    ref = _fd(b, _g(kind, amp, scale), t, xs)
    assert np.all(np.abs(us - ref) < Z * ses), (us, ref)


def test_shared_trees_heat_kernel_2d(orc):
    """Linear f = -u (no offspring): c_0(x) = e^{-t} E g(x + sqrt(2t) Z) is the
    heat kernel at every node, d = 2."""
    import closed_forms as cfm
    eq = W._eq(2, (0.0, -1.0), W.G_GAUSS, 0.4, 1.0, K=4, shared=1)
    pts = np.array([[0.0, 0.0], [0.5, -0.4], [1.2, 0.3]])
    c, se, *_ = orc.estimate(eq, pts, 1.0, 100_000, seed=12)
    ref = cfm.heat(pts, 1.0, 1.0, 1.0, 0.4)
    assert np.all(np.abs(c[:, 0] - ref) < Z * se[:, 0]), (c[:, 0], ref)


def test_shared_rejects_variable_coefficients(orc):
    with pytest.raises(ValueError):
        orc.normalize(_eq((0.0, 0.0, -1.0), W.STRAT_A_SHIFT, shared=1, coef_kind=[0, 0, 1]))


def test_strategy_b_ternary_law_and_mean_leaves(orc):
    """m = 3 single term (Fig. pkcompare's m = 3 case): a tree
    with Ne splits has 2Ne + 1 leaves and there are FussCatalan(Ne) =
    C(3Ne, Ne)/(2Ne + 1) of them, so P(Ne = n) = q^{2n+1} (1-q)^n C(3n,n)/(2n+1);
    mean leaves (Eq. aproxTb2 context) = q/(1 - m(1-q)) for
    the unpruned law (q = 0.8 > (m-1)/m keeps it finite)."""
    from math import comb
    q = 0.8
    eq = _eq((0.0, 0.0, 0.0, 1.0), W.STRAT_B, q=q, K=40)
    qh = orc.normalize(eq)["q_hat"]
    rec = orc.trees(eq, np.array([[0.0]]), 1.0, 200_000, seed=23)[0]
    assert np.all(rec["leaves"][rec["pruned"] == 0] == 2 * rec["ne"][rec["pruned"] == 0] + 1)
    nmax = 8
    p = np.array([qh ** (2 * n + 1) * (1 - qh) ** n * comb(3 * n, n) / (2 * n + 1) for n in range(nmax)])
    obs = np.array([np.sum((rec["ne"] == n) & (rec["pruned"] == 0)) for n in range(nmax)])
    z = (obs - rec.size * p) / np.sqrt(rec.size * p * (1 - p))
    assert np.all(np.abs(z) < Z), z
    mean_leaves = qh / (1.0 - 3.0 * (1.0 - qh))
    se = rec["leaves"].std() / np.sqrt(rec.size)
    assert abs(rec["leaves"].mean() - mean_leaves) < Z * se + 1e-3, (rec["leaves"].mean(), mean_leaves)
