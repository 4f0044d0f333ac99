"""Pins of the oracle's Strategy-A SAMPLING (R29) against mathematics
other than itself.

R29 draws a particle's exponential clock and the radii of
its Box–Muller increments from ONE Gamma(m+1) variate split
by the spacings of m sorted uniforms.  Its laws are exact (Beta–Gamma
algebra), but checking that by eye needs the identity, so these tests pin it
from three sides, each naming the plausible mistakes it catches (every one was
checked by mutating rt_oracle.c and watching the test fail):

* test_poisson_bins_multid — a k = 1 offspring at rate 1 makes the splits of a
  tree a Poisson process along ONE Brownian path, so the order-n coefficient
  is e^{-t}(a t)^n/n! x heat(x, t) in every dimension.  Orders n >= 1 are
  built from increments over split lifetimes (the clock's own event), which
  the root-leaf pins of test_oracle_rng.py never see.  Catches: a radius that
  reuses the clock's share (e1 := e0), a spacing taken from unsorted words
  (d = 3: e1 = G(v2 - v1) < 0), a wrong spacing (e2 := G(1 - v1)), the
  increment over τ instead of min(S, τ).
* test_lorentzian_scale — cfg4's initial data g = A/(1 + |x|²/s²)
   at s != 1 in d = 1, 2, 3 against a closed-form integral
  of the heat kernel (closed_forms.lorentz_heat).  Catches a dropped /s² (at
  s = 1, the only scale cfg4 uses, that mistake is invisible).
* test_r29_equals_textbook_in_law — the oracle's textbook mode (sampling = 1:
  S = -ln(u)/λ by inversion and r = sqrt(-2 ln v), 53-bit uniforms; SURVEY
  §8(c)'s original definition, which shares none of R29's algebra) and R29
  estimate the same per-order coefficients c_n, second moments E[C² 1{Ne=n}]
  and order law P(Ne = n) at cfg2 and cfg4, constant and spatial data, 1e6
  trees each: per-order z-scores within 4 and pooled chi-square p > 1e-3.
"""
import math

import numpy as np
import pytest
from scipy import stats

import closed_forms as cf
import workloads as W

Z = 4.0


def _lin_eq(dim, b1, lam, kind, amp, scale, K, D=1.0):
    return dict(dim=dim, D=D, degree=1, b=[0.0, b1] + [0.0] * 7, lam=lam, offspring=0,
                init_kind=kind, init_amp=amp, init_scale=scale, K=K)


@pytest.mark.parametrize("dim,D,s", [(2, 1.0, 1.3), (3, 0.5, 0.9), (3, 1.0, 1.6)])
def test_poisson_bins_multid(orc, dim, D, s):
    """f = -0.5u with λ overridden to 1: a_1 = 0.5 is a k = 1 offspring of
    weight 0.5, the rings form a Poisson(λt) process on one Brownian path, so
    c_n = e^{-t} (0.5 t)^n / n! x E[g(x + sqrt(2Dt) Z)] for Gaussian g of
    scale s (the heat kernel without decay) — in d = 2 and 3, where R29's
    split-event radii (e1, e2 of the clock's Gamma variate) move the
    particle."""
    eq = _lin_eq(dim, -0.5, 1.0, W.G_GAUSS, 0.6, s, K=8, D=D)
    nz = orc.normalize(eq)
    assert nz["support"] == [1] and nz["w"] == [0.5]
    t, N = 1.2, 200_000
    pts = W.random_nodes(3, dim, 40 + dim)
    pts[0] = 0.0
    c, se, us, ses, st = orc.estimate(eq, pts, t, N, seed=101 + dim)
    h = cf.heat(pts, t, D, 0.0, 0.6, s)
    zs = []
    for n in range(5):
        ex = math.exp(-t) * (0.5 * t) ** n / math.factorial(n) * h
        z = (c[:, n] - ex) / se[:, n]
        assert np.all(np.abs(z) < Z), (n, z)
        zs.extend(z)
    assert stats.chi2.sf(np.sum(np.square(zs)), len(zs)) > 1e-3
    # the Poisson law of the order bins themselves (structure only)
    p = np.array([math.exp(-t) * t ** n / math.factorial(n) for n in range(9)])
    s_, _ = orc.sums(eq, pts[:1], t, N, seed=101 + dim)
    cnt = s_[0, :9, 2]
    keep = p * N > 20
    e = p[keep] * N
    o = cnt[keep]
    e = np.append(e, N - e.sum()); o = np.append(o, N - o.sum())
    assert stats.chisquare(o, e).pvalue > 1e-3


@pytest.mark.parametrize("dim,s", [(1, 0.7), (2, 1.5), (3, 0.7), (3, 1.5)])
def test_lorentzian_scale(orc, dim, s):
    """f = -u (empty support): c_0 = e^{-t} E[g(x + sqrt(2Dt) Z)] for the
    Lorentzian g = A/(1 + |x|²/s²) at s != 1 (closed_forms.lorentz_heat, the
    Laplace representation of 1/(1+a)); c_n = 0 for n >= 1."""
    eq = _lin_eq(dim, -1.0, 0.0, W.G_LORENTZ, 0.5, s, K=3)
    pts = W.random_nodes(4, dim, 60 + dim)
    pts[0] = 0.0
    t, N = 1.0, 100_000
    c, se, *_ = orc.estimate(eq, pts, t, N, seed=61)
    ex = cf.lorentz_heat(pts, t, 1.0, 1.0, 0.5, s)
    z = (c[:, 0] - ex) / se[:, 0]
    assert np.all(np.abs(z) < Z), z
    assert stats.chi2.sf(np.sum(z * z), len(z)) > 1e-3
    assert np.all(c[:, 1:] == 0.0)
    # the closed form itself: s -> the heat kernel's Gaussian limit is not
    # available, so anchor it at x = 0, d = 1 against direct quadrature
    if dim == 1:
        from scipy.integrate import quad
        v = 2.0 * t
        direct = quad(lambda y: 0.5 / (1 + y * y / s ** 2) * math.exp(-y * y / (2 * v)) /
                      math.sqrt(2 * math.pi * v), -60, 60, epsabs=1e-14, limit=400)[0]
        assert abs(cf.lorentz_heat([[0.0]], t, 1.0, 0.0, 0.5, s)[0] - direct) < 1e-12


def _moments(rec, K):
    """Per order n: sample mean of C 1{Ne=n} and of C² 1{Ne=n} with their
    standard errors, and the bin counts (pruned trees in bin K+1)."""
    C = np.where(rec["pruned"] == 1, 0.0, rec["C"])
    ne = np.where(rec["pruned"] == 1, K + 1, rec["ne"])
    N = len(C)
    out = []
    for n in range(K + 1):
        x = np.where(ne == n, C, 0.0)
        x2 = x * x
        out.append((x.mean(), x.std() / math.sqrt(N), x2.mean(), x2.std() / math.sqrt(N)))
    cnt = np.bincount(ne, minlength=K + 2)
    return np.array(out), cnt


@pytest.mark.parametrize("name,const", [("cfg2", False), ("cfg2", True), ("cfg4", False),
                                        ("cfg4", True)])
def test_r29_equals_textbook_in_law(orc, name, const):
    """R29 (the contract) and the textbook sampler are two samplings of the
    same laws: Exp(λ) clock independent of the iid N(0,1) increment
    components.  Independent streams, 1e6 trees each: the per-order means
    (all orders with >= 2000 trees in both samples) and second moments
    (orders <= 6, where C² is not heavy-tailed) agree within 4 combined
    standard errors, pooled chi-square p > 1e-3, and the order law (bin
    counts incl. the pruned bin) passes a two-sample chi-square test."""
    cfg = W.get(name)
    eq = dict(cfg["eq"])
    if const:
        eq.update(init_kind=W.G_CONST, init_amp=0.45)
    K, t, N = eq["K"], cfg["t"], 1_000_000
    x = np.full((1, eq["dim"]), 0.25)
    ra = orc.trees(eq, x, t, N, seed=2024)[0]
    rb = orc.trees(dict(eq, sampling=1), x, t, N, seed=2024)[0]
    ma, ca = _moments(ra, K)
    mb, cb = _moments(rb, K)
    zs = []
    for n in range(K + 1):
        if min(ca[n], cb[n]) < 2000:
            continue
        z1 = (ma[n, 0] - mb[n, 0]) / math.hypot(ma[n, 1], mb[n, 1])
        assert abs(z1) < Z, (n, "mean", z1)
        zs.append(z1)
        if n <= 6:
            z2 = (ma[n, 2] - mb[n, 2]) / math.hypot(ma[n, 3], mb[n, 3])
            assert abs(z2) < Z, (n, "second moment", z2)
            zs.append(z2)
    assert len(zs) >= 12
    assert stats.chi2.sf(np.sum(np.square(zs)), len(zs)) > 1e-3
    keep = (ca + cb) > 40
    table = np.array([np.append(ca[keep], ca[~keep].sum()), np.append(cb[keep], cb[~keep].sum())])
    table = table[:, table.sum(0) > 0]
    assert stats.chi2_contingency(table)[1] > 1e-3
    # the textbook mode is a genuinely different stream (not R29 relabelled)
    assert not np.array_equal(ra["C"], rb["C"])


def test_textbook_mode_rejected_for_strategy_b(orc):
    """Strategy B keeps its own textbook draws (R8); the switch is A-only."""
    eq = dict(W.get("ex3B")["eq"], sampling=1)
    with pytest.raises(ValueError):
        orc.normalize(eq)
