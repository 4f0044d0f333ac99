"""Pins of the oracle's random-number layer (reading R1, R8).

* Philox4x32-10 against the Random123 known-answer vectors (golden file) and
  against PyTorch's host-callable at::philox_engine (a library routine).
* unif53 against its exact end points and bit-level definition.
* The exponential clock and Box–Muller normals of the oracle's trees against
  their laws (E[S] = 1/λ; Var(displacement) = 2Dh).
"""
import math
import os
import subprocess

import numpy as np
import pytest
from scipy import stats

HERE = os.path.dirname(os.path.abspath(__file__))


def _kat():
    rows = []
    for line in open(os.path.join(HERE, "golden", "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(w, 16) for w in line.split()]
        rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answers(orc):
    for ctr, key, out in _kat():
        assert list(orc.philox(key, ctr)) == out


@pytest.fixture(scope="module")
def torch_philox(tmp_path_factory):
    import torch
    inc = os.path.join(os.path.dirname(torch.__file__), "include")
    exe = str(tmp_path_factory.mktemp("tp") / "torch_philox")
    subprocess.check_call(["g++", "-O1", "-std=c++17", "-I" + inc,
                           os.path.join(HERE, "helpers", "torch_philox.cpp"), "-o", exe])
    return exe


def test_philox_matches_torch_engine(orc, torch_philox):
    rng = np.random.default_rng(1234)
    rows = rng.integers(0, 2 ** 32, size=(200, 6), dtype=np.uint64)
    rows[:20, 3] = 0                      # include small counters too
    inp = "\n".join(" ".join(str(int(v)) for v in r) for r in rows) + "\n"
    out = subprocess.run([torch_philox], input=inp, capture_output=True, text=True,
                         check=True).stdout.split("\n")
    for r, line in zip(rows, out):
        ref = [int(w) for w in line.split()]
        got = list(orc.philox([r[0], r[1]], [r[2], r[3], r[4], r[5]]))
        assert got == ref


def test_unif53_exact(orc):
    assert orc.unif53(0, 0) == 2.0 ** -53
    assert orc.unif53(0xFFFFFFFF, 0xFFFFFFFF) == 1.0 - 2.0 ** -53
    # 2*(x>>12)+1 over 2^53 for an arbitrary word pair
    lo, hi = 0x89ABCDEF, 0x01234567
    x = (hi << 32) | lo
    assert orc.unif53(lo, hi) == (2 * (x >> 12) + 1) / 2.0 ** 53
    assert 0.0 < orc.unif53(0, 0) < orc.unif53(0xFFFFFFFF, 0xFFFFFFFF) < 1.0


def test_unif32_exact(orc):
    """32-bit uniforms (the d = 3 Box–Muller angles, R8): (2w+1)/2^33."""
    assert orc.unif32(0) == 2.0 ** -33
    assert orc.unif32(0xFFFFFFFF) == 1.0 - 2.0 ** -33
    assert orc.unif32(12345) == (2 * 12345 + 1) / 2.0 ** 33


def test_root_particle_laws(orc):
    """Root lifetime S ~ Exp(λ) and Gaussian displacement over min(S, t).

    With f = -u (b = (0,-1), λ = 1, empty support) every tree is the root
    particle alone: it is a leaf iff S > t.  P(leaf) = e^{-λt} and, for
    constant g, c_0 = A e^{-λt}; the displacement of a leaf over h = t has
    variance 2Dt — checked through Gaussian data, where
    E[g(x + sqrt(2Dt) ξ)] has the closed form of tests/closed_forms.heat."""
    eq = dict(dim=1, D=1.0, degree=1, b=[0.0, -1.0] + [0.0] * 7, lam=0.0, offspring=0,
              init_kind=0, init_amp=1.0, init_scale=1.0, K=4)
    t, N = 0.7, 200_000
    rec = orc.trees(eq, np.zeros((1, 1)), t, N, seed=5)[0]
    leaf = rec["ne"] == 0
    p = math.exp(-t)
    assert abs(leaf.mean() - p) < 4 * math.sqrt(p * (1 - p) / N)
    assert np.all(rec["ne"][~leaf] == 1) and np.all(rec["C"][~leaf] == 0.0)
    assert np.all(rec["particles"] == 1)


def test_box_muller_normality(orc):
    """Leaves of linear-f trees at x = 0 with g(x) = exp(-x^2/s^2) sample
    exp(-(sqrt(2Dt) ξ)^2/s^2).  Recover ξ² = -s² log(g) / (2Dt) and test it
    against the chi-square(1) law (KS), i.e. ξ is standard normal in |ξ|."""
    D, t, s = 0.5, 1.0, 3.0
    eq = dict(dim=1, D=D, degree=1, b=[0.0, -1e-9] + [0.0] * 7, lam=0.0, offspring=0,
              init_kind=2, init_amp=1.0, init_scale=s, K=4)
    rec = orc.trees(eq, np.zeros((1, 1)), t, 40_000, seed=11)[0]
    leaf = rec["ne"] == 0
    xi2 = -s * s * np.log(rec["C"][leaf]) / (2 * D * t)
    assert leaf.mean() > 0.99
    assert stats.kstest(xi2, stats.chi2(1).cdf).pvalue > 1e-3


@pytest.mark.parametrize("dim", [2, 3])
def test_box_muller_multid(orc, dim):
    """Same as above in d = 2, 3: |ξ|² ~ chi-square(d) (independent components,
    the d = 3 layout draws a second Philox block, R8)."""
    D, t, s = 0.5, 1.0, 3.0
    eq = dict(dim=dim, D=D, degree=1, b=[0.0, -1e-9] + [0.0] * 7, lam=0.0, offspring=0,
              init_kind=2, init_amp=1.0, init_scale=s, K=4)
    rec = orc.trees(eq, np.zeros((1, dim)), t, 40_000, seed=13)[0]
    leaf = rec["ne"] == 0
    r2 = -s * s * np.log(rec["C"][leaf]) / (2 * D * t)
    assert stats.kstest(r2, stats.chi2(dim).cdf).pvalue > 1e-3


@pytest.mark.parametrize("dim", [1, 2, 3])
def test_clock_and_radii_independent(orc, dim):
    """DESIGN.md R29 draws the clock and the Box–Muller radii from ONE Gamma
    variate split by uniform spacings; they must still be independent.  With
    λ = 1 and t = 1 a root particle is a leaf iff its clock exceeds t
    (probability e^{-1}); among those leaves the displacement must remain
    sqrt(2Dt) ξ with |ξ|² ~ chi-square(d) — a radius correlated with the
    clock (e.g. sharing e0) would be inflated exactly on this event."""
    D, t, s = 0.5, 1.0, 3.0
    eq = dict(dim=dim, D=D, degree=1, b=[0.0, -1.0] + [0.0] * 7, lam=0.0, offspring=0,
              init_kind=2, init_amp=1.0, init_scale=s, K=4)
    rec = orc.trees(eq, np.zeros((1, dim)), t, 60_000, seed=17 + dim)[0]
    leaf = rec["ne"] == 0
    p = math.exp(-t)
    assert abs(leaf.mean() - p) < 4 * math.sqrt(p * (1 - p) / len(leaf))
    r2 = -s * s * np.log(rec["C"][leaf]) / (2 * D * t)
    assert stats.kstest(r2, stats.chi2(dim).cdf).pvalue > 1e-3
