"""Pins of the oracle's [L/M] Padé.

* SPEC.md's fixtures and exact rational reconstructions (golden file).
* mpmath.pade at 50 digits (a library routine) on random and config-shaped
  coefficient vectors.
* The exact per-order series of the configs' constant-data ODEs resummed by
  [5/5] / [7/7] reproduces u' = f(u) (to ~1e-13).
* Flag semantics (R12): a zero pivot falls back to the largest
  regular [L/M'] with bit0 and M' in bits 8..15; |Q(1)| tiny
  -> bit1; Q changing sign on (0,1] -> bit2; Padé value more than 10 se_sum
  from the partial sum -> bit3.
"""
import math
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import closed_forms as cf
import workloads as W

HERE = os.path.dirname(os.path.abspath(__file__))


def _fixtures():
    out = []
    for line in open(os.path.join(HERE, "golden", "pade_fixtures.txt")):
        if line.startswith("#") or not line.strip():
            continue
        head, tail = line.split("|")
        L, M, val = head.split()
        c = [float(Fraction(w)) for w in tail.split()]
        out.append((int(L), int(M), float(Fraction(val)), c))
    return out


@pytest.mark.parametrize("L,M,val,c", _fixtures())
def test_pade_fixtures(orc, L, M, val, c):
    u, fl, p, q = orc.pade(c, L, M)
    assert abs(u - val) <= 1e-13 * abs(val), (u, val)
    assert fl & 1 == 0
    assert q[0] == 1.0


def _mp_pade_at1(c, L, M):
    with mpmath.workdps(50):
        p, q = mpmath.pade([mpmath.mpf(x) for x in c[: L + M + 1]], L, M)
        return float(mpmath.polyval(p[::-1], 1) / mpmath.polyval(q[::-1], 1)), p, q


@pytest.mark.parametrize("seed", range(6))
def test_pade_vs_mpmath_random(orc, seed):
    rng = np.random.default_rng(seed)
    L, M = [(1, 1), (2, 2), (3, 2), (5, 5), (2, 4), (7, 7)][seed]
    # geometric-ish decay keeps the Toeplitz system well conditioned
    c = rng.normal(size=L + M + 1) * 0.6 ** np.arange(L + M + 1)
    u, fl, p, q = orc.pade(c, L, M)
    ref, pr, qr = _mp_pade_at1(c, L, M)
    assert abs(u - ref) <= 1e-9 * max(1.0, abs(ref)), (u, ref)
    np.testing.assert_allclose(q, [float(x) for x in qr], rtol=1e-7, atol=1e-9)


@pytest.mark.parametrize("name,u0,K", [("cfg2", 0.4, 12), ("cfg4", 0.5, 16)])
def test_pade_exact_series_reproduces_ode(orc, name, u0, K):
    """[L/M] of the exact z^n coefficients of the constant-data ODE at z = 1
    equals u(t) of u' = f(u) (the configs' series are Padé-summable)."""
    cfg = W.get(name)
    b = cfg["eq"]["b"]
    a = [b[k] + (1.0 if k == 1 else 0.0) for k in range(9)]
    c = cf.ode_orders(a, 1.0, u0, cfg["t"], K)
    u, fl, _, _ = orc.pade(c, cfg["L"], cfg["M"])
    ref = cf.ode_u(b, u0, cfg["t"])
    assert abs(u - ref) < 1e-10 * abs(ref), (u, ref)
    ref_mp, _, _ = _mp_pade_at1(c, cfg["L"], cfg["M"])
    assert abs(u - ref_mp) < 1e-10 * abs(ref)


def test_pade_exact_kpp_is_degenerate(orc):
    """cfg1's exact series is geometric (type [0/1]); for M >= 2 the Toeplitz
    matrix is singular.  [1/1] and [0/1] are exact; an
    exactly singular [5/5] falls back to [5/1] — the highest regular order
     — which reconstructs the rational function exactly."""
    c0, r = 0.3 * math.exp(-0.5), 0.3 * (1 - math.exp(-0.5))
    c = [c0 * r ** n for n in range(13)]
    u, fl, _, _ = orc.pade(c, 0, 1)
    assert abs(u - cf.kpp_const(0.3, 0.5)) < 1e-15
    u, fl, _, _ = orc.pade(c, 1, 1)
    assert abs(u - cf.kpp_const(0.3, 0.5)) < 1e-15
    # exact zero pivot needs exactly-representable geometric coefficients:
    # 1/(1 - z/2) = 2 at z = 1
    c2 = [0.5 ** n for n in range(11)]
    u, fl, p, q = orc.pade(c2, 5, 5)
    assert fl & 1 and (fl >> 8) & 0xFF == 1
    assert u == 2.0
    assert q[0] == 1.0 and q[1] == -0.5 and np.all(q[2:] == 0.0)


def test_pade_degenerate_table_falls_back_to_partial_sum(orc):
    """at early PDD time levels no tree reaches L splits and
    c_5..c_10 are exactly 0; every [5/M'] system with M' >= 1 then has a zero
    first column, so the value is [5/0] = c_0 + ... + c_5 (M' = 0), finite."""
    c = [0.31, 0.04, 0.006, 7e-4, 5e-5, 0.0] + [0.0] * 5
    u, fl, p, q = orc.pade(c, 5, 5)
    assert fl & 1 and (fl >> 8) & 0xFF == 0
    acc = 0.0
    for v in c[:6]:          # (not sum(): Python >= 3.12 compensates)
        acc += v
    assert u == acc and math.isfinite(u)
    # M' = 2: c_n of 1/(1 - z²/4) = (1, 0, 1/4, 0, 1/16, ...) (type [0/2],
    # dyadic, so elimination is exact): the [2/4] and [2/3] Toeplitz matrices
    # have rank 2 and exact zero pivots, [2/2] is regular and exact: 4/3
    g = [0.25 ** (n // 2) if n % 2 == 0 else 0.0 for n in range(12)]
    u, fl, p, q = orc.pade(g, 2, 4)
    assert fl & 1 and (fl >> 8) & 0xFF == 2
    assert abs(u - 4.0 / 3.0) < 1e-15
    assert np.array_equal(q, [1.0, 0.0, -0.25, 0.0, 0.0])


def test_pade_node_divergence_flag(orc):
    """bit3: |u - Σ_{n<=K} c_n| > 10 se_sum.  The exp
    series' [2/2] (19/7) differs from the partial sum 1+1+1/2+1/6+1/24 by
    0.0060: flagged at se_sum = 1e-4, not at 1e-2."""
    c = [1, 1, 0.5, 1 / 6, 1 / 24]
    u, fl = orc.pade_node(c, 4, 2, 2, 1e-4)
    assert abs(u - 19 / 7) < 1e-14 and fl == 8
    u, fl = orc.pade_node(c, 4, 2, 2, 1e-2)
    assert fl == 0
    # bit3 compares with ALL K+1 coefficients, not only the L+M+1 Padé uses
    c6 = c + [1 / 120]
    u6, fl6 = orc.pade_node(c6, 5, 2, 2, 5e-4)
    assert u6 == u and abs(u - sum(c6)) < 10 * 5e-4 and fl6 == 0


def test_pade_flags(orc):
    # 1/(1 - 2z): pole at z = 1/2 inside (0, 1]  -> bit2
    u, fl, _, _ = orc.pade([1.0, 2.0, 4.0], 0, 1)
    assert fl & 4 and not fl & 1
    assert u == pytest.approx(-1.0)
    # 1/(1 - z): Q(1) = 0 -> bit1 (and bit2)
    u, fl, _, _ = orc.pade([1.0, 1.0], 0, 1)
    assert fl & 2 and fl & 4
    # well-behaved: exp series [2/2]
    u, fl, _, _ = orc.pade([1, 1, 0.5, 1 / 6, 1 / 24], 2, 2)
    assert fl == 0


def test_pade_m0_is_partial_sum(orc):
    """M = 0: the approximant is the truncated series."""
    c = [0.3, -0.2, 0.1, 0.05]
    u, fl, p, q = orc.pade(c, 3, 0)
    assert u == pytest.approx(sum(c), rel=1e-15)
