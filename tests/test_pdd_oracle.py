"""Pins of oracle/pdd_oracle.py (NEXT row f1: PDD splines and local solver)
against mathematics and library routines other than itself:

  not-a-knot spline  -> scipy.interpolate.CubicSpline(bc_type="not-a-knot")
                        (the library routine), exact reproduction of cubics
  tensor spline      -> exact reproduction of s^3 t^2, t^3 s
  Strang/PR-ADI      -> the 2-D heat kernel (f = 0, exact Dirichlet data),
                        second-order convergence, the ODE for spatially
                        constant data (f != 0)
  single-domain FD   -> the pinned Monte Carlo oracle at cfg3's equation and
                        interface points (within 4 standard errors)
"""
import math

import numpy as np
import pytest
from scipy.interpolate import CubicSpline

import closed_forms as cf
import workloads as W
from oracle import pdd_oracle as PO


@pytest.mark.parametrize("n", [4, 5, 7, 12, 20])
def test_nak_spline_vs_scipy(n):
    rng = np.random.default_rng(n)
    x0, h = -1.3, 0.37
    xs = x0 + h * np.arange(n)
    y = rng.normal(size=n)
    M = PO.nak_second_derivatives(y, h)
    q = rng.uniform(xs[0], xs[-1], 500)
    ref = CubicSpline(xs, y, bc_type="not-a-knot")(q)
    got = PO.nak_eval(y, M, x0, h, q)
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
    assert np.allclose(PO.nak_eval(y, M, x0, h, xs), y, rtol=0, atol=1e-13)


def test_nak_reproduces_cubics_and_tensor_polynomials():
    x0, h, n = 0.0, 0.25, 9
    xs = x0 + h * np.arange(n)
    y = xs ** 3 - 2 * xs
    q = np.linspace(0, 2, 101)
    assert np.max(np.abs(PO.nak_eval(y, PO.nak_second_derivatives(y, h), x0, h, q) - (q ** 3 - 2 * q))) < 1e-12
    s = -2.0 + 0.5 * np.arange(9)
    t = 0.1 * np.arange(6)
    for fn in (lambda S, T: S ** 3 * T ** 2, lambda S, T: T ** 3 * S - S ** 2):
        V = fn(s[None, :], t[:, None])
        se, te = np.linspace(-2, 2, 17), np.linspace(0, 0.5, 11)
        W = PO.tensor_table(V, -2.0, 0.5, 0.0, 0.1, se, te)
        assert np.max(np.abs(W - fn(se[None, :], te[:, None]))) < 1e-10


def _heat2d(X, Y, t, D=1.0):
    return 1.0 / (1.0 + 4 * D * t) * np.exp(-(X ** 2 + Y ** 2) / (1.0 + 4 * D * t))


def _adi_heat_err(h, dt, T=0.25):
    x = np.arange(-1.0, 1.0 + 0.5 * h, h)
    y = np.arange(-0.5, 1.5 + 0.5 * h, h)
    X, Y = np.meshgrid(x, y, indexing="ij")

    def bc(m):
        tt = m * dt
        return dict(x0=_heat2d(x[0], y, tt), x1=_heat2d(x[-1], y, tt),
                    y0=_heat2d(x, y[0], tt), y1=_heat2d(x, y[-1], tt))

    n = int(round(T / dt))
    u = PO.strang_adi(_heat2d(X, Y, 0.0), [0.0], 1.0, h, dt, n, bc)
    return np.max(np.abs(u - _heat2d(X, Y, T)))


def test_adi_heat_kernel_second_order():
    e1 = _adi_heat_err(0.1, 0.01)
    e2 = _adi_heat_err(0.05, 0.005)
    assert e1 < 2e-3 and e2 < 6e-4
    assert 3.0 < e1 / e2 < 5.0, (e1, e2)        # second order in (h, dt)


def test_adi_constant_data_is_the_ode():
    """Spatially constant data with the ODE's boundary values stays the ODE
    solution (cfg2/3's f): the diffusion step is exact on constants."""
    b = W.B_CFG2
    u0, T, n = 0.5, 0.5, 100
    dt = T / n
    ts = dt * np.arange(n + 1)
    ode = np.array([cf.ode_u(b, u0, tt) if tt > 0 else u0 for tt in ts])
    # the scheme's own reaction (RK4 half steps) applied to the constant
    x = np.linspace(0, 1, 11)
    u = PO.strang_adi(np.full((11, 11), u0), b, 1.0, 0.1, dt, n,
                      lambda m: {k: np.full(11, ode[m]) for k in ("x0", "x1", "y0", "y1")})
    assert np.max(np.abs(u - ode[-1])) < 1e-9


def test_single_domain_matches_monte_carlo_cfg3(orc):
    """The reference FD (zero Dirichlet on [-6, 6]²) against the pinned Monte
    Carlo oracle for cfg3's equation at interface points (within 4 s.e.)."""
    cfg = W.get("cfg3")
    eq, t = cfg["eq"], cfg["t"]
    g = lambda X, Y: eq["init_amp"] * np.exp(-(X ** 2 + Y ** 2))   # noqa: E731
    x, u = PO.single_domain(g, eq["b"][: eq["degree"] + 1], 1.0, 6.0, 0.05, t, 500)
    pts = np.array([[0.0, 0.0], [0.0, 1.0], [-1.25, 0.0], [0.0, -1.75]])
    _, _, us, ses, _ = orc.estimate(eq, pts, t, 100_000, seed=31)
    ix = [np.argmin(np.abs(x - p)) for p in pts.ravel()]
    ref = np.array([u[ix[2 * q], ix[2 * q + 1]] for q in range(len(pts))])
    z = (us - ref) / ses
    assert np.all(np.abs(z) < 4.0), (us, ref, z)


PDD_CFG = dict(lo=-2.0, hi=2.0, T=0.5, n_cells=40, n_steps=100, n_s=17, n_t=6, boundary=1,
               L=5, M=5, n_trees=100_000, seed=0)


def test_pdd_downstream_exact_heat_data():
    """The whole downstream with exact interface/edge data of the heat equation
    (f = 0, Gaussian data) reproduces the 2-D heat kernel to the spline + ADI
    error (and the t = 0 table is g exactly)."""
    cfg = dict(PDD_CFG)
    eq = W._eq(2, (0.0,), W.G_GAUSS, 1.0, 1.0, K=12)
    eq["degree"] = 0
    nodes = PO.pdd_nodes(cfg)
    tk = cfg["T"] * np.arange(cfg["n_t"]) / (cfg["n_t"] - 1)
    V = np.stack([[_heat2d(nodes[l, :, 0], nodes[l, :, 1], t) for t in tk] for l in range(6)])
    F, Wt = PO.pdd_downstream(V, cfg, eq)
    x = np.linspace(-2, 2, cfg["n_cells"] + 1)
    X, Y = np.meshgrid(x, x, indexing="ij")
    assert np.max(np.abs(F - _heat2d(X, Y, cfg["T"]))) < 2e-3
    assert np.max(np.abs(Wt[0, 0] - _heat2d(0.0, x, 0.0))) < 1e-3


def test_product_pdd_nodes_layout():
    """rt_pdd_nodes (host-side layout in the C ABI) equals the oracle's."""
    import paper_2402_06491_b200 as P
    assert np.array_equal(P.pdd_nodes(PDD_CFG), PO.pdd_nodes(PDD_CFG))
