"""Independent mathematics the oracle (and, through it, the CUDA path) is
pinned to.  Nothing here samples trees or calls oracle/ or the product: these
are closed forms, ODE integrations and a finite-difference PDE solver derived
directly from the PDE u_t = D Δu + f(u), u(x,0) = g(x).

* ``ode_u``: spatially constant data reduce the PDE to u' = f(u)
  (BASELINE.json configs[0]: for f = u^2 - u, u = u0 / (u0 + (1-u0) e^t)).
* ``ode_orders``: the z-graded series of the same ODE, U' = -λU + z Σ a_k U^k,
  whose z^n coefficient is the expected contribution of trees with n splitting
  events (grouping by splits).  Integrated with DOP853.
* ``heat``: the heat-kernel solution for linear f = -λu with Gaussian data
  (Green's function of Eq. green2).
* ``fd_solve_1d``: Strang-split Crank–Nicolson finite differences on a large
  box — the paper's own validation route ("implicit finite difference scheme
  with a very fine mesh").
"""
from __future__ import annotations

import math

import numpy as np
from scipy.integrate import solve_ivp
from scipy.linalg import solve_banded


def poly_f(b):
    b = list(b)
    return lambda u: sum(bk * u ** k for k, bk in enumerate(b))


def kpp_const(u0: float, t: float) -> float:
    """BASELINE.json configs[0]: u = u0 / (u0 + (1 - u0) e^t) for f = u^2 - u."""
    return u0 / (u0 + (1.0 - u0) * math.exp(t))


def ode_u(b, u0: float, t: float) -> float:
    """u(t) for u' = f(u), u(0) = u0 (DOP853, rtol 1e-13)."""
    f = poly_f(b)
    sol = solve_ivp(lambda _t, y: [f(y[0])], (0.0, t), [u0], method="DOP853",
                    rtol=1e-13, atol=1e-16)
    return float(sol.y[0, -1])


def _series_pow(c: np.ndarray, k: int, nmax: int) -> np.ndarray:
    out = np.zeros(nmax + 1)
    out[0] = 1.0
    for _ in range(k):
        out = np.convolve(out, c)[: nmax + 1]
    return out


def ode_orders(a, lam: float, u0: float, t: float, K: int) -> np.ndarray:
    """c_0..c_K(t): z^n coefficients of U_z solving U' = -λU + z Σ_k a_k U^k,
    U(0) = u0.  ``a`` are the coefficients of f(u) + λu (a_1 = b_1 + λ)."""
    a = list(a)

    def rhs(_t, c):
        d = -lam * c
        for k, ak in enumerate(a):
            if ak == 0.0:
                continue
            pk = _series_pow(c, k, K)
            d[1:] += ak * pk[:K]
        return d

    c0 = np.zeros(K + 1)
    c0[0] = u0
    sol = solve_ivp(rhs, (0.0, t), c0, method="DOP853", rtol=1e-13, atol=1e-18)
    return sol.y[:, -1].copy()


def heat(x, t: float, D: float, lam: float, A: float, s: float = 1.0) -> np.ndarray:
    """u for u_t = DΔu - λu, u(x,0) = A exp(-|x|²/s²):
    e^{-λt} A (1 + 4Dt/s²)^{-d/2} exp(-|x|²/(s² + 4Dt))."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    d = x.shape[1]
    r2 = np.sum(x * x, axis=1)
    return math.exp(-lam * t) * A * (1.0 + 4.0 * D * t / s ** 2) ** (-d / 2.0) * \
        np.exp(-r2 / (s ** 2 + 4.0 * D * t))


def heat_1d_quadrature(g, x: float, t: float, D: float, lam: float) -> float:
    """e^{-λt} ∫ g(x + sqrt(2Dt) z) φ(z) dz by Gauss–Hermite quadrature (200 nodes)."""
    z, w = np.polynomial.hermite_e.hermegauss(200)
    vals = g(x + math.sqrt(2.0 * D * t) * z)
    return math.exp(-lam * t) * float(np.sum(w * vals) / math.sqrt(2.0 * math.pi))


def fd_solve_1d(b, g, t: float, D: float = 1.0, L: float = 12.0, dx: float = 0.02,
                dt: float = 2e-3) -> tuple[np.ndarray, np.ndarray]:
    """Crank–Nicolson diffusion + exact-ish (RK4) reaction, Strang splitting,
    on [-L, L] with boundary values following the ODE of the boundary data."""
    f = poly_f(b)
    x = np.arange(-L, L + 0.5 * dx, dx)
    n = x.size
    u = g(x).astype(np.float64)
    nsteps = int(round(t / dt))
    dt = t / nsteps
    r = D * dt / dx ** 2
    m = n - 2
    ab = np.zeros((3, m))
    ab[0, 1:] = -0.5 * r
    ab[1, :] = 1.0 + r
    ab[2, :-1] = -0.5 * r

    def react(v, h):
        sub = 4
        hh = h / sub
        for _ in range(sub):
            k1 = f(v); k2 = f(v + 0.5 * hh * k1); k3 = f(v + 0.5 * hh * k2); k4 = f(v + hh * k3)
            v = v + hh / 6.0 * (k1 + 2 * k2 + 2 * k3 + k4)
        return v

    for _ in range(nsteps):
        u = react(u, 0.5 * dt)
        ul, ur = u[0], u[-1]
        rhs = u[1:-1] + 0.5 * r * (u[:-2] - 2 * u[1:-1] + u[2:])
        rhs[0] += 0.5 * r * ul
        rhs[-1] += 0.5 * r * ur
        inner = solve_banded((1, 1), ab, rhs)
        u = np.concatenate([[ul], inner, [ur]])
        u = react(u, 0.5 * dt)
    return x, u


def fd_at(b, g, t: float, pts, **kw) -> np.ndarray:
    x, u = fd_solve_1d(b, g, t, **kw)
    return np.interp(np.asarray(pts, dtype=np.float64), x, u)


def fd_solve_1d_xt(fxt, g, t: float, D: float = 1.0, L: float = 12.0, dx: float = 0.02,
                   dt: float = 2e-3) -> tuple[np.ndarray, np.ndarray]:
    """As fd_solve_1d for a reaction f(u, x, t) depending on space and time
    (variable coefficients): Strang splitting, the reaction
    half-steps integrated by RK4 in time at fixed x, CN diffusion."""
    x = np.arange(-L, L + 0.5 * dx, dx)
    n = x.size
    u = g(x).astype(np.float64)
    nsteps = int(round(t / dt))
    dt = t / nsteps
    r = D * dt / dx ** 2
    m = n - 2
    ab = np.zeros((3, m))
    ab[0, 1:] = -0.5 * r
    ab[1, :] = 1.0 + r
    ab[2, :-1] = -0.5 * r

    def react(v, t0, h):
        sub = 4
        hh = h / sub
        tt = t0
        for _ in range(sub):
            k1 = fxt(v, x, tt)
            k2 = fxt(v + 0.5 * hh * k1, x, tt + 0.5 * hh)
            k3 = fxt(v + 0.5 * hh * k2, x, tt + 0.5 * hh)
            k4 = fxt(v + hh * k3, x, tt + hh)
            v = v + hh / 6.0 * (k1 + 2 * k2 + 2 * k3 + k4)
            tt += hh
        return v

    for s in range(nsteps):
        t0 = s * dt
        u = react(u, t0, 0.5 * dt)
        ul, ur = u[0], u[-1]
        rhs = u[1:-1] + 0.5 * r * (u[:-2] - 2 * u[1:-1] + u[2:])
        rhs[0] += 0.5 * r * ul
        rhs[-1] += 0.5 * r * ur
        inner = solve_banded((1, 1), ab, rhs)
        u = np.concatenate([[ul], inner, [ur]])
        u = react(u, t0 + 0.5 * dt, 0.5 * dt)
    return x, u


def catalan(n: int) -> int:
    return math.comb(2 * n, n) // (n + 1)


def lorentz_heat(x, t: float, D: float, lam: float, A: float, s: float) -> np.ndarray:
    """u for u_t = DΔu - λu, u(x,0) = A / (1 + |x|²/s²) in any dimension d.

    Derived without the radial density used elsewhere: write
    1/(1 + a) = ∫_0^∞ e^{-w(1 + a)} dw and average the Gaussian factor
    e^{-w|X|²/s²} over X ~ N(x, 2Dt I_d) in closed form,
    E e^{-w|X|²/s²} = (1 + 4Dtw/s²)^{-d/2} exp(-w|x|² / (s² + 4Dtw)),
    so u = e^{-λt} A ∫_0^∞ e^{-w} (1 + 4Dtw/s²)^{-d/2}
    exp(-w|x|²/(s² + 4Dtw)) dw (one smooth, exponentially decaying integral,
    scipy quad)."""
    from scipy.integrate import quad
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    d = x.shape[1]
    v = 2.0 * D * t
    out = np.empty(x.shape[0])
    for i, xi in enumerate(x):
        r2 = float(np.sum(xi * xi))
        f = lambda w: math.exp(-w) * (1.0 + 2.0 * v * w / s ** 2) ** (-d / 2.0) * \
            math.exp(-w * r2 / (s ** 2 + 2.0 * v * w))   # noqa: E731
        val, _ = quad(f, 0.0, math.inf, epsabs=1e-15, epsrel=1e-13, limit=400)
        out[i] = math.exp(-lam * t) * A * val
    return out
