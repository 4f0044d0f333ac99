"""Probabilistic domain decomposition downstream (NEXT row f1) — TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py for who may import it).

Plain numpy implementations, written from PAPER.md:936-950 and 1007-1012,
of what the CUDA path (`rt_pdd_solve`) computes after the interface values:

* ``nak_second_derivatives`` / ``nak_eval``: 1-D cubic spline through uniform
  nodes with the not-a-knot condition ("a not-a-knot condition is imposed",
  PAPER.md:941).  Written from the definition: C² piecewise cubic, third
  derivative continuous at the first and last interior nodes.  Pinned in
  tests/test_pdd_oracle.py against scipy's CubicSpline(bc_type="not-a-knot").
* ``tensor_table``: the tensor-product spline in (s, t) on one interface line
  ("tensor product interpolation based on cubic spline")
  evaluated at grid nodes s_i and times t_m: splines in s per time node, then
  a spline in t through those values.
* ``strang_adi``: the local solver on one rectangle — Strang splitting of
  u_t = D Δu + f(u): half a reaction step (classical RK4 on u' = f(u)),
  a Peaceman–Rachford ADI diffusion step (Crank–Nicolson in each direction,
  the paper's "Crank-Nicolson (implicit) finite difference method",
  PAPER.md:971-973) with Dirichlet data carried through the same splitting,
  half a reaction step.  Pinned against
  the heat kernel (f = 0), the ODE (spatially constant data, exact boundary
  data) and second-order self-convergence.
* ``single_domain``: the same solver on a large box with zero Dirichlet data
  (the paper's artificial boundary choice for Example 4):
  the reference a PDD field is checked against.
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import solve_banded


# ---------------------------------------------------------------------------
# not-a-knot cubic spline on uniform nodes
def nak_second_derivatives(y: np.ndarray, h: float) -> np.ndarray:
    """Second derivatives M_0..M_{n-1} of the C² cubic spline through y on a
    uniform grid of spacing h with the not-a-knot conditions
    M_0 - 2 M_1 + M_2 = 0 and M_{n-3} - 2 M_{n-2} + M_{n-1} = 0 (third
    derivative continuous at the first and last interior nodes).  Solved as
    one banded system, exactly as the conditions are written (n >= 4)."""
    y = np.asarray(y, dtype=np.float64)
    n = y.size
    if n < 4:
        raise ValueError("not-a-knot needs >= 4 nodes")
    A = np.zeros((n, n))
    r = np.zeros(n)
    A[0, 0:3] = (1.0, -2.0, 1.0)
    A[n - 1, n - 3:n] = (1.0, -2.0, 1.0)
    for i in range(1, n - 1):
        # C² continuity: M_{i-1} + 4 M_i + M_{i+1} = 6 (y_{i+1} - 2 y_i + y_{i-1}) / h²
        A[i, i - 1:i + 2] = (1.0, 4.0, 1.0)
        r[i] = 6.0 * (y[i + 1] - 2.0 * y[i] + y[i - 1]) / (h * h)
    return np.linalg.solve(A, r)


def nak_eval(y: np.ndarray, M: np.ndarray, x0: float, h: float, x) -> np.ndarray:
    """Evaluate the spline (nodes x0 + j h) at x (inside [x0, x0 + (n-1)h])."""
    x = np.asarray(x, dtype=np.float64)
    n = y.size
    j = np.clip(np.floor((x - x0) / h).astype(int), 0, n - 2)
    a = x0 + j * h
    b = a + h
    return (M[j] * (b - x) ** 3 / (6.0 * h) + M[j + 1] * (x - a) ** 3 / (6.0 * h)
            + (y[j] / h - M[j] * h / 6.0) * (b - x) + (y[j + 1] / h - M[j + 1] * h / 6.0) * (x - a))


def tensor_table(V: np.ndarray, s0: float, hs: float, t0: float, ht: float,
                 s_eval: np.ndarray, t_eval: np.ndarray) -> np.ndarray:
    """V[k, j] = value at (t_k, s_j).  Returns W[m, i] = tensor spline at
    (t_eval[m], s_eval[i]): splines in s for every time node, then, at each
    s_eval[i], the spline in t through those values."""
    nt = V.shape[0]
    A = np.empty((nt, s_eval.size))
    for k in range(nt):
        A[k] = nak_eval(V[k], nak_second_derivatives(V[k], hs), s0, hs, s_eval)
    W = np.empty((t_eval.size, s_eval.size))
    for i in range(s_eval.size):
        W[:, i] = nak_eval(A[:, i], nak_second_derivatives(A[:, i], ht), t0, ht, t_eval)
    return W


# ---------------------------------------------------------------------------
# local solver: Strang splitting, RK4 reaction, Peaceman–Rachford ADI
def poly(b):
    b = list(b)
    return lambda u: sum(bk * u ** k for k, bk in enumerate(b))


def react(u: np.ndarray, f, h: float) -> np.ndarray:
    """One classical RK4 step of u' = f(u) (pointwise)."""
    k1 = f(u)
    k2 = f(u + 0.5 * h * k1)
    k3 = f(u + 0.5 * h * k2)
    k4 = f(u + h * k3)
    return u + h / 6.0 * (k1 + 2.0 * k2 + 2.0 * k3 + k4)


def _tri_solve(r: float, rhs: np.ndarray, axis: int) -> np.ndarray:
    """(I - r/2 δ²) w = rhs along `axis` for the interior unknowns; rhs already
    carries the Dirichlet contributions."""
    m = rhs.shape[axis]
    ab = np.zeros((3, m))
    ab[0, 1:] = -0.5 * r
    ab[1, :] = 1.0 + r
    ab[2, :-1] = -0.5 * r
    if axis == 0:
        return solve_banded((1, 1), ab, rhs)
    return solve_banded((1, 1), ab, rhs.T).T


def strang_adi(u0: np.ndarray, b, D: float, h: float, dt: float, n_steps: int, bc) -> np.ndarray:
    """March u0 (shape [nx+1, ny+1], index [i, j] = (x_i, y_j)) n_steps steps.

    bc(n) returns the Dirichlet data at t_n = n dt as a dict with keys 'x0',
    'x1' (arrays over j: the edges x = x_0, x = x_nx) and 'y0', 'y1' (arrays
    over i).  Step n:
      1. half reaction R_{dt/2} (RK4 on u' = f(u)) of every node, the
         boundary holding u_b(t_n): the boundary is now bA = R_{dt/2} u_b(t_n);
      2. bB = R_{-dt/2} u_b(t_{n+1}) (one RK4 step backwards): the boundary
         value that the final half reaction carries to u_b(t_{n+1});
      3. Peaceman–Rachford diffusion, r = D dt/h²:
         x-sweep (I - r/2 δx²) u* = (I + r/2 δy²) u, u* = (bA + bB)/2 on the
         boundary; y-sweep (I - r/2 δy²) v = (I + r/2 δx²) u*, v = bB on the
         boundary;
      4. half reaction, then the boundary is set to u_b(t_{n+1}).
    Transforming the boundary data with the same splitting keeps the scheme
    consistent at the boundary: spatially constant data reproduce the ODE to
    RK4 accuracy and f = 0 reduces to Peaceman–Rachford with the data at
    t_n, t_{n+1/2} (to O(dt²)), t_{n+1}."""
    f = poly(b)
    r = D * dt / (h * h)
    u = np.array(u0, dtype=np.float64)

    def impose(w, e):
        w[0, :] = e["x0"]; w[-1, :] = e["x1"]; w[:, 0] = e["y0"]; w[:, -1] = e["y1"]
        return w

    u = impose(u, bc(0))
    for n in range(n_steps):
        u = react(u, f, 0.5 * dt)                                   # boundary -> bA
        bA = dict(x0=u[0, :].copy(), x1=u[-1, :].copy(), y0=u[:, 0].copy(), y1=u[:, -1].copy())
        bB = {k: react(v, f, -0.5 * dt) for k, v in bc(n + 1).items()}
        bM = {k: 0.5 * (bA[k] + bB[k]) for k in bA}
        # x-sweep: unknowns u*[1:-1, 1:-1]; explicit part in y
        rhs = u[1:-1, 1:-1] + 0.5 * r * (u[1:-1, :-2] - 2.0 * u[1:-1, 1:-1] + u[1:-1, 2:])
        rhs[0, :] += 0.5 * r * bM["x0"][1:-1]
        rhs[-1, :] += 0.5 * r * bM["x1"][1:-1]
        us = np.empty_like(u)
        us[1:-1, 1:-1] = _tri_solve(r, rhs, axis=0)
        us = impose(us, bM)
        # y-sweep: unknowns v[1:-1, 1:-1]; explicit part in x
        rhs = us[1:-1, 1:-1] + 0.5 * r * (us[:-2, 1:-1] - 2.0 * us[1:-1, 1:-1] + us[2:, 1:-1])
        rhs[:, 0] += 0.5 * r * bB["y0"][1:-1]
        rhs[:, -1] += 0.5 * r * bB["y1"][1:-1]
        v = np.empty_like(u)
        v[1:-1, 1:-1] = _tri_solve(r, rhs, axis=1)
        v = impose(v, bB)
        u = impose(react(v, f, 0.5 * dt), bc(n + 1))
    return u


def single_domain(g, b, D: float, L: float, h: float, T: float, n_steps: int):
    """Reference: the same scheme on [-L, L]² with zero Dirichlet data."""
    x = np.linspace(-L, L, int(round(2 * L / h)) + 1)
    X, Y = np.meshgrid(x, x, indexing="ij")
    z = np.zeros(x.size)
    u = strang_adi(g(X, Y), b, D, x[1] - x[0], T / n_steps, n_steps,
                   lambda n: dict(x0=z, x1=z, y0=z, y1=z))
    return x, u


# ---------------------------------------------------------------------------
# the PDD downstream of rt_pdd_downstream_dev, written plainly
def g_fn(eq):
    """u(x, y, 0) for the equation dict (the four data shapes)."""
    a, s = eq["init_amp"], eq["init_scale"]
    k = eq["init_kind"]
    if k == 0:
        return lambda X, Y: a + 0.0 * X
    if k == 1:
        return lambda X, Y: a * 0.5 * (1.0 + np.tanh(X / s))
    if k == 2:
        return lambda X, Y: a * np.exp(-(X * X + Y * Y) / (s * s))
    return lambda X, Y: a / (1.0 + (X * X + Y * Y) / (s * s))


def pdd_nodes(cfg: dict) -> np.ndarray:
    """[6, n_s, 2]: lines 0 x = mid, 1 y = mid, 2 x = lo, 3 x = hi, 4 y = lo,
    5 y = hi; s_j = lo + (hi - lo) j/(n_s - 1)."""
    lo, hi, ns = cfg["lo"], cfg["hi"], cfg["n_s"]
    mid = 0.5 * (lo + hi)
    s = lo + (hi - lo) * (np.arange(ns) / (ns - 1))
    c = np.full(ns, 1.0)
    xy = [(mid * c, s), (s, mid * c), (lo * c, s), (hi * c, s), (s, lo * c), (s, hi * c)]
    return np.stack([np.stack(p, axis=1) for p in xy])


def pdd_downstream(V: np.ndarray, cfg: dict, eq: dict):
    """V [6, n_t, n_s] nodal values -> (field [(n+1), (n+1)] at T, W tables
    [6, n_steps + 1, n + 1]).  Each line's table is the tensor spline at
    (x_i, t_n); each quadrant is marched by strang_adi with its edges' tables,
    then written into the global field in quadrant order q = qx + 2 qy."""
    lo, hi, n, T, N = cfg["lo"], cfg["hi"], cfg["n_cells"], cfg["T"], cfg["n_steps"]
    ns, nt = cfg["n_s"], cfg["n_t"]
    h = (hi - lo) / n
    x = lo + h * np.arange(n + 1)
    tn = (T / N) * np.arange(N + 1)
    hs, ht = (hi - lo) / (ns - 1), T / (nt - 1)
    W = np.stack([tensor_table(V[l], lo, hs, 0.0, ht, x, tn) for l in range(6)])
    m = n // 2
    b = eq["b"][: eq["degree"] + 1]
    g = g_fn(eq)
    F = np.zeros((n + 1, n + 1))
    for q in range(4):
        qx, qy = q & 1, q >> 1
        i0, j0 = qx * m, qy * m
        lx0, lx1 = (2, 0) if qx == 0 else (0, 3)
        ly0, ly1 = (4, 1) if qy == 0 else (1, 5)
        xs, ys = x[i0:i0 + m + 1], x[j0:j0 + m + 1]
        X, Y = np.meshgrid(xs, ys, indexing="ij")
        bc = (lambda st, lx0=lx0, lx1=lx1, ly0=ly0, ly1=ly1, i0=i0, j0=j0:
              dict(x0=W[lx0, st, j0:j0 + m + 1], x1=W[lx1, st, j0:j0 + m + 1],
                   y0=W[ly0, st, i0:i0 + m + 1], y1=W[ly1, st, i0:i0 + m + 1]))
        F[i0:i0 + m + 1, j0:j0 + m + 1] = strang_adi(g(X, Y), b, eq["D"], h, T / N, N, bc)
    return F, W
