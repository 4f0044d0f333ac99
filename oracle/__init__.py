"""ctypes binding of the CPU oracle (rt_oracle.c) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_2402_06491_b200) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "rt_oracle.c")
CFLAGS = ["-O2", "-std=gnu11", "-fPIC", "-shared", "-ffp-contract=off",
          "-fno-fast-math", "-Wall", "-Wextra", "-Wno-unused-parameter"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "rt_oracle.h"))):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class Params(C.Structure):
    _fields_ = [("dim", C.c_int32), ("D", C.c_double), ("degree", C.c_int32),
                ("b", C.c_double * 9), ("lam", C.c_double), ("offspring", C.c_int32),
                ("init_kind", C.c_int32), ("init_amp", C.c_double),
                ("init_scale", C.c_double), ("K", C.c_int32), ("precision", C.c_int32),
                ("strategy", C.c_int32), ("q", C.c_double), ("coef_kind", C.c_int32 * 9),
                ("coef_axis", C.c_int32), ("coef_scale", C.c_double), ("coef_t0", C.c_double),
                ("shared", C.c_int32), ("sampling", C.c_int32)]


class Norm(C.Structure):
    _fields_ = [("lam", C.c_double), ("inv_lambda", C.c_double), ("sigma", C.c_double),
                ("a", C.c_double * 9), ("n_support", C.c_int32), ("support", C.c_int32 * 9),
                ("thresh", C.c_uint64 * 9), ("p_hat", C.c_double * 9), ("w", C.c_double * 9),
                ("beta", C.c_int32), ("tq", C.c_uint64), ("q_hat", C.c_double)]


class TreeRec(C.Structure):
    _fields_ = [("ne", C.c_int32), ("leaves", C.c_int32), ("particles", C.c_int32),
                ("pruned", C.c_int32), ("C", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("trees", C.c_int64), ("pruned", C.c_int64), ("particles", C.c_int64),
                ("leaves", C.c_int64), ("splits", C.c_int64)]


TREE_DTYPE = np.dtype([("ne", np.int32), ("leaves", np.int32), ("particles", np.int32),
                       ("pruned", np.int32), ("C", np.float64)])

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        _lib.or_philox.argtypes = [C.POINTER(C.c_uint32)] * 3
        _lib.or_unif53.argtypes = [C.c_uint32, C.c_uint32]
        _lib.or_unif53.restype = C.c_double
        _lib.or_unif32.argtypes = [C.c_uint32]
        _lib.or_unif32.restype = C.c_double
        _lib.or_normalize.argtypes = [C.POINTER(Params), C.POINTER(Norm)]
        _lib.or_tree.argtypes = [C.POINTER(Params), dp, C.c_int64, C.c_int64, C.c_double,
                                 C.c_uint64, C.POINTER(TreeRec)]
        _lib.or_trees.argtypes = [C.POINTER(Params), dp, C.c_int64, C.c_double, C.c_int64,
                                  C.c_int64, C.c_uint64, C.c_void_p]
        _lib.or_trees_at.argtypes = [C.POINTER(Params), dp, C.c_int64, C.c_double, C.c_void_p,
                                     C.c_int64, C.c_uint64, C.c_void_p]
        _lib.or_sums.argtypes = [C.POINTER(Params), dp, C.c_int64, C.c_double, C.c_int64,
                                 C.c_int64, C.c_uint64, dp, C.POINTER(Stats)]
        _lib.or_finalize.argtypes = [dp, C.c_int64, C.c_int32, C.c_int64, dp, dp, dp, dp]
        _lib.or_finalize.restype = None
        _lib.or_pade.argtypes = [dp, C.c_int32, C.c_int32, dp, C.POINTER(C.c_uint32), dp, dp]
        _lib.or_pade_node.argtypes = [dp, C.c_int32, C.c_int32, C.c_int32, C.c_double, dp,
                                      C.POINTER(C.c_uint32)]
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def params(eq: dict) -> Params:
    p = Params()
    p.dim = eq["dim"]; p.D = eq["D"]; p.degree = eq["degree"]
    for k in range(9):
        p.b[k] = eq["b"][k]
    p.lam = eq.get("lam", 0.0); p.offspring = eq.get("offspring", 0)
    p.init_kind = eq["init_kind"]; p.init_amp = eq["init_amp"]
    p.init_scale = eq["init_scale"]; p.K = eq["K"]; p.precision = eq.get("precision", 0)
    p.strategy = eq.get("strategy", 0); p.q = eq.get("q", 0.5)
    ck = eq.get("coef_kind", [0] * 9)
    for k in range(9):
        p.coef_kind[k] = ck[k]
    p.coef_axis = eq.get("coef_axis", 0); p.coef_scale = eq.get("coef_scale", 1.0)
    p.coef_t0 = eq.get("coef_t0", 0.1)
    p.shared = eq.get("shared", 0)
    p.sampling = eq.get("sampling", 0)
    return p


def philox(key, ctr) -> np.ndarray:
    k = (C.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    c = (C.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    o = (C.c_uint32 * 4)()
    lib().or_philox(k, c, o)
    return np.array(list(o), dtype=np.uint32)


def unif53(lo: int, hi: int) -> float:
    return lib().or_unif53(lo, hi)


def unif32(w: int) -> float:
    return lib().or_unif32(w)


def normalize(eq: dict) -> dict:
    p = params(eq)
    n = Norm()
    e = lib().or_normalize(C.byref(p), C.byref(n))
    if e:
        raise ValueError(f"or_normalize error {e}")
    ns = n.n_support
    return dict(lam=n.lam, inv_lambda=n.inv_lambda, sigma=n.sigma, a=list(n.a),
                support=list(n.support)[:ns], thresh=list(n.thresh)[:ns],
                p_hat=list(n.p_hat)[:ns], w=list(n.w)[:ns], beta=n.beta, tq=n.tq, q_hat=n.q_hat)


def trees(eq: dict, points: np.ndarray, t: float, n_trees: int, seed: int,
          j0: int = 0) -> np.ndarray:
    """Per-tree records [n_points, n_trees] (ne, leaves, particles, pruned, C)."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    n = pts.shape[0]
    out = np.zeros((n, n_trees), dtype=TREE_DTYPE)
    e = lib().or_trees(C.byref(params(eq)), _dp(pts), n, t, j0, n_trees, seed,
                       out.ctypes.data_as(C.c_void_p))
    if e:
        raise ValueError(f"or_trees error {e}")
    return out


def trees_at(eq: dict, points: np.ndarray, t: float, js, seed: int) -> np.ndarray:
    """Per-tree records [n_points, len(js)] for the tree indices js of every node."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    jj = np.ascontiguousarray(np.asarray(js, dtype=np.int64))
    n = pts.shape[0]
    out = np.zeros((n, jj.size), dtype=TREE_DTYPE)
    e = lib().or_trees_at(C.byref(params(eq)), _dp(pts), n, t, jj.ctypes.data_as(C.c_void_p),
                          jj.size, seed, out.ctypes.data_as(C.c_void_p))
    if e:
        raise ValueError(f"or_trees_at error {e}")
    return out


def tree(eq: dict, x, i: int, j: int, t: float, seed: int) -> dict:
    xx = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))
    r = TreeRec()
    e = lib().or_tree(C.byref(params(eq)), _dp(xx), i, j, t, seed, C.byref(r))
    if e:
        raise ValueError(f"or_tree error {e}")
    return dict(ne=r.ne, leaves=r.leaves, particles=r.particles, pruned=r.pruned, C=r.C)


def sums(eq: dict, points: np.ndarray, t: float, n_trees: int, seed: int, j0: int = 0):
    """Order-binned sums [n, K+2, 3] (ΣC, ΣC², count; bin K+1 = pruned) and stats."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    n = pts.shape[0]
    K = eq["K"]
    out = np.zeros((n, K + 2, 3), dtype=np.float64)
    st = Stats()
    e = lib().or_sums(C.byref(params(eq)), _dp(pts), n, t, j0, n_trees, seed, _dp(out),
                      C.byref(st))
    if e:
        raise ValueError(f"or_sums error {e}")
    return out, dict(trees=st.trees, pruned=st.pruned, particles=st.particles,
                     leaves=st.leaves, splits=st.splits)


def finalize(s: np.ndarray, K: int, N: int):
    n = s.shape[0]
    s = np.ascontiguousarray(s, dtype=np.float64)
    c = np.zeros((n, K + 1)); se = np.zeros((n, K + 1))
    us = np.zeros(n); ses = np.zeros(n)
    lib().or_finalize(_dp(s), n, K, N, _dp(c), _dp(se), _dp(us), _dp(ses))
    return c, se, us, ses


def estimate(eq: dict, points: np.ndarray, t: float, n_trees: int, seed: int):
    """(coeffs [n,K+1], stderr [n,K+1], u_sum [n], se_sum [n], stats)."""
    s, st = sums(eq, points, t, n_trees, seed)
    c, se, us, ses = finalize(s, eq["K"], n_trees)
    return c, se, us, ses, st


def pade(c, L: int, M: int):
    """[L/M] Padé at z = 1 -> (u, flags, p, q)."""
    cc = np.ascontiguousarray(np.asarray(c, dtype=np.float64))
    u = C.c_double(); fl = C.c_uint32()
    p = np.zeros(L + 1); q = np.zeros(M + 1)
    e = lib().or_pade(_dp(cc), L, M, C.byref(u), C.byref(fl), _dp(p), _dp(q))
    if e:
        raise ValueError(f"or_pade error {e}")
    return u.value, fl.value, p, q


def pade_node(c, K: int, L: int, M: int, se_sum: float):
    """[L/M] Padé at z = 1 with the bit3 divergence flag -> (u, flags)."""
    cc = np.ascontiguousarray(np.asarray(c, dtype=np.float64))
    u = C.c_double(); fl = C.c_uint32()
    e = lib().or_pade_node(_dp(cc), K, L, M, float(se_sum), C.byref(u), C.byref(fl))
    if e:
        raise ValueError(f"or_pade_node error {e}")
    return u.value, fl.value
