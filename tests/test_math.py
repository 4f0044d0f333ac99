"""Accuracy of the product's lean FP64 math (csrc/rt_math.cuh) on the host
(same source; MUFU seeds emulated in FP32) against 64-bit-mantissa long-double
references, over the argument domains the tree walk produces.
The device build (real MUFU seeds) is checked the same way in
tests/test_gpu_math.py."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
EPS = 2.0 ** -52


@pytest.fixture(scope="module")
def m(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("m") / "math_host.so")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared",
                           os.path.join(HERE, "helpers", "math_host.cpp"), "-o", so])
    lib = C.CDLL(so)
    for f in ("m_log", "m_sqrt", "m_rcp", "m_exp", "m_exp_tab", "m_cospi2"):
        getattr(lib, f).argtypes = [C.c_void_p, C.c_long, C.c_void_p]
    lib.m_sincospi2.argtypes = [C.c_void_p, C.c_long, C.c_void_p, C.c_void_p]
    return lib


def _u53(n, seed):
    rng = np.random.default_rng(seed)
    m = rng.integers(0, 2 ** 52, size=n, dtype=np.uint64)
    return (2 * m + 1).astype(np.float64) * 2.0 ** -53


def _call(lib, name, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    getattr(lib, name)(x.ctypes.data, x.size, y.ctypes.data)
    return y


def test_log_unit_interval(m):
    x = np.concatenate([_u53(400_000, 1), [2.0 ** -53, 1 - 2.0 ** -53, 0.5, 0.6875, 1 - 2.0 ** -30,
                                           0.68749999999999989, 0.99609375, 0.70710678118654757]])
    got = _call(m, "m_log", x)
    ref = np.log(x.astype(np.longdouble))
    err = np.abs(got.astype(np.longdouble) - ref)
    rel = err / np.abs(ref)
    assert float(np.max(rel)) < 4 * EPS, float(np.max(rel))
    # general positive normals too (the routine is not specific to (0,1))
    y = np.exp(np.random.default_rng(2).uniform(-700, 700, 100_000))
    g = _call(m, "m_log", y)
    r = np.log(y.astype(np.longdouble))
    assert float(np.max(np.abs(g - r) / np.maximum(np.abs(r), 1e-300))) < 4 * EPS


def test_log_near_one_relative(m):
    """log(1 - 2^-k) keeps relative accuracy (the table entries at 1 are exact)."""
    x = 1.0 - 2.0 ** -np.arange(8, 53, dtype=np.float64)
    got = _call(m, "m_log", x)
    ref = np.log1p(-(2.0 ** -np.arange(8, 53)).astype(np.longdouble))
    assert float(np.max(np.abs(got - ref) / np.abs(ref))) < 4 * EPS


def test_sincospi2(m):
    a = np.concatenate([2 * _u53(400_000, 3), [0.0, 0.25, 0.5, 0.75, 1.0, 1.25, 1.5, 1.75, 2.0]])
    s = np.empty_like(a); c = np.empty_like(a)
    m.m_sincospi2(a.ctypes.data, a.size, s.ctypes.data, c.ctypes.data)
    pi = np.longdouble("3.14159265358979323846264338327950288")
    sr = np.sin(pi * a.astype(np.longdouble)); cr = np.cos(pi * a.astype(np.longdouble))
    assert float(np.max(np.abs(s - sr))) < 2.5 * EPS / 2
    assert float(np.max(np.abs(c - cr))) < 2.5 * EPS / 2
    # exact values at the quadrant points a = 0, 1/2, 1, 3/2, 2
    assert (s[-9], c[-9]) == (0.0, 1.0) and (s[-7], c[-7]) == (1.0, 0.0)
    assert (s[-5], c[-5]) == (0.0, -1.0) and (s[-3], c[-3]) == (-1.0, 0.0)
    assert (s[-1], c[-1]) == (0.0, 1.0)


def test_cospi2_single_polynomial(m):
    """cos(pi a) for a = 2v, v a 32-bit or 53-bit uniform (the d = 3 angle),
    absolute error < 2.5 ulp(1) against long double (one Horner polynomial on
    |f| <= 1/2 cancels near the zeros a = 1/2, 3/2; the Box-Muller normal r cos
    then carries <= 2e-15 absolute error, far inside the 1e-12 per-tree
    bound), exact at the extrema a = 0, 1, 2."""
    rng = np.random.default_rng(5)
    w = rng.integers(0, 2 ** 32, size=200_000, dtype=np.uint64)
    a = np.concatenate([2.0 * (2 * w + 1).astype(np.float64) * 2.0 ** -33, 2.0 * _u53(200_000, 6),
                        [0.0, 0.5, 1.0, 1.5, 2.0, 0.25, 0.75, 1.25, 1.75, 2.0 ** -40, 2 - 2.0 ** -40]])
    got = _call(m, "m_cospi2", a)
    pi = np.longdouble("3.14159265358979323846264338327950288")
    ref = np.cos(pi * a.astype(np.longdouble))
    assert float(np.max(np.abs(got - ref))) < 2.5 * EPS
    assert got[-11] == 1.0 and got[-9] == -1.0 and got[-7] == 1.0


def _w_edges():
    """32-bit words around every reduction boundary (quadrant / half-turn
    edges at multiples of 2^29) plus random ones."""
    e = []
    for k in range(9):
        for d in (-2, -1, 0, 1):
            v = k * 2 ** 29 + d
            if 0 <= v < 2 ** 32:
                e.append(v)
    r = np.random.default_rng(11).integers(0, 2 ** 32, size=500_000, dtype=np.uint64)
    return np.concatenate([np.array(e, dtype=np.uint64), r]).astype(np.uint32)


def test_u32_angle_reductions_bitwise(m):
    """sincos2pi_u32(w) / cos2pi_u32(w) (the integer reduction of the d = 3
    angles) equal sincospi2(2v) / cospi2(2v) bit for bit, v = (2w+1)·2^-33
    (the FP64 reduction they replace: same q, same exact f)."""
    w = _w_edges()
    a = 2.0 * (2 * w.astype(np.float64) + 1) * 2.0 ** -33
    assert np.array_equal((2 * w.astype(np.uint64) + 1).astype(np.float64), 2 * w.astype(np.float64) + 1)
    s_ref = np.empty_like(a); c_ref = np.empty_like(a)
    m.m_sincospi2(a.ctypes.data, a.size, s_ref.ctypes.data, c_ref.ctypes.data)
    s = np.empty_like(a); c = np.empty_like(a)
    m.m_sincos2pi_u32.argtypes = [C.c_void_p, C.c_long, C.c_void_p, C.c_void_p]
    m.m_sincos2pi_u32(w.ctypes.data, w.size, s.ctypes.data, c.ctypes.data)
    assert np.array_equal(s.view(np.uint64), s_ref.view(np.uint64))
    assert np.array_equal(c.view(np.uint64), c_ref.view(np.uint64))
    c1 = _call(m, "m_cospi2", a)
    c2 = np.empty_like(a)
    m.m_cos2pi_u32.argtypes = [C.c_void_p, C.c_long, C.c_void_p]
    m.m_cos2pi_u32(w.ctypes.data, w.size, c2.ctypes.data)
    assert np.array_equal(c2.view(np.uint64), c1.view(np.uint64))


def test_sqrt_pos_equals_sqrt_nr_on_positive_normals(m):
    """sqrt_pos (the kernel's Box–Muller radii, argument always > 0) is
    sqrt_nr without the zero select: bitwise equal on positive normals."""
    x = np.exp(np.random.default_rng(13).uniform(-700, 700, 300_000))
    a = _call(m, "m_sqrt", x)
    m.m_sqrt_pos.argtypes = [C.c_void_p, C.c_long, C.c_void_p]
    b = np.empty_like(x)
    m.m_sqrt_pos(x.ctypes.data, x.size, b.ctypes.data)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_sqrt_rcp(m):
    rng = np.random.default_rng(4)
    x = np.concatenate([np.exp(rng.uniform(-80, 80, 300_000)), [0.0, 1.0, 4.0, 2.0 ** -60]])
    got = _call(m, "m_sqrt", x)
    ref = np.sqrt(x.astype(np.longdouble))
    rel = np.abs(got - ref) / np.maximum(ref, 1e-300)
    assert float(np.max(rel)) < 2 * EPS and got[-4] == 0.0
    d = 1.0 + np.exp(rng.uniform(-40, 20, 300_000))
    got = _call(m, "m_rcp", d)
    ref = 1 / d.astype(np.longdouble)
    assert float(np.max(np.abs(got - ref) / ref)) < 2 * EPS


def test_exp_neg(m):
    rng = np.random.default_rng(5)
    x = np.concatenate([-rng.exponential(3.0, 300_000), -rng.uniform(0, 700, 50_000), [0.0, -1e-300, -708.0]])
    got = _call(m, "m_exp", x)
    ref = np.exp(x.astype(np.longdouble))
    assert float(np.max(np.abs(got - ref) / ref)) < 4 * EPS
    assert _call(m, "m_exp", np.array([-800.0]))[0] == 0.0


def test_mul_exp_tab(m):
    """a · e^x with the power of two applied to the product (the record-ring
    trees' C = Π e^X): < 4 eps wherever the product is normal, over |x| <=
    1400 (e^x alone over- or underflows beyond ±709); equal to a ·
    exp_neg_tab(x) bit for bit where e^x is normal and a is a power of two."""
    rng = np.random.default_rng(9)
    x = rng.uniform(-1400, 1400, 400_000)
    loga = rng.uniform(-700, 700, x.size)
    keep = np.abs(x + loga) < 700
    x, loga = x[keep], loga[keep]
    a = np.exp(loga) * rng.choice([-1.0, 1.0], x.size)
    m.m_mul_exp.argtypes = [C.c_void_p, C.c_void_p, C.c_long, C.c_void_p]
    y = np.empty_like(x)
    m.m_mul_exp(a.ctypes.data, x.ctypes.data, x.size, y.ctypes.data)
    ref = a.astype(np.longdouble) * np.exp(x.astype(np.longdouble))
    assert np.all(np.isfinite(y))
    assert float(np.max(np.abs(y - ref) / np.abs(ref))) < 4 * EPS
    xs = -rng.uniform(0, 700, 10_000)
    ones = np.ldexp(1.0, rng.integers(-60, 60, xs.size)).astype(np.float64)
    y1 = np.empty_like(xs)
    m.m_mul_exp(ones.ctypes.data, xs.ctypes.data, xs.size, y1.ctypes.data)
    assert np.array_equal(y1, ones * _call(m, "m_exp_tab", xs))


def test_exp_neg_tab(m):
    """The table-driven exp (shared-tree phase 2): same bound and domain as
    exp_neg, including every table entry's neighbourhood, the subnormal range
    (the 2^m scaling in two exact steps) and the cut-off below -745.5."""
    rng = np.random.default_rng(6)
    ln2_32 = np.log(2.0) / 32
    grid = -np.arange(0, 2000) * ln2_32
    x = np.concatenate([-rng.exponential(3.0, 300_000), -rng.uniform(0, 708, 50_000),
                        grid, grid - ln2_32 / 2, grid + ln2_32 / 2 - 1e-12, [0.0, -1e-300, -708.0]])
    x = x[x <= 0]
    got = _call(m, "m_exp_tab", x)
    ref = np.exp(x.astype(np.longdouble))
    assert float(np.max(np.abs(got - ref) / ref)) < 4 * EPS
    sub = -rng.uniform(708.5, 744.0, 20_000)             # subnormal results: absolute 2^-1074 granularity
    g2 = _call(m, "m_exp_tab", sub)
    r2 = np.exp(sub.astype(np.longdouble))
    assert float(np.max(np.abs(g2 - r2))) <= 2.0 ** -1074 * 2
    assert _call(m, "m_exp_tab", np.array([-800.0]))[0] == 0.0
