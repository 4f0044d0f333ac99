"""Device accuracy of the product's lean FP64 math (csrc/rt_math.cuh, the
routines the tree walk inlines) against 64-bit-mantissa long-double
references — the same bounds as the host build in tests/test_math.py, now
with the real MUFU.RCP64H / RSQ64H seeds and the device's FMA contraction."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
EPS = 2.0 ** -52
PI = np.longdouble("3.14159265358979323846264338327950288")


@pytest.fixture(scope="module")
def dev():
    so = os.path.join("/tmp", f"math_dev_{os.getpid()}.so")
    inc = os.path.join(os.path.dirname(HERE), "paper_2402_06491_b200", "csrc")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-O3", "-shared", "-Xcompiler", "-fPIC", "-I" + inc,
                           os.path.join(HERE, "helpers", "math_dev.cu"), "-o", so])
    lib = C.CDLL(so)
    lib.math_dev.argtypes = [C.c_int, C.c_void_p, C.c_long, C.c_void_p, C.c_void_p]
    return lib


def _run(lib, which, x, a=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    z = np.empty_like(x) if a is None else np.ascontiguousarray(a, dtype=np.float64).copy()
    assert lib.math_dev(which, x.ctypes.data, x.size, y.ctypes.data, z.ctypes.data) == 0
    return y, z


def _u53(n, seed):
    rng = np.random.default_rng(seed)
    return (2 * rng.integers(0, 2 ** 52, size=n, dtype=np.uint64) + 1).astype(np.float64) * 2.0 ** -53


def test_device_log(dev):
    x = np.concatenate([_u53(400_000, 1), [2.0 ** -53, 1 - 2.0 ** -53, 0.5, 0.6875]])
    y, _ = _run(dev, 0, x)
    ref = np.log(x.astype(np.longdouble))
    assert float(np.max(np.abs(y - ref) / np.abs(ref))) < 4 * EPS


def test_device_sincospi_and_cospi(dev):
    a = 2 * _u53(400_000, 3)
    s, c = _run(dev, 1, a)
    assert float(np.max(np.abs(s - np.sin(PI * a.astype(np.longdouble))))) < 1.25 * EPS
    assert float(np.max(np.abs(c - np.cos(PI * a.astype(np.longdouble))))) < 1.25 * EPS
    c2, _ = _run(dev, 2, a)
    assert float(np.max(np.abs(c2 - np.cos(PI * a.astype(np.longdouble))))) < 2.5 * EPS


def test_device_sqrt_rcp_exp(dev):
    rng = np.random.default_rng(7)
    x = np.exp(rng.uniform(-30, 30, 300_000))
    y, _ = _run(dev, 3, x)
    assert float(np.max(np.abs(y - np.sqrt(x.astype(np.longdouble))) / np.sqrt(x))) < 2 * EPS
    d = 1.0 + np.exp(rng.uniform(-20, 20, 300_000))
    r, _ = _run(dev, 4, d)
    assert float(np.max(np.abs(r * d.astype(np.longdouble) - 1))) < 2 * EPS
    e = -rng.uniform(0, 700, 300_000)
    v, _ = _run(dev, 5, e)
    ref = np.exp(e.astype(np.longdouble))
    assert float(np.max(np.abs(v - ref) / ref)) < 4 * EPS
    w, _ = _run(dev, 8, e)                              # the table-driven exp (shared trees)
    assert float(np.max(np.abs(w - ref) / ref)) < 4 * EPS


def test_device_mul_exp(dev):
    """a · e^x as the record-ring flush evaluates a tree's C = Π e^X (DESIGN.md
    §4): relative error < 4 eps over |x| <= 1400 whenever the product is a
    normal number, though e^x alone over- or underflows (the round-1 form
    1/e^{-x} turned x > 745 into NaN)."""
    rng = np.random.default_rng(8)
    x = rng.uniform(-1400, 1400, 400_000)
    loga = rng.uniform(-700, 700, x.size)
    keep = np.abs(x + loga) < 700                         # the product is a normal number
    x, loga = x[keep], loga[keep]
    a = np.exp(loga) * rng.choice([-1.0, 1.0], x.size)
    y, _ = _run(dev, 9, x, a)
    ref = a.astype(np.longdouble) * np.exp(x.astype(np.longdouble))
    assert np.all(np.isfinite(y))
    assert float(np.max(np.abs(y - ref) / np.abs(ref))) < 4 * EPS
    z, _ = _run(dev, 9, np.array([-5.0, 0.0, 3.0]), np.zeros(3))
    assert np.all(z == 0.0)


def test_device_u32_angles_bitwise(dev):
    """The integer-reduced d = 3 angles equal the FP64-reduced ones bit for bit
    on the device too (tests/test_math.py does the host build)."""
    e = [k * 2 ** 29 + d for k in range(9) for d in (-2, -1, 0, 1) if 0 <= k * 2 ** 29 + d < 2 ** 32]
    w = np.concatenate([np.array(e, dtype=np.float64),
                        np.random.default_rng(12).integers(0, 2 ** 32, 400_000).astype(np.float64)])
    a = 2.0 * (2 * w + 1) * 2.0 ** -33
    s_ref, c_ref = _run(dev, 1, a)
    s, c = _run(dev, 6, w)
    assert np.array_equal(s.view(np.uint64), s_ref.view(np.uint64))
    assert np.array_equal(c.view(np.uint64), c_ref.view(np.uint64))
    c1, _ = _run(dev, 2, a)
    c2, _ = _run(dev, 7, w)
    assert np.array_equal(c2.view(np.uint64), c1.view(np.uint64))
