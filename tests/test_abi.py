"""The C-ABI library loads and exports every symbol include/rt.h declares, and
host-side validation rejects bad arguments — no GPU needed (no compute call
reaches a kernel here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rtmod():
    from paper_2402_06491_b200 import build, rt
    build.build()
    return rt


def _declared():
    src = open(os.path.join(ROOT, "include", "rt.h")).read()
    return sorted(set(re.findall(r"^\s*(?:rt_status|const char\*)\s+(rt_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported(rtmod):
    names = _declared()
    assert len(names) >= 13
    lib = rtmod.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(rtmod.SYMBOLS)


def test_so_is_sm100a(rtmod):
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", rtmod.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _create(rtmod, **kw):
    eq = dict(W.get("cfg2")["eq"])
    eq.update(kw)
    p = rtmod.eq_params(eq)
    h = C.c_void_p()
    return rtmod.lib().rt_create(C.byref(p), C.byref(h)), rtmod.lib().rt_last_error().decode()


@pytest.mark.parametrize("kw,frag", [
    (dict(dim=0), "dim"), (dict(dim=4), "dim"), (dict(D=0.0), "D must"),
    (dict(D=float("nan")), "D must"), (dict(degree=9), "degree"),
    (dict(init_kind=7), "init_kind"), (dict(init_scale=0.0), "init_scale"),
    (dict(K=-1), "K must"), (dict(K=31), "K must"), (dict(offspring=5), "offspring"),
    (dict(precision=2), "precision"), (dict(init_amp=float("inf")), "init_amp"),
    (dict(K=28), "label width"),                       # β = 2 for k_max = 4: 1 + 28*2 > 56
    (dict(b=[0, -1, 1e-12, 1.0] + [0] * 5, degree=3), "zero integer"),
    (dict(strategy=3), "strategy"), (dict(strategy=2, q=0.0), "q < 1"),
    (dict(strategy=2, q=1.0), "q < 1"), (dict(strategy=1, precision=1), "FP32"),
    (dict(coef_kind=[0, 1] + [0] * 7), "k = 1"), (dict(coef_kind=[0, 0, 2] + [0] * 6), "coef_kind"),
    (dict(coef_kind=[0, 0, 1] + [0] * 6, coef_t0=0.0), "t0 > 0"),
    (dict(coef_kind=[0, 0, 1] + [0] * 6, coef_axis=1), "axis"),
    (dict(shared=2), "shared"), (dict(shared=1, precision=1), "FP64"),
    (dict(shared=1, strategy=1, coef_kind=[0, 0, 1] + [0] * 6), "constant coefficients"),
])
def test_create_rejects(rtmod, kw, frag):
    st, msg = _create(rtmod, **kw)
    assert st == rtmod.RT_E_ARG and frag in msg, (st, msg)


def test_null_pointers(rtmod):
    L = rtmod.lib()
    assert L.rt_create(None, None) == rtmod.RT_E_ARG
    assert L.rt_estimate(None, None, 1, 1.0, 10, 0, None, None) == rtmod.RT_E_ARG
    assert L.rt_get_stats(None, None) == rtmod.RT_E_ARG
    assert L.rt_destroy(None) == rtmod.RT_OK


def test_pade_arg_checks(rtmod):
    L = rtmod.lib()
    c = np.zeros(13)
    u = np.zeros(1)
    assert L.rt_pade(c.ctypes.data, 1, 12, 7, 7, None, u.ctypes.data, None) == rtmod.RT_E_ARG
    assert "L + M <= K" in L.rt_last_error().decode()
    assert L.rt_pade(c.ctypes.data, 0, 12, 1, 1, None, u.ctypes.data, None) == rtmod.RT_E_ARG
    assert L.rt_pade(c.ctypes.data, 1, 12, -1, 1, None, u.ctypes.data, None) == rtmod.RT_E_ARG
    c31 = np.zeros(32)
    assert L.rt_pade(c31.ctypes.data, 1, 31, 1, 1, None, u.ctypes.data, None) == rtmod.RT_E_ARG


def test_product_does_not_import_oracle():
    """The product package never imports or links the oracle (test infra)."""
    pkg = os.path.join(ROOT, "paper_2402_06491_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read().lower()
                assert "import oracle" not in src and "liboracle" not in src and \
                    "rt_oracle" not in src, f
