"""Thin ctypes binding of librt.so (include/rt.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module
only converts torch tensors / numpy arrays to pointers and status codes to
exceptions.  PyTorch supplies device memory and the current stream.  There is
no CPU fallback: if the library or a CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RT_LIB_VARIANT=debug selects the bounds-checked build (librt_debug.so, tests only)
LIB_PATH = os.path.join(_HERE, "librt_debug.so" if os.environ.get("RT_LIB_VARIANT") == "debug"
                        else "librt.so")

RT_OK, RT_E_ARG, RT_E_CUDA, RT_E_NOMEM, RT_E_STATE, RT_E_NUMERIC = 0, 1, 2, 3, 4, 5
G_CONST, G_TANH_STEP, G_GAUSS, G_LORENTZ = 0, 1, 2, 3
OFFSPRING_ABS, OFFSPRING_UNIFORM = 0, 1
PREC_FP64, PREC_FP32_POS = 0, 1

# every symbol include/rt.h declares
SYMBOLS = ("rt_create", "rt_destroy", "rt_estimate", "rt_estimate_dev", "rt_sums_dev",
           "rt_finalize_dev", "rt_pade", "rt_pade_dev", "rt_interface_values", "rt_trace_dev",
           "rt_get_stats", "rt_set_launch", "rt_set_pool", "rt_philox_dev", "rt_last_error",
           "rt_pdd_nodes", "rt_pdd_downstream_dev", "rt_pdd_solve", "rt_fp64_peak")


class RTError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"rt status {status}: {msg}")
        self.status = status


class EqParams(C.Structure):
    _fields_ = [("dim", C.c_int32), ("D", C.c_double), ("degree", C.c_int32),
                ("b", C.c_double * 9), ("lam", C.c_double), ("offspring", C.c_int32),
                ("init_kind", C.c_int32), ("init_amp", C.c_double), ("init_scale", C.c_double),
                ("K", C.c_int32), ("precision", C.c_int32),
                ("strategy", C.c_int32), ("q", C.c_double), ("coef_kind", C.c_int32 * 9),
                ("coef_axis", C.c_int32), ("coef_scale", C.c_double), ("coef_t0", C.c_double),
                ("shared", C.c_int32)]


class PddCfg(C.Structure):
    _fields_ = [("lo", C.c_double), ("hi", C.c_double), ("T", C.c_double), ("n_cells", C.c_int32),
                ("n_steps", C.c_int32), ("n_s", C.c_int32), ("n_t", C.c_int32),
                ("boundary", C.c_int32), ("L", C.c_int32), ("M", C.c_int32),
                ("n_trees", C.c_int64), ("seed", C.c_uint64)]


def pdd_cfg(c: dict) -> PddCfg:
    p = PddCfg()
    for k, _ in PddCfg._fields_:
        setattr(p, k, c[k])
    return p


class Stats(C.Structure):
    _fields_ = [("trees", C.c_int64), ("pruned", C.c_int64), ("particles", C.c_int64),
                ("leaves", C.c_int64), ("splits", C.c_int64), ("kernel_ms", C.c_double),
                ("total_ms", C.c_double)]


class Plane(C.Structure):
    _fields_ = [("axis", C.c_int32), ("value", C.c_double), ("lo", C.c_double),
                ("hi", C.c_double), ("n_per_dim", C.c_int32)]


TREE_REC_DTYPE = np.dtype([("ne", np.int32), ("leaves", np.int32), ("particles", np.int32),
                           ("pruned", np.int32), ("C", np.float64)])

_lib = None


def lib():
    """Load librt.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2402_06491_b200.build`")
        L = C.CDLL(LIB_PATH)
        vp, dp, i64, i32, u64 = C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_uint64
        H = C.c_void_p
        sig = {
            "rt_create": ([C.POINTER(EqParams), C.POINTER(C.c_void_p)]),
            "rt_destroy": ([H]),
            "rt_estimate": ([H, dp, i64, C.c_double, i64, u64, dp, dp]),
            "rt_estimate_dev": ([H, dp, i64, C.c_double, i64, u64, dp, dp, vp]),
            "rt_sums_dev": ([H, dp, i64, C.c_double, i64, i64, u64, dp, vp]),
            "rt_finalize_dev": ([dp, i64, i32, i64, dp, dp, dp, dp, vp]),
            "rt_pade": ([dp, i64, i32, i32, i32, dp, dp, vp]),
            "rt_pade_dev": ([dp, i64, i32, i32, i32, dp, dp, vp, vp]),
            "rt_interface_values": ([H, C.POINTER(Plane), i32, i64, C.c_double, i64, u64, i32, i32,
                                     dp, dp, dp, vp, C.POINTER(C.c_int64)]),
            "rt_trace_dev": ([H, dp, i64, C.c_double, i64, i64, u64, i32, vp, dp, vp]),
            "rt_get_stats": ([H, C.POINTER(Stats)]),
            "rt_set_launch": ([H, i32, i64]),
            "rt_set_pool": ([H, i32]),
            "rt_pdd_nodes": ([C.POINTER(PddCfg), dp]),
            "rt_pdd_downstream_dev": ([H, C.POINTER(PddCfg), dp, dp, dp, vp]),
            "rt_pdd_solve": ([H, C.POINTER(PddCfg), dp, dp, dp]),
            "rt_fp64_peak": ([C.POINTER(C.c_double), C.POINTER(C.c_double)]),
            "rt_philox_dev": ([u64, vp, i64, vp, vp]),
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.rt_last_error.argtypes = []
        L.rt_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(status: int):
    if status != RT_OK:
        raise RTError(status, lib().rt_last_error().decode())


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev_f64(x, dim: int):
    import torch
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float64:
        raise TypeError("expected a CUDA float64 tensor")
    x = x.contiguous()
    if x.dim() == 1:
        x = x.reshape(-1, dim)
    if x.shape[-1] != dim:
        raise ValueError(f"points must be [n, {dim}]")
    return x


def eq_params(eq: dict) -> EqParams:
    p = EqParams()
    p.dim = eq["dim"]; p.D = eq["D"]; p.degree = eq["degree"]
    b = list(eq["b"]) + [0.0] * 9
    for k in range(9):
        p.b[k] = b[k]
    p.lam = eq.get("lam", 0.0); p.offspring = eq.get("offspring", OFFSPRING_ABS)
    p.init_kind = eq["init_kind"]; p.init_amp = eq["init_amp"]
    p.init_scale = eq.get("init_scale", 1.0); p.K = eq["K"]
    p.precision = eq.get("precision", PREC_FP64)
    p.strategy = eq.get("strategy", 0)
    p.q = eq.get("q", 0.5)
    ck = eq.get("coef_kind", [0] * 9)
    for k in range(9):
        p.coef_kind[k] = ck[k]
    p.coef_axis = eq.get("coef_axis", 0)
    p.coef_scale = eq.get("coef_scale", 1.0)
    p.coef_t0 = eq.get("coef_t0", 0.1)
    p.shared = eq.get("shared", 0)
    return p


class Estimator:
    """A handle (rt_create) for one equation; methods mirror the C ABI."""

    def __init__(self, eq: dict):
        self.eq = dict(eq)
        self.dim = eq["dim"]
        self.K = eq["K"]
        h = C.c_void_p()
        self._p = eq_params(eq)
        _check(lib().rt_create(C.byref(self._p), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().rt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_launch(self, grid_ctas: int = 0, trees_per_task: int = 0):
        _check(lib().rt_set_launch(self._h, grid_ctas, trees_per_task))

    def set_pool(self, entries: int = 0):
        """Cap the per-warp shared-memory stack pool (0 = automatic); smaller
        pools push more stack entries to the global overflow area (tests)."""
        _check(lib().rt_set_pool(self._h, entries))

    # -- NEXT row f1: probabilistic domain decomposition (rt_pdd_*) ----------
    def pdd_solve(self, cfg: dict):
        """rt_pdd_solve: the whole PDD on host buffers.  Returns (field
        [(n+1), (n+1)], nodal values [6, n_t, n_s], {T_MC, T_INT, T_LOCAL} ms)."""
        n1 = cfg["n_cells"] + 1
        F = np.empty((n1, n1))
        V = np.empty((6, cfg["n_t"], cfg["n_s"]))
        ms = np.empty(3)
        _check(lib().rt_pdd_solve(self._h, C.byref(pdd_cfg(cfg)), _ptr(F), _ptr(V), _ptr(ms)))
        return F, V, dict(T_MC=float(ms[0]), T_INT=float(ms[1]), T_LOCAL=float(ms[2]))

    def pdd_downstream(self, cfg: dict, nodal, want_bc: bool = False, stream=None):
        """rt_pdd_downstream_dev on a CUDA tensor nodal [6, n_t, n_s]: returns
        (field [(n+1), (n+1)], boundary tables [6, n_steps+1, n+1] or None)."""
        import torch
        V = _dev_f64(nodal, cfg["n_s"]).reshape(6, cfg["n_t"], cfg["n_s"])
        n1 = cfg["n_cells"] + 1
        F = torch.empty((n1, n1), dtype=torch.float64, device=V.device)
        bc = torch.empty((6, cfg["n_steps"] + 1, n1), dtype=torch.float64, device=V.device) \
            if want_bc else None
        _check(lib().rt_pdd_downstream_dev(self._h, C.byref(pdd_cfg(cfg)), _ptr(V), _ptr(F), _ptr(bc),
                                           _stream(stream)))
        return F, bc

    # -- device API ---------------------------------------------------------
    def estimate(self, points, t: float, n_trees: int, seed: int, stream=None):
        """(coeffs, stderr) [n, K+1] CUDA float64 tensors (rt_estimate_dev)."""
        import torch
        x = _dev_f64(points, self.dim)
        n = x.shape[0]
        c = torch.empty((n, self.K + 1), dtype=torch.float64, device=x.device)
        s = torch.empty_like(c)
        _check(lib().rt_estimate_dev(self._h, _ptr(x), n, float(t), int(n_trees), int(seed),
                                     _ptr(c), _ptr(s), _stream(stream)))
        return c, s

    def sums(self, points, t: float, n_trees: int, seed: int, tree_offset: int = 0,
             stream=None, out=None):
        """Raw order-binned sums [n, K+2, 3] (rt_sums_dev)."""
        import torch
        x = _dev_f64(points, self.dim)
        n = x.shape[0]
        out = out if out is not None else torch.empty((n, self.K + 2, 3), dtype=torch.float64,
                                                      device=x.device)
        _check(lib().rt_sums_dev(self._h, _ptr(x), n, float(t), int(tree_offset), int(n_trees),
                                 int(seed), _ptr(out), _stream(stream)))
        return out

    def trace(self, points, t: float, n_trees: int, seed: int, tree_offset: int = 0,
              rec_shift: int = 0, stream=None):
        """Per-tree records of the production kernel -> (records ndarray [n, n_rec], sums)."""
        import torch
        x = _dev_f64(points, self.dim)
        n = x.shape[0]
        n_rec = (n_trees + (1 << rec_shift) - 1) >> rec_shift
        rec = torch.zeros((n, n_rec, 3), dtype=torch.float64, device=x.device)  # 24 B records
        sums = torch.empty((n, self.K + 2, 3), dtype=torch.float64, device=x.device)
        _check(lib().rt_trace_dev(self._h, _ptr(x), n, float(t), int(tree_offset), int(n_trees),
                                  int(seed), int(rec_shift), _ptr(rec), _ptr(sums),
                                  _stream(stream)))
        raw = rec.cpu().numpy().view(np.uint8).reshape(n, n_rec, 24)
        return np.ascontiguousarray(raw).view(TREE_REC_DTYPE).reshape(n, n_rec), sums

    def stats(self) -> dict:
        st = Stats()
        _check(lib().rt_get_stats(self._h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in Stats._fields_}

    # -- host API -----------------------------------------------------------
    def estimate_host(self, points: np.ndarray, t: float, n_trees: int, seed: int,
                      out_coeffs: Optional[np.ndarray] = None,
                      out_stderr: Optional[np.ndarray] = None):
        """rt_estimate on host buffers (numpy arrays or pinned CPU tensors)."""
        if isinstance(points, np.ndarray):
            pts = np.ascontiguousarray(points, dtype=np.float64)
            n = pts.size // self.dim
        else:
            pts = points
            n = pts.numel() // self.dim
        if out_coeffs is None:
            out_coeffs = np.empty((n, self.K + 1), dtype=np.float64)
        if out_stderr is None:
            out_stderr = np.empty((n, self.K + 1), dtype=np.float64)
        _check(lib().rt_estimate(self._h, _ptr(pts), n, float(t), int(n_trees), int(seed),
                                 _ptr(out_coeffs), _ptr(out_stderr)))
        return out_coeffs, out_stderr

    def interface_values(self, planes: Sequence[dict], max_points: int, t: float, n_trees: int,
                         seed: int, L: int, M: int):
        arr = (Plane * len(planes))()
        for q, pl in enumerate(planes):
            arr[q].axis = pl["axis"]; arr[q].value = pl["value"]; arr[q].lo = pl["lo"]
            arr[q].hi = pl["hi"]; arr[q].n_per_dim = pl["n_per_dim"]
        pts = np.empty((max_points, self.dim), dtype=np.float64)
        u = np.empty(max_points); se = np.empty(max_points)
        fl = np.empty(max_points, dtype=np.uint32)
        n = C.c_int64()
        _check(lib().rt_interface_values(self._h, arr, len(planes), int(max_points), float(t),
                                         int(n_trees), int(seed), int(L), int(M), _ptr(pts),
                                         _ptr(u), _ptr(se), _ptr(fl), C.byref(n)))
        k = n.value
        return pts[:k].copy(), u[:k].copy(), se[:k].copy(), fl[:k].copy()


def finalize(sums, K: int, n_total: int, stream=None):
    """(coeffs, stderr, u_sum, se_sum) from raw sums (rt_finalize_dev)."""
    import torch
    n = sums.shape[0]
    dev = sums.device
    c = torch.empty((n, K + 1), dtype=torch.float64, device=dev)
    s = torch.empty_like(c)
    us = torch.empty(n, dtype=torch.float64, device=dev)
    ses = torch.empty_like(us)
    _check(lib().rt_finalize_dev(_ptr(sums.contiguous()), n, K, int(n_total), _ptr(c), _ptr(s),
                                 _ptr(us), _ptr(ses), _stream(stream)))
    return c, s, us, ses


def pade(coeffs, L: int, M: int, se_sum=None, stream=None):
    """[L/M] Padé at z = 1 per row (rt_pade_dev) -> (u, flags) CUDA tensors;
    se_sum (CUDA tensor [n], optional) enables flag bit3."""
    import torch
    c = coeffs.contiguous()
    n, k1 = c.shape
    u = torch.empty(n, dtype=torch.float64, device=c.device)
    fl = torch.empty(n, dtype=torch.int32, device=c.device)
    se = None if se_sum is None else se_sum.contiguous()
    _check(lib().rt_pade_dev(_ptr(c), n, k1 - 1, int(L), int(M), _ptr(se), _ptr(u), _ptr(fl),
                             _stream(stream)))
    return u, fl


def pade_host(coeffs: np.ndarray, L: int, M: int, se_sum=None):
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    if c.ndim == 1:
        c = c.reshape(1, -1)
    n, k1 = c.shape
    u = np.empty(n); fl = np.empty(n, dtype=np.uint32)
    se = None if se_sum is None else np.ascontiguousarray(se_sum, dtype=np.float64).reshape(n)
    _check(lib().rt_pade(_ptr(c), n, k1 - 1, int(L), int(M), _ptr(se), _ptr(u), _ptr(fl)))
    return u, fl


def philox(key: int, ctr):
    """Library Philox4x32-10 on device: ctr uint32 [n, 4] tensor -> [n, 4] (as int32 bits)."""
    import torch
    c = ctr.contiguous()
    out = torch.empty_like(c)
    _check(lib().rt_philox_dev(int(key), _ptr(c), c.shape[0], _ptr(out), _stream()))
    return out


def pdd_nodes(cfg: dict) -> np.ndarray:
    """rt_pdd_nodes: nodal point coordinates [6, n_s, 2] of the PDD lines."""
    out = np.empty((6, cfg["n_s"], 2))
    _check(lib().rt_pdd_nodes(C.byref(pdd_cfg(cfg)), _ptr(out)))
    return out


def fp64_peak() -> dict:
    """rt_fp64_peak: measured FP64 FMA throughput (lane-ops/s) of cuda:current."""
    v, ms = C.c_double(), C.c_double()
    _check(lib().rt_fp64_peak(C.byref(v), C.byref(ms)))
    return dict(lane_ops_per_s=v.value, ms=ms.value)
