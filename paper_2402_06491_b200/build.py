"""Build the sm_100a shared library librt.so in-tree (nvcc cross-compiles
without a GPU).  ``python -m paper_2402_06491_b200.build``."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "librt.so")
SO_DEBUG = os.path.join(HERE, "librt_debug.so")   # -DRT_DEBUG_BOUNDS (tests/test_gpu_bounds.py)
SOURCES = [os.path.join(CSRC, "rt_api.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("tree_walk.cuh", "philox.cuh", "rt_math.cuh", "rt_math_tables.h", "pdd.cuh", "shared_eval.cuh", "pade.cuh")] + \
    [os.path.join(ROOT, "include", "rt.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]


def stale(so: str = SO) -> bool:
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    so = SO_DEBUG if debug else SO
    if not force and not stale(so):
        return so
    tmp = so + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *(["-DRT_DEBUG_BOUNDS"] if debug else []), *SOURCES, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build_ptxas_debug.log" if debug else "build_ptxas.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed ({r.returncode}); see {log}")
    fn = ""
    for line in r.stderr.splitlines():
        if "Compiling entry function" in line:
            fn = line
        elif not debug and "spill stores" in line and "tree_walk" in fn and \
                not line.strip().startswith("0 bytes stack frame, 0 bytes spill stores, 0 bytes spill loads"):
            raise RuntimeError("tree_walk kernel uses local memory: " + fn + " :: " + line)
    os.replace(tmp, so)
    if verbose:
        print(r.stderr)
    return so


def build_all(force: bool = False) -> None:
    """The production and the bounds-checked library, compiled concurrently."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(2) as ex:
        for f in [ex.submit(build, force, False, False), ex.submit(build, force, False, True)]:
            f.result()


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))
