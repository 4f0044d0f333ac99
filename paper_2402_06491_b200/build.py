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
SOURCES = [os.path.join(CSRC, "rt_api.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("tree_walk.cuh", "philox.cuh", "rt_math.cuh", "rt_math_tables.h", "pdd.cuh", "shared_eval.cuh")] + \
    [os.path.join(ROOT, "include", "rt.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return SO
    tmp = SO + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *SOURCES, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build_ptxas.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed ({r.returncode}); see {log}")
    fn = ""
    for line in r.stderr.splitlines():
        if "Compiling entry function" in line:
            fn = line
        elif "spill stores" in line and "tree_walk" in fn and \
                not line.strip().startswith("0 bytes stack frame, 0 bytes spill stores, 0 bytes spill loads"):
            raise RuntimeError("tree_walk kernel uses local memory: " + fn + " :: " + line)
    os.replace(tmp, SO)
    if verbose:
        print(r.stderr)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
