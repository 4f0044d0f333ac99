"""Memory-safety evidence without compute-sanitizer (closed on the GPU pool):
the parity tests that stress every index path — all tree-parity
configurations (every strategy, dimension, shared trees), the stack pool's
overflow area, 55-bit labels and K = 30 depths, the PDD downstream, the
randomised equations of test_gpu_fuzz.py — re-run
against the bounds-checked build librt_debug.so (-DRT_DEBUG_BOUNDS: device
checks on every computed pool / free-list / overflow / ring / slot / partials
index; a failed check traps the kernel).  They must pass unchanged."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def test_parity_suite_under_bounds_checks():
    sys.path.insert(0, ROOT)
    from paper_2402_06491_b200 import build as b
    b.build(debug=True)
    env = dict(os.environ, RT_LIB_VARIANT="debug")
    which = subprocess.run([sys.executable, "-c", "import paper_2402_06491_b200.rt as r; print(r.LIB_PATH)"],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert which.stdout.strip().endswith("librt_debug.so"), which.stdout + which.stderr
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                        os.path.join(HERE, "test_gpu_parity.py"), os.path.join(HERE, "test_gpu_pdd.py"),
                        os.path.join(HERE, "test_gpu_fuzz.py"),
                        "-k", "tree_parity or pool or extreme or geometry or pdd_downstream or edge or chunks or ring"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    tail = r.stdout.strip().splitlines()[-1]
    print("bounds-checked run:", tail)
    assert " passed" in tail and "failed" not in tail
