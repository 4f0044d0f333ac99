"""Host logic of bench.py's roofline accounting (no GPU): the algorithmic
FP64 cost model and its shared-tree crediting."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import workloads as W  # noqa: E402


def test_cost_model_per_unit_counts():
    """Per-unit costs follow the libdevice table: d = 3 draws one more cosine
    normal than d = 2, which draws one sin/cos pair more than d = 1's cosine."""
    u1 = bench.algo_fp64_per_unit(W.get("cfg2")["eq"])
    u3 = bench.algo_fp64_per_unit(W.get("cfg4")["eq"])
    assert u1["particle"] < u3["particle"]
    assert u3["tree"] == 3 and u1["split"] == 2
    # Lorentzian g (cfg4): r² (2d-1 ops) + two divisions + the product
    assert u3["leaf"] == 5 + 2 * bench.LD["div"] + 1 + 1


def test_shared_trees_credit_the_walk_once():
    """Shared trees walk each tree once for all nodes: particles and splits are
    credited once per tree, g evaluations and accumulations once per node."""
    eq = dict(W.get("cfg4")["eq"], shared=1)
    st = dict(particles=1000.0, leaves=600.0, splits=300.0, trees=100.0)
    u = bench.algo_fp64_per_unit(eq)
    n = 8
    got = bench.algo_fp64_ops(eq, st, n)
    want = (1000 / n) * u["particle"] + 600 * u["leaf"] + (300 / n) * u["split"] + 100 * u["tree"]
    assert abs(got - want) < 1e-9 * want
    # independent trees: no scaling whatever n_points says
    eq0 = W.get("cfg4")["eq"]
    assert bench.algo_fp64_ops(eq0, st, n) == bench.algo_fp64_ops(eq0, st)
