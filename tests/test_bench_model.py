"""Host logic of bench.py's roofline accounting (no GPU): the algorithmic
FP64 cost model and its shared-tree crediting."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import workloads as W  # noqa: E402


def test_cost_model_per_unit_counts():
    """Contract units (R29): per particle ONE Gamma(m+1)
    variate (m multiplies + 1 log), its m+1 shares (m+1 multiplies, m
    subtractions), 4 clock ops, per radius 2 multiplies + 1 sqrt, one angle
    per normal pair (+ the third normal's), d FMAs.  basis="survey" is SURVEY
    §8(d)'s textbook list: one exponential variate, ⌈d/2⌉ Box–Muller pairs,
    one sqrt, d + 3 plain ops."""
    u1 = bench.algo_fp64_per_unit(W.get("cfg2")["eq"])
    u3 = bench.algo_fp64_per_unit(W.get("cfg4")["eq"])
    assert u1["particle"] == (1 + 20) + (2 + 1) + 4 + 1 * (2 + 8) + 20 + 1 == 59
    assert u3["particle"] == (2 + 20) + (3 + 2) + 4 + 2 * (2 + 8) + 2 * 20 + 3 == 94
    s1 = bench.algo_fp64_per_unit(W.get("cfg2")["eq"], basis="survey")
    s3 = bench.algo_fp64_per_unit(W.get("cfg4")["eq"], basis="survey")
    assert s1["particle"] == 20 + 1 * (20 + 8 + 20) + 8 + 1 + 3 == 80
    assert s3["particle"] == 20 + 2 * (20 + 8 + 20) + 8 + 3 + 3 == 130
    assert u3["tree"] == 3 and u1["split"] == 1
    # Lorentzian g (cfg4): |x|² (2d-1) + /s² + 1 + reciprocal (div 8) + amp, then Π *= g
    assert u3["leaf"] == s3["leaf"] == 5 + 1 + 1 + 8 + 1 + 1
    # Gaussian g (cfg2, d = 1): the textbook per-leaf x² + /s² + exp 15 + amp,
    # then Π *= g; the kernel's closed form — x², one FMA into
    # the exponent sum, amp, Π *= amp per leaf; exp + 1 multiply per tree
    assert s1["leaf"] == 1 + 1 + 15 + 1 + 1
    assert u1["leaf"] == 1 + 1 + 1 + 1 and u1["tree"] == 3 + 15 + 1
    # FP32 positions: only the FP64 part (clock, weights, product, sums)
    u32 = bench.algo_fp64_per_unit(dict(W.get("cfg2")["eq"], precision=W.PREC_FP32_POS))
    assert u32["particle"] == (1 + 20) + (2 + 1) + 4 and u32["leaf"] == 1


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
    # Gaussian data: one exponential per (node, tree); leaves' moments once per tree
    eg = dict(W.get("cfg3")["eq"], shared=1)
    ug = bench.algo_fp64_per_unit(eg)
    got = bench.algo_fp64_ops(eg, st, n)
    want = ((1000 / n) * ug["particle"] + (600 / n) * (2 * 2 + 2) + (300 / n) * ug["split"]
            + (100 / n) * (8 + 2 * 2) + 100 * (2 * 2 + 3 + 15 + ug["tree"]))
    assert abs(got - want) < 1e-9 * want
    # independent trees: no scaling whatever n_points says
    eq0 = W.get("cfg4")["eq"]
    assert bench.algo_fp64_ops(eq0, st, n) == bench.algo_fp64_ops(eq0, st)


def test_cost_model_strategies():
    """Strategy B replaces the clock's log by two plain ops and adds η(τ) = τ
    per split and 1/q per leaf; Strategy A's shift adds e^{(k-1)λτ_c} per split
    and the root factor per tree."""
    base = W.get("ex1A")["eq"]
    ua = bench.algo_fp64_per_unit(base)                       # shift
    ub = bench.algo_fp64_per_unit(W.get("ex1B")["eq"])        # Strategy B
    up = bench.algo_fp64_per_unit(dict(base, strategy=0), basis="survey")   # potential
    assert up["particle"] - ub["particle"] == 20 - 2
    upc = bench.algo_fp64_per_unit(dict(base, strategy=0))   # potential, contract basis
    us = bench.algo_fp64_per_unit(base, basis="survey")      # shift, textbook: e^{(k-1)λτ_c} per split
    assert us["split"] == up["split"] + 15 + 2
    # the kernel's closed form: (k-1)λ and an FMA into the
    # exponent sum per split; the root factor, and e^{+X} = 1/e^{-X} per tree
    assert ua["split"] == upc["split"] + 2 and ua["tree"] == upc["tree"] + 1 + 8
    # variable coefficients: y², /s², X +=, τ_c + t0, D *= per split; 1/D and × per tree
    uv = bench.algo_fp64_per_unit(W.get("ex5A")["eq"])
    assert uv["split"] == 1 + 2 + 5 and uv["tree"] == 3 + 1 + (15 + 1) + 8 + (8 + 1)
    assert ub["split"] == up["split"] + 1 and ub["leaf"] == upc["leaf"] + 1


def test_clock_summary_from_nvidia_smi_rows():
    """The clocks object: median SM clock over samples under load, the
    throttle reasons seen, and NVML samples when nvidia-smi had none."""
    c = bench.ClockSampler(0)
    c.out = ("0, 1965, 1965, 950.1, 0x0, Not Active, Not Active, Not Active, Not Active\n"
             "0, 1950, 1965, 940.0, 0x4, Not Active, Not Active, Not Active, Active\n"
             "0, 1965, 1965, 120.0, 0x1, Not Active, Not Active, Not Active, Not Active\n")
    s = c.summary()
    assert s["sm_mhz"] == 1957.5 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"] and s["samples_under_load"] == 2
    c2 = bench.ClockSampler(0)
    c2.out = ""
    c2.nvml = [(1965, 0), (1965, 0x40), (1950, 0)]
    s2 = c2.summary()
    assert s2["sm_mhz"] == 1965.0 and s2["reasons"] == ["hw_thermal_slowdown"] and s2["source"].startswith("nvml")


def test_reference_arm_json_line():
    """`bench.py --impl reference` (the oracle on host cores, no GPU): one JSON
    line with the contract's keys, e2e with zero copies, and a sample that is a
    subset of the workload (cfg1: 16 nodes x 1e4 trees, run whole)."""
    import json
    import subprocess
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "cfg1", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["unit"] == "trees/s" and line["value"] > 0
    assert line["config"]["workload"] == "cfg1"
    assert line["e2e"] == {"value": line["value"], "unit": "trees/s",
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] == line["value"]
    assert cb["sample"].startswith("16 nodes x 10000 trees of cfg1")
