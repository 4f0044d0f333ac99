"""Write a markdown summary of one GPU cycle (tools/gpu_cycle.sh <tag>) into
profiles/<round>/<tag>.md and copy the evidence files beside it.

    python tools/profile_report.py <tag> [round]

Reads gpurun_out/{bench_cfg4,bench_cfg2}_<tag>.log (bench JSON lines),
gpurun_out/launches_<tag>.csv (ncu launch list of the default bench command)
and gpurun_out/prof_tw_<tag>.ncu-rep (ncu --set full of the tree walk)."""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def bench_line(path):
    if not os.path.exists(path):
        return None
    for ln in open(path):
        ln = ln.strip()
        if ln.startswith("{"):
            return json.loads(ln)
    return None


def launches(path):
    rows = [ln for ln in open(path) if not ln.startswith("==")]
    tot, n = collections.Counter(), collections.Counter()
    for r in csv.DictReader(rows):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0]
        tot[k] += float(r["Metric Value"])
        n[k] += 1
    return tot, n


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout


def main():
    tag = sys.argv[1]
    rnd = sys.argv[2] if len(sys.argv) > 2 else "r1"
    dst = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    md = [f"# GPU cycle `{tag}` (1 x B200)", ""]
    host = os.path.join(OUT, f"host_{tag}.txt")
    if os.path.exists(host):
        md += ["Host: " + " / ".join(x.strip() for x in open(host) if x.strip()), ""]
    tests = os.path.join(OUT, f"gpu_tests_{tag}.log")
    if os.path.exists(tests):
        md += ["`pytest -m gpu`: " + " ".join(open(tests).read().strip().splitlines()[-2:]), ""]
    md += ["## Bench lines (`python bench.py`; the others with `--config <cfg>`)", ""]
    for cfg in ("cfg4", "cfg1", "cfg2", "cfg3"):
        b = bench_line(os.path.join(OUT, f"bench_{cfg}_{tag}.log"))
        if not b:
            continue
        rf = b["roofline"]
        md.append(f"- **{cfg}**: {b['value']:.4g} trees/s, {b['leaf_evals_per_s']:.4g} leaf-evals/s, "
                  f"{b['ms_per_step']:.2f} ms/step; tree-walk launch {rf['launch_ms']:.2f} ms; "
                  f"roofline ({rf['bound']}) achieved {rf['achieved']:.3f} of {rf['peak']:.3f} {rf['unit']} "
                  f"= **{rf['frac']:.3f}**"
                  + (f" (SURVEY textbook table {rf['frac_survey_textbook_table']:.3f})"
                     if "frac_survey_textbook_table" in rf else "")
                  + f"; clocks {b['clocks']}; e2e {b['e2e']['value']:.4g} trees/s"
                  + (f"; oracle {b['cpu_baseline']['value']:.4g} trees/s on {b['cpu_baseline']['cores']} core"
                     if b.get("cpu_baseline") else ""))
        shutil.copy(os.path.join(OUT, f"bench_{cfg}_{tag}.log"), dst)
    md.append("")
    lc = os.path.join(OUT, f"launches_{tag}.csv")
    if os.path.exists(lc):
        tot, n = launches(lc)
        T = sum(tot.values())
        md += ["## Launch list (ncu `gpu__time_duration.sum`, --clock-control none; default bench command "
               "with --steps 2 --warmup 3)", "", "| kernel | launches | total ms | share | avg ms |",
               "|---|---|---|---|---|"]
        for k, v in tot.most_common():
            md.append(f"| `{k}` | {n[k]} | {v / 1e6:.3f} | {v / T * 100:.2f} % | {v / n[k] / 1e6:.3f} |")
        md.append("")
        shutil.copy(lc, dst)
    tc = os.path.join(OUT, f"traffic_cfg4_{tag}.csv")
    if os.path.exists(tc):
        md += ["## ncu hardware counters, one full-size cfg4 tree-walk launch", "", "```",
               run([sys.executable, "tools/traffic_json.py", tc, "cfg4", tag]).strip(), "```", ""]
        shutil.copy(tc, dst)
    for name, what in ((f"prof_tw_{tag}", "cfg4 equation, 1024 nodes x 2e5 trees"),
                       (f"prof_tw_cfg4_{tag}", "cfg4 equation, 1024 nodes x 2e5 trees"),
                       (f"prof_tw_cfg2_{tag}", "cfg2, 64 nodes x 1e6 trees")):
        rep = os.path.join(OUT, name + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        md += [f"## ncu --set full, tree-walk kernel ({what})", "", "```",
               run([sys.executable, "tools/ncu_summary.py", rep]).strip(), "```", "",
               "Per-iteration instruction budget (runs of equal execution count):", "", "```",
               run([sys.executable, "tools/ncu_blocks.py", rep]).strip(), "```", ""]
        if "cfg2" not in name:   # the report (30 MB with sources) travels xz-compressed
            subprocess.run(["xz", "-9", "-T8", "-c", rep], stdout=open(
                os.path.join(dst, name + ".ncu-rep.xz"), "wb"), check=True)
    path = os.path.join(dst, f"{tag}.md")
    with open(path, "w") as f:
        f.write("\n".join(md) + "\n")
    print(path)


if __name__ == "__main__":
    main()
