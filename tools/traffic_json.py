"""profiles/r2/traffic_<workload>.json from the ncu metrics CSV of one
full-size tree-walk launch (tools/gpu_perf.sh): DRAM and L2 traffic, FP64-pipe
and issue utilisation, and instructions per loop iteration (particles from
the same launch's bench stats are not available to ncu, so the iteration
count is passed in).  python tools/traffic_json.py <csv> <workload> <tag>
[iterations]"""
import csv
import json
import os
import sys

path, workload, tag = sys.argv[1:4]
iters = float(sys.argv[4]) if len(sys.argv) > 4 else None
rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("==")) if r]
h = rows[0]
m = {r[h.index("Metric Name")]: r[h.index("Metric Value")].replace(",", "") for r in rows[1:]}
kern = rows[1][h.index("Kernel Name")]
out = {
    "workload": workload,
    "kernel": kern,
    "dram_bytes_read": int(float(m["dram__bytes_read.sum"])),
    "dram_bytes_write": int(float(m["dram__bytes_write.sum"])),
    "lts_bytes": int(float(m["lts__t_bytes.sum"])),
    "launch_ns": int(float(m["gpu__time_duration.sum"])),
    "fp64_pipe_pct": float(m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
    "issue_active_pct": float(m["sm__inst_issued.avg.pct_of_peak_sustained_active"]),
    "warp_inst": int(float(m["smsp__inst_executed.sum"])),
    "threads_per_inst": float(m["smsp__thread_inst_executed_per_inst_executed.ratio"]),
    "source": f"ncu --metrics ... --clock-control none -k regex:tree_walk -s 3 -c 1 python bench.py "
              f"--steps 1 --warmup 3 --no-cpu-baseline --graph off (tools/gpu_perf.sh, round {tag})",
}
if iters:
    out["inst_per_iteration"] = out["warp_inst"] / iters
os.makedirs("profiles/r2", exist_ok=True)
with open(f"profiles/r2/traffic_{workload}.json", "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
