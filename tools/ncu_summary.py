"""Print the key tree_walk metrics of an ncu report (details page + SASS opcode mix)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
KEYS = ["Duration", "Registers Per Thread", "Achieved Active Warps Per SM", "Theoretical Occupancy",
        "Issue Slots Busy", "Executed Ipc Active", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Eligible Warps Per Scheduler", "No Eligible",
        "Compute (SM) Throughput", "Branch Efficiency"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
for row in csv.reader(out.splitlines()):
    if len(row) > 4 and row[-4] in KEYS:
        print(f"{row[-4]:40s} {row[-2]:>14s} {row[-3]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
want = ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__inst_executed.sum", "gpu__time_duration.sum"]
for h, u, v in zip(r[0], r[1], r[2]):
    if h in want:
        print(f"{h:70s} {v:>18s} {u}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
tot = 0
by = collections.Counter()
for row in rows[2:]:
    if len(row) < len(hdr):
        continue
    s = row[ix["Source"]].strip()
    t = s.split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    n = int(row[ix["Instructions Executed"]] or 0)
    by[op.split(".")[0]] += n
    tot += n
print("warp instructions executed:", tot)
print("  ".join(f"{k}:{v / tot * 100:.1f}%" for k, v in by.most_common(30)))
