"""Warp stall reasons (cycles per issued instruction) of an ncu report."""
import csv
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
out = []
for h, v in zip(r[0], r[2]):
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
        try:
            out.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
print("  ".join(f"{n}:{v:.2f}" for v, n in sorted(out, reverse=True) if v >= 0.01))
