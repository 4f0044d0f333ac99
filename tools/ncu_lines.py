"""Per-source-line instruction / stall attribution of an ncu report (cuda,sass page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None
hdr = None
agg = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] != "" and len(r) >= 8:
        try:
            n = int(r[7] or 0)
            smp = int(r[4] or 0)
        except ValueError:
            continue
        if n > 0 or smp > 0:
            agg.append((n, smp, f"{cur}:{r[0]}", r[1].strip()[:90]))
tot = sum(a[0] for a in agg)
tots = sum(a[1] for a in agg)
print(f"total warp instructions {tot:.4g}, stall samples {tots}")
for n, smp, loc, src in sorted(agg, reverse=True)[:top]:
    print(f"{n / tot * 100:5.1f}% inst {smp / tots * 100:5.1f}% stall  {loc:22s} {src}")
