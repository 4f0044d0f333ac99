"""Per-iteration instruction budget of the tree-walk loop from an ncu report:
runs of consecutive SASS instructions with equal execution counts, normalised
by the loop-head execution count."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) >= len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
cnt = [int(r[ix["Instructions Executed"]] or 0) for r in data]
ops = []
for r in data:
    t = r[ix["Source"]].strip().split()
    ops.append((t[1] if t and t[0].startswith("@") else (t[0] if t else "")))
# one iteration = one particle step = the first Philox multiply (M0 = 0xD2511F53)
src = [r[ix["Source"]] for r in data]
it = next((c for c, t in zip(cnt, src) if "IMAD.WIDE.U32" in t and "-0x2daee0ad" in t and c > 0), max(cnt))
print(f"iterations {it}, instructions/iteration {sum(cnt) / it:.1f}")
cur, start = None, 0
blocks = []
for k, c in enumerate(cnt + [None]):
    if c != cur:
        if cur is not None and cur > 0:
            blocks.append((start, k - 1, cur))
        cur, start = c, k
for a, b, c in blocks:
    w = c / it * (b - a + 1)
    if w < 0.5:
        continue
    thr = float(data[a][ix["Avg. Threads Executed"]] or 0)
    hist = collections.Counter(o.split(".")[0] for o in ops[a:b + 1])
    print(f"{a:4d}-{b:4d} x{c / it:5.2f} thr{thr:5.1f} n={b - a + 1:3d} per-iter={w:6.1f}  "
          + " ".join(f"{k}:{v}" for k, v in hist.most_common(8)))
