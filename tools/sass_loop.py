"""Static SASS census of the tree-walk main loop (no GPU needed).

    python tools/sass_loop.py [mangled-kernel-substring]   (default: <3, 3, false>)

Finds the kernel in librt.so, the largest backward branch (the particle
loop) and prints the opcode histogram of the straight-line body."""
import collections
import re
import subprocess
import sys

so = "paper_2402_06491_b200/librt.so"
want = sys.argv[1] if len(sys.argv) > 1 else "tree_walk_kernelILi3ELi3ELb0E"
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
body = next(f for f in funcs if f.startswith("_ZN3rtk16" + want) or want in f.split("\n")[0])
ins = []
for ln in body.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
print("kernel instructions:", len(ins))
loops = []
for a, t in ins:
    m = re.search(r"BRA\s.*?(0x[0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        loops.append((a - int(m.group(1), 16), int(m.group(1), 16), a))
loops.sort(reverse=True)
for span, lo, hi in loops[:6]:
    print(f"backward branch {hi:#x} -> {lo:#x}: {span // 16} instructions")
span, lo, hi = max((l for l in loops if not any(x in dict(ins)[l[2]] for x in ("BRA 0x",)) or True),
                   key=lambda l: l[0])
c = collections.Counter()
for a, t in ins:
    if lo <= a <= hi:
        op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0]
        c[op] += 1
print(f"loop body {lo:#x}..{hi:#x}: {sum(c.values())} instructions")
print("  ".join(f"{k}:{v}" for k, v in c.most_common(40)))
