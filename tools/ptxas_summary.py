"""Summarise registers / spills per tree_walk instantiation from build_ptxas.log."""
import re
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "paper_2402_06491_b200/build_ptxas.log"
fn = sp = None
for line in open(path):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        fn = m.group(1)
        continue
    if fn and "tree_walk" in fn:
        m = re.search(r"(\d+) bytes spill stores", line)
        if m:
            sp = m.group(1)
        m2 = re.search(r"Used (\d+) registers", line)
        if m2:
            name = re.sub(r"_ZN3rtk16tree_walk_kernelI|EEvNS_10WalkParamsE", "", fn)
            print(f"{name:28s} spill={sp} regs={m2.group(1)}")
            fn = None
