#!/usr/bin/env python
"""Per-kernel registers / spills from an nvcc -Xptxas -v log (fused kernels)."""
import re
import subprocess
import sys

txt = open(sys.argv[1]).read().splitlines()
cur = None
for i, line in enumerate(txt):
    m = re.search(r"Compiling entry function '(\S+)'", line) or re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
    m2 = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m2 and cur and "fused" in cur:
        regs = None
        for l2 in txt[i + 1:i + 3]:
            r = re.search(r"Used (\d+) registers", l2)
            if r:
                regs = r.group(1)
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        name = re.sub(r".*Cfg<(.*?)>.*", r"Cfg<\1>", name)
        print(f"{name:28s} regs {regs}  spill st {m2.group(2)} ld {m2.group(3)}")
        cur = None
