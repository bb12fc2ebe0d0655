#!/usr/bin/env python
"""Summarise an `ncu --page source --csv --print-source sass` dump of the fused
kernel by barrier-delimited segment (= kernel stage): stall samples per
reason, executed instructions.  Usage: sass_segments.py dump.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
iS = h.index("Source")
iE = h.index("Instructions Executed")
reasons = ["stall_barrier", "stall_long_sb", "stall_short_sb", "stall_wait", "stall_math", "stall_mio",
           "stall_selected", "stall_not_selected", "stall_branch_resolving", "stall_no_inst", "stall_lg"]
idx = {r: h.index(r) for r in reasons}
segs, cur, n, ex = [], {r: 0.0 for r in reasons}, 0, 0.0
for r in data:
    for k, i in idx.items():
        cur[k] += float(r[i] or 0)
    ex += float(r[iE] or 0)
    n += 1
    if "BAR.SYNC" in r[iS]:
        segs.append((n, ex, cur))
        cur, n, ex = {k: 0.0 for k in reasons}, 0, 0.0
segs.append((n, ex, cur))
tot = sum(sum(c.values()) for _, _, c in segs)
print("seg  instr   exec(M)  samples%  " + " ".join(r.replace("stall_", "")[:9].rjust(9) for r in reasons))
for k, (n, ex, c) in enumerate(segs):
    s = sum(c.values())
    print(f"{k:3d} {n:6d} {ex / 1e6:8.1f} {100 * s / tot:8.1f}  " +
          " ".join(f"{100 * c[r] / tot:9.1f}" for r in reasons))
