#!/usr/bin/env python
"""Warp-stall samples of one ncu capture of the fused kernel attributed to source lines.

ncu's SASS source page (per-instruction stall samples) is matched by offset to the
line table of the same kernel in the in-tree build (`nvdisasm -g` of the cubin
extracted with `cuobjdump -xelf`), so the build must be the profiled one.

  python tools/ncu_stall_lines.py REPORT.ncu-rep [KERNEL_MANGLED_NAME] [TOP]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.environ.get("COMMET_LIB") or os.path.join(ROOT, "paper_2510_00884_b200", "libcommet.so")
CSRC = os.path.join(ROOT, "paper_2510_00884_b200", "csrc")
DEFAULT_K = "_ZN6commet12fused_kernelINS_3CfgILi64ELi16ELi8ELi8ELi3ELi0ELi0ELi0ELi4ELi0EEEEEvNS_7AsmArgsE"


def line_table(kernel):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "kernel_fused", LIB], cwd=d, check=True, capture_output=True)
        cubin = [f for f in os.listdir(d) if f.startswith("kernel_fused")][0]
        out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cubin)], capture_output=True, text=True).stdout
    i = out.find(".text." + kernel)
    j = out.find("//---------------------", i + 300)
    line, table = None, {}
    for ln in out[i:j].splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            line = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            table[int(m.group(1), 16)] = line
    return table


def main():
    rep = sys.argv[1]
    kernel = sys.argv[2] if len(sys.argv) > 2 else DEFAULT_K
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    data = [r for r in rows[2:] if r and r[0].startswith("0x")]
    a0 = int(data[0][0], 16)
    stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    table = line_table(kernel)
    total = collections.Counter()
    by_line = collections.defaultdict(collections.Counter)
    for r in data:
        key = table.get(int(r[0], 16) - a0)
        for c in stalls:
            v = int(r[h.index(c)] or 0)
            total[c] += v
            by_line[key][c] += v
    T = sum(total.values())
    print(f"{rep}: {T} warp samples")
    print("stall reasons: " + ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in total.most_common(10)))
    srcs = {}
    for key in by_line:
        if key and key[0] not in srcs:
            p = os.path.join(CSRC, key[0])
            srcs[key[0]] = open(p).read().splitlines() if os.path.exists(p) else []
    print(f"\ntop {top} source lines (share of all samples; main reasons):")
    for key, cnt in sorted(by_line.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
        n = sum(cnt.values())
        text = srcs.get(key[0], [])[key[1] - 1].strip()[:70] if key and srcs.get(key[0]) else ""
        why = ", ".join(f"{k[6:]} {100 * v / n:.0f}%" for k, v in cnt.most_common(3))
        print(f"{100 * n / T:5.2f}%  {key[0] if key else '?'}:{key[1] if key else '?'}  [{why}]  {text}")


if __name__ == "__main__":
    main()
