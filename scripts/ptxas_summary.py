#!/usr/bin/env python
"""Registers / spills per kernel from a ptxas -v log:  python scripts/ptxas_summary.py LOG [substring]"""
import re
import subprocess
import sys

log, pat = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
cur, out = None, {}
for line in open(log):
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"Function properties for (\w+)", line)
    if m:
        cur = m.group(1)
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        out.setdefault(cur, {})["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        out.setdefault(cur, {})["regs"] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(out), capture_output=True, text=True).stdout.split("\n")
for (k, v), n in zip(out.items(), names):
    if pat in n:
        print(f"{v.get('regs', '?'):>4} regs  spill {v.get('spill', (0, 0))}  {n[:150]}")
