#!/usr/bin/env python
"""Summarise `nvcc -Xptxas -v` output (stdin): one line per kernel with registers, stack,
spills and shared memory.  usage: nvcc ... -Xptxas -v 2>&1 | python tools/ptxas_summary.py [filter]"""
import re
import subprocess
import sys

filt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
info = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        info[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        info[cur].update(stack=int(m.group(1)), sst=int(m.group(2)), sld=int(m.group(3)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        info[cur]["regs"] = int(m.group(1))
        m2 = re.search(r"(\d+) bytes smem", line)
        info[cur]["smem"] = int(m2.group(1)) if m2 else 0
names = list(info)
try:
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
except Exception:
    dem = names
for n, d in zip(names, dem):
    if filt and filt not in d:
        continue
    d = re.sub(r"lfds::\(anonymous namespace\)::", "", d)
    d = d.split("(")[0]
    i = info[n]
    print(f"{d:60s} regs {i.get('regs', '?'):>4} stack {i.get('stack', 0):>4} spill {i.get('sst', 0)}/{i.get('sld', 0)} smem {i.get('smem', 0)}")
