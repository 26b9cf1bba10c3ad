#!/usr/bin/env python
"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel: total time,
launch count and share.  usage: summarize_launches.py launches.csv [steps_profiled]"""
import collections
import csv
import sys


def main(path, steps=1):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        k = d["Kernel Name"].replace("(anonymous namespace)::", "")
        k = k.split("(")[0] if not k.startswith("void") else k.split("(")[0]
        agg.setdefault(k, [0.0, 0])
        agg[k][0] += float(d["Metric Value"])
        agg[k][1] += 1
    tot = sum(v[0] for v in agg.values())
    print(f"# {path}: {len(data)} launches, {tot/1e6:.3f} ms total (cold-cache, serialised)")
    print(f"{'ms/step':>9} {'launches':>8} {'share':>6}  kernel")
    for k, (v, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{v/1e6/steps:9.3f} {n:8d} {100*v/tot:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1)
