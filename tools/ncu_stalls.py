#!/usr/bin/env python
"""Top warp-stall reasons (pc-sampling share) of `ncu --page raw --csv` exports.
usage: ncu_stalls.py raw.csv [raw2.csv ...]"""
import csv
import sys

for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr, vals = rows[0], rows[2]
    st = {}
    for h, v in zip(hdr, vals):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v.replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    top = sorted(st.items(), key=lambda kv: -kv[1])[:8]
    print(f.split("/")[-1] + ": " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
