#!/usr/bin/env python
"""Add the k_xplane entry of a config to profiles/ncu_traffic.json["<config>"]["kernels"] from an
`ncu --set full` raw export holding one launch of each form of one direction (forward): DRAM bytes
per solve pass over all right-hand sides (bench.py's unit) = 2 directions x the sum over the forms
x the RHS chunks per pass (C5: 64 right-hand sides in chunks of 16 -> 4).
usage: xplane_traffic.py <config> <ncu_k_xplane_raw.csv> [chunks]"""
import csv
import json
import os
import sys


def main(cfg, path, chunks=1):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    seen, total, ns = set(), 0.0, 0.0
    for r in rows[2:]:
        row, unit = dict(zip(hdr, r)), dict(zip(hdr, units))
        name = row.get("Kernel Name", "")
        if "k_xplane" not in name or name in seen:
            continue
        seen.add(name)
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            total += float(row[m].replace(",", "")) * scale.get(unit[m], 1.0)
        tu = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "ns": 1.0, "us": 1e3, "ms": 1e6}
        ns += float(row["gpu__time_duration.sum"].replace(",", "")) * tu.get(unit["gpu__time_duration.sum"], 1.0)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
    data = json.load(open(out)) if os.path.exists(out) else {}
    ent = data.setdefault(cfg, {}).setdefault("kernels", {})
    total, ns = total * chunks, ns * chunks
    ent["k_xplane"] = {"dram_bytes_per_pass": 2 * total, "launches_per_pass": 2.0 * len(seen) * chunks, "ns_per_pass": 2 * ns,
                       "source": os.path.relpath(path, os.path.join(os.path.dirname(out), ".."))}
    json.dump(data, open(out, "w"), indent=1)
    print(cfg, "k_xplane forms", len(seen), "dram GB per pass", 2 * total / 1e9, "ms per pass", 2 * ns / 1e6)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 1)
