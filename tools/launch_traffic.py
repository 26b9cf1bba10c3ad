#!/usr/bin/env python
"""Per-kernel-kind DRAM traffic and device-time shares of one solve pass, from an ncu launch list
taken with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum over a
bench.py run (profiles/README.md).  Writes profiles/ncu_traffic.json[config]["kernels"][kind] =
{dram_bytes_per_pass, launches_per_pass, ns_per_pass} (bench.py's roofline.kernels traffic ratio)
and prints the share table.  ncu times are cold-cache and serialised: compare SHARES.
usage: launch_traffic.py <config> <launches.csv> [--write]"""
import csv
import json
import os
import re
import sys

KINDS = [(r"k_xform3m<", "k_xform3m"), (r"k_xform<|k_xsmall<", "k_xform"), (r"k_xplane<", "k_xplane"), (r"k_dstw<", "k_dstw"), (r"k_dst2<", "k_dst2"), (r"k_dstt<", "k_dstt"),
         (r"k_dst<", "k_dst"), (r"k_zs1<", "k_zs1"), (r"k_zs2<", "k_zs2"), (r"k_zs3<", "k_zs3"),
         (r"k_proj_rows<|k_proj<", "k_proj_rows"), (r"k_projm", "k_projm"), (r"k_s5m<|k_p2sum", "k_s5m"),
         (r"k_iface_res", "k_iface_res"), (r"k_write_iface", "k_write_iface"), (r"k_gemm", "k_gemm"),
         (r"k_zsw", "k_zsw"), (r"k_fold|k_unfold", "k_fold"), (r"k_residual", "k_residual"), (r"k_axpy", "k_axpy")]


def kind_of(name):
    for rx, k in KINDS:
        if re.search(rx, name):
            return k
    return None


def main(cfg, path, write):
    rows = {}
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        key = r["ID"]
        ent = rows.setdefault(key, {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            ent["ns"] = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        else:
            ent[r["Metric Name"]] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    # solve passes in the capture: one step-2 z-solve each
    npass = sum(1 for e in rows.values() if kind_of(e["name"]) == "k_zs1") or 1
    agg = {}
    for e in rows.values():
        k = kind_of(e["name"])
        if k is None:
            continue
        a = agg.setdefault(k, {"dram_bytes_per_pass": 0.0, "launches_per_pass": 0.0, "ns_per_pass": 0.0})
        a["dram_bytes_per_pass"] += (e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)) / npass
        a["launches_per_pass"] += 1.0 / npass
        a["ns_per_pass"] += e.get("ns", 0) / npass
    tot = sum(a["ns_per_pass"] for a in agg.values()) or 1
    print(f"{cfg}: {npass} solve passes in {path}")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns_per_pass"]):
        a["share"] = a["ns_per_pass"] / tot
        print(f"  {k:14s} {a['ns_per_pass'] / 1e6:8.3f} ms  share {a['share']:.3f}  "
              f"dram {a['dram_bytes_per_pass'] / 1e9:7.2f} GB  launches {a['launches_per_pass']:.0f}")
    if write:
        out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
        data = json.load(open(out)) if os.path.exists(out) else {}
        data.setdefault(cfg, {})["kernels"] = agg
        data[cfg]["kernels_source"] = os.path.basename(path)
        json.dump(data, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], "--write" in sys.argv)
