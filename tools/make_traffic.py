#!/usr/bin/env python
"""Build profiles/ncu_traffic.json (per config, per bench stage: DRAM bytes read + written per
launch, from `ncu --set full` raw exports) for bench.py's roofline.traffic field.
usage: make_traffic.py <config> <raw.csv>... (stage inferred from the kernel name)"""
import csv
import json
import os
import re
import sys

STAGES = [  # (regex on the demangled kernel name, bench stages it stands for)
    (r"k_s5m<", ["step5_global_zsolve"]),
    (r"k_zs3", ["step5_global_zsolve"]),
    (r"k_dstw<", ["step1_x_sine", "step7_x_sine"]),
    (r"k_dst2<", ["step1_plane_sine", "step7_plane_sine"]),
    (r"k_zs2", ["step6_zsolve_lift"]),
    (r"k_zs1", ["step2_zsolve"]),
    (r"k_dst<.*, (1|true)>", ["step1_x_sine", "step7_x_sine"]),
    (r"k_dst<.*, (0|false)>", ["step1_y_sine", "step7_y_sine"]),
    (r"k_xform3m<(1|true)>", ["step1_x_dense", "step7_x_dense"]),
    (r"k_xform3m<(0|false)>", ["step1_y_dense", "step7_y_dense"]),
    (r"k_projm<", ["step5_projection"]),
    (r"k_proj(_rows)?<", ["step3_edge_projection"]),
]


def main(cfg, paths):
    out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    d = data.setdefault(cfg, {})
    for path in paths:
        rows = list(csv.reader(open(path)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            row = dict(zip(hdr, r))
            unit = dict(zip(hdr, units))
            name = row.get("Kernel Name", "")

            def val(k):
                v = float(row[k].replace(",", ""))
                u = unit.get(k, "byte").lower()
                return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}.get(u, 1)
            b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
            for rx, stages in STAGES:
                if re.search(rx, name):
                    for s in stages:
                        d[s] = {"dram_bytes_per_launch": b, "kernel": name[:120], "source": os.path.basename(path)}
                    break
    json.dump(data, open(out_path, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
