#!/usr/bin/env python
"""Print the key counters of an `ncu --page raw --csv` export (one or more kernels).
usage: ncu_summary.py raw.csv [raw2.csv ...]"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__t_bytes.sum", "L1 bytes"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 inst %"),
    ("sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma inst %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem"),
    ("smsp__inst_executed.sum", "inst"),
    ("local_load", "local"),
]


def main(paths):
    for path in paths:
        rows = list(csv.reader(open(path)))
        if len(rows) < 3:
            print(path, "empty")
            continue
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            print(f"== {path}: {d.get('Kernel Name', '?')[:110]}")
            for k, name in KEYS:
                if k in d:
                    print(f"   {name:14s} {d[k]:>18s} {u.get(k, '')}")
            stalls = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled") or
                      k.startswith("smsp__warp_issue_stalled") and k.endswith("per_warp_active.pct")]
            vals = []
            for k, v in stalls:
                try:
                    vals.append((float(v.replace(",", "")), k))
                except ValueError:
                    pass
            for v, k in sorted(vals, reverse=True)[:6]:
                print(f"   stall {k.replace('smsp__warp_issue_stalled_', '')[:60]:60s} {v:8.2f}")


if __name__ == "__main__":
    main(sys.argv[1:])
