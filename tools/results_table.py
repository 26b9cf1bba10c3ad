#!/usr/bin/env python
"""Markdown rows of DESIGN.md §11 from the bench JSON lines of an evidence run.
usage: python tools/results_table.py [dir]   (default profiles/r01/bench_final)"""
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else os.path.join("profiles", "r01", "bench_final")
for c in ["c4", "c4j", "c4q", "c3", "c2", "c1", "c5", "c4h"]:
    p = os.path.join(d, f"bench_{c}.json")
    if not os.path.exists(p):
        continue
    j = json.loads(open(p).read().strip().splitlines()[-1])
    r = j["roofline"]
    e2e = j.get("e2e") or {}
    cpu = j.get("cpu_baseline") or {}
    sol = r.get("solve") or {}
    res = j["config"].get("rel_residual_dd") or j["config"].get("rel_residual_preconditioned")
    mg = (j["config"].get("resonance_margin") or {}).get("margin_global_rel")
    share = r.get("share")
    print(f"| {c} | {j['ms_per_step']:.3f} | {j['value']:.3g} | {e2e.get('value', float('nan')):.3g} "
          f"({e2e.get('ms_per_step', float('nan')):.1f} ms) | {cpu.get('value', float('nan')):.2g} | "
          f"{r.get('kernel')} ({share if share is None else f'{share:.0%}'} of the step, {r['frac']:.2f} of "
          f"{r['bound']}) | {sol.get('frac', float('nan')):.3f} ({sol.get('t_roof_ms', float('nan')):.2f} ms) | "
          f"{res if res is None else f'{res:.1e}'} | {mg if mg is None else f'{mg:.1e}'} |")
