#!/usr/bin/env python
"""Sine-transform stage times of the C4 grid under uniform partitions of spacing s (core blocks
of s-1 nodes, L = 2s), with the plane transform (options.plane_dst) on and off.
usage: python tools/plane_dst_ab.py [s ...]   (default 32 64 128)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_01299_b200 import Plan  # noqa: E402
from workloads import make_problem  # noqa: E402

base = make_problem("c4")
f = torch.from_numpy(base.rhs(0)[None]).cuda()
for s in [int(a) for a in sys.argv[1:]] or [32, 64, 128]:
    j = [s * b for b in range(1, base.nx // s)]
    p = base.with_partition(j, j)
    for pd in (1, 0):
        plan = Plan.from_problem(p, profile=True, plane_dst=bool(pd), graph=True)
        for _ in range(2):
            u = plan.solve(f)
        torch.cuda.synchronize()
        plan.stage_times()
        n = 5
        for _ in range(n):
            u = plan.solve(f)
        torch.cuda.synchronize()
        st = plan.stage_times()
        sine = {k: v[0] / n for k, v in st.items() if "sine" in k and v[1]}
        tot = sum(v[0] for v in st.values()) / n
        print(f"s={s} L={2 * s} plane_dst={pd}: stages total {tot:.3f} ms, sine {sum(sine.values()):.3f} ms",
              " ".join(f"{k}={v:.3f}" for k, v in sine.items()), flush=True)
        del plan, u
        torch.cuda.empty_cache()
