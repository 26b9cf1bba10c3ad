#!/usr/bin/env python
"""GMRES convergence of the heterogeneous C4 problem for a few anomaly sizes / contrasts."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_01299_b200 import Plan  # noqa: E402
from paper_1909_01299_b200.lfds import LfdsError  # noqa: E402
from workloads import anomaly, make_problem  # noqa: E402

p = make_problem(sys.argv[1] if len(sys.argv) > 1 else "c4")
plan = Plan.from_problem(p)
f = torch.from_numpy(p.rhs(0)).cuda()
for eps, lo, hi, zlo, zhi in [(-0.03, 0.45, 0.55, 0.4, 0.6), (-0.1, 0.45, 0.55, 0.4, 0.6), (-0.03, 0.375, 0.625, 0.375, 0.625),
                              (-0.01, 0.375, 0.625, 0.375, 0.625)]:
    dl = torch.from_numpy(anomaly(p, eps=eps, box=((zlo, zhi), (lo, hi), (lo, hi)))).cuda()
    t = time.time()
    try:
        u, rep = plan.solve_hetero(f, dl, tol=1e-10, restart=16, maxit=160)
        torch.cuda.synchronize()
        print(f"eps {eps} box xy [{lo},{hi}) z [{zlo},{zhi}): {rep} {time.time() - t:.2f} s", flush=True)
    except LfdsError as e:
        print(f"eps {eps} box xy [{lo},{hi}) z [{zlo},{zhi}): {e} {time.time() - t:.2f} s", flush=True)
