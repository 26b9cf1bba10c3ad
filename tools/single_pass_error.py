#!/usr/bin/env python
"""Single-pass (no refinement) forward error of the GPU solve against the oracle's refined
solution on a full-size config, for the z-modal and the z-sweep step 5 (R13 evidence).
usage: python tools/single_pass_error.py c5 [rhs_index]"""
import dataclasses
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1909_01299_b200 import Plan  # noqa: E402
from workloads import make_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
r = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = make_problem(name)
p = dataclasses.replace(p, nrhs=max(p.nrhs, r + 1)) if p.nrhs <= r else p
F = p.rhs(r)[None]
t0 = time.time()
ref = oracle.solve(p, F[0])
print(f"{name} oracle (ii) + 80-bit refinement: {time.time() - t0:.1f} s")
f = torch.from_numpy(F).cuda()
cases = [(True, 0, True), (True, 1, True), (True, 1, False), (False, 0, True), (False, 1, True)]
for modal, refine, dd in cases:
    plan = Plan.from_problem(p, s5_modal=modal, refine=refine, residual_dd=dd)
    u = plan.solve(f).cpu().numpy()[0]
    err = float(np.linalg.norm(u - ref) / np.linalg.norm(ref))
    _, norms = plan.residual(torch.from_numpy(u[None]).cuda(), f, dd=True)
    print(f"{name} s5_modal={int(modal)} refine={refine} residual_dd={int(dd)}: rel error {err:.3e}, "
          f"rel residual {float(norms[0, 0] / norms[0, 1]):.3e}")
    plan.close()
