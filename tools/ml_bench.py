"""Multi-level vs two-level solve time at full size (PAPER.md:77-79 remark; DESIGN §8 row 4).

python tools/ml_bench.py --config c4q --coarse 256 [--steps 5 --warmup 3]
  coarse = stride of the coarse interfaces along x and y (every config interface that is a
  multiple of it), the fine ones are the config's own.  Device time per solve with CUDA events
  on the solve stream (inputs > L2, so no flush), and the relative residual in double-double
  through the two-level plan's lfds_residual.  Prints one JSON line.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_01299_b200 import MLPlan, Plan  # noqa: E402
from workloads import make_problem  # noqa: E402


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4q")
    ap.add_argument("--coarse", type=int, nargs="+", default=[256])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--two-level", type=int, default=1, dest="two")
    a = ap.parse_args()
    p = make_problem(a.config)
    rng = np.random.default_rng(1)
    F = (rng.standard_normal(p.shape) + 1j * rng.standard_normal(p.shape)).astype(np.complex128)
    f = torch.from_numpy(F).cuda()
    del F
    u = torch.empty_like(f)
    plan = Plan.from_problem(p)
    out = {"workload": a.config, "shape": list(p.shape), "fine_x": list(p.iface_x)}
    if a.two:
        out["two_level_ms"] = timed(lambda: plan.solve(f, out=u), a.steps, a.warmup)
        _, nr = plan.residual(u, f)
        out["two_level_rel_residual"] = float(nr[0, 0] / nr[0, 1])
    for c in a.coarse:
        cx = [i for i in p.iface_x if i % c == 0]
        cy = [i for i in p.iface_y if i % c == 0]
        ml = MLPlan(p.hx, p.hy, p.hz, p.sigma_node, p.sigma_edge, p.lam, cx, cy, p.iface_x, p.iface_y)
        ms = timed(lambda: ml.solve(f, out=u), a.steps, a.warmup)
        _, nr = plan.residual(u, f)
        out[f"ml_{c}"] = {"coarse_x": cx, "coarse_blocks": ml.n_coarse_blocks(), "ms": ms,
                          "rel_residual": float(nr[0, 0] / nr[0, 1]),
                          "workspace_gb": ml.workspace().numel() / 1e9}
        ml.close()
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
