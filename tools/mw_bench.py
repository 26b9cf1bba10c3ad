"""Lebedev-grid Maxwell solve at full size (§3): device time per solve,
per-kernel-group times and rooflines, residual.  Prints one JSON line.

python tools/mw_bench.py [--config mw1] [--steps 10 --warmup 3]
Inputs: workloads.maxwell (seeded, drawn on the device); the fields (3.2 GB each) exceed L2.
Roofline: the transform groups are FP64 tensor-pipe (DMMA) bound — algorithmic flops 8 per
complex x complex MAC (complex bases) or 4 per real x complex MAC (real bases), against the
in-run DMMA peak (lfds.fp64_peak); gather / scatter / z-solve are HBM bound — algorithmic bytes
read once + written once, against MEASURED_PEAKS.json.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_01299_b200 import MWPlan  # noqa: E402
from paper_1909_01299_b200 import lfds  # noqa: E402
from workloads.maxwell import make_mw, rhs_torch  # noqa: E402


def hbm_peak():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        for k in ("hbm_gbs", "hbm_GBps", "hbm"):
            if k in d:
                v = d[k]
                return float(v["value"] if isinstance(v, dict) else v), "MEASURED_PEAKS.json " + k
    except Exception:
        pass
    return 7700.0, "nominal (MEASURED_PEAKS.json missing)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mw1")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--two-level", type=int, nargs="*", default=[], dest="two",
                    help="also time the two-level solve with B x B blocks for each B given")
    a = ap.parse_args()
    p = make_mw(a.config)
    nz, ny, nx = p.shape
    f = rhs_torch(p)
    t0 = torch.cuda.Event(enable_timing=True)
    plan = MWPlan.from_problem(p)
    H = torch.empty_like(f)
    for _ in range(a.warmup):
        plan.solve(f, out=H)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        plan.solve(f, out=H)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    r = plan.residual(H, f)
    rel = float(torch.linalg.vector_norm(r) / torch.linalg.vector_norm(f))
    del r
    # per-kernel groups (untimed profiled solves after the timed region)
    prof = MWPlan.from_problem(p, profile=True)
    for _ in range(3):
        prof.solve(f, out=H)
    kt = prof.kernel_times()
    prof.close()
    two = {}
    for B in a.two:
        from paper_1909_01299_b200 import MW2Plan
        step = (nx - 1) // B
        ix = [b * step - (b * step) % 2 for b in range(1, B)]
        stepy = (ny - 1) // B
        iy = [b * stepy - (b * stepy) % 2 for b in range(1, B)]
        p2 = MW2Plan.from_problem(p, ix, iy)
        H2 = torch.empty_like(f)
        for _ in range(a.warmup):
            p2.solve(f, out=H2)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.steps):
            p2.solve(f, out=H2)
        e1.record()
        torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1) / a.steps
        r2 = plan.residual(H2, f)
        two[f"{B}x{B}"] = {"ix": ix, "iy": iy, "ms": ms2, "rel_residual": float(torch.linalg.vector_norm(r2) /
                                                                              torch.linalg.vector_norm(f)),
                           "rel_diff_vs_layered": float(torch.linalg.vector_norm(H2 - H) / torch.linalg.vector_norm(H)),
                           "workspace_gb": p2.workspace().numel() / 1e9}
        del r2, H2
        p2.close()
        torch.cuda.empty_cache()
    plan.close()
    n = (nx - 1) // 2, (ny - 1) // 2, (nz - 1) // 2
    # unknowns: 3 components on the interior P nodes (i + j + k even, 1 <= i <= N - 2)
    par = [[sum(1 for i in range(1, N - 1) if i % 2 == q) for q in (0, 1)] for N in (nx, ny, nz)]
    unknowns = 3 * sum(par[0][a] * par[1][b] * par[2][c] for a in (0, 1) for b in (0, 1) for c in (0, 1)
                       if (a + b + c) % 2 == 0)
    realx = all(complex(h).imag == 0 for h in p.hx)
    realy = all(complex(h).imag == 0 for h in p.hy)
    hx_, hy_, hz_ = n
    # family sizes: nodes per axis family (primary n-1, dual n); levels: even n_z-1, odd n_z
    fams = [(hx_ - 1, hy_ - 1, hz_ - 1), (hx_, hy_, hz_ - 1), (hx_ - 1, hy_, hz_), (hx_, hy_ - 1, hz_)]
    def xflops(real):
        per = 4 if real else 8
        return sum(per * fx * fx * 3 * lev * fy for fx, fy, lev in fams)
    def yflops(real):
        per = 4 if real else 8
        return sum(per * fy * fy * 3 * lev * hx_ for fx, fy, lev in fams)
    coef = sum(3 * lev * hx_ * hy_ for _, _, lev in fams)
    full = 3 * nz * ny * nx
    alg = {"k_mw_xfwd": ("tensor", xflops(realx)), "k_mw_xinv": ("tensor", xflops(realx)),
           "k_mw_yfwd": ("tensor", yflops(realy)), "k_mw_yinv": ("tensor", yflops(realy)),
           "k_mw_gather": ("hbm", 16 * (full + coef)), "k_mw_scatter": ("hbm", 16 * (full + coef)),
           "k_mw_zsolve": ("hbm", 16 * 2 * coef)}
    peak_fp64 = lfds.fp64_peak()
    hbm, hsrc = hbm_peak()
    total = sum(v[0] for v in kt.values())
    kernels = {}
    for k, (t, cnt) in kt.items():
        per = t / max(cnt, 1)
        b, w = alg[k]
        if b == "tensor":
            ach, pk, unit = w / (per * 1e-3) / 1e12, peak_fp64, "TFLOP/s"
        else:
            ach, pk, unit = w / (per * 1e-3) / 1e9, hbm, "GB/s"
        kernels[k] = {"ms": per, "share": t / total, "bound": b, "achieved": ach, "peak": pk, "unit": unit,
                      "frac": ach / pk, "algorithmic": w}
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    out = {"metric": "unknowns solved/sec (Maxwell H, complex128 direct solve)", "value": unknowns / (ms * 1e-3),
           "unit": "unknowns/s", "ms_per_step": ms, "steps": a.steps, "warmup": a.warmup, "dtype": "c128",
           "config": {"workload": a.config, "grid_nodes": [nx, ny, nz], "unknowns": unknowns,
                      "real_bases": [realx, realy], "rel_residual": rel, "l2": "inputs > L2 (3.2 GB fields)"},
           "roofline": dict(kernels[dom], kernel=dom), "kernels": kernels, "fp64_peak_tflops_in_run": peak_fp64,
           "hbm_peak_source": hsrc, "two_level": two, "kernel_times_from": "CUDA events per launch group, profiled solves after the timed region"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
