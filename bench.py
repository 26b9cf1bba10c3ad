#!/usr/bin/env python
"""Benchmark: unknowns solved per second of the blocked separable Helmholtz solve on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One *step* = one lfds_solve of the whole hot path (steps 1-7 of PAPER.md:63-73, plus the
refinement passes the config needs) over one batch of right-hand sides already resident
in HBM.  Default workload: BASELINE.json configs[3] ("c4", 1024 x 1024 x 256, 8 x 8
blocks, complex128) — the largest config, the one north_star's roofline and scaling
targets are quoted on; it fits one GPU (4.3 GB per array, larger than the 126 MB L2, so
no L2 flush is needed between steps).  N > 1 (torchrun): every rank solves its own
share of the blocks S^ij of the same problem (block sharding, north_star: LPT block ownership,
step-5 global modes split by x-mode, two NCCL all-reduces for the interface exchange;
"scaling": "strong"); C5's 64 right-hand sides are split across ranks instead (no collective,
"weak").  The time is the max over ranks.

The reference arm (--impl reference) is the CPU oracle (oracle/, test infrastructure) on
the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import make_problem  # noqa: E402

METRIC = "unknowns solved/sec (complex128 direct solve)"
UNIT = "unknowns/s"
# refinement passes each config needs for the 1e-9 parity bar (DESIGN.md §2 R12/R13): C2's
# BJ-fixed quadratic PML profile has cond(V) ~ 1e5; C5 is near-resonant (single pass 1.6e-9 from
# the refined solution, tests/test_gpu_parity.py::test_full_size_c5_chunked_vs_oracle) -> one
# double-double refinement pass each; C1, C3, C4 need none.
REFINE = {"c1": 0, "c2": 1, "c3": 0, "c4": 0, "c5": 1}
# the refinement residual in fp64 already meets the 1e-9 bar on both (tools/single_pass_error.py:
# C5 2.5e-10, C2 1.9e-16 against the oracle's 80-bit-refined solution; double-double reaches
# 4.4e-14 / 3.6e-18 at ~6x the residual cost), so the timed step uses the fp64 residual
RESIDUAL_DD = {"c2": False, "c5": False}
# right-hand sides per pipeline pass (workspace scales with it): C5's 64 RHS x 0.84 GB per
# array do not fit next to f and u in one pass; 16 per pass keeps the workspace at ~35 GB
RHS_CHUNK = {"c5": 16}
# multi-GPU split (north_star: blocks S^ij over the GPUs, NCCL for the interface exchange);
# C5's 64 independent right-hand sides are split across GPUs instead (no exchange needed)
DEFAULT_SHARD = {"c5": "rhs"}
# FP64 peaks: derived 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz = 37.2 TF/s;
# measured on this pool (profiles/r01_fp64_peaks.log): DMMA 37.1, DFMA 34.2 TF/s.
FP64_PEAK_TFLOPS = 37.2
# LFDS_XPLANE=0 (A/B knob of the library): no plane dense transforms (k_xplane)
XPLANE = os.environ.get("LFDS_XPLANE", "1") != "0"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            mp = json.load(fh)
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def sample_problem(p, nz_sample: int):
    """The same x/y grid, partition, lambda and sigma recipe with N_z reduced (CPU sample)."""
    from workloads.configs import sigma_layers
    nz = p.nz
    # keep the layer structure: resample the cell -> layer map onto nz_sample + 1 cells
    layer_vals = []
    for c in range(nz + 1):
        v = complex(p.sigma_edge[c]).real
        if not layer_vals or layer_vals[-1] != v:
            layer_vals.append(v)
    hz, se, sn = sigma_layers(nz_sample, np.array(layer_vals))
    rng = np.random.default_rng(np.random.SeedSequence([1909, 1299, 900, nz_sample]))
    shape = (nz_sample, p.ny, p.nx)

    def rhs(r):
        out = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / math.sqrt(2)
        return out

    return dataclasses.replace(p, hz=hz, sigma_edge=se, sigma_node=sn, nrhs=1, _rhs=rhs,
                               name=p.name + f"_nz{nz_sample}")


def cpu_oracle_sample(p, nz_sample: int, steps: int = 1):
    """Time the oracle's global separable solve (ii) (setup excluded) on the sample."""
    import oracle
    from oracle.solve import global_bases
    ps = sample_problem(p, nz_sample)
    g = global_bases(ps)
    f = ps.rhs(0)
    b = oracle.mass_rhs(ps, f)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.solve_separable(ps, b, g)
        times.append(time.perf_counter() - t0)
    try:
        from threadpoolctl import threadpool_info
        threads = max([d.get("num_threads", 1) for d in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    return ps, times, threads


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.lines = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def stage_algorithmic(p, R: int, plan=None):
    """Algorithmic (flops, bytes) per launch of each timed stage (DESIGN.md §5 table).

    Dense transform stages: a complex eigenvector matrix (C blocks) costs 8 flops per complex
    MAC, a real one (R blocks) 4 (real matrix x complex data); each element moves 32 B.
    Sine stages (uniform blocks, FFT-based DST): HBM-bound, 32 B per element.
    z-solves: 32 B per unknown (read + write).  Step 5: the rank-|I| contraction costs
    8 (|I_x| + |I_y|) flops per global unknown (RHS build and projection each; both in k_s5m
    in the z-modal form)."""
    def sizes(n, iface):
        cuts = [0] + list(iface) + [n + 1]
        return [cuts[i + 1] - cuts[i] - 1 for i in range(len(cuts) - 1)]
    bx, by = sizes(p.nx, p.iface_x), sizes(p.ny, p.iface_y)
    kx = [plan.basis(0, i)[2] if plan else 2 for i in range(len(bx))]
    ky = [plan.basis(1, j)[2] if plan else 2 for j in range(len(by))]
    nz = p.nz

    def is_sine(kind, n):  # mirrors dst_supported() in lfds_dst.cu
        L = 2 * (n + 1)
        return kind == 0 and (L in (16, 32, 64, 128, 256, 512) or (L % 16 == 0 and L // 16 in (3, 5, 6, 10, 12, 20)))

    esz = 8.0 if p.real else 16.0  # bytes per value (f64 path: real data, real bases)

    def dense(kinds, sz, axis):
        fl, el = 0.0, 0.0
        for i in range(len(bx)):
            for j in range(len(by)):
                k, n = (kinds[i], bx[i]) if axis == 0 else (kinds[j], by[j])
                if xfused(i, j):
                    continue
                if p.real or not is_sine(k, n):  # the f64 path has no sine kernels
                    e = bx[i] * by[j] * nz * R
                    fl += (2.0 if p.real else 8.0 if k == 2 else 4.0) * n * e
                    el += e
        return fl, 2 * esz * el

    plane_dst = bool(getattr(plan, "plane_dst", True)) if plan else True

    def fused(i, j):  # mirrors fused2() in lfds_host.cpp / dst2_supported() in lfds_dst.cu
        return (plane_dst and not p.real and is_sine(kx[i], bx[i]) and is_sine(ky[j], by[j])
                and bx[i] == by[j] and 2 * (bx[i] + 1) in (32, 64, 128))

    def xcand(i, j):  # mirrors xplane() in lfds_host.cpp: two bases of <= 32 nodes, no sine form
        return (XPLANE and not p.real and not fused(i, j)
                and not is_sine(kx[i], bx[i]) and not is_sine(ky[j], by[j]) and bx[i] <= 32 and by[j] <= 32)
    # ... used when such blocks hold at least half of the block unknowns (lfds_host.cpp, setup)
    xp_ok = 2 * sum(bx[i] * by[j] for i in range(len(bx)) for j in range(len(by)) if xcand(i, j)) \
        >= sum(bx[i] * by[j] for i in range(len(bx)) for j in range(len(by)))

    def xfused(i, j):
        return xp_ok and xcand(i, j)

    def sine(kinds, axis):
        el = 0.0
        for i in range(len(bx)):
            for j in range(len(by)):
                k, n = (kinds[i], bx[i]) if axis == 0 else (kinds[j], by[j])
                if is_sine(k, n) and not p.real and not fused(i, j):
                    el += bx[i] * by[j] * nz * R
        return None, 32.0 * el

    # plane sine transform (both axes in one pass): 32 B per element of the fused blocks
    psine = (None, 32.0 * sum(bx[i] * by[j] * nz * R for i in range(len(bx)) for j in range(len(by))
                              if fused(i, j)))
    nf = plan.info().get("n_plane_dst") if plan else None
    if nf is not None and nf != sum(fused(i, j) for i in range(len(bx)) for j in range(len(by))):
        raise RuntimeError(f"plane-transform block count {nf} (library) != bench accounting")
    nxf = plan.info().get("n_plane_dense") if plan else None
    if nxf is not None and nxf != sum(xfused(i, j) for i in range(len(bx)) for j in range(len(by))):
        raise RuntimeError(f"plane-dense block count {nxf} (library) != bench accounting")
    # plane dense transform (k_xplane: both axes in one pass): 4 n flops per element for a real
    # basis, 8 n for a complex one, and 32 B per element
    pdense = (sum(((8.0 if kx[i] == 2 else 4.0) * bx[i] + (8.0 if ky[j] == 2 else 4.0) * by[j])
                  * bx[i] * by[j] * nz * R for i in range(len(bx)) for j in range(len(by))
                  if xfused(i, j)) or None,
              32.0 * sum(bx[i] * by[j] * nz * R for i in range(len(bx)) for j in range(len(by)) if xfused(i, j)))
    el_blk = sum(nx * ny * nz * R for nx in bx for ny in by)
    el_all = p.nx * p.ny * nz * R
    nifx, nify = len(p.iface_x), len(p.iface_y)
    nif = nifx + nify
    cm = 2.0 if p.real else 8.0  # flops per multiply-add (real or complex)
    plane = cm * (nifx * p.ny * p.ny + nify * p.nx * p.nx) * nz * R
    xd, yd = dense(kx, bx, 0), dense(ky, by, 1)
    modal = bool(plan.info().get("s5_modal", 0)) if plan else False
    # z-modal step 5: plane data to and from z-modes, real Z x complex data
    # (4 nz flops per plane element); k_s5m: r^ (8 |I| flops) plus both projections (8 |I|)
    # per global unknown
    zpl = 4.0 * nz * (nifx * p.ny + nify * p.nx) * nz * R
    xs, ys = sine(kx, 0), sine(ky, 1)
    return {
        "step1_x_sine": xs, "step1_x_dense": xd, "step1_y_sine": ys, "step1_y_dense": yd,
        "step2_zsolve": (None, 2 * esz * el_blk),
        "step3_edge_projection": (None, esz * el_blk),
        "step5_plane_forward": ((plane + zpl) if modal else plane, None),
        "step5_global_zsolve": (16.0 * nif * el_all, None) if modal else (cm * nif * el_all, esz * el_all),
        "step5_projection": (zpl, None) if modal else (cm * nif * el_all, esz * el_all),
        "step5_plane_inverse": (plane, None),
        "step6_zsolve_lift": (None, 2 * esz * el_blk),
        "step7_y_sine": ys, "step7_y_dense": yd, "step7_x_sine": xs, "step7_x_dense": xd,
        "step1_plane_sine": psine, "step7_plane_sine": psine,
        "step1_plane_dense": pdense, "step7_plane_dense": pdense,
        # refinement: r = Mf - Au reads u and f and writes r; u += r reads both, writes u
        "refine_residual": (None, 48.0 * el_all), "refine_axpy": (None, 48.0 * el_all),
    }


def kernel_algorithmic(p, R: int, plan=None):
    """Algorithmic (flops, bytes) per solve pass of each kernel kind (DESIGN.md §5 table), the
    same accounting as stage_algorithmic regrouped by the kernel that does the work:

    k_xform3m (complex eigenvector matrix, DMMA 3M): the dense passes of C blocks (8 n flops per
    element and direction), the step-5 plane transforms W^T R / W P (8 N flops per plane element),
    step 3's edge values (W_y G, W_x H: 8 n^2 per edge column) and step 6's face transforms
    (F w-face: 8 n^2 per face column); 32 B per element of the dense passes and planes.
    k_xform (real matrix): dense passes of R blocks (4 n) and the step-5 z-transforms (4 N_z per
    plane element, both directions).  Sine kernels, z-solves, edge projection, refinement: bytes."""
    alg = stage_algorithmic(p, R, plan)

    def sizes(n, iface):
        cuts = [0] + list(iface) + [n + 1]
        return [cuts[i + 1] - cuts[i] - 1 for i in range(len(cuts) - 1)]
    bx, by = sizes(p.nx, p.iface_x), sizes(p.ny, p.iface_y)
    kx = [plan.basis(0, i)[2] if plan else 2 for i in range(len(bx))]
    ky = [plan.basis(1, j)[2] if plan else 2 for j in range(len(by))]
    nz = p.nz
    esz = 8.0 if p.real else 16.0

    def is_sine(kind, n):
        L = 2 * (n + 1)
        return kind == 0 and (L in (16, 32, 64, 128, 256, 512) or (L % 16 == 0 and L // 16 in (3, 5, 6, 10, 12, 20)))

    def xfused(i, j):  # stage_algorithmic's rule (k_xplane blocks)
        fz = (bool(getattr(plan, "plane_dst", True)) if plan else True) and is_sine(kx[i], bx[i]) \
            and is_sine(ky[j], by[j]) and bx[i] == by[j] and 2 * (bx[i] + 1) in (32, 64, 128)
        return (XPLANE and not p.real and not fz
                and not is_sine(kx[i], bx[i]) and not is_sine(ky[j], by[j]) and bx[i] <= 32 and by[j] <= 32)
    xcand = xfused
    xp_ok = 2 * sum(bx[i] * by[j] for i in range(len(bx)) for j in range(len(by)) if xcand(i, j)) \
        >= sum(bx[i] * by[j] for i in range(len(bx)) for j in range(len(by)))

    def xfused(i, j):  # noqa: F811 (the rule above, gated by the plan-level share test)
        return xp_ok and xcand(i, j)

    fc = bc = fr = br = 0.0  # complex-S / real-S dense passes (4 per block: x, y forward + inverse)
    for i in range(len(bx)):
        for j in range(len(by)):
            e = bx[i] * by[j] * nz * R
            if xfused(i, j):
                continue
            for k, n in ((kx[i], bx[i]), (ky[j], by[j])):
                if p.real or is_sine(k, n):
                    continue
                if k == 2:
                    fc += 2 * 8.0 * n * e
                    bc += 2 * 2 * esz * e
                else:
                    fr += 2 * 4.0 * n * e
                    br += 2 * 2 * esz * e
    nifx, nify = len(p.iface_x), len(p.iface_y)
    plane_el = (nifx * p.ny + nify * p.nx) * nz * R
    if nifx + nify and not p.real:
        # forward + inverse plane transforms; a palindromic global axis contracts folded data at
        # half length (lfds_info.global_fold: bit 0 x, bit 1 y)
        gf = plan.info().get("global_fold", 0) if plan else 0
        fy, fxx = (0.5 if gf & 2 else 1.0), (0.5 if gf & 1 else 1.0)
        fc += 2 * 8.0 * (nifx * p.ny * p.ny * fy + nify * p.nx * p.nx * fxx) * nz * R
        bc += 2 * 2 * esz * plane_el
        # step 3 edge values (two edge rows per block side) and step 6 face transforms (one per interior face)
        for i in range(len(bx)):
            for j in range(len(by)):
                fc += 8.0 * (by[j] ** 2 + bx[i] ** 2) * 2 * nz * R
                nfx = (i > 0) + (i < len(bx) - 1)
                nfy = (j > 0) + (j < len(by) - 1)
                fc += 8.0 * (nfx * by[j] ** 2 + nfy * bx[i] ** 2) * nz * R
    modal = bool(plan.info().get("s5_modal", 0)) if plan else False
    if modal:
        fr += 2 * 4.0 * nz * plane_el
        br += 2 * 2 * esz * plane_el
    out = {
        "k_xform3m": (fc or None, bc or None), "k_xform": (fr or None, br or None),
        "k_dstw": (None, (alg["step1_x_sine"][1] or 0) + (alg["step7_x_sine"][1] or 0) or None),
        "k_dst": (None, (alg["step1_y_sine"][1] or 0) + (alg["step7_y_sine"][1] or 0) or None),
        "k_dstt": (None, (alg["step1_y_sine"][1] or 0) + (alg["step7_y_sine"][1] or 0) or None),
        "k_dst2": (None, (alg["step1_plane_sine"][1] or 0) + (alg["step7_plane_sine"][1] or 0) or None),
        "k_xplane": (2 * (alg["step1_plane_dense"][0] or 0) or None, 2 * (alg["step1_plane_dense"][1] or 0) or None),
        "k_zs1": alg["step2_zsolve"], "k_zsw": alg["step2_zsolve"], "k_zs2": alg["step6_zsolve_lift"],
        "k_proj_rows": alg["step3_edge_projection"],
        "k_s5m": (alg["step5_global_zsolve"][0], None) if modal else (None, None),
        "k_zs3": (None, None) if modal else alg["step5_global_zsolve"],
        "k_projm": (None, None) if modal else alg["step5_projection"],
        "k_residual": alg["refine_residual"], "k_axpy": alg["refine_axpy"],
    }
    return out


def kernel_roofline(p, nrhs, plan, kernels, steps, config, passes=1, fp64_peak=None):
    """Per-kernel-kind roofline table: device ms per step (CUDA events around every launch of the
    kind, inside the timed region), share of the summed kernel time, algorithmic work ÷ time
    against the bound that governs it (FP64 tensor for the DMMA contractions, HBM otherwise), and
    ncu DRAM bytes per launch ÷ algorithmic bytes where a capture exists."""
    alg = kernel_algorithmic(p, nrhs, plan)
    hbm_peak, hbm_src = _peaks()
    fpk = fp64_peak or FP64_PEAK_TFLOPS
    try:  # per kernel kind: ncu dram read + write bytes summed over one pass's launches
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh_:
            ncu = json.load(fh_).get(config, {}).get("kernels", {})
    except Exception:
        ncu = {}
    tot = sum(v[0] for v in kernels.values()) or 1.0
    table = {}
    for name, (ms, nl) in kernels.items():
        if not nl:
            continue
        mult = max(1, passes - 1) if name in ("k_residual", "k_axpy") else passes
        per_step_ms = ms / max(1, steps)
        flops, nbytes = alg.get(name, (None, None))
        t_tensor = (flops or 0) / (fpk * 1e12)
        t_hbm = (nbytes or 0) / (hbm_peak * 1e9)
        ent = {"ms_per_step": per_step_ms, "share": ms / tot, "launches_per_step": nl / max(1, steps)}
        if flops and t_tensor >= t_hbm:
            a = flops * mult / (per_step_ms * 1e-3) / 1e12
            ent.update(bound="tensor", achieved=a, peak=fpk, unit="TFLOP/s", frac=a / fpk, alg_flops=flops * mult)
        elif nbytes:
            a = nbytes * mult / (per_step_ms * 1e-3) / 1e9
            ent.update(bound="hbm", achieved=a, peak=hbm_peak, unit="GB/s", frac=a / hbm_peak, alg_bytes=nbytes * mult)
        tr = ncu.get(name)
        if tr:
            ent["ncu_dram_bytes_per_launch"] = tr["dram_bytes_per_pass"] / max(1, tr["launches_per_pass"])
            if nbytes:  # dram traffic of one pass vs its algorithmic bytes (> 1: re-reads)
                ent["ncu_traffic_ratio"] = tr["dram_bytes_per_pass"] / nbytes
        table[name] = ent
    return table


def roofline_summary(p, nrhs, plan, stages, steps, config, ms_max, passes=1, kernels=None, fp64_peak=None):
    """Roofline of the dominant stage and of the whole solve.  Stage work is per
    solve pass over all nrhs right-hand sides; a step runs `passes` of them (1 + refinement
    passes, or the fast solves inside a GMRES solve)."""
    # roofline of the dominant stage (the kernel kind with the largest device time per step);
    # governing bound = whichever of flops/peak and bytes/peak is the larger time
    alg = stage_algorithmic(p, nrhs, plan)
    hbm_peak, hbm_src = _peaks()
    # (stages with a stated algorithmic work; plane-sized glue stages have none)
    cand = {k: v for k, v in stages.items() if any(x for x in alg.get(k, (None, None)))} or stages
    dom = max(cand.items(), key=lambda kv: kv[1][0])
    name, (st_ms, st_launch) = dom
    per_step_ms = st_ms / max(1, steps)
    flops, nbytes = alg.get(name, (None, None))
    # a solve stage runs once per pass; the refinement stages once per refinement
    mult = max(1, passes - 1) if name.startswith("refine_") else passes
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh_:
            ent = json.load(fh_).get(config, {}).get(name)
            traffic = ent["dram_bytes_per_launch"] if ent else None  # ncu dram read+write, one launch
    except Exception:
        pass
    t_tensor = (flops or 0) / (FP64_PEAK_TFLOPS * 1e12)
    t_hbm = (nbytes or 0) / (hbm_peak * 1e9)
    if t_tensor >= t_hbm and flops:
        achieved = flops * mult / (per_step_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic, "kernel": name,
                "peak_source": "FP64 tensor (DMMA) = 148 SMs x 64 FMA/clk x 2 x 1.965 GHz (DESIGN.md §5); "
                               "measured DMMA 37.1 TF/s (profiles/r01_fp64_peaks.log)"}
    else:
        achieved = (nbytes or 0) * mult / (per_step_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic, "kernel": name,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({hbm_src})"}
    # whole-solve roofline: T_roof = max(64 B/unknown / HBM, F_alg / FP64)
    f_alg = sum(v[0] or 0 for k, v in alg.items() if "dense" in k or k.startswith("step5_"))
    b_alg = (64.0 if not p.real else 32.0) * p.unknowns * nrhs
    t_roof = passes * max(b_alg / (hbm_peak * 1e9), f_alg / (FP64_PEAK_TFLOPS * 1e12)) * 1e3
    roof["solve"] = {"t_roof_ms": t_roof, "frac": t_roof / ms_max, "alg_bytes": b_alg, "alg_flops": f_alg}
    roof["stage_ms_per_step"] = {k: v[0] / max(1, steps) for k, v in stages.items() if v[1]}
    roof["passes_per_step"] = passes
    if kernels:
        # the dominant KERNEL (largest device time per step over all its launches) is the one the
        # top-level fields report; the stage view above stays for reference
        table = kernel_roofline(p, nrhs, plan, kernels, steps, config, passes, fp64_peak)
        roof["kernels"] = table
        cand = {k: v for k, v in table.items() if "frac" in v}
        if cand:
            name, ent = max(cand.items(), key=lambda kv: kv[1]["ms_per_step"])
            tr = ent.get("ncu_dram_bytes_per_launch")  # average over the kind's launches
            roof.update(bound=ent["bound"], achieved=ent["achieved"], peak=ent["peak"], unit=ent["unit"],
                        frac=ent["frac"], traffic=tr, kernel=name, share=ent["share"],
                        peak_source=("in-run DMMA loop (lfds_fp64_peak)" if ent["bound"] == "tensor" and fp64_peak
                                     else roof["peak_source"] if ent["bound"] == roof["bound"]
                                     else f"MEASURED_PEAKS.json hbm_gbs ({hbm_src})"))
    return roof


def run_reference(args, rank, world):
    if rank != 0:
        return
    if args.config in HETERO:  # oracle: sparse LU of A_het on the shrunken analog, per step
        import oracle
        from workloads import anomaly, shrunken
        base, eps = HETERO[args.config]
        ps = shrunken(base, nrhs=1)
        dls, fs = anomaly(ps, eps=eps), ps.rhs(0)
        ts = []
        for _ in range(args.warmup + args.steps):
            t1 = time.perf_counter()
            oracle.solve_hetero_direct(ps, dls, fs)
            ts.append(time.perf_counter() - t1)
        t = statistics.mean(ts[args.warmup:])
        val = ps.unknowns / t
        smp = f"{ps.name} analog {ps.shape} with the same anomaly recipe, sparse LU of A_het"
        print(json.dumps({
            "impl": "reference", "metric": METRIC.replace("direct solve", "heterogeneous solve, GMRES + fast-solver preconditioner"),
            "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic", "config": {"workload": args.config, "sample": smp},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "sample": smp},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)
        return
    p = make_problem(args.config)
    nz_s = args.cpu_nz
    ps, ts, threads = cpu_oracle_sample(p, nz_s, args.warmup + args.steps)
    t = statistics.mean(ts[args.warmup:])
    val = ps.unknowns / t
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": args.config, "sample": f"{p.name} with N_z={nz_s} (same x/y grid, blocks, lambda, "
                   f"sigma layers), 1 RHS, oracle (ii) solve only", "nx": p.nx, "ny": p.ny, "nz": nz_s},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{p.name} x/y grid with N_z={nz_s}: {ps.unknowns} unknowns per step"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1909_01299_b200 import Plan
    from paper_1909_01299_b200 import dist as lfds_dist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    p = make_problem(args.config)
    shard = args.shard or DEFAULT_SHARD.get(args.config, "blocks")
    blocks = shard == "blocks" and (world > 1 or args.shard == "blocks")  # --shard blocks: phased path at N=1 too
    allreduce = None if world > 1 else (lambda t: None)
    # blocks: every rank works on the same right-hand sides, owning a share of the blocks and
    # of the step-5 modes (strong scaling); rhs: rank r solves its own right-hand sides
    nrhs = p.nrhs if args.nrhs <= 0 else args.nrhs
    pw = dataclasses.replace(p, nrhs=nrhs * (1 if blocks else world))
    rhs0 = 0 if blocks else rank * nrhs
    refine = REFINE.get(args.config, 0) if args.refine is None else args.refine
    # block-sharded refinement runs in dist.solve_sharded_refined (u completed by a sum over the
    # ranks between the passes); the library plan itself does not refine then
    t0 = time.perf_counter()
    # the timed solve replays a CUDA graph of its launches (options.graph; stage events are graph
    # nodes); the sharded path runs phase by phase with the exchanges in between
    res_dd = RESIDUAL_DD.get(args.config, True)
    # per-kernel events inside the timed region for the long steps; for the short (launch-bound)
    # configs they would perturb the step, so the kernel table comes from separate profiled steps
    kprof_timed = args.config not in SHORT_STEP
    plan = Plan.from_problem(p, device=local_rank, refine=0 if blocks else refine, residual_dd=res_dd,
                             profile=2 if kprof_timed else 1,
                             graph=not blocks, rhs_chunk=0 if blocks else RHS_CHUNK.get(args.config, 0),
                             plane_dst=bool(args.plane_dst), dst_tma=bool(args.dst_tma))
    setup_s = time.perf_counter() - t0
    info0 = plan.info()
    part = lfds_dist.shard(plan, rank, world) if blocks else None
    exchange = args.exchange if blocks and world > 1 else None
    if exchange == "library":
        try:  # both exchanges as ncclAllReduce on the solve stream, inside lfds_solve
            lfds_dist.attach_nccl(plan, rank, world)
        except Exception as exc:  # no usable NCCL in the process: the torch.distributed exchanges
            print(f"rank {rank}: in-library exchanges unavailable ({exc}); using torch.distributed", file=sys.stderr)
            exchange = "torch"
            plan.set_comm(None)
    dt = torch.float64 if p.real else torch.complex128
    # right-hand sides generated one at a time straight into device memory (C5: 64 x 0.84 GB)
    f = torch.empty((nrhs,) + p.shape, dtype=dt, device=dev)
    for r in range(nrhs):
        f[r].copy_(torch.from_numpy(pw.rhs(rhs0 + r)))
    u = torch.zeros_like(f)
    ws = plan.workspace(nrhs) if blocks else None

    def sharded_solve(f_, u_):
        if refine:
            lfds_dist.solve_sharded_refined(plan, f_, u_, ws, refine, allreduce, dd=res_dd)
        else:
            lfds_dist.solve_sharded(plan, f_, u_, ws, allreduce)

    def step():
        if blocks:
            sharded_solve(f, u)
        else:
            plan.solve(f, out=u)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    plan.stage_times()  # reset
    plan.kernel_times()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    stages = plan.stage_times()
    kernels = plan.kernel_times()
    rep0 = plan.report()
    if not kprof_timed:  # untimed profiled steps for the per-kernel table (same launches)
        plan.set_profile(2)
        for _ in range(max(3, args.steps)):
            step()
        torch.cuda.synchronize()
        plan.stage_times()
        kernels = plan.kernel_times()
        plan.set_profile(1)
    launches_per_step = rep0["n_kernel_launches"]
    piv = rep0["min_pivot_ratio"]
    tmax = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    units = p.unknowns * nrhs * (1 if blocks else world)
    value = units / (ms_max * 1e-3)
    # correctness of what was timed: relative residual in double-double (sharded: the ranks'
    # parts of u are disjoint, their sum is the solution)
    if blocks:
        if world > 1 and not refine:  # (the refined path leaves the whole u on every rank)
            dist.all_reduce(u)
        plan.set_partition(None)
    rel_res = 0.0
    for r0 in range(0, nrhs, 4):  # a few right-hand sides at a time (C5: 64 x 0.84 GB)
        _, norms = plan.residual(u[r0:r0 + 4], f[r0:r0 + 4], dd=True)
        rel_res = max(rel_res, float(max(norms[:, 0] / norms[:, 1])))
    if not blocks:  # device u and the solve workspace are not needed any more (e2e has its own)
        del u
        plan._ws.clear()
        torch.cuda.empty_cache()
    if blocks:
        lfds_dist.shard(plan, rank, world)
        ws = plan.workspace(nrhs)
    # e2e: host (pinned) buffers through the public API, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        ne = min(nrhs, args.e2e_rhs) if not blocks else nrhs
        fh = f[:ne].cpu().pin_memory()
        NSL = 3  # solves in flight: H2D of one, compute of another, D2H of a third
        uhs = [torch.empty_like(fh).pin_memory() for _ in range(NSL)]
        streams = [torch.cuda.Stream(device=dev) for _ in range(NSL)]

        def step_host(i):
            if blocks:  # H2D of f, sharded solve, D2H of u (this rank's part)
                f.copy_(fh, non_blocking=True)
                sharded_solve(f, u)
                uhs[0].copy_(u, non_blocking=True)
                torch.cuda.current_stream().synchronize()
            else:
                # consecutive solves rotate over NSL streams and workspaces, so the host-to-device
                # copy, the compute and the device-to-host copy of different solves overlap
                plan.solve_host(fh, out=uhs[i % NSL], stream=streams[i % NSL], sync=False, slot=i % NSL)
        for i in range(2 * NSL):  # warm-up: two rounds over the slots (first-touch of the pinned buffers)
            step_host(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        k2 = max(9, args.steps)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for s_ in streams:
            s_.wait_stream(stream)
        for i in range(k2):
            step_host(i)
        for s_ in streams:
            stream.wait_stream(s_)
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / k2], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        nbytes = fh.numel() * fh.element_size()
        e2e = {"value": p.unknowns * ne * (1 if blocks else world) / (float(t.item()) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "ms_per_step": float(t.item()),
               "nrhs_per_gpu": ne}
    fp64_peak = None
    try:  # in-run FP64 tensor peak (the DMMA kernels' denominator), after the timed region
        from paper_1909_01299_b200.lfds import fp64_peak as _fp64_peak
        fp64_peak = _fp64_peak()
    except Exception:
        pass
    roof = roofline_summary(p, nrhs, plan, stages, args.steps, args.config, ms_max, passes=1 + refine,
                            kernels=kernels, fp64_peak=fp64_peak)
    roof["fp64_peak_tflops_in_run"] = fp64_peak
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        ps, ts, threads = cpu_oracle_sample(p, args.cpu_nz, 1)
        cpu = {"value": ps.unknowns / ts[0], "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"{p.name} x/y grid, N_z={args.cpu_nz}, 1 RHS, oracle (ii) solve only "
                         f"({ps.unknowns} unknowns, {ts[0]:.1f} s)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong" if blocks else "weak",
            "vs_baseline": None, "dtype": "c128" if not p.real else "f64", "data": "synthetic",
            "config": {"workload": args.config, "nx": p.nx, "ny": p.ny, "nz": p.nz,
                       "blocks": [len(p.iface_x) + 1, len(p.iface_y) + 1], "nrhs_per_gpu": nrhs,
                       "refine_passes": refine,
                       "refine_residual": ("double-double" if res_dd else "fp64") if refine else None,
                       "parallelism": (f"block-sharded x{world} (LPT blocks, step-5 modes, 2 NCCL all-reduces, "
                                       f"{'in-library' if exchange == 'library' else 'torch.distributed'})"
                                       if blocks else f"rhs-sharded x{world}" if world > 1 else "1 gpu"),
                       "l2": "inputs larger than L2 (no flush)" if p.unknowns * 16 > 126e6 else "L2-resident",
                       "setup_s": setup_s, "rel_residual_dd": rel_res,
                       # reading R13: min |lambda_l + mu_m + theta_t| of the global and block
                       # z-systems (relative to the family's spectral scale), from lfds_info
                       "resonance_margin": {k: info0[k] for k in ("margin_global", "margin_global_rel",
                                                                  "margin_block", "margin_block_rel")},
                       "min_pivot_ratio": piv},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(),
        }
        line["roofline"]["kernel_times_from"] = ("CUDA events around every launch in the timed region" if kprof_timed
                                                 else "CUDA events around every launch in untimed profiled steps "
                                                      "after the timed region (short step)")
        print(json.dumps(line), flush=True)
    plan.close()


# launch-bound configs (steps of ~0.3-1.5 ms): per-launch events would perturb the timed region
SHORT_STEP = {"c1", "c2", "c3"}

# heterogeneous workload: the C4 grid and background with an
# embedded velocity anomaly (workloads.anomaly: a box over the middle quarter of every axis at
# c_bg (1 + eps)); solved by lfds_gmres (right-preconditioned GMRES, the fast solve as the
# preconditioner) to HETERO_TOL
HETERO = {"c4h": ("c4", -0.01)}
HETERO_TOL, HETERO_RESTART = 1e-10, 16


def run_hetero(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1909_01299_b200 import Plan
    from workloads import anomaly, shrunken
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    base, eps = HETERO[args.config]
    p = make_problem(base)
    dl = anomaly(p, eps=eps)
    t0 = time.perf_counter()
    plan = Plan.from_problem(p, device=local_rank, profile=2, plane_dst=bool(args.plane_dst))
    setup_s = time.perf_counter() - t0
    f = torch.from_numpy(p.rhs(0)).to(dev)
    dlam = torch.from_numpy(dl).to(dev)
    u = torch.empty_like(f)
    reps = []

    def step():
        _, r = plan.solve_hetero(f, dlam, tol=HETERO_TOL, restart=HETERO_RESTART, maxit=400, out=u)
        reps.append(r)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    plan.stage_times()  # reset
    plan.kernel_times()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    stages = plan.stage_times()
    kernels = plan.kernel_times()
    tmax = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    value = p.unknowns * world / (ms_max * 1e-3)  # replicas: every rank solves its own copy
    solves = stages.get("step2_zsolve", (0.0, args.steps))[1] / max(1, args.steps)  # one k_zs1 per solve
    roof = roofline_summary(p, 1, plan, stages, args.steps, args.config, ms_max, passes=max(1.0, solves),
                            kernels=kernels)
    e2e = None
    if not args.no_e2e:  # pinned host f -> device, solve, u -> host, every step
        fh = f.cpu().pin_memory()
        uh = torch.empty_like(fh).pin_memory()
        fd = torch.empty_like(f)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k2 = max(2, min(args.steps, 3))
        a.record(stream)
        for _ in range(k2):
            fd.copy_(fh, non_blocking=True)
            plan.solve_hetero(fd, dlam, tol=HETERO_TOL, restart=HETERO_RESTART, maxit=400, out=u)
            uh.copy_(u, non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        t_e2e = a.elapsed_time(b) / k2
        nb = fh.numel() * fh.element_size()
        e2e = {"value": p.unknowns * world / (t_e2e * 1e-3), "unit": UNIT, "h2d_bytes_per_step": nb,
               "d2h_bytes_per_step": nb, "ms_per_step": t_e2e, "nrhs_per_gpu": 1}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:  # oracle: sparse LU of A_het on the shrunken analog
        import oracle
        ps = shrunken(base, nrhs=1)
        dls = anomaly(ps, eps=eps)
        t1 = time.perf_counter()
        oracle.solve_hetero_direct(ps, dls, ps.rhs(0))
        tc = time.perf_counter() - t1
        cpu = {"value": ps.unknowns / tc, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"{ps.name} analog {ps.shape} with the same anomaly recipe, sparse LU of A_het "
                         f"({ps.unknowns} unknowns, {tc:.2f} s)"}
    last = reps[-1]
    if rank == 0:
        line = {
            "metric": METRIC.replace("direct solve", "heterogeneous solve, GMRES + fast-solver preconditioner"),
            "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic",
            "config": {"workload": args.config, "nx": p.nx, "ny": p.ny, "nz": p.nz,
                       "blocks": [len(p.iface_x) + 1, len(p.iface_y) + 1], "anomaly_eps": eps,
                       "tol": HETERO_TOL, "restart": HETERO_RESTART, "krylov_iterations": last["iterations"],
                       "krylov_cycles": last["cycles"], "rel_residual_preconditioned": last["rel_residual"],
                       "parallelism": "1 gpu" if world == 1 else f"replicas x{world}",
                       "l2": "inputs larger than L2 (no flush)", "setup_s": setup_s},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": plan.report()["n_kernel_launches"] * args.steps, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    plan.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5", "c4j", "c4q", "c4h"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nrhs", type=int, default=0, help="RHS per GPU (0 = the config's)")
    ap.add_argument("--refine", type=int, default=None)
    ap.add_argument("--cpu-nz", type=int, default=16, dest="cpu_nz")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shard", choices=["blocks", "rhs"], default=None,
                    help="N > 1: block sharding with two NCCL exchanges (default) or RHS sharding")
    ap.add_argument("--e2e-rhs", type=int, default=4, dest="e2e_rhs", help="RHS per e2e step (memory bound)")
    ap.add_argument("--exchange", choices=["library", "torch"], default="library",
                    help="block sharding: exchanges inside lfds_solve (NCCL, lfds_set_comm) or torch.distributed")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dst-tma", type=int, default=1, choices=[0, 1], dest="dst_tma",
                    help="1: TMA-fed strided sine passes (options.dst_tma)")
    ap.add_argument("--plane-dst", type=int, default=1, choices=[0, 1], dest="plane_dst",
                    help="1: plane sine transforms on uniform x uniform blocks (options.plane_dst)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.config in HETERO:
            run_hetero(args, rank, world, local_rank)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
