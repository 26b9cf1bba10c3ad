#!/usr/bin/env python
"""Per-rank compute time of the block-sharded solve, measured on ONE GPU: the plan is set up as
rank r of `world` (LPT blocks, step-5 x-modes) and its three phases are timed back to back with
CUDA events (the two exchanges are not performed: this is the compute each rank does between
them).  The max over ranks, plus the all-reduce time of the two exchange buffers at an assumed
NVLink bus bandwidth, estimates the world-GPU step; the 1-GPU step is timed the same way.
usage: python tools/shard_rank_time.py [config] [worlds...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_01299_b200 import Plan, dist  # noqa: E402
from workloads import make_problem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
worlds = [int(a) for a in sys.argv[2:]] or [2, 4, 8]
BUS_GBS = float(os.environ.get("BUS_GBS", "725"))  # 8-rank NCCL all-reduce bus bandwidth measured on this pool (B200_PROFILING.md)
p = make_problem(cfg)
f = torch.from_numpy(p.rhs(0)[None]).cuda()
u = torch.zeros_like(f)
plan = Plan.from_problem(p)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


t1 = timed(lambda: plan.solve(f, out=u))
out = {"config": cfg, "t_1gpu_ms": t1, "worlds": {}}
for world in worlds:
    ranks = []
    xbytes = 0
    for r in range(world):
        dist.shard(plan, r, world)
        ws = plan.workspace(1)
        xbytes = sum(plan.exchange_view(ws, 1, w).numel() * 8 for w in (1, 2))

        phases = (1, 4, 5, 3) if plan.formation else (1, 2, 3)
        xbytes = sum(plan.exchange_view(ws, 1, w).numel() * 8 for w in ((1, 2, 3) if plan.formation else (1, 2)))

        def run():
            for ph in phases:
                plan.solve_phase(ph, f, u, ws)
        ranks.append(timed(run))
    # ring all-reduce volume per rank: exchanges 1 and 2 over all ranks; exchange 3 (formation
    # split) within its groups (R1~ over the W_l ranks of a y-mode group, R2~ over the W_m of an
    # x-mode group: lfds_set_comm_groups)
    x12 = sum(plan.exchange_view(ws, 1, w).numel() * 8 for w in (1, 2))
    comm = 2 * (world - 1) / world * x12 / (BUS_GBS * 1e9) * 1e3
    if plan.formation:
        wm, wl = dist.mode_grid(world, True)
        inf = plan.info()
        x3m = inf["n_if_x"] * inf["nz"] * inf["ny"] * 16  # R1~ bytes (one right-hand side)
        x3l = inf["n_if_y"] * inf["nz"] * inf["nx"] * 16  # R2~ bytes
        comm += (2 * (wl - 1) / wl * x3m + 2 * (wm - 1) / wm * x3l) / (BUS_GBS * 1e9) * 1e3
    est = max(ranks) + comm
    out["worlds"][world] = {"rank_ms": [round(x, 3) for x in ranks], "max_rank_ms": max(ranks),
                            "exchange_bytes": xbytes, "comm_ms_est": comm, "step_ms_est": est,
                            "speedup_est": t1 / est}
    print(f"{cfg} world {world}: ranks max {max(ranks):.2f} ms (min {min(ranks):.2f}), "
          f"comm est {comm:.2f} ms -> {est:.2f} ms, speed-up {t1 / est:.2f}x (1 GPU {t1:.2f} ms)", flush=True)
plan.set_partition(None)
print(json.dumps(out))
if os.environ.get("SHARD_STAGES"):  # stage breakdown of rank 0 of the largest world
    pp = Plan.from_problem(p, profile=True)
    W = max(worlds)
    dist.shard(pp, 0, W)
    ws = pp.workspace(1)
    phs = (1, 4, 5, 3) if pp.formation else (1, 2, 3)
    for ph in phs:
        pp.solve_phase(ph, f, u, ws)
    torch.cuda.synchronize()
    pp.stage_times()
    for _ in range(3):
        for ph in phs:
            pp.solve_phase(ph, f, u, ws)
    torch.cuda.synchronize()
    st = {k: v[0] / 3 for k, v in pp.stage_times().items() if v[1]}
    print(f"{cfg} world {W} rank 0 stages (ms):", " ".join(f"{k}={v:.3f}" for k, v in st.items()),
          f"sum={sum(st.values()):.3f}", flush=True)
