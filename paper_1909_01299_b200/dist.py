"""Block sharding of the two-level solve over ranks (BASELINE.json north_star: "Work is
partitioned across the 8 B200s of one box by blocks S^ij, with NCCL over NVLink only for the
interface exchange").

Blocks S^ij are independent in the two block passes ("for each
i,j"), so each rank computes a subset, chosen by longest-processing-time-first on a cost model
(dense complex transform directions cost ~8n flops per element and direction, dense real ~4n,
sine-transform directions ~O(log n)).  The interface step is one exchange: every rank adds the
contributions of its own blocks to the residual on the interface planes and the
residuals are summed over the ranks (exchange 1).  Step 5 is split by global
x-modes l (and, in the z-modal form, by global y-modes m): each rank handles its (m, l) range and
the plane projections are summed (exchange 2); the plane data R1~ / R2~ that a group of ranks
reads in common is formed in parts and summed (exchange 3).
Both sums run either inside the library (attach_nccl: ncclAllReduce on the solve stream, no
host round trip) or as `torch.distributed.all_reduce` on views of the library workspace
(`allreduce` can be replaced: tests use an in-process emulation and gloo).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import numpy as np


def block_costs(nx_blocks: Sequence[int], ny_blocks: Sequence[int], kinds_x: Sequence[int],
                kinds_y: Sequence[int]) -> np.ndarray:
    """Modelled cost of each block (row-major [j][i]): elements x per-direction transform cost
    (+ the z-solves and edge work, ~60 units per element)."""
    def dcost(kind, n):
        L = 2 * (n + 1)
        if kind == 0 and (L in (16, 32, 64, 128, 256, 512) or (L % 16 == 0 and L // 16 in (3, 5, 6, 10, 12, 20))):
            return 40.0                                   # sine transform, HBM-bound
        return (8.0 if kind == 2 else 4.0) * n             # dense DMMA contraction
    c = np.zeros((len(ny_blocks), len(nx_blocks)))
    for j, (ny, ky) in enumerate(zip(ny_blocks, kinds_y)):
        for i, (nx, kx) in enumerate(zip(nx_blocks, kinds_x)):
            c[j, i] = nx * ny * (dcost(kx, nx) + dcost(ky, ny) + 60.0)
    return c


def lpt_partition(costs: np.ndarray, world: int) -> np.ndarray:
    """Owner rank of every block: longest processing time first (deterministic tie-break)."""
    flat = costs.ravel()
    order = sorted(range(flat.size), key=lambda b: (-flat[b], b))
    load = [0.0] * world
    owner = np.zeros(flat.size, dtype=np.int32)
    for b in order:
        r = min(range(world), key=lambda q: (load[q], q))
        owner[b] = r
        load[r] += flat[b]
    return owner.reshape(costs.shape)


def mode_ranges(nx: int, world: int, align: int = 32) -> List[tuple]:
    """Contiguous global x-mode ranges [l0, l1) per rank, aligned to warp tiles."""
    units = (nx + align - 1) // align
    out, start = [], 0
    for r in range(world):
        cnt = units // world + (1 if r < units % world else 0)
        l0 = min(start * align, nx)
        l1 = min((start + cnt) * align, nx)
        out.append((l0, l1))
        start += cnt
    return out


def mode_grid(world: int, modal: bool) -> tuple:
    """(W_m, W_l): ranks along the step-5 y-modes and x-modes.  The z-modal step 5 splits both
    (W_m = the largest divisor of world not above sqrt(world)), so that R1 = W_y^T RX is also
    formed per rank; the per-mode z-sweeps split x-modes only."""
    if not modal:
        return 1, world
    wm = max(d for d in range(1, int(world ** 0.5) + 1) if world % d == 0)
    return wm, world // wm


def shard(plan, rank: int, world: int, formation: bool = True) -> dict:
    """Configure `plan` for `rank` of `world` (LPT block ownership, step-5 mode ranges).
    formation: split the FORMING of R1~ (W_y^T RX and its z-transform) among the ranks that read
    the same y-modes, and of R2~ among those that read the same x-modes (a third exchange sums
    the parts); without it every rank of a group forms the same rows (the z-modal step 5 only)."""
    info = plan.info()
    nbx, nby = info["nbx"], info["nby"]
    bx = [plan.basis(0, i) for i in range(nbx)]
    by = [plan.basis(1, j) for j in range(nby)]
    costs = block_costs([b[1].shape[0] for b in bx], [b[1].shape[0] for b in by], [b[2] for b in bx],
                        [b[2] for b in by])
    owner = lpt_partition(costs, world)
    wm, wl = mode_grid(world, bool(info.get("s5_modal", 0)))
    rm, rl = rank // wl, rank % wl
    l0, l1 = mode_ranges(info["nx"], wl)[rl]
    plan.set_partition(owner == rank, l0, l1, rank == 0)
    m0, m1 = 0, info["ny"]
    if wm > 1:
        m0, m1 = mode_ranges(info["ny"], wm, align=64)[rm]
        plan.set_mode_rows(m0, m1)
    fm, fl = (m0, m1), (l0, l1)
    if formation and world > 1 and info.get("s5_modal", 0):
        # the W_l ranks of this y-mode group share [m0, m1): rank rl forms part rl; the W_m ranks
        # of this x-mode group share [l0, l1): rank rm forms part rm
        fm = tuple(m0 + x for x in mode_ranges(m1 - m0, wl, align=8)[rl])
        fl = tuple(l0 + x for x in mode_ranges(l1 - l0, wm, align=8)[rm])
        plan.set_formation_rows(fm[0], fm[1], fl[0], fl[1])
    return {"owner": owner, "l_range": (l0, l1), "m_range": (m0, m1), "form_m": fm, "form_l": fl, "costs": costs,
            "grid": (rm, rl)}


def attach_nccl(plan, rank: int, world: int, broadcast: Optional[Callable] = None) -> bytes:
    """In-library exchanges for a sharded plan: rank 0 makes the NCCL group id, `broadcast`
    (default: torch.distributed.broadcast of a uint8 tensor from rank 0) shares it, and every
    rank joins (lfds_set_comm).  lfds_solve then runs the phases and both all-reduces on the
    solve stream."""
    from .lfds import nccl_unique_id
    uid = bytes(128)
    if rank == 0:
        try:
            uid = nccl_unique_id()
        except Exception:  # broadcast the empty id anyway: every rank then fails the same way
            uid = bytes(128)
    if world > 1:
        if broadcast is None:
            import torch
            import torch.distributed as tdist
            dev = torch.device("cuda", torch.cuda.current_device()) if tdist.get_backend() == "nccl" else "cpu"
            t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
            tdist.broadcast(t, 0)
            uid = bytes(t.cpu().tolist())
        else:
            uid = broadcast(uid)
    if uid == bytes(128):
        raise RuntimeError("no NCCL group id (lfds_nccl_unique_id failed on rank 0)")
    plan.set_comm(uid, rank, world)
    if getattr(plan, "formation", False) and world > 1:
        # exchange 3 within the groups that share R1~ rows (same y-mode range) / R2~ rows
        info = plan.info()
        wm, wl = mode_grid(world, bool(info.get("s5_modal", 0)))
        plan.set_comm_groups(rank // wl, rank % wl)
    return uid


def solve_sharded(plan, f, u, ws, allreduce: Optional[Callable] = None, stream=None):
    """One block-sharded solve: phase 1, sum of exchange 1, phase 2, sum of exchange 2, phase 3.
    `allreduce(tensor)` sums in place over the ranks (default: torch.distributed.all_reduce).
    A plan with an in-library communicator (attach_nccl) does all of it in one lfds_solve."""
    if getattr(plan, "has_comm", False) and allreduce is None:
        return plan.solve(f, out=u, stream=stream)
    if allreduce is None:
        import torch.distributed as dist

        def allreduce(t):
            dist.all_reduce(t)
    nrhs = f.shape[0]
    plan.solve_phase(1, f, u, ws, stream)
    allreduce(plan.exchange_view(ws, nrhs, 1))
    if getattr(plan, "formation", False):  # step 5 in two halves around exchange 3 ([R1~, R2~])
        plan.solve_phase(4, f, u, ws, stream)
        allreduce(plan.exchange_view(ws, nrhs, 3))
        plan.solve_phase(5, f, u, ws, stream)
    else:
        plan.solve_phase(2, f, u, ws, stream)
    allreduce(plan.exchange_view(ws, nrhs, 2))
    plan.solve_phase(3, f, u, ws, stream)
    return u


def solve_sharded_refined(plan, f, u, ws, passes: int, allreduce: Optional[Callable] = None, stream=None,
                          dd: bool = False):
    """Block-sharded solve with `passes` refinement passes (reading R13: u += S(f - M^-1 A u)).

    A sharded solve writes u only on the rank's blocks and its segments of the interface planes
    (lfds_solve_phase), so u starts at zero and one sum over the ranks completes it; every rank
    then forms the f-units residual of the whole grid (lfds_residual_f, the stencil reads u
    across the block boundaries), solves for the correction with the same block sharding, and
    completes the correction by a second sum before adding it (lfds_axpy).  Two volume sums per
    pass: meant for the small, refinement-needing configs (C2: 17 MB per field)."""
    import torch
    if allreduce is None:
        import torch.distributed as dist

        def allreduce(t):
            dist.all_reduce(t)
    real = torch.view_as_real if u.is_complex() else (lambda t: t)
    u.zero_()
    solve_sharded(plan, f, u, ws, None if getattr(plan, "has_comm", False) else allreduce, stream)
    allreduce(real(u))
    for _ in range(passes):
        r = plan.residual_f(u, f, dd=dd, stream=stream)
        rf = r if u.is_complex() else r.real.contiguous()
        d = torch.zeros_like(u)
        solve_sharded(plan, rf, d, ws, None if getattr(plan, "has_comm", False) else allreduce, stream)
        allreduce(real(d))
        plan.axpy(d.to(torch.complex128) if not d.is_complex() else d, u, stream=stream)
    return u
