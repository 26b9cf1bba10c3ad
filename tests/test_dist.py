"""Host-side logic of the block-sharded multi-GPU path (paper_1909_01299_b200/dist.py):
LPT block ownership, step-5 x-mode ranges, and the phase / exchange protocol of
solve_sharded run by two gloo ranks on CPU (the CUDA library is replaced by a recording
stand-in whose exchanges carry rank-specific partial sums)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist_mod
import torch.multiprocessing as mp

from paper_1909_01299_b200 import dist


def test_lpt_balances_c4_blocks():
    nb = [127] * 7 + [128]
    kinds = [2] + [0] * 6 + [2]
    c = dist.block_costs(nb, nb, kinds, kinds)
    for world in (2, 4, 8):
        owner = dist.lpt_partition(c, world)
        loads = np.array([c[owner == r].sum() for r in range(world)])
        assert owner.shape == (8, 8) and set(np.unique(owner)) == set(range(world))
        assert loads.max() / loads.mean() < 1.05


def test_lpt_single_rank_owns_everything():
    c = np.arange(1, 13, dtype=float).reshape(3, 4)
    assert (dist.lpt_partition(c, 1) == 0).all()


@pytest.mark.parametrize("nx,world", [(1024, 8), (128, 3), (9, 2), (33, 4)])
def test_mode_ranges_partition_all_modes(nx, world):
    rs = dist.mode_ranges(nx, world)
    assert rs[0][0] == 0 and rs[-1][1] == nx
    for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
        assert a1 == b0 and a0 <= a1
    assert all(l0 % 32 == 0 for l0, _ in rs if l0 < nx)


class _FakePlan:
    """Records the phase order and exposes exchange buffers holding rank-specific partials."""

    def __init__(self, rank):
        self.rank, self.calls = rank, []
        self.ex = {1: torch.full((6,), float(rank + 1), dtype=torch.float64),
                   2: torch.arange(4, dtype=torch.float64) * (rank + 1)}

    def solve_phase(self, phase, f, u, ws, stream=None):
        self.calls.append(phase)
        if phase == 2:  # phase 2 sees the summed exchange 1
            self.seen1 = self.ex[1].clone()

    def exchange_view(self, ws, nrhs, which):
        self.calls.append(("x", which))
        return self.ex[which]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist_mod.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fp = _FakePlan(rank)
        f = torch.zeros(1, 2, 2, 2)
        dist.solve_sharded(fp, f, f.clone(), None)
        out[rank] = (fp.calls, fp.seen1.tolist(), fp.ex[2].tolist())
    finally:
        dist_mod.destroy_process_group()


def test_solve_sharded_protocol_gloo_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        calls, seen1, ex2 = out[r]
        assert calls == [1, ("x", 1), 2, ("x", 2), 3]
        assert seen1 == [3.0] * 6                     # 1 + 2: exchange 1 summed before phase 2
        assert ex2 == [0.0, 3.0, 6.0, 9.0]            # (1 + 2) * arange: exchange 2 summed


class _OraclePlan:
    """Stand-in whose phase 1 is the interface residual of PAPER.md:52/:69 computed by the ORACLE
    for this rank's own blocks only: -A v_b restricted to the planes for every owned block b
    (v_b = the oracle's block solution, zero elsewhere), plus b = M f on the planes on rank 0.
    Summed over the ranks (exchange 1) it must equal r_b = b - A v on the planes for the whole
    partition, whatever the LPT ownership."""

    def __init__(self, p, rank, world, owner):
        import oracle
        from oracle.solve import block_ranges
        b = oracle.mass_rhs(p, p.rhs(0))
        v = oracle.block_solutions(p, b)
        own = np.zeros(p.shape, bool)
        bxr, byr = block_ranges(p.nx, p.iface_x), block_ranges(p.ny, p.iface_y)
        for j, (y0, y1) in enumerate(byr):
            for i, (x0, x1) in enumerate(bxr):
                if owner[j, i] == rank:
                    own[:, y0 - 1:y1, x0 - 1:x1] = True
        part = -oracle.apply_stencil(p, np.where(own, v, 0))
        if rank == 0:
            part = part + b
        self.p, self.full = p, b - oracle.apply_stencil(p, v)
        self.ex1 = torch.from_numpy(self._planes(part).view(np.float64).copy())
        self.ex2 = torch.zeros(2, dtype=torch.float64)

    def _planes(self, r):
        return np.concatenate([r[:, :, a - 1].ravel() for a in self.p.iface_x] +
                              [r[:, bb - 1, :].ravel() for bb in self.p.iface_y])

    def solve_phase(self, phase, f, u, ws, stream=None):
        if phase == 2:
            self.seen1 = self.ex1.numpy().view(np.complex128).copy()

    def exchange_view(self, ws, nrhs, which):
        return self.ex1 if which == 1 else self.ex2


def _oracle_worker(rank, world, port, out):
    from workloads import shrunken
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist_mod.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = shrunken("c3", nrhs=1)
        nb = [len(p.iface_x) + 1, len(p.iface_y) + 1]
        # ownership as dist.shard assigns it (LPT on the modelled costs, here all blocks real)
        owner = dist.lpt_partition(dist.block_costs([1] * nb[0], [1] * nb[1], [1] * nb[0], [1] * nb[1]) +
                                   np.arange(nb[0] * nb[1]).reshape(nb[1], nb[0]), world)
        fp = _OraclePlan(p, rank, world, owner)
        dist.solve_sharded(fp, torch.zeros(1, 1, 1, 1), None, None)
        out[rank] = float(np.abs(fp.seen1 - fp._planes(fp.full)).max() / np.abs(fp.full).max())
    finally:
        dist_mod.destroy_process_group()


def test_exchange1_sums_the_ranks_partial_interface_residuals_gloo_world2():
    """Two gloo ranks, each owning the LPT half of the blocks of the shrunken C3 analog: the
    summed exchange 1 equals the oracle's interface residual of the whole partition."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_oracle_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] < 1e-13 and out[1] < 1e-13, dict(out)


class _RefinePlan:
    """Stand-in for the refinement protocol of dist.solve_sharded_refined: its sharded 'solve' is
    the ORACLE's direct solve scaled by (1 + 1e-6) (an approximate inverse, so that refinement
    has work to do), written only on this rank's slab of x nodes (the disjoint support a sharded
    solve leaves in u); residual_f is the oracle's f - M^-1 A u on the whole grid."""

    def __init__(self, p, rank, world):
        self.p, self.rank, self.world = p, rank, world
        self.has_comm = False
        n = p.nx
        self.x0, self.x1 = rank * n // world, (rank + 1) * n // world

    def solve_phase(self, phase, f, u, ws, stream=None):
        if phase == 3:  # (the separable oracle: scipy's splu runs ~100x slower in spawned workers)
            import oracle
            from oracle.solve import global_bases
            self.g = getattr(self, "g", None) or global_bases(self.p)
            sol = oracle.solve_separable(self.p, oracle.mass_rhs(self.p, f.numpy()[0]), self.g) * (1 + 1e-6)
            u[0, :, :, self.x0:self.x1] = torch.from_numpy(np.ascontiguousarray(sol[:, :, self.x0:self.x1]))

    def exchange_view(self, ws, nrhs, which):
        return torch.zeros(4, dtype=torch.float64)

    def residual_f(self, u, f, dd=False, stream=None):
        import oracle
        U, Fv = u.numpy()[0], f.numpy()[0]
        V = oracle.mass_rhs(self.p, np.ones(self.p.shape, complex))
        r = (oracle.mass_rhs(self.p, Fv) - oracle.apply_stencil(self.p, U)) / V
        return torch.from_numpy(r[None].astype(np.complex128))

    def axpy(self, d, u, stream=None):
        u += d
        return u


def _refine_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist_mod.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)  # two ranks' BLAS / SuperLU thread pools on one host would oversubscribe it
        torch.set_num_threads(1)
        from workloads import shrunken
        p = shrunken("c2", nrhs=1)
        f = torch.from_numpy(p.rhs_all())
        u = torch.full_like(f, 7.0)  # garbage: the protocol must zero it first
        dist.solve_sharded_refined(_RefinePlan(p, rank, world), f, u, None, passes=1)
        out[rank] = u.numpy()
    finally:
        dist_mod.destroy_process_group()


def test_solve_sharded_refined_protocol_gloo_world2():
    """Two gloo ranks: u completed by a sum over the ranks, the whole-grid f-units residual, the
    sharded correction solve and its sum: one pass takes the 1e-6 approximate inverse to the
    oracle's solution at ~1e-12 on every rank."""
    import oracle
    from workloads import shrunken
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_refine_worker, args=(2, port, out), nprocs=2, join=True)
    p = shrunken("c2", nrhs=1)
    ref = oracle.solve(p, p.rhs(0))  # separable + 80-bit refinement
    for r in range(2):
        u = out[r][0]
        err = np.linalg.norm(u - ref) / np.linalg.norm(ref)
        assert err < 1e-11, (r, err)
    assert np.array_equal(out[0], out[1])
