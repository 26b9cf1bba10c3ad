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
