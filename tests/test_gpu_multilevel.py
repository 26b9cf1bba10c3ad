"""Multi-level (nested) partition, lfds_ml_* (PAPER.md:77-79 remark):
coarse interfaces take the global step 5, every coarse block is solved by the two-level method of
its own fine partition.  The method is exact like the two-level one, so the bar is the same:
the oracle's sparse-LU solution (oracle.solve_direct) to north_star's 1e-9, per-block and
per-plane max-norms included, and the plain two-level solve of the fine partition."""
import numpy as np
import pytest

import oracle
from workloads import shrunken

from test_gpu_parity import assert_parity, rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ml(p, cx, cy, fx=None, fy=None, **kw):
    from paper_1909_01299_b200 import MLPlan
    return MLPlan(p.hx, p.hy, p.hz, p.sigma_node, p.sigma_edge, p.lam, cx, cy,
                  p.iface_x if fx is None else fx, p.iface_y if fy is None else fy, **kw)


@pytest.mark.parametrize("name,cx,cy", [
    ("c4j", [24], [24]),          # 2 x 2 coarse blocks, each with one fine interface per axis
    ("c3", [18], [27]),           # graded steps, uneven coarse blocks (2 + 1 / 3 + 0 fine ones)
    ("c5", [16], [8, 24]),        # 2 x 3 coarse blocks, a coarse block without fine interfaces
    ("c2", [], [20]),             # coarse cut along y only: the whole x extent in every block
])
def test_multilevel_matches_oracle(name, cx, cy):
    p = shrunken(name, nrhs=1)
    F = p.rhs_all()
    ml = _ml(p, cx, cy)
    assert ml.n_coarse_blocks() == (len(cx) + 1) * (len(cy) + 1)
    f = torch.from_numpy(np.ascontiguousarray(F[0])).cuda()
    u = ml.solve(f)
    torch.cuda.synchronize()
    U = u.cpu().numpy()
    ref = oracle.solve_direct(p, oracle.mass_rhs(p, F[0]))
    assert_parity(p, U, ref)
    assert oracle.rel_residual(p, U, F[0], np.clongdouble) < 1e-10
    # the two-level solve of the fine partition reaches the same solution
    from paper_1909_01299_b200 import Plan
    u2 = Plan.from_problem(p).solve(f)
    assert rel(U, u2.cpu().numpy()) < 1e-11


def test_multilevel_repeat_and_new_rhs():
    """The coarse-block plans replay as CUDA graphs: a second solve with other data through the
    same buffers must not reuse stale results."""
    p = shrunken("c4j", nrhs=1)
    ml = _ml(p, [24], [24])
    rng = np.random.default_rng(7)
    f = torch.empty(p.shape, dtype=torch.complex128, device="cuda")
    u = torch.empty_like(f)
    for _ in range(2):
        F = rng.standard_normal(p.shape) + 1j * rng.standard_normal(p.shape)
        f.copy_(torch.from_numpy(F))
        ml.solve(f, out=u)
        torch.cuda.synchronize()
        ref = oracle.solve_direct(p, oracle.mass_rhs(p, F))
        assert_parity(p, u.cpu().numpy(), ref)


def test_multilevel_rejects_coarse_interface_outside_fine_set():
    from paper_1909_01299_b200.lfds import LfdsError
    p = shrunken("c4j", nrhs=1)
    with pytest.raises(LfdsError, match="not in the fine set"):
        _ml(p, [20], [24])
