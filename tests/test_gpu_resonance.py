"""The failure contract of SURVEY §8(b) (reading R13): a resonant lambda
is reported with its harmonic, never regularised; the pivot monitor reaches lfds_get_report
without a synchronisation inside the solve."""
import math

import numpy as np
import pytest

from workloads import shrunken
from workloads.configs import Problem

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _uniform_problem(nx, ny, nz, ix, iy, lam):
    """sigma = 1, unit steps: every 1-D pencil has the closed-form sine eigenvalues
    -4 sin^2(pi k / (2 (N + 1))), and theta_t = that of z plus lambda (M_z^sigma = M_z)."""
    return Problem(name="res", hx=np.ones(nx + 1, complex), hy=np.ones(ny + 1, complex),
                   hz=np.ones(nz + 1, complex), sigma_edge=np.ones(nz + 1, complex),
                   sigma_node=np.ones(nz, complex), lam=lam, iface_x=list(ix), iface_y=list(iy), nrhs=1,
                   real=False, _rhs=None)


def _ev(k, n):
    return -4.0 * math.sin(math.pi * k / (2 * (n + 1))) ** 2


def test_lambda_at_a_global_eigenvalue_is_reported_with_its_harmonic():
    from paper_1909_01299_b200 import LfdsError, Plan
    nx, ny, nz = 20, 17, 8
    l, m, t = 3, 5, 2  # 1-based sine indices
    lam_res = -(_ev(l, nx) + _ev(m, ny) + _ev(t, nz))
    p = _uniform_problem(nx, ny, nz, [10], [8], lam_res * (1 + 1e-13))
    with pytest.raises(LfdsError) as ei:
        Plan.from_problem(p)
    assert ei.value.code == 3, str(ei.value)
    msg = str(ei.value)
    # global bases of unit steps: natural sine order (index l - 1); theta ascending: t -> nz - t
    assert "global" in msg and "(l, m) = (2, 4)" in msg and f"t = {nz - t}" in msg, msg
    # with the check off the plan builds and lfds_info carries the same margin
    plan = Plan.from_problem(p, resonance_tol=0.0)
    info = plan.info()
    assert info["margin_global_lmt"] == [l - 1, m - 1, nz - t]
    assert info["margin_global"] < 1e-12 and info["margin_global_rel"] < 1e-13
    assert info["margin_block_rel"] > 1e-4  # the blocks' own spectra are far from it
    plan.close()
    # a lambda between the eigenvalues: no error, a finite margin
    p2 = _uniform_problem(nx, ny, nz, [10], [8], lam_res + 1e-3)
    plan = Plan.from_problem(p2)
    assert plan.info()["margin_global"] == pytest.approx(1e-3, rel=1e-6)
    plan.close()


def test_lambda_at_a_block_eigenvalue_names_the_block():
    from paper_1909_01299_b200 import LfdsError, Plan
    nx, ny, nz = 20, 17, 8
    # block (1, 0): x nodes 11..20 (n = 10), y nodes 1..7 (n = 7)
    lam_res = -(_ev(2, 10) + _ev(3, 7) + _ev(4, nz))
    p = _uniform_problem(nx, ny, nz, [10], [8], lam_res)
    with pytest.raises(LfdsError) as ei:
        Plan.from_problem(p)
    msg = str(ei.value)
    assert ei.value.code == 3 and "block (1, 0)" in msg and "(l, m) = (1, 2)" in msg, msg


def test_margins_reported_for_a_regular_config_and_pivot_monitor_read_back():
    from paper_1909_01299_b200 import Plan
    p = shrunken("c5", nrhs=1)
    plan = Plan.from_problem(p, graph=True)
    info = plan.info()
    assert 0 < info["margin_global_rel"] < 1 and 0 < info["margin_block_rel"] < 1
    assert all(v >= 0 for v in info["margin_global_lmt"] + info["margin_block_ij"] + info["margin_block_lmt"])
    f = torch.from_numpy(p.rhs_all()).cuda()
    for _ in range(2):  # capture + replay: the monitor's copy is a node of the graph
        plan.solve(f)
        rep = plan.report()
        assert 1e-14 < rep["min_pivot_ratio"] <= 1.0
    plan.close()
