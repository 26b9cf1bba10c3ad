"""GPU parity of the heterogeneous-medium solve (lfds_gmres: right-preconditioned GMRES with the
fast layered solver) against the oracle's sparse LU of A_het."""
import numpy as np
import pytest

import oracle
from workloads import anomaly, shrunken

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _plan(p, **kw):
    from paper_1909_01299_b200 import Plan
    return Plan.from_problem(p, **kw)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name,eps", [("c2", -0.1), ("c4", -0.15), ("c4j", 0.1), ("c5", -0.1)])
def test_gmres_matches_oracle(name, eps):
    p = shrunken(name, nrhs=1)
    dl = anomaly(p, eps=eps)
    F = p.rhs(0)
    plan = _plan(p)
    u, rep = plan.solve_hetero(torch.from_numpy(F).cuda(), torch.from_numpy(dl).cuda(), tol=1e-12, restart=20)
    ref = oracle.solve_hetero_direct(p, dl, F)
    U = u.cpu().numpy()
    print(name, rep, rel(U, ref))
    assert rep["rel_residual"] <= 1e-12 and rep["iterations"] >= 2
    assert rel(U, ref) < 1e-9, rel(U, ref)
    assert oracle.rel_residual_hetero(p, dl, U, F, np.clongdouble) < 1e-10


def test_zero_perturbation_is_one_fast_solve():
    p = shrunken("c4", nrhs=1)
    F = torch.from_numpy(p.rhs(0)).cuda()
    plan = _plan(p)
    u, rep = plan.solve_hetero(F, torch.zeros_like(F), tol=1e-12)
    assert rep["iterations"] == 1
    assert rel(u.cpu().numpy(), plan.solve(F).cpu().numpy()) < 1e-13


def test_restarts_and_determinism():
    p = shrunken("c2", nrhs=1)
    dl = torch.from_numpy(anomaly(p, eps=-0.2)).cuda()
    F = torch.from_numpy(p.rhs(0)).cuda()
    plan = _plan(p)
    u1, r1 = plan.solve_hetero(F, dl, tol=1e-11, restart=3, maxit=300)
    u2, r2 = plan.solve_hetero(F, dl, tol=1e-11, restart=3, maxit=300)
    assert r1["cycles"] > 1 and r1 == r2 and torch.equal(u1, u2)
    u3, _ = plan.solve_hetero(F, dl, tol=1e-11, restart=30)
    assert rel(u1.cpu().numpy(), u3.cpu().numpy()) < 1e-9


def test_not_converged_and_bad_arguments():
    from paper_1909_01299_b200.lfds import LfdsError
    p = shrunken("c2", nrhs=1)
    dl = torch.from_numpy(anomaly(p, eps=-0.3)).cuda()
    F = torch.from_numpy(p.rhs(0)).cuda()
    plan = _plan(p)
    with pytest.raises(LfdsError) as e:
        plan.solve_hetero(F, dl, tol=1e-14, maxit=2)
    assert e.value.code == 7  # LFDS_ENOTCONVERGED
    with pytest.raises(ValueError):
        plan.solve_hetero(F, dl, restart=0)
