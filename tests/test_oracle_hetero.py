"""Pins of the heterogeneous-medium oracle (oracle/hetero.py): the node-wise
lambda enters Eq. (fd) exactly like lambda does; checked against the homogeneous operator and
against the oracle's independent separable solver through the Lippmann-Schwinger identity."""
import dataclasses

import numpy as np

import oracle
from workloads import anomaly, shrunken


def test_zero_perturbation_is_the_layered_operator():
    p = shrunken("c2")
    d = oracle.assemble_hetero(p, np.zeros(p.shape, complex)) - oracle.assemble(p)
    assert d.nnz == 0 or abs(d).max() == 0


def test_constant_perturbation_is_a_shifted_lambda():
    """dlam = c everywhere is the homogeneous operator of lambda + c (Eq. (fd) lambda term)."""
    p = shrunken("c4")
    c = 0.37 - 0.05j
    A1 = oracle.assemble_hetero(p, np.full(p.shape, c))
    A2 = oracle.assemble(dataclasses.replace(p, lam=p.lam + c))
    assert abs(A1 - A2).max() <= 1e-14 * abs(A2).max()


def test_hetero_operator_is_complex_symmetric():
    p = shrunken("c3")
    A = oracle.assemble_hetero(p, anomaly(p, eps=-0.2))
    assert abs(A - A.T).max() == 0


def test_lippmann_schwinger_identity():
    """u_het = S(f - dlam u_het) with S the oracle's separable layered solver:
    sparse LU of A_het on one side, the eigen-route of the background on the other."""
    p = shrunken("c4")
    dl = anomaly(p, eps=-0.15)
    f = p.rhs(0)
    u = oracle.solve_hetero_direct(p, dl, f)
    v = oracle.solve_separable(p, oracle.mass_rhs(p, f - dl * u))
    assert np.linalg.norm(v - u) <= 1e-10 * np.linalg.norm(u)
    assert oracle.rel_residual_hetero(p, dl, u, f, np.clongdouble) < 1e-12
    # and the anomaly matters: the background solution is different
    u0 = oracle.solve_direct(p, oracle.mass_rhs(p, f))
    assert np.linalg.norm(u0 - u) > 1e-3 * np.linalg.norm(u)


def test_anomaly_recipe():
    p = shrunken("c2")
    dl = anomaly(p, eps=-0.1)
    inside = dl != 0
    assert inside.any() and not inside.all()
    assert np.allclose(dl[inside], p.lam * (0.9 ** -2 - 1))
