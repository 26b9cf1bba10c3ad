"""Pins for oracle/solve.py: brute force, manufactured discrete solutions, closed forms, invariants."""
import numpy as np
import pytest

import oracle
from oracle.solve import block_ranges
from workloads import make_problem, shrunken

from test_oracle_operator import tiny_problem


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_direct_equals_separable_on_analogs(name):
    """(i) sparse LU == (ii) global separable eigen-solve (+ refinement) on every config's analog."""
    p = shrunken(name)
    f = p.rhs(0)
    b = oracle.mass_rhs(p, f)
    u1 = oracle.solve_direct(p, b)
    u2 = oracle.solve(p, f)
    assert rel(u2, u1) < 1e-12
    assert oracle.rel_residual(p, u1, f, np.clongdouble) < 1e-13
    assert oracle.rel_residual(p, u2, f, np.clongdouble) < 1e-14


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_manufactured_discrete_solution(name):
    """Random u*, b = A u* with the literally assembled A, solve -> u* (pins exactness)."""
    p = shrunken(name)
    rng = np.random.default_rng(11)
    us = rng.standard_normal(p.shape) + 1j * rng.standard_normal(p.shape)
    b = (oracle.assemble(p) @ us.ravel()).reshape(p.shape)
    f = b / oracle.mass_rhs(p, np.ones(p.shape))
    u = oracle.solve(p, f)
    assert rel(u, us) < 1e-11


def test_manufactured_poisson_c1_grid():
    """north_star's manufactured Poisson case: lam = 0, C1 grid and sigma layers,
    u* = sin(pi p i/(N+1)) sin(pi q j/(N+1)) g(k), b = A u* by the plain stencil."""
    p = make_problem("c1").with_lambda(0.0)
    n = p.nx
    i = np.arange(1, n + 1)
    g = np.exp(-((np.arange(1, p.nz + 1) - 7.0) / 4.0) ** 2)
    us = g[:, None, None] * np.sin(np.pi * 2 * i / (n + 1))[None, :, None] * np.sin(np.pi * 3 * i / (n + 1))[None, None, :]
    b = oracle.apply_stencil(p, us.astype(np.complex128))
    f = b / oracle.mass_rhs(p, np.ones(p.shape))
    assert rel(oracle.solve(p, f, method="separable"), us) < 1e-13
    assert rel(oracle.solve(p, f, method="direct"), us) < 1e-13


def test_exact_discrete_eigenfunction():
    """sigma = 1 on uniform steps: f = sin_p (x) sin_q (x) sin_r  =>  u = f / (lam_p + mu_q + nu_r + lam)."""
    nx, ny, nz, h = 9, 7, 6, 0.8
    p = tiny_problem(nx, ny, nz, hx=np.full(nx + 1, h), hy=np.full(ny + 1, h), hz=np.full(nz + 1, h),
                     sig=1.0, lam=0.45)
    P, Q, R = 3, 5, 2
    ev = lambda n, l: -(4.0 / h ** 2) * np.sin(np.pi * l / (2 * (n + 1))) ** 2
    s = lambda n, l: np.sin(np.pi * np.arange(1, n + 1) * l / (n + 1))
    f = s(nz, R)[:, None, None] * s(ny, Q)[None, :, None] * s(nx, P)[None, None, :]
    u_exact = f / (ev(nx, P) + ev(ny, Q) + ev(nz, R) + 0.45)
    assert rel(oracle.solve(p, f.astype(np.complex128)), u_exact) < 1e-13


def test_reciprocity_and_linearity():
    p = shrunken("c2")
    rng = np.random.default_rng(3)
    cn = lambda: rng.standard_normal(p.shape) + 1j * rng.standard_normal(p.shape)
    f1, f2 = cn(), cn()
    u1, u2 = oracle.solve(p, f1), oracle.solve(p, f2)
    b1, b2 = oracle.mass_rhs(p, f1), oracle.mass_rhs(p, f2)
    # complex symmetry A = A^T => b2^T A^{-1} b1 = b1^T A^{-1} b2 (no conjugation)
    lhs, rhs = np.sum(b2 * u1), np.sum(b1 * u2)
    assert abs(lhs - rhs) < 1e-12 * abs(lhs)
    a, c = 0.3 - 1.2j, 2.1 + 0.5j
    assert rel(oracle.solve(p, a * f1 + c * f2), a * u1 + c * u2) < 1e-12


@pytest.mark.parametrize("name", ["c1", "c3", "c5"])
def test_interface_support_invariant(name):
    """after the block solves (step 2) the residual b - A v lives on the interfaces only."""
    p = shrunken(name)
    b = oracle.mass_rhs(p, p.rhs(0))
    A = oracle.assemble(p)
    v = oracle.block_solutions(p, b, A)
    r = b - (A @ v.ravel()).reshape(p.shape)
    mask = oracle.interface_mask(p)
    assert np.abs(r[~mask]).max() < 1e-12 * np.abs(b).max()
    assert np.abs(r[mask]).max() > 1e-3 * np.abs(b).max()
    assert np.all(v[mask] == 0)


def test_single_block_partition_is_global_solve():
    p = shrunken("c4").with_partition([], [])
    b = oracle.mass_rhs(p, p.rhs(0))
    v = oracle.block_solutions(p, b)
    assert rel(v, oracle.solve_direct(p, b)) < 1e-13


def test_block_ranges():
    assert block_ranges(24, [12]) == [(1, 11), (13, 24)]
    assert block_ranges(128, [32, 64, 96]) == [(1, 31), (33, 63), (65, 95), (97, 128)]
    assert block_ranges(5, []) == [(1, 5)]


def test_multi_rhs_batch():
    p = shrunken("c5")
    F = p.rhs_all()
    U = oracle.solve(p, F)
    for r in range(p.nrhs):
        assert rel(U[r], oracle.solve(p, F[r])) < 1e-14
