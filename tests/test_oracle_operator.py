"""Pins for oracle/operator.py against the paper (Eq. (fd)/(fdmtr)/(wave2)) — not the oracle itself."""
import dataclasses
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle.operator import axis_pencil, z_pencil
from workloads import shrunken
from workloads.configs import Problem, sigma_layers


def _golden(golden_dir):
    with open(os.path.join(golden_dir, "hand_values.json")) as fh:
        return json.load(fh)


def tiny_problem(nx, ny, nz, hx=None, hy=None, hz=None, sig=None, lam=0.0, seed=0, complex_steps=False):
    rng = np.random.default_rng(seed)
    mk = lambda n: (rng.uniform(0.5, 2.0, n + 1) + (1j * rng.uniform(0, 1, n + 1) if complex_steps else 0)).astype(np.complex128)
    hx = mk(nx) if hx is None else np.asarray(hx, np.complex128)
    hy = mk(ny) if hy is None else np.asarray(hy, np.complex128)
    hz = mk(nz) if hz is None else np.asarray(hz, np.complex128)
    if sig is None:
        se = rng.uniform(0.2, 5.0, nz + 1).astype(np.complex128)
    else:
        se = np.full(nz + 1, sig, np.complex128)
    k = np.arange(1, nz + 1)
    sn = (hz[k - 1] * se[k - 1] + hz[k] * se[k]) / (hz[k - 1] + hz[k])
    return Problem(name="tiny", hx=hx, hy=hy, hz=hz, sigma_edge=se, sigma_node=sn, lam=complex(lam),
                   iface_x=[], iface_y=[], nrhs=1, real=False, _rhs=None)


def test_axis_pencil_hand_values(golden_dir):
    g = _golden(golden_dir)
    A, m = axis_pencil(g["axis_uniform3"]["steps"])
    np.testing.assert_array_equal(A, np.array(g["axis_uniform3"]["A"]))
    np.testing.assert_array_equal(m, np.array(g["axis_uniform3"]["M"]))
    A, m = axis_pencil(g["axis_steps12"]["steps"])
    np.testing.assert_array_equal(A, np.array(g["axis_steps12"]["A"]))
    np.testing.assert_array_equal(m, np.array(g["axis_steps12"]["M"]))
    z = g["z_sigma23"]
    Az, mz, _ = z_pencil(z["steps"], z["sigma_half"], [1.0])
    np.testing.assert_array_equal(Az, np.array(z["A_z"]))


def test_single_node_value(golden_dir):
    g = _golden(golden_dir)
    p = tiny_problem(1, 1, 1, hx=[1, 1], hy=[1, 1], hz=[1, 1], sig=1.0, lam=0.0)
    A = oracle.assemble(p).toarray()
    assert A.shape == (1, 1) and A[0, 0] == g["node_1x1x1"]["A"]
    assert oracle.apply_stencil(p, np.ones((1, 1, 1)))[0, 0, 0] == g["node_1x1x1"]["A"]


@pytest.mark.parametrize("seed,cplx", [(0, False), (1, True), (2, True)])
def test_stencil_equals_kronecker(seed, cplx):
    """Eq. (fd) row-by-row == Eq. (fdmtr) with sigma folded into M_z^sigma (reading R1)."""
    p = tiny_problem(5, 4, 6, seed=seed, lam=0.37 - 0.2j, complex_steps=cplx)
    A = oracle.assemble(p).toarray()
    K = oracle.assemble_kron(p).toarray()
    assert np.abs(A - K).max() <= 1e-14 * np.abs(A).max()


def test_operator_complex_symmetric():
    """A = A^T exactly (symmetric stencil of Eq. (fd)); also for PML configs."""
    for name in ("c2", "c4"):
        A = oracle.assemble(shrunken(name))
        assert abs(A - A.T).max() == 0.0


def test_apply_matches_assembled():
    p = tiny_problem(6, 5, 4, seed=3, lam=1.3, complex_steps=True)
    rng = np.random.default_rng(0)
    u = rng.standard_normal(p.shape) + 1j * rng.standard_normal(p.shape)
    Au = (oracle.assemble(p) @ u.ravel()).reshape(p.shape)
    ap = oracle.apply_stencil(p, u)
    assert np.linalg.norm(ap - Au) <= 1e-14 * np.linalg.norm(Au)
    ape = oracle.apply_stencil(p, u, np.clongdouble).astype(np.complex128)
    assert np.linalg.norm(ape - Au) <= 1e-14 * np.linalg.norm(Au)


def test_linears_annihilated():
    """sigma = 1, lam = 0, unit steps: second differences annihilate linear functions."""
    n = 7
    p = tiny_problem(n, n, n, hx=np.ones(n + 1), hy=np.ones(n + 1), hz=np.ones(n + 1), sig=1.0, lam=0.0)
    K, J, I = np.meshgrid(*(np.arange(1, n + 1),) * 3, indexing="ij")
    u = 0.3 + 1.1 * I - 0.7 * J + 2.0 * K
    Au = oracle.apply_stencil(p, u.astype(np.complex128))
    assert np.abs(Au[1:-1, 1:-1, 1:-1]).max() < 1e-12


def _continuum_error(n, lam):
    L = 1.0
    h = L / (n + 1)
    st = np.full(n + 1, h)
    p = tiny_problem(n, n, n, hx=st, hy=st, hz=st, sig=1.0, lam=lam)
    x = h * np.arange(1, n + 1)
    K, J, I = np.meshgrid(x, x, x, indexing="ij")
    u = np.sin(np.pi * I) * np.sin(np.pi * J) * np.sin(np.pi * K)
    # Eq. (wave2): sigma(u_xx + u_yy) + (sigma u_z)_z + lam u = f  with sigma = 1
    f = (-3.0 * np.pi ** 2 + lam) * u
    uh = oracle.solve_separable(p, oracle.mass_rhs(p, f))
    return np.abs(uh - u).max()


@pytest.mark.parametrize("lam", [0.0, 4.0])
def test_second_order_convergence_to_wave2(lam):
    """Pins sign and scale of Eq. (fd) against the continuum equation (wave2)."""
    e1, e2 = _continuum_error(7, lam), _continuum_error(15, lam)
    ratio = e1 / e2
    assert 3.3 < ratio < 4.7, (e1, e2)
    assert e2 < 0.02


def test_workload_sigma_node_is_control_volume_average():
    hz, se, sn = sigma_layers(16, np.array([1.0, 4.0, 0.25]))
    # C1 layer boundaries per SURVEY §8(d): cells 0-5 / 6-11 / 12-16
    assert list(se.real) == [1.0] * 6 + [4.0] * 6 + [0.25] * 5
    assert sn[5] == 0.5 * (1.0 + 4.0) and sn[0] == 1.0
