"""Pins for oracle/eig.py: closed-form sine eigenpairs, SPEC worked examples, invariants."""
import json
import os

import numpy as np
import pytest

from oracle.eig import gen_eig, sine_basis
from oracle.operator import axis_pencil
from workloads.configs import axis_steps


def _golden(golden_dir):
    with open(os.path.join(golden_dir, "hand_values.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("n,h", [(11, 1.0), (31, 0.7), (127, 1.0), (128, 2.5)])
def test_uniform_steps_give_sine_modes(n, h):
    """W_il = sqrt(2/(h(n+1))) sin(pi i l/(n+1)), lam_l = -(4/h^2) sin^2(pi l/(2(n+1))) (closed form)."""
    lam, W = gen_eig(np.full(n + 1, h))
    i = np.arange(1, n + 1)
    lam_cf = np.sort(-(4.0 / h ** 2) * np.sin(np.pi * i / (2 * (n + 1))) ** 2)
    np.testing.assert_allclose(lam.real, lam_cf, rtol=0, atol=1e-12 / h ** 2)
    assert np.abs(lam.imag).max() == 0
    # eigenvalues sorted ascending: column c is sine mode l = n - c
    for c in range(n):
        l = n - c
        w = np.sqrt(2.0 / (h * (n + 1))) * np.sin(np.pi * i * l / (n + 1))
        s = np.sign(np.dot(W[:, c].real, w))
        assert np.abs(s * W[:, c] - w).max() < 1e-11


def test_sine_basis_helper_matches_closed_form():
    lam, W = sine_basis(9, 1.0)
    A, m = axis_pencil(np.ones(10))
    assert np.abs(A @ W - (m[:, None] * W) * lam[None, :]).max() < 1e-13


def test_spec_examples(golden_dir):
    g = _golden(golden_dir)
    lam, _ = gen_eig(g["eig_uniform3"]["steps"])
    np.testing.assert_allclose(lam.real, g["eig_uniform3"]["lambda"], atol=1e-14)
    lam, W = gen_eig(g["eig_1x1_a"]["steps"])
    np.testing.assert_allclose(lam.real, g["eig_1x1_a"]["lambda"], atol=1e-15)
    np.testing.assert_allclose(np.abs(W[:, 0]), g["eig_1x1_a"]["absW"], atol=1e-15)
    h0 = 2 + np.sqrt(4 - 4.0 / 3.0); h1 = 4 - h0
    lam, W = gen_eig([h0, h1])
    np.testing.assert_allclose(lam.real, g["eig_1x1_b"]["lambda"], atol=1e-14)
    np.testing.assert_allclose(np.abs(W[:, 0]), g["eig_1x1_b"]["absW"], atol=1e-15)


STEP_CASES = {
    "c2_pml_quad": axis_steps(96, 0, 1.0, 16, "quad"),
    "c3_graded_pml": axis_steps(192, 24, 1.2, 8, "quad"),
    "c4_pml_const": axis_steps(960, 0, 1.0, 32, "const"),
    "c4_block_edge": axis_steps(960, 0, 1.0, 32, "const")[:128],
    "random_real": np.random.default_rng(5).uniform(0.5, 2, 40),
    "odd_palindrome": axis_steps(23, 3, 1.3, 4, "quad"),
}


@pytest.mark.parametrize("case", list(STEP_CASES))
def test_pencil_invariants(case):
    """A W = M W Lambda and W^T M W = I (transpose, reading R4)."""
    h = STEP_CASES[case]
    lam, W = gen_eig(h)
    A, m = axis_pencil(h)
    res = np.abs(A @ W - (m[:, None] * W) * lam[None, :]).max() / (np.abs(A).max() * np.abs(W).max())
    bio = np.abs(W.T @ (m[:, None] * W) - np.eye(len(m))).max()
    # PML bases are intrinsically non-normal (cond(V) up to ~1e5 for the C2 quadratic ramp, SURVEY
    # Appendix), so their W^T M W error scales with that condition number.
    tol_bio = 1e-7 if case == "c2_pml_quad" else 1e-9
    assert res < 1e-12, res
    assert bio < tol_bio, bio


def test_parity_split_beats_plain_eig_on_palindromic_pml():
    """The mirror-symmetric PML pencil is numerically degenerate for plain eig."""
    h = axis_steps(96, 0, 1.0, 16, "quad")
    A, m = axis_pencil(h)
    _, W = gen_eig(h, parity=True)
    _, Wp = gen_eig(h, parity=False)
    bio = lambda W: np.abs(W.T @ (m[:, None] * W) - np.eye(len(m))).max()
    assert bio(W) < 1e-7
    assert bio(W) < bio(Wp)
