"""ORACLE (test infrastructure): 1D generalized eigenpairs A_d W = M_d W Lambda.

Method: symmetrise S = M^{-1/2} A M^{-1/2} with the principal
complex square root; for a palindromic step sequence (h_t = h_{N-t}) split S into its
even and odd (mirror-symmetric / antisymmetric) halves and solve each separately (the
halves' eigenvalues interleave and would otherwise be numerically degenerate under PML);
normalise v^T v = 1 (complex-symmetric, transpose not conjugate, reading R4);
W = M^{-1/2} V, so W^T M W = I and A W = M W Lambda.  Eigenpairs are sorted by
(Re, Im) of the eigenvalue (reading R14).  LAPACK (scipy.linalg.eig / eigh) is the
library primitive; nothing here is shared with the host eigensolver of the C library.

Pins: tests/test_oracle_eig.py (closed-form sine eigenpairs on uniform steps,
SPEC S:195 eigenvalues -2 +- sqrt 2, -2, 1x1 pencils, pencil residual and
biorthonormality invariants on PML / graded steps).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .operator import axis_pencil


def _sym_tridiag(h):
    A, m = axis_pencil(h)
    s = 1.0 / np.sqrt(m.astype(np.complex128))
    d = np.diag(A) * s * s
    e = np.diag(A, 1) * s[:-1] * s[1:]
    return d, e, m, s


def _eig_sym_dense(S, real):
    if real:
        lam, V = np.linalg.eigh(S.real)
        return lam.astype(np.complex128), V.astype(np.complex128)
    lam, V = sla.eig(S)
    nrm = np.sqrt(np.sum(V * V, axis=0))          # v^T v (no conjugation)
    return lam, V / nrm[None, :]


def _tridiag(d, e):
    n = len(d)
    S = np.diag(d).astype(np.complex128)
    if n > 1:
        S += np.diag(e, 1) + np.diag(e, -1)
    return S


def gen_eig(h, parity: bool = True):
    """Eigenpairs of the Dirichlet pencil of steps h (N+1 steps, N nodes).

    Returns (lam (N,), W (N, N)) with A W = M W diag(lam), W^T M W = I."""
    h = np.asarray(h, dtype=np.complex128)
    d, e, m, s = _sym_tridiag(h)
    n = len(d)
    real = bool(np.all(h.imag == 0) and np.all(h.real > 0))
    palin = parity and n >= 2 and bool(np.all(h == h[::-1]))
    if not palin:
        lam, V = _eig_sym_dense(_tridiag(d, e), real)
    else:
        k = n // 2
        r2 = np.sqrt(2.0)
        if n % 2 == 0:
            de = d[:k].copy(); de[k - 1] += e[k - 1]
            do = d[:k].copy(); do[k - 1] -= e[k - 1]
            le, Ye = _eig_sym_dense(_tridiag(de, e[:k - 1]), real)
            lo, Yo = _eig_sym_dense(_tridiag(do, e[:k - 1]), real)
            Ve = np.vstack([Ye, Ye[::-1, :]]) / r2
            Vo = np.vstack([Yo, -Yo[::-1, :]]) / r2
        else:
            # even block on (y, gamma), gamma = c/sqrt2, coupling sqrt2 * e_{k-1}
            de = d[:k + 1].copy()
            ee = e[:k].copy(); ee[k - 1] = r2 * e[k - 1]
            le, Ye = _eig_sym_dense(_tridiag(de, ee), real)
            Ve = np.vstack([Ye[:k], r2 * Ye[k:k + 1], Ye[:k][::-1]]) / r2
            if k > 0:
                lo, Yo = _eig_sym_dense(_tridiag(d[:k], e[:k - 1]), real)
                Vo = np.vstack([Yo, np.zeros((1, k)), -Yo[::-1, :]]) / r2
            else:
                lo, Vo = np.zeros(0, np.complex128), np.zeros((1, 0), np.complex128)
        lam = np.concatenate([le, lo])
        V = np.hstack([Ve, Vo])
    order = np.lexsort((lam.imag, lam.real))
    lam, V = lam[order], V[:, order]
    W = s[:, None] * V
    return lam, W


def sine_basis(n: int, hstep: float):
    """Closed form for uniform real steps h:
    W_il = sqrt(2/(h(n+1))) sin(pi i l/(n+1)), lam_l = -(4/h^2) sin^2(pi l/(2(n+1)))."""
    i = np.arange(1, n + 1)[:, None]
    l = np.arange(1, n + 1)[None, :]
    W = np.sqrt(2.0 / (hstep * (n + 1))) * np.sin(np.pi * i * l / (n + 1))
    lam = -(4.0 / hstep ** 2) * np.sin(np.pi * np.arange(1, n + 1) / (2 * (n + 1))) ** 2
    order = np.argsort(lam)
    return lam[order].astype(np.complex128), W[:, order].astype(np.complex128)
