"""ORACLE (test infrastructure): horizontally heterogeneous media.

The paper's motivating use: layered background media "with several embedded inhomogeneities"
(PAPER.md:20), where iterative solvers are needed and the layered-medium solver serves as the
preconditioner.  Model: a node-wise lambda (a velocity anomaly in the
Helmholtz shift), lambda_ijk = lambda + dlam_ijk, in Eq. (fd).  Its lambda
term  lambda u hx^_i hy^_j hz^_k  becomes  (lambda + dlam_ijk) u hx^_i hy^_j hz^_k, so

    A_het = A + diag(dlam_ijk hx^_i hy^_j hz^_k),        u = A_het^{-1} M f.

``solve_hetero_direct`` is that definition: sparse LU (scipy SuperLU) of the assembled A_het —
tiny grids only.  The CUDA path (lfds_gmres) reaches the same u by preconditioned GMRES; it
shares nothing with this module.

Pins: tests/test_oracle_hetero.py (dlam = 0 gives A exactly; a constant dlam = c gives the
matrix of lambda + c; A_het symmetric; the Lippmann-Schwinger identity u = S(f - dlam u) with
the oracle's independent separable solver S).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .operator import assemble, apply_stencil, control_volumes, mass_rhs


def _volumes(p) -> np.ndarray:
    cx, cy, cz = (control_volumes(np.asarray(h, dtype=np.complex128)) for h in (p.hx, p.hy, p.hz))
    return cz[:, None, None] * cy[None, :, None] * cx[None, None, :]


def assemble_hetero(p, dlam: np.ndarray) -> sp.csr_matrix:
    """A_het = A + diag(dlam hx^ hy^ hz^) (Eq. (fd) with lambda_ijk = lambda + dlam_ijk)."""
    d = (np.asarray(dlam, dtype=np.complex128) * _volumes(p)).ravel()
    return (assemble(p) + sp.diags(d)).tocsr()


def solve_hetero_direct(p, dlam: np.ndarray, f: np.ndarray) -> np.ndarray:
    """u = A_het^{-1} M f by sparse LU (partial pivoting); f, dlam, u are [k][j][i]."""
    b = mass_rhs(p, f).ravel()
    u = spla.splu(assemble_hetero(p, dlam).tocsc()).solve(b)
    return u.reshape(p.shape)


def rel_residual_hetero(p, dlam: np.ndarray, u: np.ndarray, f: np.ndarray, dtype=np.complex128) -> float:
    """||A_het u - M f|| / ||M f||, matrix-free (Eq. (fd) term by term plus the dlam term)."""
    b = mass_rhs(p, f, dtype)
    uu = np.asarray(u, dtype=dtype)
    r = apply_stencil(p, uu, dtype) + np.asarray(dlam, dtype=dtype) * uu * _volumes(p).astype(dtype) - b
    return float(np.linalg.norm(r.astype(np.complex128)) / np.linalg.norm(b.astype(np.complex128)))
