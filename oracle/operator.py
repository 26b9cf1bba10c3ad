"""ORACLE (test infrastructure): the 7-point finite-volume operator of Eq. (fd).

Conventions (DESIGN.md §2 readings):
  R3  N_d unknown nodes per axis, 1..N_d; N_d+1 steps h_0..h_{N_d}; step h_t joins node t
      and t+1; nodes 0 and N_d+1 carry the homogeneous Dirichlet condition (R10).
  P:36 control-volume edge  hat h_i = (h_{i-1} + h_i)/2.
  R1  the Kronecker form folds sigma_k into the z-mass of the horizontal terms:
      A = A_x(x)M_y(x)M_z^s + M_x(x)A_y(x)M_z^s + M_x(x)M_y(x)A_z + lam M_x(x)M_y(x)M_z,
      M_z^s = diag(sigma_k hat h^z_k).  Eq. (fd) is the authority.
  Arrays are [k][j][i] (z slowest, x fastest); flat index (k*Ny + j)*Nx + i.

Pins: tests/test_oracle_operator.py (SPEC hand values S:134-136 in tests/golden,
stencil == Kronecker, exact symmetry, 1x1x1 value, linear annihilation, O(h^2)
convergence to Eq. (wave2)'s continuum solution).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def control_volumes(h: np.ndarray) -> np.ndarray:
    """hat h_i = (h_{i-1} + h_i)/2, i = 1..N, from the N+1 steps."""
    h = np.asarray(h)
    return 0.5 * (h[:-1] + h[1:])


def axis_pencil(h: np.ndarray):
    """Dense (A_d, diag M_d) of one horizontal axis.

    Row of node i: A[i,i-1] = 1/h_{i-1}, A[i,i] = -(1/h_{i-1} + 1/h_i), A[i,i+1] = 1/h_i
    (the x-bracket of Eq. (fd) without its sigma_k hat h^y hat h^z factor)."""
    h = np.asarray(h, dtype=np.complex128)
    n = len(h) - 1
    A = np.zeros((n, n), dtype=np.complex128)
    for i in range(n):            # row i <-> node i+1: left step h[i], right step h[i+1]
        A[i, i] = -(1.0 / h[i] + 1.0 / h[i + 1])
        if i > 0:
            A[i, i - 1] = 1.0 / h[i]
        if i + 1 < n:
            A[i, i + 1] = 1.0 / h[i + 1]
    return A, control_volumes(h)


def z_pencil(hz: np.ndarray, sigma_edge: np.ndarray, sigma_node: np.ndarray):
    """(A_z, diag M_z, diag M_z^sigma) from the z-bracket of Eq. (fd) and reading R1."""
    hz = np.asarray(hz, dtype=np.complex128)
    se = np.asarray(sigma_edge, dtype=np.complex128)
    n = len(hz) - 1
    A = np.zeros((n, n), dtype=np.complex128)
    for k in range(n):            # row k <-> node k+1: sigma_{k+1/2 - 1} = se[k], sigma_{k+1+1/2} = se[k+1]
        A[k, k] = -(se[k] / hz[k] + se[k + 1] / hz[k + 1])
        if k > 0:
            A[k, k - 1] = se[k] / hz[k]
        if k + 1 < n:
            A[k, k + 1] = se[k + 1] / hz[k + 1]
    mz = control_volumes(hz)
    return A, mz, np.asarray(sigma_node, dtype=np.complex128) * mz


def assemble(p) -> sp.csr_matrix:
    """Assemble A literally from Eq. (fd), row by row (vectorised over nodes).

    For node (i,j,k) the off-diagonal couplings are
      x:  sigma_k hat h^y_j hat h^z_k / h^x_i      (to i+1),  ... / h^x_{i-1}  (to i-1)
      y:  sigma_k hat h^x_i hat h^z_k / h^y_j      (to j+1),  ... / h^y_{j-1}  (to j-1)
      z:  sigma_{k+1/2} hat h^x_i hat h^y_j / h^z_k (to k+1), sigma_{k-1/2} ... / h^z_{k-1} (to k-1)
    and the diagonal is minus their sum (including couplings to Dirichlet nodes, whose
    values are zero) plus lam hat h^x hat h^y hat h^z."""
    nx, ny, nz = p.nx, p.ny, p.nz
    hx, hy, hz = (np.asarray(a, dtype=np.complex128) for a in (p.hx, p.hy, p.hz))
    cx, cy, cz = control_volumes(hx), control_volumes(hy), control_volumes(hz)
    se = np.asarray(p.sigma_edge, dtype=np.complex128)
    sn = np.asarray(p.sigma_node, dtype=np.complex128)
    K, J, I = np.meshgrid(np.arange(1, nz + 1), np.arange(1, ny + 1), np.arange(1, nx + 1), indexing="ij")
    K, J, I = K.ravel(), J.ravel(), I.ravel()
    row = ((K - 1) * ny + (J - 1)) * nx + (I - 1)
    hhx, hhy, hhz = cx[I - 1], cy[J - 1], cz[K - 1]
    sig = sn[K - 1]
    # (neighbour offset, coefficient, neighbour-in-domain mask, flat column)
    terms = [
        (sig * hhy * hhz / hx[I], I + 1 <= nx, row + 1),
        (sig * hhy * hhz / hx[I - 1], I - 1 >= 1, row - 1),
        (sig * hhx * hhz / hy[J], J + 1 <= ny, row + nx),
        (sig * hhx * hhz / hy[J - 1], J - 1 >= 1, row - nx),
        (se[K] * hhx * hhy / hz[K], K + 1 <= nz, row + nx * ny),
        (se[K - 1] * hhx * hhy / hz[K - 1], K - 1 >= 1, row - nx * ny),
    ]
    rows, cols, vals = [], [], []
    diag = p.lam * hhx * hhy * hhz
    for coef, inside, col in terms:
        diag = diag - coef
        rows.append(row[inside]); cols.append(col[inside]); vals.append(coef[inside])
    rows.append(row); cols.append(row); vals.append(diag)
    n = nx * ny * nz
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    return A.tocsr()


def assemble_kron(p) -> sp.csr_matrix:
    """The Kronecker form Eq. (fdmtr) with reading R1 (sigma folded into M_z^sigma)."""
    Ax, mx = axis_pencil(p.hx)
    Ay, my = axis_pencil(p.hy)
    Az, mz, mzs = z_pencil(p.hz, p.sigma_edge, p.sigma_node)
    Ax, Ay, Az = sp.csr_matrix(Ax), sp.csr_matrix(Ay), sp.csr_matrix(Az)
    Mx, My, Mz, Mzs = sp.diags(mx), sp.diags(my), sp.diags(mz), sp.diags(mzs)
    k3 = lambda z, y, x: sp.kron(z, sp.kron(y, x))  # flat order (k, j, i)
    A = k3(Mzs, My, Ax) + k3(Mzs, Ay, Mx) + k3(Az, My, Mx) + p.lam * k3(Mz, My, Mx)
    return A.tocsr()


def mass_rhs(p, f: np.ndarray, dtype=np.complex128) -> np.ndarray:
    """b = (M_x (x) M_y (x) M_z) f, the right side of Eq. (fd)/(fdmtr); f is [..., k, j, i]."""
    cx = control_volumes(np.asarray(p.hx, dtype=dtype))
    cy = control_volumes(np.asarray(p.hy, dtype=dtype))
    cz = control_volumes(np.asarray(p.hz, dtype=dtype))
    w = cz[:, None, None] * cy[None, :, None] * cx[None, None, :]
    return np.asarray(f, dtype=dtype) * w


def apply_stencil(p, u: np.ndarray, dtype=np.complex128) -> np.ndarray:
    """A u, matrix-free, term by term as Eq. (fd) is written; u is [k][j][i].

    ``dtype=np.clongdouble`` evaluates every product and sum in 80-bit extended
    precision (used for the refinement residual, reading R13)."""
    hx = np.asarray(p.hx, dtype=dtype); hy = np.asarray(p.hy, dtype=dtype)
    hz = np.asarray(p.hz, dtype=dtype)
    se = np.asarray(p.sigma_edge, dtype=dtype); sn = np.asarray(p.sigma_node, dtype=dtype)
    lam = np.asarray(p.lam, dtype=dtype)
    cx, cy, cz = control_volumes(hx), control_volumes(hy), control_volumes(hz)
    nz, ny, nx = u.shape
    up = np.zeros((nz + 2, ny + 2, nx + 2), dtype=dtype)
    up[1:-1, 1:-1, 1:-1] = u
    c = up[1:-1, 1:-1, 1:-1]
    # x-term: sigma_k ((u_{i+1}-u_i)/h^x_i - (u_i-u_{i-1})/h^x_{i-1}) hat h^y_j hat h^z_k
    tx = (up[1:-1, 1:-1, 2:] - c) / hx[None, None, 1:] - (c - up[1:-1, 1:-1, :-2]) / hx[None, None, :-1]
    tx = sn[:, None, None] * tx * cy[None, :, None] * cz[:, None, None]
    # y-term: sigma_k ((u_{j+1}-u_j)/h^y_j - (u_j-u_{j-1})/h^y_{j-1}) hat h^x_i hat h^z_k
    ty = (up[1:-1, 2:, 1:-1] - c) / hy[None, 1:, None] - (c - up[1:-1, :-2, 1:-1]) / hy[None, :-1, None]
    ty = sn[:, None, None] * ty * cx[None, None, :] * cz[:, None, None]
    # z-term: (sigma_{k+1/2}(u_{k+1}-u_k)/h^z_k - sigma_{k-1/2}(u_k-u_{k-1})/h^z_{k-1}) hat h^x_i hat h^y_j
    tz = (se[1:, None, None] * (up[2:, 1:-1, 1:-1] - c) / hz[1:, None, None]
          - se[:-1, None, None] * (c - up[:-2, 1:-1, 1:-1]) / hz[:-1, None, None])
    tz = tz * cx[None, None, :] * cy[None, :, None]
    tl = lam * c * cx[None, None, :] * cy[None, :, None] * cz[:, None, None]
    return tx + ty + tz + tl


def rel_residual(p, u: np.ndarray, f: np.ndarray, dtype=np.complex128) -> float:
    """||A u - M f||_2 / ||M f||_2 (the north-star residual, SURVEY.md §8(b) 'Units')."""
    b = mass_rhs(p, f, dtype)
    r = apply_stencil(p, np.asarray(u, dtype=dtype), dtype) - b
    return float(np.linalg.norm(r.astype(np.complex128)) / np.linalg.norm(b.astype(np.complex128)))
