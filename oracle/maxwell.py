"""ORACLE (test infrastructure): the Lebedev-grid Maxwell system of PAPER.md §3 (lines 81-246).

What it computes, written as the plain definitions (no harmonic decomposition, no blocking):
  * grid M: nodes r_{ijk} = (x_i, y_j, z_k), 0-based i = 0..N_x-1 (N_x odd), from the steps
    h_t = x_{t+1} - x_t (complex steps allowed, the coordinate stretching of a PML);
  * Lebedev P-grid = nodes with i + j + k even, R-grid = the others (read
    0-based: reading M2 of DESIGN.md §13);
  * the finite difference Eq. (fin): (f_x)_i = (f_{i+1} - f_{i-1}) /
    (x_{i+1} - x_{i-1}) at every node with both neighbours; it maps P to R and back;
  * Eq. (abstr): A_h H = curl_h(rho curl_h H) - i omega mu H, with
    rho = diag(c1, c2, c3)(z) applied pointwise on the R nodes ("c^k_i =
    c_i(z_k)"), H on P, E = rho curl_h H on R;
  * boundary conditions: H x n = 0 on the P nodes of dOmega and
    E x n = 0 on its R nodes.  Read here (M3): every component of E on a boundary R node is
    zero (its normal component never enters an interior equation), the unknowns are the three
    components of H on the interior P nodes, and H = 0 on the boundary P nodes (the normal
    component vanishes there too: (curl E)_n on a face only sees tangential E);
  * the solution H = A_h^{-1} f by sparse LU (scipy), f on the interior P nodes.

Fields are arrays (3, N_z, N_y, N_x) (component, z, y, x), complex128; entries off the
interior P nodes are ignored on input and zero on output.  Flat node index (k N_y + j) N_x + i.

Pins: tests/test_oracle_maxwell.py — parity rule examples (SPEC [OP] build_lebedev), curl of
linear fields exact on graded grids, curl grad = 0, the P -> R support rule, the control-volume
adjoint symmetry of the curl pair (W A_h = (W A_h)^T with W = d_x d_y d_z), the omega-term
check on curl-free fields, a hand-evaluated diagonal entry, and the manufactured round trip.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def nodes(h: np.ndarray) -> np.ndarray:
    """Node coordinates x_0 = 0, x_{t+1} = x_t + h_t (complex for stretched steps)."""
    h = np.asarray(h, dtype=np.complex128)
    return np.concatenate([[0.0], np.cumsum(h)])


def diff_matrix(h: np.ndarray) -> sp.csr_matrix:
    """Eq. (fin) on one axis as an N x N matrix: row i (1 <= i <= N-2) takes
    (f_{i+1} - f_{i-1}) / (x_{i+1} - x_{i-1}); the boundary rows are empty."""
    x = nodes(h)
    n = len(x)
    rows, cols, vals = [], [], []
    for i in range(1, n - 1):
        d = x[i + 1] - x[i - 1]
        rows += [i, i]
        cols += [i + 1, i - 1]
        vals += [1.0 / d, -1.0 / d]
    return sp.csr_matrix((np.array(vals, dtype=np.complex128), (rows, cols)), shape=(n, n))


def parity_masks(nx: int, ny: int, nz: int):
    """(P, R, interior) boolean arrays of shape (N_z, N_y, N_x): P = even i + j + k."""
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    P = (i + j + k) % 2 == 0
    inner = (i > 0) & (i < nx - 1) & (j > 0) & (j < ny - 1) & (k > 0) & (k < nz - 1)
    return P, ~P, inner


class Grid:
    """The tensor grid M of PAPER.md:96-103 with its three (fin) operators on flat vectors."""

    def __init__(self, hx, hy, hz):
        self.hx, self.hy, self.hz = (np.asarray(h, dtype=np.complex128) for h in (hx, hy, hz))
        self.nx, self.ny, self.nz = len(self.hx) + 1, len(self.hy) + 1, len(self.hz) + 1
        Ix, Iy, Iz = (sp.identity(n, dtype=np.complex128, format="csr") for n in (self.nx, self.ny, self.nz))
        self.Dx = sp.kron(Iz, sp.kron(Iy, diff_matrix(self.hx))).tocsr()
        self.Dy = sp.kron(Iz, sp.kron(diff_matrix(self.hy), Ix)).tocsr()
        self.Dz = sp.kron(diff_matrix(self.hz), sp.kron(Iy, Ix)).tocsr()
        P, R, inner = parity_masks(self.nx, self.ny, self.nz)
        self.P, self.R, self.inner = P, R, inner
        self.shape = (self.nz, self.ny, self.nx)
        self.nn = self.nx * self.ny * self.nz

    def curl(self) -> sp.csr_matrix:
        """curl_h on stacked (x, y, z) component vectors of length 3 N (no masking)."""
        Z = sp.csr_matrix((self.nn, self.nn), dtype=np.complex128)
        return sp.bmat([[Z, -self.Dz, self.Dy], [self.Dz, Z, -self.Dx], [-self.Dy, self.Dx, Z]]).tocsr()

    def weights(self) -> np.ndarray:
        """Control-volume weights W_{ijk} = d_x(i) d_y(j) d_z(k), d(i) = x_{i+1} - x_{i-1}
        (boundary nodes: 1; they carry no unknowns), flat."""
        def d(h):
            x = nodes(h)
            w = np.ones(len(x), dtype=np.complex128)
            w[1:-1] = x[2:] - x[:-2]
            return w
        return np.einsum("k,j,i->kji", d(self.hz), d(self.hy), d(self.hx)).ravel()


def unknown_mask(g: Grid) -> np.ndarray:
    """Interior P nodes (the unknowns of each component), shape (N_z, N_y, N_x)."""
    return g.P & g.inner


def operator(g: Grid, c1, c2, c3, mu, omega) -> sp.csr_matrix:
    """A_h on the full stacked field (3 N): Pi_P [curl rho Pi_R curl - i omega mu] Pi_P, with
    Pi_P = interior-P projector on H, Pi_R = interior-R projector on E (E = 0 on the boundary
    R nodes), rho = diag(c1, c2, c3) of the node's z level."""
    c = [np.asarray(v, dtype=np.complex128) for v in (c1, c2, c3)]
    kk = np.broadcast_to(np.arange(g.nz)[:, None, None], g.shape).ravel()
    pm = np.tile(unknown_mask(g).ravel(), 3).astype(np.complex128)
    rm = np.tile((g.R & g.inner).ravel(), 3).astype(np.complex128)
    rho = np.concatenate([c[0][kk], c[1][kk], c[2][kk]])
    C = g.curl()
    PiP, PiRrho = sp.diags(pm), sp.diags(rm * rho)
    return (PiP @ C @ PiRrho @ C @ PiP - 1j * omega * mu * PiP).tocsr()


def apply(g: Grid, H: np.ndarray, c1, c2, c3, mu, omega) -> np.ndarray:
    """A_h H on the interior P nodes (zero elsewhere); H of shape (3, N_z, N_y, N_x)."""
    A = operator(g, c1, c2, c3, mu, omega)
    return (A @ np.asarray(H, dtype=np.complex128).ravel()).reshape((3,) + g.shape)


def solve(g: Grid, f: np.ndarray, c1, c2, c3, mu, omega) -> np.ndarray:
    """H = A_h^{-1} f by sparse LU on the unknowns (3 components x interior P nodes)."""
    A = operator(g, c1, c2, c3, mu, omega)
    idx = np.flatnonzero(np.tile(unknown_mask(g).ravel(), 3))
    Auu = A[idx][:, idx].tocsc()
    x = spla.splu(Auu).solve(np.asarray(f, dtype=np.complex128).ravel()[idx])
    H = np.zeros(3 * g.nn, dtype=np.complex128)
    H[idx] = x
    return H.reshape((3,) + g.shape)


def rel_residual(g: Grid, H, f, c1, c2, c3, mu, omega) -> float:
    """||f - A_h H|| / ||f|| over the unknowns."""
    m = np.broadcast_to(unknown_mask(g), (3,) + g.shape)
    r = (np.asarray(f) - apply(g, H, c1, c2, c3, mu, omega))[m]
    return float(np.linalg.norm(r) / np.linalg.norm(np.asarray(f)[m]))
