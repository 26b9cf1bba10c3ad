"""ORACLE (test infrastructure): the discrete solution u = A^{-1} M f of Eq. (fd).

The paper's two-level method is a direct solver: in exact arithmetic it returns this
u (PAPER.md:24 "compute the solution u", :58-60 u = v + w).  So the oracle
is that definition written out, two ways:

 (i)  ``solve_direct``   sparse LU (scipy SuperLU, partial pivoting) of the literally
      assembled matrix — tiny grids only.
 (ii) ``solve_separable`` the global separable eigen-solve of Eq. (fdmtrprjfrerr)
       with the WHOLE grid as one block: b^ = (W_x^T (x) W_y^T (x) I) b,
      one tridiagonal z-solve [A_z + lam M_z + (lam_l + mu_m) M_z^sigma] u^_lm = b^_lm per
      mode (LAPACK zgtsv, partial pivoting, reading R15), u = (W_x (x) W_y (x) I) u^.

``solve`` adds iterative refinement with an 80-bit (clongdouble) residual of the
literal stencil (reading R13): u <- u + S(b - A u) until ||r||/||b|| stops decreasing.

``block_solutions`` gives the pass-1 quantity v of PAPER.md:43-44 by definition
(sparse LU of each block's restricted matrix, v = 0 on the interfaces), used to pin
the interface-support invariant and, through r_b = b - A v on the planes,
the CUDA path's steps 1-4 (tests/test_gpu_parity.py::
test_pass1_interface_residual_matches_oracle_block_solutions).

Pins: tests/test_oracle_solve.py ((i) == (ii) on shrunken analogs of every config,
random manufactured discrete solutions, exact discrete eigenfunction, reciprocity,
linearity, interface-support invariant, O(h^2) continuum convergence).
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.sparse.linalg as spla
from scipy.linalg import lapack

from .operator import assemble, apply_stencil, mass_rhs, z_pencil
from .eig import gen_eig


@dataclasses.dataclass
class GlobalBases:
    lam_x: np.ndarray
    W_x: np.ndarray
    lam_y: np.ndarray
    W_y: np.ndarray
    az_sub: np.ndarray   # A_z[k, k-1]
    az_diag: np.ndarray  # A_z[k, k] + lam * M_z[k]
    az_sup: np.ndarray   # A_z[k, k+1]
    mzs: np.ndarray      # M_z^sigma


def global_bases(p) -> GlobalBases:
    lx, Wx = gen_eig(p.hx)
    if np.array_equal(p.hx, p.hy):
        ly, Wy = lx, Wx
    else:
        ly, Wy = gen_eig(p.hy)
    Az, mz, mzs = z_pencil(p.hz, p.sigma_edge, p.sigma_node)
    return GlobalBases(lx, Wx, ly, Wy, np.diag(Az, -1).copy(), np.diag(Az) + p.lam * mz,
                       np.diag(Az, 1).copy(), mzs)


def _zsolve(dl, d, du, rhs):
    """LAPACK zgtsv (Gaussian elimination with partial pivoting) for one tridiagonal system."""
    _, _, _, x, info = lapack.zgtsv(dl.copy(), d.copy(), du.copy(), rhs.copy())
    if info != 0:
        raise np.linalg.LinAlgError(f"zgtsv info={info}")
    return x


def solve_separable(p, b: np.ndarray, bases: GlobalBases | None = None) -> np.ndarray:
    """(ii): b is [nrhs?][k][j][i] in b-units; returns u of the same shape."""
    g = bases or global_bases(p)
    single = b.ndim == 3
    B = b[None] if single else b
    nr, nz, ny, nx = B.shape
    # forward: b^[r,k,m,l] = sum_q sum_p W_y[q,m] W_x[p,l] b[r,k,q,p]
    t = B.astype(np.complex128) @ g.W_x                         # contract p
    bh = np.einsum("qm,rkql->rkml", g.W_y, t, optimize=True)   # contract q
    bh = np.ascontiguousarray(bh.transpose(3, 2, 1, 0))        # [l, m, k, r]
    uh = np.empty_like(bh)
    for l in range(nx):
        for m in range(ny):
            d = g.az_diag + (g.lam_x[l] + g.lam_y[m]) * g.mzs
            uh[l, m] = _zsolve(g.az_sub, d, g.az_sup, bh[l, m])
    uh = np.ascontiguousarray(uh.transpose(3, 2, 1, 0))        # [r, k, m, l]
    # inverse: u[r,k,q,p] = sum_m W_y[q,m] sum_l W_x[p,l] u^[r,k,m,l]
    t = uh @ g.W_x.T
    u = np.einsum("qm,rkmp->rkqp", g.W_y, t, optimize=True)
    return u[0] if single else u


def solve_direct(p, b: np.ndarray, A=None) -> np.ndarray:
    """(i): sparse LU of the assembled Eq. (fd) matrix (tiny grids)."""
    A = assemble(p) if A is None else A
    lu = spla.splu(A.tocsc().astype(np.complex128))
    single = b.ndim == 3
    B = b[None] if single else b
    u = np.stack([lu.solve(x.ravel().astype(np.complex128)).reshape(x.shape) for x in B])
    return u[0] if single else u


def residual_ext(p, u: np.ndarray, b_ext: np.ndarray) -> np.ndarray:
    """b - A u in clongdouble (80-bit) arithmetic; b_ext already clongdouble."""
    return b_ext - apply_stencil(p, np.asarray(u, dtype=np.clongdouble), np.clongdouble)


def solve(p, f: np.ndarray, method: str = "separable", max_refine: int = 6, bases=None,
          return_info: bool = False):
    """u = A^{-1} M f with clongdouble-residual refinement (reading R13).

    f: [k][j][i] or [r][k][j][i] (density units of Eq. (fd))."""
    single = f.ndim == 3
    F = f[None] if single else f
    if method == "separable":
        g = bases or global_bases(p)
        S = lambda b: solve_separable(p, b, g)
    elif method == "direct":
        A = assemble(p)
        S = lambda b: solve_direct(p, b, A)
    else:
        raise ValueError(method)
    out, infos = [], []
    for fr in F:
        b_ext = mass_rhs(p, fr, np.clongdouble)
        bn = float(np.linalg.norm(b_ext.astype(np.complex128)))
        u = S(b_ext.astype(np.complex128))
        hist, best, best_rn = [], u, np.inf
        for it in range(max_refine + 1):
            r = residual_ext(p, u, b_ext)
            rn = float(np.linalg.norm(r.astype(np.complex128))) / (bn if bn > 0 else 1.0)
            hist.append(rn)
            if rn < best_rn:
                best, best_rn = u, rn
            else:
                break                                   # stopped decreasing
            if it == max_refine or rn == 0.0 or (len(hist) > 1 and rn > 0.5 * hist[-2]):
                break                                   # stagnated at the rounding floor
            u = u + S(r.astype(np.complex128))
        out.append(best)
        infos.append({"residual_history": hist})
    u = out[0] if single else np.stack(out)
    if return_info:
        return u, (infos[0] if single else infos)
    return u


def block_ranges(n: int, iface):
    """Contiguous 1-based node ranges [lo, hi] between the interface nodes (reading R9)."""
    cuts = [0] + list(iface) + [n + 1]
    return [(cuts[a] + 1, cuts[a + 1] - 1) for a in range(len(cuts) - 1) if cuts[a + 1] - 1 >= cuts[a] + 1]


def interface_mask(p) -> np.ndarray:
    """True on the union of interface planes (all z)."""
    m = np.zeros(p.shape, dtype=bool)
    for a in p.iface_x:
        m[:, :, a - 1] = True
    for b in p.iface_y:
        m[:, b - 1, :] = True
    return m


def block_solutions(p, b: np.ndarray, A=None) -> np.ndarray:
    """v of PAPER.md:43-44: each block solved with homogeneous Dirichlet data, v = 0 on
    the interfaces (definition Eq. (fdmtrprj): the restriction P A P of A to the block)."""
    A = (assemble(p) if A is None else A).tocsr()
    v = np.zeros(p.shape, dtype=np.complex128)
    K = np.arange(p.nz)
    for (x0, x1) in block_ranges(p.nx, p.iface_x):
        for (y0, y1) in block_ranges(p.ny, p.iface_y):
            kk, jj, ii = np.meshgrid(K, np.arange(y0 - 1, y1), np.arange(x0 - 1, x1), indexing="ij")
            idx = ((kk * p.ny + jj) * p.nx + ii).ravel()
            sub = A[idx][:, idx].tocsc()
            v.ravel()[idx] = spla.splu(sub).solve(b.ravel()[idx].astype(np.complex128))
    return v
