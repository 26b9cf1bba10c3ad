"""Seeded synthetic inputs of the Lebedev-grid Maxwell solve (§3).

No arithmetic of the method here: only grid steps, the layered diagonal resistivity
rho = diag(c1, c2, c3)(z), mu, omega and the right-hand side f.

Recipe:
* every axis has N = 2n + 1 nodes (odd, so both ends are primary nodes, reading M1) and
  N - 1 steps: a unit core, G outward-graded steps (ratio q) and P stretched steps
  h (1 + 2i (s/P)^2) on each side (the complex coordinate stretching of a PML; the paper gives
  no profile), or all unit steps (``pml=0``);
* z: unit core steps with G graded steps at the bottom, L layers over the N_z nodes with
  horizontal resistivity c1 = c2 = 10**U(-0.5, 1) and vertical c3 = c1 * U(1, 3) (anisotropic
  layers, the diagonal rho of PAPER.md:346-348);
* mu = 1, omega = 2 / delta^2 for a skin depth delta (in cells) of the most conductive layer;
* f: ``nsrc`` unit point sources (CN(0,1) amplitudes, random component) at interior P nodes of
  the core + 1e-3 CN(0,1) on every interior P node; zero elsewhere.  Shape (3, N_z, N_y, N_x).
Seeds: default_rng(SeedSequence([1909, 1299, 900 + cfg, stream])).
"""
from __future__ import annotations

import dataclasses

import numpy as np

MW_CONFIGS = {
    # name: (cfg id, n_x, n_y, n_z, G, q, P, layers, delta, nsrc)
    "mw_tiny": (1, 3, 3, 3, 0, 1.0, 1, 2, 3.0, 2),
    "mw_s": (2, 8, 7, 6, 1, 1.3, 2, 3, 4.0, 4),
    "mw_s2": (3, 12, 9, 8, 2, 1.2, 3, 4, 5.0, 6),
    "mw_u": (4, 8, 8, 5, 0, 1.0, 0, 1, 4.0, 3),      # uniform real steps, one layer
    "mw1": (10, 256, 256, 128, 8, 1.1, 16, 6, 12.0, 16),
}


def _rng(cfg: int, stream: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([1909, 1299, 900 + cfg, stream]))


def axis_steps(n: int, G: int, q: float, P: int, bottom_only: bool = False) -> np.ndarray:
    """The 2n complex steps of an axis with 2n + 1 nodes (core unit steps, G graded, P PML)."""
    N = 2 * n + 1
    h = np.ones(N - 1, dtype=np.complex128)
    tail = []
    for s in range(1, G + 1):
        tail.append(complex(q ** s))
    base = q ** G
    for s in range(1, P + 1):
        tail.append(base * (1.0 + 2.0j * (s / P) ** 2))
    T = len(tail)
    assert 2 * T < N - 1, "tails longer than the axis"
    if T == 0:
        return h
    # right tail: the last T steps grow outward; left tail (unless bottom_only): its mirror
    h[N - 1 - T:] = tail
    if not bottom_only:
        h[:T] = tail[::-1]
    return h


@dataclasses.dataclass
class MWProblem:
    name: str
    hx: np.ndarray
    hy: np.ndarray
    hz: np.ndarray
    c1: np.ndarray      # (N_z,) per z level
    c2: np.ndarray
    c3: np.ndarray
    mu: complex
    omega: float
    nsrc: int
    cfg: int

    @property
    def shape(self):
        return (len(self.hz) + 1, len(self.hy) + 1, len(self.hx) + 1)

    def rhs(self) -> np.ndarray:
        nz, ny, nx = self.shape
        f = np.zeros((3, nz, ny, nx), dtype=np.complex128)
        k, j, i = np.ogrid[:nz, :ny, :nx]
        unk = ((i + j + k) % 2 == 0) & (i > 0) & (i < nx - 1) & (j > 0) & (j < ny - 1) & (k > 0) & (k < nz - 1)
        rn = _rng(self.cfg, 4)
        noise = rn.standard_normal((3, nz, ny, nx)) + 1j * rn.standard_normal((3, nz, ny, nx))
        f += 1e-3 * noise * unk
        rs = _rng(self.cfg, 3)
        placed = 0
        while placed < self.nsrc:
            c = int(rs.integers(0, 3))
            kk = int(rs.integers(1, nz - 1))
            jj = int(rs.integers(max(1, ny // 4), max(2, 3 * ny // 4)))
            ii = int(rs.integers(max(1, nx // 4), max(2, 3 * nx // 4)))
            if not unk[kk, jj, ii]:
                continue
            f[c, kk, jj, ii] += rs.standard_normal() + 1j * rs.standard_normal()
            placed += 1
        return f


def make_mw(name: str) -> MWProblem:
    cfg, nx, ny, nz, G, q, P, L, delta, nsrc = MW_CONFIGS[name]
    hx = axis_steps(nx, G, q, P)
    hy = axis_steps(ny, G, q, P)
    hz = axis_steps(nz, G, q, 0, bottom_only=True).real.astype(np.complex128)
    r = _rng(cfg, 0)
    rh = 10.0 ** r.uniform(-0.5, 1.0, L)
    rv = rh * r.uniform(1.0, 3.0, L)
    Nz = 2 * nz + 1
    layer = (np.arange(Nz) * L) // Nz
    c1 = rh[layer].astype(np.complex128)
    c2 = c1.copy()
    c3 = rv[layer].astype(np.complex128)
    omega = 2.0 * rh.min() / delta ** 2
    return MWProblem(name, hx, hy, hz, c1, c2, c3, 1.0 + 0j, float(omega), nsrc, cfg)


def rhs_torch(p: MWProblem, device="cuda"):
    """The same recipe as MWProblem.rhs() drawn on the device with torch's generator (seed
    1909 * 1000 + cfg): full-size fields (3 x 257 x 513 x 513 complex128 = 3.2 GB) are not built
    in numpy.  Only the layout (interior P nodes) is used, no arithmetic of the method."""
    import torch
    nz, ny, nx = p.shape
    g = torch.Generator(device=device)
    g.manual_seed(1909 * 1000 + p.cfg)
    f = torch.randn((3, nz, ny, nx), dtype=torch.complex128, device=device, generator=g) * 1e-3
    k = torch.arange(nz, device=device)[:, None, None]
    j = torch.arange(ny, device=device)[None, :, None]
    i = torch.arange(nx, device=device)[None, None, :]
    unk = ((i + j + k) % 2 == 0) & (i > 0) & (i < nx - 1) & (j > 0) & (j < ny - 1) & (k > 0) & (k < nz - 1)
    f *= unk
    rs = _rng(p.cfg, 3)
    placed = 0
    while placed < p.nsrc:
        c = int(rs.integers(0, 3))
        kk = int(rs.integers(1, nz - 1))
        jj = int(rs.integers(max(1, ny // 4), max(2, 3 * ny // 4)))
        ii = int(rs.integers(max(1, nx // 4), max(2, 3 * nx // 4)))
        if (ii + jj + kk) % 2:
            continue
        f[c, kk, jj, ii] += complex(rs.standard_normal(), rs.standard_normal())
        placed += 1
    return f
