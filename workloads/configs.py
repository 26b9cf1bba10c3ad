"""BASELINE.json configs C1..C5 (and shrunken analogs) as seeded synthetic inputs.

Recipe (restated in DESIGN.md §3):

* Axis grid (x and y): N unknown nodes = C core + 2T tail nodes, T = G graded + P PML.
  N+1 steps h_0..h_N; step h_t joins node t and t+1 (nodes 0 and N+1 are the
  Dirichlet boundary, reading R3 of DESIGN.md).  Core steps (t = T+1..T+C-1) are 1,
  or U[0.8, 1.2] for C5.  Outward tail step s = 1..T+1 (s = 1 is the real step that
  joins the core to the tail) is ``q**(s-1)`` for s <= G+1 and a PML step after that;
  the left tail puts step s at t = T+1-s, the right tail at t = T+C+s-1.
* PML profiles (the paper gives none): ``quad`` = base*(1+2i((s-G-1)/P)^2)
  with base = q**G (C2 as BASELINE.json states it; C3, C5), ``const`` = base*(1+0.5i) (C4).
* z: N_z unknowns, unit steps, Dirichlet top/bottom.  sigma: L layers over the N_z+1
  z-cells (cell c -> layer floor(c*L/(N_z+1))), values 10**U(a, b); sigma_edge[c] is
  sigma_{c+1/2}; sigma_node[k] is the control-volume average (reading R2), computed here
  because it is part of the *input* (the C-ABI takes both arrays).
* Interfaces: nodes floor(b*(N+1)/B), b = 1..B-1 (1-based, width-1 planes, reading R9).
* lambda = (2*pi/ppw)**2 (sigma_ref = 1); C1 lambda = -0.5.
* Seeds: numpy default_rng(SeedSequence([1909, 1299, cfg, stream])); streams
  0 = sigma layers, 1 = x core steps, 2 = y core steps, 3 = point sources, 4+r = RHS r.
* RHS f (the density of Eq. (fd), before the mass weight): C1 N(0,1) real; C2 a unit
  point source at (64,64,32) + 1e-3 CN(0,1); C3 CN(0,1); C4 16 point sources with
  CN(0,1) amplitudes uniform over the core (x,y) and all z + 1e-3 CN(0,1); C5 64 x CN(0,1).

Arrays: f[r] has shape (N_z, N_y, N_x) (x fastest), matching the C-ABI layout
[nrhs][nz][ny][nx].
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, List, Optional

import numpy as np

CONFIG_NAMES = ("c1", "c2", "c3", "c4", "c5", "c4j", "c4q")


def _rng(cfg: int, stream: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([1909, 1299, cfg, stream]))


def axis_steps(C: int, G: int = 0, q: float = 1.0, P: int = 0, pml: str = "none",
               core: Optional[np.ndarray] = None) -> np.ndarray:
    """Return the N+1 complex steps of one horizontal axis (see module docstring)."""
    T = G + P
    N = C + 2 * T
    h = np.ones(N + 1, dtype=np.complex128)
    if core is not None:
        assert core.shape == (C - 1,)
        h[T + 1:T + C] = core
    for s in range(1, T + 2):
        if s <= G + 1:
            val = complex(q ** (s - 1))
        else:
            base = q ** G
            if pml == "quad":
                val = base * (1.0 + 2.0j * ((s - G - 1) / P) ** 2)
            elif pml == "const":
                val = base * (1.0 + 0.5j)
            else:
                raise ValueError(pml)
        h[T + 1 - s] = val
        h[T + C + s - 1] = val
    return h


def sigma_layers(nz: int, layer_values: np.ndarray):
    """sigma_edge (nz+1 cells) and sigma_node (nz nodes, control-volume average, reading R2)."""
    L = len(layer_values)
    cells = np.arange(nz + 1)
    sigma_edge = np.asarray(layer_values, dtype=np.complex128)[(cells * L) // (nz + 1)]
    hz = np.ones(nz + 1, dtype=np.complex128)
    k = np.arange(1, nz + 1)
    sigma_node = (hz[k - 1] * sigma_edge[k - 1] + hz[k] * sigma_edge[k]) / (hz[k - 1] + hz[k])
    return hz, sigma_edge, sigma_node


def interfaces(N: int, B: int) -> List[int]:
    return [(b * (N + 1)) // B for b in range(1, B)]


@dataclasses.dataclass
class Problem:
    name: str
    hx: np.ndarray          # (Nx+1,) complex128 steps
    hy: np.ndarray          # (Ny+1,)
    hz: np.ndarray          # (Nz+1,)
    sigma_edge: np.ndarray  # (Nz+1,) sigma_{k+1/2}, k = 0..Nz
    sigma_node: np.ndarray  # (Nz,)   sigma_k, k = 1..Nz
    lam: complex
    iface_x: List[int]      # sorted 1-based interface nodes
    iface_y: List[int]
    nrhs: int
    real: bool              # C1: every input real, float64 path
    _rhs: Callable[[int], np.ndarray] = dataclasses.field(repr=False, default=None)
    description: str = ""

    @property
    def nx(self) -> int:
        return len(self.hx) - 1

    @property
    def ny(self) -> int:
        return len(self.hy) - 1

    @property
    def nz(self) -> int:
        return len(self.hz) - 1

    @property
    def shape(self):
        return (self.nz, self.ny, self.nx)

    @property
    def unknowns(self) -> int:
        return self.nx * self.ny * self.nz

    def rhs(self, r: int = 0) -> np.ndarray:
        """Right-hand side r, shape (Nz, Ny, Nx); float64 if ``real`` else complex128."""
        assert 0 <= r < self.nrhs
        return self._rhs(r)

    def rhs_all(self) -> np.ndarray:
        return np.stack([self.rhs(r) for r in range(self.nrhs)])

    def with_partition(self, iface_x, iface_y, name=None) -> "Problem":
        return dataclasses.replace(self, iface_x=list(iface_x), iface_y=list(iface_y),
                                   name=name or self.name)

    def with_lambda(self, lam) -> "Problem":
        return dataclasses.replace(self, lam=lam)


def _cn(rng, shape):
    out = np.empty(shape, dtype=np.complex128)
    v = out.view(np.float64).reshape(shape + (2,))
    rng.standard_normal(out=v)
    out *= 1.0 / math.sqrt(2.0)
    return out


def _build(cfg_id, name, *, C, G, q, P, pml, nz, layers, lrange, lam, B, nrhs,
           rhs_kind, core_jitter=False, real=False, description="", fixed_layers=None):
    if core_jitter:
        cx = _rng(cfg_id, 1).uniform(0.8, 1.2, C - 1).astype(np.complex128)
        cy = _rng(cfg_id, 2).uniform(0.8, 1.2, C - 1).astype(np.complex128)
    else:
        cx = cy = None
    hx = axis_steps(C, G, q, P, pml, cx)
    hy = axis_steps(C, G, q, P, pml, cy)
    if fixed_layers is not None:
        vals = np.asarray(fixed_layers, dtype=np.float64)
    else:
        vals = 10.0 ** _rng(cfg_id, 0).uniform(lrange[0], lrange[1], layers)
    hz, sig_e, sig_n = sigma_layers(nz, vals)
    N = len(hx) - 1
    T = G + P
    shape = (nz, N, N)

    def rhs(r):
        if rhs_kind == "real_normal":
            return _rng(cfg_id, 4 + r).standard_normal(shape)
        if rhs_kind == "cn":
            return _cn(_rng(cfg_id, 4 + r), shape)
        if rhs_kind == "point_center":
            f = 1e-3 * _cn(_rng(cfg_id, 4 + r), shape)
            # unit point source at 1-based node (N/2, N/2, nz/2)
            f[nz // 2 - 1, N // 2 - 1, N // 2 - 1] += 1.0
            return f
        if rhs_kind == "points16":
            f = 1e-3 * _cn(_rng(cfg_id, 4 + r), shape)
            g = _rng(cfg_id, 3)
            px = g.integers(T + 1, T + C + 1, 16)
            py = g.integers(T + 1, T + C + 1, 16)
            pz = g.integers(1, nz + 1, 16)
            amp = _cn(g, (16,))
            for a in range(16):
                f[pz[a] - 1, py[a] - 1, px[a] - 1] += amp[a]
            return f
        raise ValueError(rhs_kind)

    return Problem(name=name, hx=hx, hy=hy, hz=hz, sigma_edge=sig_e, sigma_node=sig_n,
                   lam=complex(lam), iface_x=interfaces(N, B), iface_y=interfaces(N, B),
                   nrhs=nrhs, real=real, _rhs=rhs, description=description)


def _lam(ppw):
    return (2.0 * math.pi / ppw) ** 2


def make_problem(name: str) -> Problem:
    """Full-size BASELINE.json configs c1..c5."""
    if name == "c1":
        return _build(1, "c1", C=24, G=0, q=1.0, P=0, pml="none", nz=16, layers=3, lrange=None,
                      fixed_layers=(1.0, 4.0, 0.25), lam=-0.5, B=2, nrhs=1, rhs_kind="real_normal",
                      real=True, description="tiny real Poisson-Helmholtz 24x24x16, 2x2 blocks")
    if name == "c2":
        return _build(2, "c2", C=96, G=0, q=1.0, P=16, pml="quad", nz=64, layers=5, lrange=(-1, 1),
                      lam=_lam(10), B=4, nrhs=1, rhs_kind="point_center",
                      description="complex PML 128x128x64, 4x4 blocks")
    if name == "c3":
        return _build(3, "c3", C=192, G=24, q=1.2, P=8, pml="quad", nz=128, layers=20, lrange=(-2, 2),
                      lam=_lam(8), B=16, nrhs=1, rhs_kind="cn",
                      description="graded geophysical grid 256x256x128, 16x16 blocks")
    if name == "c4":
        return _build(4, "c4", C=960, G=0, q=1.0, P=32, pml="const", nz=256, layers=50, lrange=(-1, 1),
                      lam=_lam(10), B=8, nrhs=1, rhs_kind="points16",
                      description="large uniform survey 1024x1024x256, 8x8 blocks")
    if name == "c5":
        return _build(5, "c5", C=448, G=24, q=1.2, P=8, pml="quad", nz=200, layers=30, lrange=(-1, 1),
                      lam=_lam(10), B=16, nrhs=64, rhs_kind="cn", core_jitter=True,
                      description="multi-RHS 512x512x200 x 64 RHS, 16x16 blocks")
    if name == "c4j":
        # C4 with the paper's partition strategy for grids with a uniform survey core (PAPER.md:75,
        # "three subgrids": thin non-uniform / PML tails, uniform core computed by FFT), kept at
        # BASELINE.json's 8 x 8 block count: interfaces at the last left-PML node and the last core
        # node, six uniform core blocks of 159 nodes (sine transforms of length 320) between
        j = [32, 192, 352, 512, 672, 832, 992]
        return make_problem("c4").with_partition(j, j, name="c4j")
    if name == "c4q":
        # C4 with the sqrt(N)-block partition (SPEC S:68-85's second cost regime): 32 x 32 blocks of
        # 31 nodes, interfaces at multiples of 32 (the first and last blocks are the PML tails)
        j = [32 * b for b in range(1, 32)]
        return make_problem("c4").with_partition(j, j, name="c4q")
    raise KeyError(name)


def shrunken(name: str, nrhs: Optional[int] = None) -> Problem:
    """Small analogs with the same step/PML/grading/sigma structure (oracle (i) feasible)."""
    if name == "c1":
        return make_problem("c1")
    if name == "c2":
        return _build(102, "c2s", C=24, G=0, q=1.0, P=8, pml="quad", nz=8, layers=5, lrange=(-1, 1),
                      lam=_lam(10), B=4, nrhs=nrhs or 1, rhs_kind="point_center")
    if name == "c3":
        return _build(103, "c3s", C=24, G=6, q=1.2, P=4, pml="quad", nz=10, layers=6, lrange=(-2, 2),
                      lam=_lam(8), B=5, nrhs=nrhs or 1, rhs_kind="cn")
    if name == "c4":
        return _build(104, "c4s", C=30, G=0, q=1.0, P=8, pml="const", nz=12, layers=5, lrange=(-1, 1),
                      lam=_lam(10), B=4, nrhs=nrhs or 1, rhs_kind="points16")
    if name == "c4j":  # tails 7 / 8 PML nodes, two uniform core blocks of 15 (L = 32)
        j = [8, 24, 40]
        return _build(106, "c4js", C=32, G=0, q=1.0, P=8, pml="const", nz=12, layers=5, lrange=(-1, 1),
                      lam=_lam(10), B=4, nrhs=nrhs or 1, rhs_kind="points16").with_partition(j, j, name="c4js")
    if name == "c5":
        return _build(105, "c5s", C=20, G=6, q=1.2, P=4, pml="quad", nz=9, layers=5, lrange=(-1, 1),
                      lam=_lam(10), B=5, nrhs=nrhs or 3, rhs_kind="cn", core_jitter=True)
    raise KeyError(name)


def anomaly(p: Problem, eps: float = -0.1, box=((0.375, 0.625), (0.375, 0.625), (0.375, 0.625))) -> np.ndarray:
    """Node-wise shift perturbation dlam of an embedded inhomogeneity: a box of
    velocity c_bg (1 + eps) in the layered background, so lambda = omega^2 / c^2 becomes
    lambda (1 + eps)^-2 inside.  ``box`` holds (lo, hi) fractions of the unknown nodes along
    (z, y, x).  Returns dlam with the field layout (N_z, N_y, N_x), complex128."""
    dl = np.zeros(p.shape, dtype=np.complex128)
    sl = tuple(slice(int(lo * n), max(int(lo * n) + 1, int(hi * n))) for (lo, hi), n in zip(box, p.shape))
    dl[sl] = complex(p.lam) * ((1.0 + eps) ** -2 - 1.0)
    return dl
