"""GPU parity of the Lebedev-grid Maxwell solve (lfds_mw_*, §3) against the Maxwell
oracle (oracle/maxwell.py: the curl-curl system of Eq. (abstr) assembled from Eq. (fin), sparse
LU).  The separable route is exact, so the bar is north_star's complex128 1e-9 (relative 2-norm),
with per-component / per-level max-norm checks beside it."""
import math

import numpy as np
import pytest

from oracle import maxwell as mx
from workloads.maxwell import make_mw

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _plan(p, **kw):
    from paper_1909_01299_b200 import MWPlan
    return MWPlan.from_problem(p, **kw)


def _oracle(p, f):
    g = mx.Grid(p.hx, p.hy, p.hz)
    return g, mx.solve(g, f, p.c1, p.c2, p.c3, p.mu, p.omega)


def _check(p, g, H, ref, tol=1e-9):
    e2 = np.linalg.norm(H - ref) / np.linalg.norm(ref)
    # per component and per z level, relative to that slice's own max |H|
    loc = 0.0
    for c in range(3):
        for k in range(1, g.nz - 1):
            s = np.abs(ref[c, k]).max()
            if s > 0:
                loc = max(loc, np.abs(H[c, k] - ref[c, k]).max() / s)
    print(f"{p.name}: rel2 {e2:.2e}  slice max-norm {loc:.2e}")
    assert e2 < tol and loc < 10 * tol, (e2, loc)
    off = ~np.broadcast_to(mx.unknown_mask(g), H.shape)
    assert np.abs(H[off]).max() == 0.0


@pytest.mark.parametrize("name", ["mw_tiny", "mw_u", "mw_s", "mw_s2"])
def test_maxwell_matches_oracle(name):
    p = make_mw(name)
    f = p.rhs()
    g, ref = _oracle(p, f)
    plan = _plan(p)
    H = plan.solve(torch.from_numpy(f).cuda()).cpu().numpy()
    _check(p, g, H, ref)
    assert mx.rel_residual(g, H, f, p.c1, p.c2, p.c3, p.mu, p.omega) < 1e-10


def test_maxwell_residual_kernel_matches_oracle_apply():
    """lfds_mw_residual (direct stencil) against the oracle's assembled A_h on random fields,
    including junk on the R and boundary nodes of H (which A_h must ignore)."""
    p = make_mw("mw_s2")
    g = mx.Grid(p.hx, p.hy, p.hz)
    rng = np.random.default_rng(3)
    H = rng.standard_normal((3,) + g.shape) + 1j * rng.standard_normal((3,) + g.shape)
    f = rng.standard_normal((3,) + g.shape) + 1j * rng.standard_normal((3,) + g.shape)
    m = np.broadcast_to(mx.unknown_mask(g), H.shape)
    ref = np.where(m, f - mx.apply(g, H * m, p.c1, p.c2, p.c3, p.mu, p.omega), 0)
    plan = _plan(p)
    r = plan.residual(torch.from_numpy(H).cuda(), torch.from_numpy(f).cuda()).cpu().numpy()
    assert np.abs(r - ref).max() < 1e-13 * np.abs(ref).max()


def test_maxwell_manufactured_and_repeat():
    """f = A_h H* (oracle) -> the GPU solve returns H*; a second solve through the same buffers
    with another f is not contaminated by the first (workspace reuse)."""
    p = make_mw("mw_s")
    g = mx.Grid(p.hx, p.hy, p.hz)
    plan = _plan(p)
    rng = np.random.default_rng(5)
    fd = torch.empty((3,) + g.shape, dtype=torch.complex128, device="cuda")
    Hd = torch.empty_like(fd)
    for _ in range(2):
        Hs = (rng.standard_normal((3,) + g.shape) + 1j * rng.standard_normal((3,) + g.shape)) * mx.unknown_mask(g)
        f = mx.apply(g, Hs, p.c1, p.c2, p.c3, p.mu, p.omega)
        fd.copy_(torch.from_numpy(f))
        plan.solve(fd, out=Hd)
        H = Hd.cpu().numpy()
        assert np.abs(H - Hs).max() < 1e-10 * np.abs(Hs).max()
    fd.zero_()
    assert plan.solve(fd, out=Hd).abs().max().item() == 0.0


def test_maxwell_uniform_grid_single_harmonic():
    """Uniform unit steps, one layer: the dual (Neumann) modes are psi_l(i) = cos(pi l i / (2n))
    at the odd nodes, psi_0 = const.  H = (0, psi_1(x) psi_0(y) g(z), 0) on the dd nodes is the
    harmonic (l, m) = (1, 0) of the system {H^pp_x, H^dd_y, H^dp_z}, whose H^pp_x and H^dp_z
    partners do not exist for m = 0 (reading M5): the oracle's f = A_h H must then be a y
    field on the dd nodes only, and the GPU solve must return H."""
    p = make_mw("mw_u")
    g = mx.Grid(p.hx, p.hy, p.hz)
    nz, ny, nx = g.shape
    n = (nx - 1) // 2
    x = np.arange(nx)
    H = np.zeros((3,) + g.shape, dtype=np.complex128)
    rng = np.random.default_rng(2)
    gz = rng.standard_normal(nz)
    for k in range(1, nz - 1):
        for j in range(1, ny - 1):
            for i in range(1, nx - 1):
                if (i + j + k) % 2 == 0 and i % 2 == 1 and j % 2 == 1:   # dd nodes on even levels
                    H[1, k, j, i] = math.cos(math.pi * (i // 2 + 0.5) / n) * gz[k]
    f = mx.apply(g, H, p.c1, p.c2, p.c3, p.mu, p.omega)
    P, _, _ = mx.parity_masks(nx, ny, nz)
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    dd = P & (i % 2 == 1) & (j % 2 == 1)
    assert np.abs(f[0]).max() < 1e-13 * np.abs(f).max() and np.abs(f[2]).max() < 1e-13 * np.abs(f).max()
    assert np.abs(f[1][~dd]).max() < 1e-13 * np.abs(f).max()
    Hg = _plan(p).solve(torch.from_numpy(f).cuda()).cpu().numpy()
    assert np.abs(Hg - H).max() < 1e-10 * np.abs(H).max()


def test_maxwell_resonant_elimination_is_reported():
    """c1 = i omega mu / nu_1^2 (c2 = 3 c1) makes c2 lambda_0^2 + c1 nu_1^2 - i omega mu = 0 for
    the harmonic (l, m) = (0, 1) only: setup must fail with LFDS_ERESONANCE naming it."""
    from paper_1909_01299_b200 import MWPlan, LfdsError
    p = make_mw("mw_u")
    ny = len(p.hy) + 1
    n = (ny - 1) // 2
    nu1 = math.sin(math.pi / (2 * n)) ** 2             # steps 2: (4 / 2^2) sin^2(pi m / (2n))
    c = 1j * p.omega * complex(p.mu) / nu1
    c1 = np.full(len(p.hz) + 1, c)
    with pytest.raises(LfdsError, match=r"\(0, 1\)") as ei:
        MWPlan(p.hx, p.hy, p.hz, c1, 3 * c1, p.c3, p.mu, p.omega)
    assert ei.value.code == 3


def test_maxwell_rejects_even_node_counts():
    from paper_1909_01299_b200 import MWPlan, LfdsError
    p = make_mw("mw_tiny")
    with pytest.raises(LfdsError, match="odd"):
        MWPlan(np.ones(7), p.hy, p.hz, p.c1, p.c2, p.c3, p.mu, p.omega)


@pytest.mark.parametrize("name,ix,iy", [
    ("mw_s", [8], [6]),          # 2 x 2 blocks
    ("mw_s2", [8, 16], [10]),    # 3 x 2 blocks, PML in the outer blocks
    ("mw_s", [4, 10], []),       # x-interfaces only (a 5-node block)
    ("mw_s2", [], [6, 12]),      # y-interfaces only
    ("mw_s", [], []),            # one block: step 5 has nothing to do
])
def test_two_level_maxwell_matches_oracle(name, ix, iy):
    """H = H^1 + H^2 through lfds_mw2_*: the oracle's sparse-LU solution to
    the 1e-9 bar, and the layered (single-block) GPU solve to 1e-11."""
    from paper_1909_01299_b200 import MW2Plan
    p = make_mw(name)
    f = p.rhs()
    g, ref = _oracle(p, f)
    plan = MW2Plan.from_problem(p, ix, iy)
    assert plan.n_blocks() == (len(ix) + 1) * (len(iy) + 1)
    fd = torch.from_numpy(f).cuda()
    H = plan.solve(fd).cpu().numpy()
    _check(p, g, H, ref)
    H1 = _plan(p).solve(fd).cpu().numpy()
    assert np.linalg.norm(H - H1) / np.linalg.norm(H1) < 1e-11


def test_two_level_maxwell_rejects_odd_interfaces():
    from paper_1909_01299_b200 import MW2Plan, LfdsError
    p = make_mw("mw_s")
    with pytest.raises(LfdsError, match="even"):
        MW2Plan.from_problem(p, [7], [])
