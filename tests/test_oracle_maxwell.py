"""Pins of the Maxwell oracle (oracle/maxwell.py) against what PAPER.md §3 and the mathematics
fix — not against itself (no formula is retyped here; each check fails a plausible mistake:
a transposed curl block, a sign, a wrong z level for rho, a missing boundary projection)."""
import numpy as np
import pytest

from oracle import maxwell as mx
from workloads.maxwell import make_mw, axis_steps


def _grid(n=(4, 3, 3), complex_steps=True, seed=0):
    rng = np.random.default_rng(seed)
    hs = []
    for m in n:
        h = rng.uniform(0.7, 1.4, 2 * m).astype(np.complex128)
        if complex_steps:
            h[0] *= 1 + 0.7j
            h[-1] *= 1 + 1.1j
        hs.append(h)
    return mx.Grid(*hs)


def test_parity_rule_examples():
    """P = even i + j + k (SPEC [OP] build_lebedev examples)."""
    P, R, _ = mx.parity_masks(7, 5, 9)
    assert P[5, 3, 2] and R[1, 1, 1]
    assert P.sum() + R.sum() == 7 * 5 * 9 and not (P & R).any()


@pytest.mark.parametrize("field,expect", [
    ((0, 0, "x"), (0, -1, 0)),   # curl (0, 0, x) = (d_y x, -d_x x, 0)
    ((0, "x", 0), (0, 0, 1)),
    (("y", 0, 0), (0, 0, -1)),
    ((0, "z", 0), (-1, 0, 0)),
    (("z", 0, 0), (0, 1, 0)),
])
def test_curl_of_linear_fields_is_exact(field, expect):
    """Eq. (fin) is exact on linear functions of the stretched coordinates, so curl_h of a
    linear field equals the continuous curl at every interior node (graded complex steps)."""
    g = _grid()
    x, y, z = (mx.nodes(h) for h in (g.hx, g.hy, g.hz))
    coord = {"x": np.broadcast_to(x[None, None, :], g.shape), "y": np.broadcast_to(y[None, :, None], g.shape),
             "z": np.broadcast_to(z[:, None, None], g.shape)}
    H = np.stack([coord[c] if isinstance(c, str) else np.zeros(g.shape) for c in field]).astype(np.complex128)
    cH = (g.curl() @ H.ravel()).reshape((3,) + g.shape)
    for c in range(3):
        assert np.allclose(cH[c][g.inner], expect[c], atol=1e-13)


def test_curl_of_gradient_vanishes():
    """D_a D_b = D_b D_a (tensor-product differences): curl_h grad_h phi = 0 at interior nodes."""
    g = _grid(seed=1)
    rng = np.random.default_rng(5)
    phi = (rng.standard_normal(g.shape) + 1j * rng.standard_normal(g.shape)) * g.R
    phi[[0, -1], :, :] = 0; phi[:, [0, -1], :] = 0; phi[:, :, [0, -1]] = 0
    p = phi.ravel()
    grad = np.concatenate([g.Dx @ p, g.Dy @ p, g.Dz @ p])
    cg = (g.curl() @ grad).reshape((3,) + g.shape)
    # interior nodes at distance >= 2 from the boundary see only computed differences
    sl = (slice(None), slice(2, -2), slice(2, -2), slice(2, -2))
    assert np.abs(cg[sl]).max() < 1e-12 * np.abs(grad).max()


def test_curl_maps_P_fields_to_R_nodes():
    """Eq. (fin) maps the P-grid to the R-grid and vice versa."""
    g = _grid(seed=2)
    rng = np.random.default_rng(3)
    H = rng.standard_normal((3,) + g.shape) * g.P
    cH = (g.curl() @ H.ravel()).reshape((3,) + g.shape)
    assert np.abs(cH[:, g.P]).max() == 0.0
    E = rng.standard_normal((3,) + g.shape) * g.R
    cE = (g.curl() @ E.ravel()).reshape((3,) + g.shape)
    assert np.abs(cE[:, g.R]).max() == 0.0


def _medium(nz, seed=4):
    rng = np.random.default_rng(seed)
    c = [rng.uniform(0.5, 3.0, nz) * (1 + 0.2j * rng.standard_normal(nz)) for _ in range(3)]
    return c


def test_weighted_symmetry_of_the_curl_curl_operator():
    """The (fin) pair is skew-adjoint under W = d_x d_y d_z (summation by parts with the
    boundary values removed by the two projections), so W A_h is (complex) symmetric for any
    steps and any diagonal rho — a transposed or mis-signed curl block breaks it."""
    g = _grid(seed=6)
    c1, c2, c3 = _medium(g.nz)
    A = mx.operator(g, c1, c2, c3, 1.0, 0.37)
    W = np.tile(g.weights(), 3)
    S = (A.multiply(W[:, None])).tocsr()
    d = abs(S - S.T).max()
    assert d < 1e-13 * abs(S).max(), d


def test_curl_free_fields_see_only_the_omega_term():
    """A_h grad_h phi = -i omega mu grad_h phi (SPEC [OP] apply_curl_curl omega-term check)."""
    g = _grid(seed=7)
    c1, c2, c3 = _medium(g.nz, seed=8)
    rng = np.random.default_rng(9)
    phi = (rng.standard_normal(g.shape) + 1j * rng.standard_normal(g.shape)) * g.R
    for ax in range(3):  # support two nodes away from the boundary: grad phi = 0 on dOmega
        idx = [slice(None)] * 3
        for e in (0, 1, -1, -2):
            idx[ax] = e
            phi[tuple(idx)] = 0
    p = phi.ravel()
    H = np.concatenate([g.Dx @ p, g.Dy @ p, g.Dz @ p]).reshape((3,) + g.shape) * g.P
    omega, mu = 0.61, 1.3
    AH = mx.apply(g, H, c1, c2, c3, mu, omega)
    m = np.broadcast_to(mx.unknown_mask(g), AH.shape)
    assert np.abs(AH[m] - (-1j * omega * mu) * H[m]).max() < 1e-12 * np.abs(H).max()


def test_hand_evaluated_entries_uniform_grid():
    """Unit steps (d = 2), layered rho: for H_x at an interior P node (i, j, k) whose
    neighbours are interior, (curl rho curl H)_x = d_y(c3 (d_x H_y - d_y H_x)) - d_z(c2 (d_z H_x
    - d_x H_z)) gives, by hand, the diagonal c3(k)/2 + (c2(k-1) + c2(k+1))/4 - i omega mu and
    the H_y coupling to node (i+1, j+1, k) of c3(k)/4, the H_z one to (i+1, j, k+1) of
    c2(k+1)/4 (E_z at level k, E_y at levels k +- 1)."""
    n = 7
    g = mx.Grid(*(np.ones(n - 1) for _ in range(3)))
    c1 = np.array([1, 1.5, 2, 2.5, 3, 3.5, 4.0])
    c2 = np.array([5, 6, 7, 8, 9, 10, 11.0])
    c3 = np.array([0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7])
    omega, mu = 0.5, 1.0
    A = mx.operator(g, c1, c2, c3, mu, omega)
    N = n ** 3
    i, j, k = 3, 3, 2
    p = (k * n + j) * n + i
    q = (k * n + j + 1) * n + i + 1
    assert abs(A[p, p] - (c3[k] / 2 + (c2[k - 1] + c2[k + 1]) / 4 - 1j * omega * mu)) < 1e-14
    assert abs(A[p, N + q] - c3[k] / 4) < 1e-14
    # the H_z coupling to (i+1, j, k+1): -d_z(c2 (-d_x H_z)) -> +c2(k+1)/4
    r = ((k + 1) * n + j) * n + i + 1
    assert abs(A[p, 2 * N + r] - c2[k + 1] / 4) < 1e-14


@pytest.mark.parametrize("name", ["mw_tiny", "mw_s"])
def test_manufactured_round_trip(name):
    """f = A_h H* for a random H* on the unknowns; the LU solve returns H*."""
    p = make_mw(name)
    g = mx.Grid(p.hx, p.hy, p.hz)
    rng = np.random.default_rng(11)
    H = (rng.standard_normal((3,) + g.shape) + 1j * rng.standard_normal((3,) + g.shape)) * mx.unknown_mask(g)
    f = mx.apply(g, H, p.c1, p.c2, p.c3, p.mu, p.omega)
    Hs = mx.solve(g, f, p.c1, p.c2, p.c3, p.mu, p.omega)
    assert np.abs(Hs - H).max() < 1e-10 * np.abs(H).max()
    assert mx.rel_residual(g, Hs, f, p.c1, p.c2, p.c3, p.mu, p.omega) < 1e-12


def test_workload_axis_steps_shape():
    h = axis_steps(5, 1, 1.3, 2)
    assert len(h) == 10 and np.allclose(h[:3], h[-3:][::-1]) and (h[3:7] == 1).all()
