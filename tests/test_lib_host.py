"""CPU-side tests of the C-ABI library: it loads, exports every symbol include/lfds.h declares,
validates its inputs, and its host eigensolver (setup) meets the paper's
closed forms and the pencil invariants — compared with the oracle's independent LAPACK route.
No compute call is made (host-only plans, options.device = -1)."""
import ctypes
import dataclasses
import os
import re

import numpy as np
import pytest

import oracle
from oracle.eig import gen_eig
from oracle.operator import axis_pencil
from workloads import make_problem, shrunken
from workloads.configs import axis_steps

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lfds():
    import paper_1909_01299_b200.lfds as m
    return m


def test_library_exports_every_header_symbol(lfds):
    with open(os.path.join(ROOT, "include", "lfds.h")) as fh:
        hdr = fh.read()
    declared = set(re.findall(r"\b(lfds_[a-z_0-9]+)\s*\(", hdr))
    assert "lfds_solve" in declared and "lfds_setup_grid" in declared
    lib = ctypes.CDLL(lfds._LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(lfds.EXPORTED)
    assert "sm_100a" in lfds.version()


def test_library_is_built_for_sm100a(lfds):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lfds._LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def host_plan(p, **kw):
    from paper_1909_01299_b200 import Plan
    return Plan.from_problem(p, device=-1, **kw)


def test_host_only_plan_refuses_compute(lfds):
    """A host-only plan returns LFDS_ENODEVICE from the C ABI before touching any pointer."""
    plan = host_plan(shrunken("c2"))
    P = ctypes.c_void_p
    rc = lfds._lib.lfds_solve(plan._h, P(256), P(512), 1, P(1024), 4096, None)
    assert rc == 8 and b"host-only" in lfds._lib.lfds_last_error()
    assert lfds._lib.lfds_workspace_bytes(plan._h, 1) == 0


@pytest.mark.parametrize("bad", [dict(iface_x=[5, 6]), dict(iface_x=[1]), dict(iface_x=[44]),
                                 dict(iface_x=[9, 4])])
def test_setup_rejects_bad_partitions(lfds, bad):
    p = shrunken("c3")
    with pytest.raises(lfds.LfdsError) as e:
        host_plan(p.with_partition(bad.get("iface_x", []), []))
    assert e.value.code == 1


def test_setup_rejects_nonpositive_steps(lfds):
    from paper_1909_01299_b200 import Plan
    p = shrunken("c2")
    hx = p.hx.copy()
    hx[3] = -1.0
    with pytest.raises(lfds.LfdsError):
        Plan(hx, p.hy, p.hz, p.sigma_node, p.sigma_edge, p.lam, p.iface_x, p.iface_y, device=-1)
    with pytest.raises(lfds.LfdsError):
        Plan(p.hx, p.hy, p.hz, -p.sigma_node, p.sigma_edge, p.lam, p.iface_x, p.iface_y, device=-1)


def test_f64_plan_requires_real_inputs(lfds):
    from paper_1909_01299_b200 import Plan
    p = shrunken("c2")
    with pytest.raises(lfds.LfdsError):
        Plan(p.hx, p.hy, p.hz, p.sigma_node, p.sigma_edge, p.lam, p.iface_x, p.iface_y, device=-1, dtype="f64")


@pytest.mark.parametrize("n,h", [(15, 1.0), (127, 1.0), (96, 0.5)])
def test_uniform_blocks_are_exact_sine_modes(n, h):
    """Kind U (uniform real steps) uses the closed form of PAPER.md:47/:75."""
    from paper_1909_01299_b200 import Plan
    one = np.ones(3)
    plan = Plan(np.full(n + 1, h), one, one, [1.0, 1.0], [1.0, 1.0, 1.0], 0.3, device=-1)
    lam, W, kind, lo = plan.basis(0, 0)
    assert kind == 0 and lo == 1
    i = np.arange(1, n + 1)
    lam_cf = -(4.0 / h ** 2) * np.sin(np.pi * i / (2 * (n + 1))) ** 2
    np.testing.assert_allclose(lam.real, lam_cf, atol=1e-13 / h ** 2)
    for c in range(n):
        l = c + 1  # natural sine order for U blocks (the fast sine transform's order)
        w = np.sqrt(2.0 / (h * (n + 1))) * np.sin(np.pi * i * l / (n + 1))
        s = np.sign(np.dot(W[:, c].real, w))
        assert np.abs(s * W[:, c] - w).max() < 4e-14


CASES = {
    "c2_pml_quad": axis_steps(96, 0, 1.0, 16, "quad"),
    "c3_graded_pml": axis_steps(192, 24, 1.2, 8, "quad"),
    "c4_pml_const": axis_steps(960, 0, 1.0, 32, "const"),
    "c4_edge_block": axis_steps(960, 0, 1.0, 32, "const")[:128],
    "c5_jittered": make_problem("c5").hx,
    "random_real": np.random.default_rng(7).uniform(0.5, 2.0, 61),
}


@pytest.mark.parametrize("case", list(CASES))
def test_host_eigensolver_invariants_and_oracle_agreement(case):
    """A W = M W Lambda, W^T M W = I, and the spectrum agrees with the oracle's LAPACK route."""
    from paper_1909_01299_b200 import Plan
    h = CASES[case]
    one = np.ones(3)
    plan = Plan(h, one, one, [1.0, 1.0], [1.0, 1.0, 1.0], 0.3, device=-1)
    lam, W, kind, _ = plan.basis(0, 0)
    A, m = axis_pencil(h)
    res = np.abs(A @ W - (m[:, None] * W) * lam[None, :]).max() / (np.abs(A).max() * np.abs(W).max())
    bio = np.abs(W.T @ (m[:, None] * W) - np.eye(len(m))).max()
    assert res < 1e-13, res
    assert bio < 1e-9, bio
    lo, _ = gen_eig(h)
    # eigenvalues are simple here; compare as sorted sets (ordering convention R14)
    d = np.abs(np.sort_complex(lam) - np.sort_complex(lo)).max() / np.abs(lo).max()
    assert d < 1e-9, d


def test_partition_blocks_and_kinds():
    """C2: blocks 31,31,31,32 with kinds C U U C."""
    plan = host_plan(make_problem("c2"))
    info = plan.info()
    assert (info["nbx"], info["nby"], info["n_if_x"]) == (4, 4, 3)
    kinds, sizes = [], []
    for b in range(4):
        lam, W, kind, lo = plan.basis(0, b)
        kinds.append(kind)
        sizes.append(len(lam))
    assert sizes == [31, 31, 31, 32] and kinds == [2, 0, 0, 2]
    assert info["eig_max_residual"] < 1e-13 and info["eig_max_biorth"] < 1e-10


def test_single_block_global_basis_equals_block_basis():
    p = shrunken("c3").with_partition([], [])
    plan = host_plan(p)
    lam_g, W_g, _, _ = plan.basis(0, -1)
    lam_b, W_b, _, _ = plan.basis(0, 0)
    assert np.array_equal(lam_g, lam_b) and np.array_equal(W_g, W_b)


@pytest.mark.parametrize("name", ["c2", "c3", "c5"])
def test_z_modal_basis_of_the_step5_pencil(name):
    """Setup diagonalises the real step-5 z pencil T(s) = A' + s E (reading R1): A' Z = E Z Theta,
    Z^T E Z = I (long-double implicit QL with accumulated rotations), checked on the rounded basis."""
    info = host_plan(make_problem(name)).info()
    assert info["real_z"] == 1 and info["s5_modal"] == 1
    assert info["z_eig_residual"] < 1e-15 and info["z_eig_orth"] < 1e-14


def test_z_modal_form_needs_real_z_tables():
    """Complex sigma (or lambda) makes the z pencil complex symmetric: step 5 keeps the sweeps."""
    p = shrunken("c2")
    pc = dataclasses.replace(p, sigma_node=p.sigma_node * (1 + 0.1j), sigma_edge=p.sigma_edge * (1 + 0.1j))
    assert host_plan(pc).info()["s5_modal"] == 0
    assert host_plan(dataclasses.replace(p, lam=p.lam + 0.01j)).info()["s5_modal"] == 0
    assert host_plan(p, s5_modal=False).info()["s5_modal"] == 0


def test_interface_count_limits():
    """Up to 32 interfaces per axis with the z-modal step 5 (KA = 32 on the tensor pipe); more
    than 16 with complex z tables (per-mode sweeps) or s5_modal = 0 is rejected at setup."""
    from paper_1909_01299_b200.lfds import LfdsError
    p = shrunken("c3").with_partition(list(range(2, 38, 2)), [])  # 18 interfaces
    assert host_plan(p).info()["s5_modal"] == 1
    for bad in (dict(s5_modal=False),):
        with pytest.raises(LfdsError) as e:
            host_plan(p, **bad)
        assert e.value.code == 1
    pc = dataclasses.replace(p, sigma_node=p.sigma_node * (1 + 0.1j), sigma_edge=p.sigma_edge * (1 + 0.1j))
    with pytest.raises(LfdsError) as e:
        host_plan(pc)
    assert e.value.code == 1


def test_plane_transform_block_count(lfds):
    """lfds_info.n_plane_dst: the blocks whose steps 1 and 7 run as one plane sine transform —
    uniform on both axes with one length L = 2(n+1) <= 128 (C4q: the 30 x 30 core blocks of 31
    nodes; C4: its 127-node core blocks stay on the two 1-D passes; off with plane_dst=False,
    and for the real f64 path, which has no sine kernels)."""
    import bench
    from workloads import make_problem
    q = make_problem("c4q")
    pq = host_plan(q)
    assert pq.info()["n_plane_dst"] == 30 * 30
    assert host_plan(q, plane_dst=False).info()["n_plane_dst"] == 0
    assert host_plan(make_problem("c4")).info()["n_plane_dst"] == 0
    assert host_plan(shrunken("c1")).info()["n_plane_dst"] == 0
    # bench.py's byte accounting agrees with the library's rule (it raises otherwise)
    alg = bench.stage_algorithmic(q, 1, pq)
    assert alg["step1_plane_sine"][1] == 32.0 * 900 * 31 * 31 * q.nz


def test_plane_dense_block_count(lfds):
    """lfds_info.n_plane_dense: the blocks whose steps 1 and 7 run as one plane transform on DMMA
    (k_xplane) — at most 32 nodes on both axes, neither axis on the fast sine transform (C5: all
    16 x 16 blocks, 14 x 14 graded real ones and the PML ones with a complex basis on an axis; C4:
    none, its blocks have 127 nodes; C4q / C3: none, their few complex corner blocks hold less than
    half of the block unknowns; the f64 path: none).  bench.py's accounting follows the same rule (it raises when
    the counts differ)."""
    import bench
    from workloads import make_problem
    c5 = make_problem("c5")
    p5 = host_plan(c5)
    assert p5.info()["n_plane_dense"] == 16 * 16
    assert host_plan(make_problem("c4")).info()["n_plane_dense"] == 0
    for name in ("c4q", "c3"):  # a few small complex corner blocks among sine blocks: not worth the launches
        q = make_problem(name)
        pq = host_plan(q)
        assert pq.info()["n_plane_dense"] == 0
        assert bench.stage_algorithmic(q, 1, pq)["step1_plane_dense"][1] == 0
    assert host_plan(shrunken("c1")).info()["n_plane_dense"] == 0
    alg = bench.stage_algorithmic(c5, 1, p5)
    assert alg["step1_plane_dense"][1] == 32.0 * c5.unknowns - 32.0 * c5.nz * (2 * 15 * 512 - 15 * 15)
    n = [31] * 15 + [32]
    k = [2] + [1] * 14 + [2]
    fl = sum(((8.0 if k[i] == 2 else 4.0) * n[i] + (8.0 if k[j] == 2 else 4.0) * n[j]) * n[i] * n[j]
             for i in range(16) for j in range(16)) * c5.nz
    assert alg["step1_plane_dense"][0] == fl
    ka = bench.kernel_algorithmic(c5, 1, p5)
    assert ka["k_xplane"] == (2 * fl, 2 * alg["step1_plane_dense"][1])
    assert ka["k_xform"][0] == 2 * 4.0 * c5.nz * (15 * 512 * 2) * c5.nz  # only the step-5 z-transforms are left
