"""CPU checks of bench.py's accounting (no GPU): the algorithmic work per stage and the roofline
arithmetic that the JSON line reports."""
import bench
from workloads import make_problem


def test_stage_algorithmic_c4_matches_the_survey_totals():
    """C4 grid: dense-transform flops (8 per complex MAC) and z-solve bytes (32 per unknown) per
    stage, from the block sizes."""
    p = make_problem("c4")
    alg = bench.stage_algorithmic(p, 1, None)  # plan=None: every block counted as complex dense
    # with plan=None all 64 blocks are dense in both directions (block sizes 7 x 127 and 128):
    # per direction sum_ij n_i n_j nz x 8 n_dir flops
    b = [127] * 7 + [128]
    per_dir = sum(bi * bj * 256 * 8 * bi for bi in b for bj in b)
    dense = sum(alg[k][0] for k in ("step1_x_dense", "step1_y_dense", "step7_y_dense", "step7_x_dense"))
    assert abs(dense - 4 * per_dir) < 1e-9 * dense
    assert alg["step2_zsolve"] == (None, 32.0 * sum(bi * bj for bi in b for bj in b) * 256)


def test_roofline_counts_passes_per_step():
    p = make_problem("c2")
    stages = {"step2_zsolve": (2.0, 2), "step6_zsolve_lift": (4.0, 2), "refine_residual": (1.0, 1)}
    r1 = bench.roofline_summary(p, 1, None, stages, 1, "c2", 10.0, passes=1)
    r2 = bench.roofline_summary(p, 1, None, stages, 1, "c2", 10.0, passes=2)
    assert r1["kernel"] == r2["kernel"] == "step6_zsolve_lift"
    assert abs(r2["achieved"] - 2 * r1["achieved"]) < 1e-9 * r1["achieved"]
    assert abs(r2["solve"]["t_roof_ms"] - 2 * r1["solve"]["t_roof_ms"]) < 1e-12
    assert r1["unit"] == "GB/s" and r1["bound"] == "hbm" and 0 < r1["frac"] == r1["achieved"] / r1["peak"]


def test_refinement_stage_counted_once_per_refinement():
    p = make_problem("c2")
    stages = {"refine_residual": (5.0, 1), "step2_zsolve": (1.0, 2)}
    r = bench.roofline_summary(p, 1, None, stages, 1, "c2", 10.0, passes=2)
    alg = bench.stage_algorithmic(p, 1, None)
    assert r["kernel"] == "refine_residual"
    assert abs(r["achieved"] - alg["refine_residual"][1] / 5e-3 / 1e9) < 1e-6 * r["achieved"]


class _KindsPlan:
    """Stand-in for a Plan: every block uniform (kind 0) except the first and last (PML, kind 2)."""

    def __init__(self, nblocks, plane_dst):
        self.nb, self.plane_dst = nblocks, plane_dst

    def basis(self, axis, b):
        return None, None, 2 if b in (0, self.nb - 1) else 0

    def info(self):
        return {"s5_modal": 1}


def test_plane_sine_bytes_replace_the_two_passes():
    """C4q (31-node blocks, L = 64): with plane_dst the uniform x uniform blocks move 32 B per
    element once (step1_plane_sine) instead of in the x pass and again in the y pass; the sine
    passes keep only the blocks uniform along one axis.  Total sine bytes drop by exactly the
    fused volume."""
    p = make_problem("c4q")
    nb = len(p.iface_x) + 1
    on = bench.stage_algorithmic(p, 1, _KindsPlan(nb, True))
    off = bench.stage_algorithmic(p, 1, _KindsPlan(nb, False))
    cuts = [0] + list(p.iface_x) + [p.nx + 1]
    n = [cuts[i + 1] - cuts[i] - 1 for i in range(nb)]
    fused = sum(n[i] * n[j] * p.nz for i in range(1, nb - 1) for j in range(1, nb - 1))
    assert on["step1_plane_sine"][1] == on["step7_plane_sine"][1] == 32.0 * fused
    assert off["step1_plane_sine"][1] == 0
    for st in ("step1_x_sine", "step1_y_sine", "step7_x_sine", "step7_y_sine"):
        assert off[st][1] - on[st][1] == 32.0 * fused
    # dense passes are untouched
    assert on["step1_x_dense"] == off["step1_x_dense"]


def test_kernel_roofline_names_the_kernel_with_the_largest_time():
    """The top-level roofline reports the kernel KIND with the largest summed device time (all
    its launches across stages), not the largest stage; its share and frac come from the table."""
    p = make_problem("c4")
    plan = _KindsPlan(len(p.iface_x) + 1, True)
    stages = {"step6_zsolve_lift": (2.5, 1), "step1_x_dense": (2.0, 1), "step7_x_dense": (2.0, 1)}
    kernels = {"k_zs2": (2.5, 1), "k_xform3m": (10.5, 20), "k_zs1": (2.3, 1)}
    r = bench.roofline_summary(p, 1, plan, stages, 1, "c4", 25.0, passes=1, kernels=kernels, fp64_peak=37.0)
    assert r["kernel"] == "k_xform3m" and r["bound"] == "tensor" and r["unit"] == "TFLOP/s"
    alg = bench.kernel_algorithmic(p, 1, plan)
    assert abs(r["achieved"] - alg["k_xform3m"][0] / 10.5e-3 / 1e12) < 1e-9 * r["achieved"]
    assert abs(r["share"] - 10.5 / 15.3) < 1e-12
    assert r["kernels"]["k_zs2"]["bound"] == "hbm"


def test_kernel_algorithmic_dense_flops_c4():
    """C4 with its PML blocks first and last on each axis (kind 2) and uniform (sine) blocks in
    between: the complex dense passes are exactly the blocks whose x or y block is a PML block,
    8 n flops per element and direction, forward and inverse."""
    p = make_problem("c4")
    nb = len(p.iface_x) + 1
    alg = bench.kernel_algorithmic(p, 1, _KindsPlan(nb, True))
    cuts = [0] + list(p.iface_x) + [p.nx + 1]
    n = [cuts[i + 1] - cuts[i] - 1 for i in range(nb)]
    pml = {0, nb - 1}
    dense = sum(2 * 8.0 * n[i] * n[i] * n[j] * p.nz + 2 * 8.0 * n[j] * n[i] * n[j] * p.nz * 0
                for i in pml for j in range(nb))  # x passes of blocks in a PML column
    dense += sum(2 * 8.0 * n[j] * n[i] * n[j] * p.nz for i in range(nb) for j in pml)  # y passes
    nif = len(p.iface_x)
    plane = 2 * 8.0 * 2 * nif * p.nx * p.nx * p.nz
    edges = sum(8.0 * (n[i] ** 2 + n[j] ** 2) * 2 * p.nz for i in range(nb) for j in range(nb))
    faces = sum(8.0 * (((i > 0) + (i < nb - 1)) * n[j] ** 2 + ((j > 0) + (j < nb - 1)) * n[i] ** 2) * p.nz
                for i in range(nb) for j in range(nb))
    assert abs(alg["k_xform3m"][0] - (dense + plane + edges + faces)) < 1e-9 * alg["k_xform3m"][0]
