"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation (numpy/scipy, fp64 with an
80-bit ``clongdouble`` residual) of what the hot path computes: the solution
u = A^{-1} (M_x (x) M_y (x) M_z) f of the 7-point finite-volume system Eq. (fd)
(PAPER.md:32-35), assembled literally, solved (i) by sparse direct elimination on
tiny grids and (ii) by the global separable eigen-solve on any size.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_1909_01299_b200``) and never imports it; its only shared input
is the seeded generator package ``workloads``.

``oracle.maxwell`` is the same for the Lebedev-grid Maxwell system of PAPER.md §3 (the curl-curl
operator of Eq. (abstr) assembled from Eq. (fin), solved by sparse LU).

Parity status per function is stated in each module header (all pinned; see
DESIGN.md §4 for the pin list).
"""
from .operator import (control_volumes, axis_pencil, z_pencil, assemble, assemble_kron,  # noqa: F401
                       apply_stencil, mass_rhs, rel_residual)
from .eig import gen_eig, sine_basis  # noqa: F401
from .solve import (solve_direct, solve_separable, solve, block_solutions,  # noqa: F401
                    residual_ext, interface_mask, GlobalBases)
from .hetero import assemble_hetero, solve_hetero_direct, rel_residual_hetero  # noqa: F401
