"""Thin ctypes binding of the C ABI in include/lfds.h (argument marshalling only).

Every step of the solve runs in the sm_100a kernels of ``_lib/liblfds.so``; PyTorch only
provides device memory (tensors, the workspace) and the CUDA stream.  There is no
fallback: if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "liblfds.so")

if not os.path.exists(_LIB_PATH):
    raise ImportError(f"liblfds.so not built ({_LIB_PATH}); run __graft_entry__.build() "
                      "or python paper_1909_01299_b200/build.py")
_lib = ctypes.CDLL(_LIB_PATH)

LFDS_C128, LFDS_F64 = 0, 1
STATUS = {0: "OK", 1: "EINVAL", 2: "EEIG", 3: "ERESONANCE", 4: "ENOMEM", 5: "ECUDA", 6: "ENCCL",
          7: "ENOTCONVERGED", 8: "ENODEVICE"}


class LfdsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"lfds {STATUS.get(code, code)}: {msg}")
        self.code = code


class _Z(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class Options(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int), ("refine", ctypes.c_int), ("refine_tol", ctypes.c_double),
                ("residual_dd", ctypes.c_int), ("device", ctypes.c_int), ("rhs_chunk", ctypes.c_int),
                ("profile", ctypes.c_int), ("s5_modal", ctypes.c_int), ("graph", ctypes.c_int),
                ("plane_dst", ctypes.c_int), ("resonance_tol", ctypes.c_double),
                ("zs_warp", ctypes.c_int), ("dst_tma", ctypes.c_int)]


class Report(ctypes.Structure):
    _fields_ = [("passes", ctypes.c_int), ("rel_residual", ctypes.c_double * 9),
                ("min_pivot_ratio", ctypes.c_double), ("n_kernel_launches", ctypes.c_int)]


class KrylovReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("cycles", ctypes.c_int), ("rel_residual", ctypes.c_double)]


class Info(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int), ("nbx", ctypes.c_int),
                ("nby", ctypes.c_int), ("n_if_x", ctypes.c_int), ("n_if_y", ctypes.c_int), ("real_z", ctypes.c_int),
                ("setup_seconds", ctypes.c_double), ("eig_max_residual", ctypes.c_double),
                ("eig_max_biorth", ctypes.c_double), ("device_table_bytes", ctypes.c_size_t),
                ("s5_modal", ctypes.c_int), ("z_eig_residual", ctypes.c_double), ("z_eig_orth", ctypes.c_double),
                ("n_plane_dst", ctypes.c_int),
                ("margin_global", ctypes.c_double), ("margin_global_rel", ctypes.c_double),
                ("margin_global_lmt", ctypes.c_int * 3),
                ("margin_block", ctypes.c_double), ("margin_block_rel", ctypes.c_double),
                ("margin_block_ij", ctypes.c_int * 2), ("margin_block_lmt", ctypes.c_int * 3),
                ("global_fold", ctypes.c_int), ("n_plane_dense", ctypes.c_int)]


_P = ctypes.c_void_p
_lib.lfds_default_options.argtypes = [ctypes.POINTER(Options)]
_lib.lfds_setup_grid.argtypes = [ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int, _P, _P, _P, _Z,
                                 ctypes.c_int, _P, ctypes.c_int, _P, ctypes.POINTER(Options), ctypes.POINTER(_P)]
_lib.lfds_workspace_bytes.argtypes = [_P, ctypes.c_int]
_lib.lfds_workspace_bytes.restype = ctypes.c_size_t
_lib.lfds_workspace_bytes_host.argtypes = [_P, ctypes.c_int]
_lib.lfds_workspace_bytes_host.restype = ctypes.c_size_t
_lib.lfds_solve.argtypes = [_P, _P, _P, ctypes.c_int, _P, ctypes.c_size_t, _P]
_lib.lfds_solve_host.argtypes = [_P, _P, _P, ctypes.c_int, _P, ctypes.c_size_t, _P]
_lib.lfds_solve_host_async.argtypes = [_P, _P, _P, ctypes.c_int, _P, ctypes.c_size_t, _P]
_lib.lfds_residual.argtypes = [_P, _P, _P, _P, ctypes.c_int, ctypes.c_int, _P, _P]
_lib.lfds_residual_f.argtypes = [_P, _P, _P, _P, ctypes.c_int, ctypes.c_int, _P]
_lib.lfds_axpy.argtypes = [_P, _P, _P, ctypes.c_int, _P]
_lib.lfds_get_report.argtypes = [_P, ctypes.POINTER(Report)]
_lib.lfds_get_info.argtypes = [_P, ctypes.POINTER(Info)]
_lib.lfds_get_basis.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), _P, _P]
_lib.lfds_set_partition.argtypes = [_P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int]
_lib.lfds_exchange_layout.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t),
                                      ctypes.POINTER(ctypes.c_size_t)]
_lib.lfds_solve_phase.argtypes = [_P, ctypes.c_int, _P, _P, ctypes.c_int, _P, ctypes.c_size_t, _P]
_lib.lfds_set_mode_rows.argtypes = [_P, ctypes.c_int, ctypes.c_int]
_lib.lfds_set_formation_rows.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
_lib.lfds_gmres_workspace_bytes.argtypes = [_P, ctypes.c_int]
_lib.lfds_gmres_workspace_bytes.restype = ctypes.c_size_t
_lib.lfds_gmres.argtypes = [_P, _P, _P, _P, ctypes.c_double, ctypes.c_int, ctypes.c_int, _P, ctypes.c_size_t, _P,
                            ctypes.POINTER(KrylovReport)]
_lib.lfds_destroy.argtypes = [_P]
_lib.lfds_stage_count.restype = ctypes.c_int
_lib.lfds_stage_name.argtypes = [ctypes.c_int]
_lib.lfds_stage_name.restype = ctypes.c_char_p
_lib.lfds_stage_times.argtypes = [_P, _P, _P]
_lib.lfds_kernel_count.restype = ctypes.c_int
_lib.lfds_kernel_name.argtypes = [ctypes.c_int]
_lib.lfds_kernel_name.restype = ctypes.c_char_p
_lib.lfds_kernel_times.argtypes = [_P, _P, _P]
_lib.lfds_set_profile.argtypes = [_P, ctypes.c_int]
_lib.lfds_fp64_peak.argtypes = [_P, ctypes.POINTER(ctypes.c_double)]
_lib.lfds_nccl_unique_id.argtypes = [_P]
_lib.lfds_set_comm.argtypes = [_P, _P, ctypes.c_int, ctypes.c_int]
_lib.lfds_set_comm_groups.argtypes = [_P, ctypes.c_int, ctypes.c_int]
_lib.lfds_last_error.restype = ctypes.c_char_p
_lib.lfds_version.restype = ctypes.c_char_p
_lib.lfds_ml_setup.argtypes = [ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int, _P, _P, _P, _Z,
                               ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int, _P, _P, _P]
_lib.lfds_ml_workspace_bytes.argtypes = [_P]
_lib.lfds_ml_workspace_bytes.restype = ctypes.c_size_t
_lib.lfds_ml_solve.argtypes = [_P, _P, _P, _P, ctypes.c_size_t, _P]
_lib.lfds_ml_get_plans.argtypes = [_P, ctypes.POINTER(ctypes.c_int)]
_lib.lfds_ml_destroy.argtypes = [_P]
_lib.lfds_ml_last_error.restype = ctypes.c_char_p
_lib.lfds_mw_setup.argtypes = [ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int, _P, _P, _P, _P, _Z, ctypes.c_double,
                               ctypes.c_int, ctypes.c_int, _P]
_lib.lfds_mw_workspace_bytes.argtypes = [_P]
_lib.lfds_mw_workspace_bytes.restype = ctypes.c_size_t
_lib.lfds_mw_solve.argtypes = [_P, _P, _P, _P, ctypes.c_size_t, _P]
_lib.lfds_mw_residual.argtypes = [_P, _P, _P, _P, _P, ctypes.c_size_t, _P]
_lib.lfds_mw_kernel_name.argtypes = [ctypes.c_int]
_lib.lfds_mw_kernel_name.restype = ctypes.c_char_p
_lib.lfds_mw_kernel_times.argtypes = [_P, _P, _P]
_lib.lfds_mw_destroy.argtypes = [_P]
_lib.lfds_mw_last_error.restype = ctypes.c_char_p
_lib.lfds_mw2_setup.argtypes = [ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int, _P, _P, _P, _P, _Z, ctypes.c_double,
                                ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int, _P]
_lib.lfds_mw2_workspace_bytes.argtypes = [_P]
_lib.lfds_mw2_workspace_bytes.restype = ctypes.c_size_t
_lib.lfds_mw2_solve.argtypes = [_P, _P, _P, _P, ctypes.c_size_t, _P]
_lib.lfds_mw2_blocks.argtypes = [_P, ctypes.POINTER(ctypes.c_int)]
_lib.lfds_mw2_destroy.argtypes = [_P]

EXPORTED = ["lfds_default_options", "lfds_setup_grid", "lfds_workspace_bytes", "lfds_solve",
            "lfds_workspace_bytes_host", "lfds_solve_host", "lfds_solve_host_async", "lfds_residual", "lfds_residual_f",
            "lfds_axpy", "lfds_get_report",
            "lfds_get_info", "lfds_get_basis", "lfds_destroy", "lfds_last_error", "lfds_version",
            "lfds_stage_count", "lfds_stage_name", "lfds_stage_times", "lfds_set_partition",
            "lfds_exchange_layout", "lfds_solve_phase", "lfds_gmres_workspace_bytes", "lfds_gmres",
            "lfds_set_mode_rows", "lfds_kernel_count", "lfds_kernel_name", "lfds_kernel_times",
            "lfds_fp64_peak", "lfds_nccl_unique_id", "lfds_set_comm", "lfds_set_formation_rows",
            "lfds_set_comm_groups", "lfds_set_profile", "lfds_ml_setup", "lfds_ml_workspace_bytes",
            "lfds_ml_solve", "lfds_ml_get_plans", "lfds_ml_destroy", "lfds_ml_last_error",
            "lfds_mw_setup", "lfds_mw_workspace_bytes", "lfds_mw_solve", "lfds_mw_residual",
            "lfds_mw_kernel_count", "lfds_mw_kernel_name", "lfds_mw_kernel_times", "lfds_mw_destroy",
            "lfds_mw_last_error", "lfds_mw2_setup", "lfds_mw2_workspace_bytes", "lfds_mw2_solve",
            "lfds_mw2_blocks", "lfds_mw2_destroy"]


def _check(rc):
    if rc != 0:
        raise LfdsError(rc, _lib.lfds_last_error().decode())


def _zarr(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    return a, a.ctypes.data_as(_P)


def version() -> str:
    return _lib.lfds_version().decode()


class Plan:
    """A setup_grid plan (per-grid tables resident on the device)."""

    def __init__(self, hx, hy, hz, sigma_node, sigma_edge, lam, iface_x: Sequence[int] = (),
                 iface_y: Sequence[int] = (), *, dtype: str = "c128", refine: int = 0,
                 refine_tol: float = 1e-13, residual_dd: bool = True, device: int = 0, rhs_chunk: int = 0,
                 profile: int = 0, s5_modal: bool = True, graph: bool = False,
                 plane_dst: bool = True, resonance_tol: float = 1e-13, zs_warp: bool = False,
                 dst_tma: bool = True):
        opt = Options()
        _lib.lfds_default_options(ctypes.byref(opt))
        opt.dtype = LFDS_F64 if dtype in ("f64", "float64") else LFDS_C128
        opt.refine, opt.refine_tol, opt.residual_dd = int(refine), float(refine_tol), int(bool(residual_dd))
        opt.device, opt.rhs_chunk, opt.profile = int(device), int(rhs_chunk), int(profile)
        opt.s5_modal = int(bool(s5_modal))
        opt.graph = int(bool(graph))
        opt.plane_dst = int(bool(plane_dst))
        opt.resonance_tol = float(resonance_tol)
        opt.zs_warp = int(bool(zs_warp))
        opt.dst_tma = int(bool(dst_tma))
        self.plane_dst = bool(plane_dst)
        self.device = int(device)
        self.has_comm = False
        self.formation = False
        self.dtype = opt.dtype
        hx_, px = _zarr(hx); hy_, py = _zarr(hy); hz_, pz = _zarr(hz)
        sn_, psn = _zarr(sigma_node); se_, pse = _zarr(sigma_edge)
        ix = np.ascontiguousarray(np.asarray(list(iface_x), dtype=np.int32))
        iy = np.ascontiguousarray(np.asarray(list(iface_y), dtype=np.int32))
        lam = complex(lam)
        h = _P()
        _check(_lib.lfds_setup_grid(len(hx_) - 1, px, len(hy_) - 1, py, len(hz_) - 1, pz, psn, pse,
                                    _Z(lam.real, lam.imag), len(ix), ix.ctypes.data_as(_P), len(iy),
                                    iy.ctypes.data_as(_P), ctypes.byref(opt), ctypes.byref(h)))
        self._h = h
        self.shape = (len(hz_) - 1, len(hy_) - 1, len(hx_) - 1)
        self._ws = {}

    @classmethod
    def from_problem(cls, p, **kw):
        """Plan for a workloads.Problem (seeded synthetic config)."""
        if p.real and "dtype" not in kw:
            kw["dtype"] = "f64"
        return cls(p.hx, p.hy, p.hz, p.sigma_node, p.sigma_edge, p.lam, p.iface_x, p.iface_y, **kw)

    # ------------------------------------------------------------------ queries
    def workspace_bytes(self, nrhs: int = 1) -> int:
        return int(_lib.lfds_workspace_bytes(self._h, nrhs))

    def workspace_bytes_host(self, nrhs: int = 1) -> int:
        return int(_lib.lfds_workspace_bytes_host(self._h, nrhs))

    def info(self) -> dict:
        i = Info()
        _check(_lib.lfds_get_info(self._h, ctypes.byref(i)))
        out = {}
        for k, _ in Info._fields_:
            v = getattr(i, k)
            out[k] = list(v) if isinstance(v, ctypes.Array) else v
        return out

    def report(self, check: bool = False) -> dict:
        """Last solve's report (waits for its pivot-monitor copy).  check=True raises LfdsError
        (ERESONANCE) when the monitor saw a pivot below 1e-14 of its row norm."""
        r = Report()
        rc = _lib.lfds_get_report(self._h, ctypes.byref(r))
        if rc != 3 or check:
            _check(rc)
        return {"passes": r.passes, "rel_residual": list(r.rel_residual)[:max(r.passes, 1)],
                "min_pivot_ratio": r.min_pivot_ratio, "n_kernel_launches": r.n_kernel_launches}

    def basis(self, axis: int, block: int = -1):
        """(lam, W, kind, lo) of a block (or the global, block=-1) basis: A W = M W diag(lam)."""
        n, kind, lo = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(_lib.lfds_get_basis(self._h, axis, block, ctypes.byref(n), ctypes.byref(kind), ctypes.byref(lo),
                                   None, None))
        lam = np.empty(n.value, np.complex128)
        W = np.empty((n.value, n.value), np.complex128)
        _check(_lib.lfds_get_basis(self._h, axis, block, None, None, None, lam.ctypes.data_as(_P),
                                   W.ctypes.data_as(_P)))
        return lam, W, kind.value, lo.value

    def stage_times(self) -> dict:
        """{stage: (device ms, launches)} accumulated since the last call (profile=True plans)."""
        n = _lib.lfds_stage_count()
        ms = np.zeros(n, np.float64)
        la = np.zeros(n, np.int32)
        _check(_lib.lfds_stage_times(self._h, ms.ctypes.data_as(_P), la.ctypes.data_as(_P)))
        return {_lib.lfds_stage_name(i).decode(): (float(ms[i]), int(la[i])) for i in range(n)}

    def set_profile(self, level: int):
        """0 none, 1 stage events, 2 stage + per-kernel-kind events (for later solves)."""
        _check(_lib.lfds_set_profile(self._h, int(level)))

    def kernel_times(self) -> dict:
        """{kernel kind: (device ms, launches)} accumulated since the last call (profile=True)."""
        n = _lib.lfds_kernel_count()
        ms = np.zeros(n, np.float64)
        la = np.zeros(n, np.int32)
        _check(_lib.lfds_kernel_times(self._h, ms.ctypes.data_as(_P), la.ctypes.data_as(_P)))
        return {_lib.lfds_kernel_name(i).decode(): (float(ms[i]), int(la[i])) for i in range(n)}

    # ------------------------------------------------------------------ compute
    def _torch(self):
        import torch
        return torch

    def workspace(self, nrhs: int, host: bool = False, slot: int = 0):
        """Cached device workspace (slot: independent workspaces for concurrent solves)."""
        torch = self._torch()
        key = (nrhs, host, slot)
        nb = self.workspace_bytes_host(nrhs) if host else self.workspace_bytes(nrhs)
        if nb == 0:
            raise LfdsError(5, _lib.lfds_last_error().decode() or "workspace query failed")
        ws = self._ws.get(key)
        if ws is None or ws.numel() < nb:
            ws = torch.empty(nb, dtype=torch.uint8, device=torch.device("cuda", max(self.device, 0)))
            self._ws[key] = ws
        return ws

    def _check_out(self, out, like, single, host=False):
        """The library writes nrhs*nz*ny*nx elements through out's raw pointer: same shape and
        dtype as f, contiguous, and on f's device (pinned CPU memory for host solves)."""
        if out is None:
            return
        O = out.unsqueeze(0) if single else out
        if tuple(O.shape) != tuple(like.shape) or O.dtype != like.dtype or not O.is_contiguous():
            raise ValueError(f"out must be a contiguous {like.dtype} tensor of shape {tuple(like.shape)}")
        if host:
            if O.is_cuda:
                raise ValueError("out must be a CPU tensor for solve_host")
        elif O.device != like.device:
            raise ValueError(f"out is on {O.device}, f on {like.device}")

    def _fdtype(self):
        torch = self._torch()
        return torch.float64 if self.dtype == LFDS_F64 else torch.complex128

    def solve(self, f, out=None, stream=None):
        """u = A^{-1} M f for f of shape (nrhs, nz, ny, nx) or (nz, ny, nx), on the device."""
        torch = self._torch()
        single = f.dim() == 3
        F = f.unsqueeze(0) if single else f
        if not (F.is_cuda and F.is_contiguous() and F.dtype == self._fdtype()):
            raise ValueError(f"f must be a contiguous CUDA {self._fdtype()} tensor")
        if tuple(F.shape[1:]) != self.shape:
            raise ValueError(f"f shape {tuple(F.shape)} does not match grid {self.shape}")
        nrhs = F.shape[0]
        self._check_out(out, F, single)
        U = torch.empty_like(F) if out is None else (out.unsqueeze(0) if single else out)
        ws = self.workspace(nrhs)
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _check(_lib.lfds_solve(self._h, _P(F.data_ptr()), _P(U.data_ptr()), nrhs, _P(ws.data_ptr()),
                               ws.numel(), _P(st)))
        return U[0] if single else U

    def solve_hetero(self, f, dlam, tol: float = 1e-10, maxit: int = 200, restart: int = 20, out=None,
                     stream=None):
        """Heterogeneous medium lambda_ijk = lambda + dlam_ijk (lfds_gmres): right-preconditioned
        GMRES with this plan's fast solve.  f, dlam: contiguous CUDA complex128 (nz, ny, nx).
        Returns (u, report dict)."""
        torch = self._torch()
        for name, t in (("f", f), ("dlam", dlam)):
            if not (t.is_cuda and t.is_contiguous() and t.dtype == torch.complex128 and tuple(t.shape) == self.shape):
                raise ValueError(f"{name} must be a contiguous CUDA complex128 tensor of shape {self.shape}")
        self._check_out(out, f, False)
        U = torch.empty_like(f) if out is None else out
        nb = int(_lib.lfds_gmres_workspace_bytes(self._h, int(restart)))
        if nb == 0:
            raise ValueError("lfds_gmres: restart must be in 1..64 on a device plan")
        key = ("gmres", int(restart))
        ws = self._ws.get(key)
        if ws is None or ws.numel() < nb or ws.device != f.device:  # cached like the solve workspace
            self._ws.pop(key, None)
            ws = self._ws[key] = torch.empty(nb, dtype=torch.uint8, device=f.device)
        st = (stream or torch.cuda.current_stream()).cuda_stream
        rep = KrylovReport()
        _check(_lib.lfds_gmres(self._h, _P(dlam.data_ptr()), _P(f.data_ptr()), _P(U.data_ptr()), float(tol),
                               int(maxit), int(restart), _P(ws.data_ptr()), nb, _P(st), ctypes.byref(rep)))
        return U, {"iterations": rep.iterations, "cycles": rep.cycles, "rel_residual": rep.rel_residual}

    def solve_host(self, f_host, out=None, stream=None, sync: bool = True, slot: int = 0):
        """End-to-end: host f (pinned CPU tensor) -> device -> solve -> host u.  sync=False
        only enqueues (lfds_solve_host_async); concurrent solves need distinct `slot`s."""
        torch = self._torch()
        single = f_host.dim() == 3
        F = f_host.unsqueeze(0) if single else f_host
        if F.is_cuda or not F.is_contiguous() or F.dtype != self._fdtype():
            raise ValueError("f_host must be a contiguous CPU tensor of the plan dtype")
        nrhs = F.shape[0]
        self._check_out(out, F, single, host=True)
        U = torch.empty_like(F, pin_memory=F.is_pinned()) if out is None else (out.unsqueeze(0) if single else out)
        ws = self.workspace(nrhs, host=True, slot=slot)
        st = (stream or torch.cuda.current_stream()).cuda_stream
        fn = _lib.lfds_solve_host if sync else _lib.lfds_solve_host_async
        _check(fn(self._h, _P(F.data_ptr()), _P(U.data_ptr()), nrhs, _P(ws.data_ptr()), ws.numel(), _P(st)))
        return U[0] if single else U

    # ------------------------------------------------------------------ block sharding
    def set_partition(self, block_owned=None, l_begin: int = 0, l_end: int = -1, rank0: bool = True):
        """Blocks this rank computes (flags [nby][nbx] or None for all), its global x-modes
        [l_begin, l_end) of step 5, and whether it adds the b-terms / writes the planes."""
        if block_owned is None:
            _check(_lib.lfds_set_partition(self._h, None, 0, 0, 1))
        else:
            own = np.ascontiguousarray(np.asarray(block_owned, dtype=np.int32).ravel())
            _check(_lib.lfds_set_partition(self._h, own.ctypes.data_as(_P), int(l_begin), int(l_end), int(rank0)))
        self._ws = {}
        self.formation = False

    def set_mode_rows(self, m_begin: int, m_end: int):
        """Second split of the z-modal step 5: this rank's global y-modes [m_begin, m_end)."""
        _check(_lib.lfds_set_mode_rows(self._h, int(m_begin), int(m_end)))
        self._ws = {}

    def set_comm(self, uid: Optional[bytes], rank: int = 0, world: int = 1):
        """In-library exchanges: join the NCCL group `uid` (128 bytes from nccl_unique_id(),
        the same on every rank; collective).  None releases it."""
        if uid is None:
            _check(_lib.lfds_set_comm(self._h, None, 0, 1))
            self.has_comm = False
            return
        buf = (ctypes.c_ubyte * 128).from_buffer_copy(bytes(uid))
        _check(_lib.lfds_set_comm(self._h, ctypes.cast(buf, _P), int(rank), int(world)))
        self.has_comm = True

    def set_formation_rows(self, m_begin: int, m_end: int, l_begin: int, l_end: int):
        """Formation split of the z-modal step 5 (exchange 3); m_begin < 0 switches it off."""
        _check(_lib.lfds_set_formation_rows(self._h, int(m_begin), int(m_end), int(l_begin), int(l_end)))
        self._ws = {}
        self.formation = m_begin >= 0

    def set_comm_groups(self, color_m: int, color_l: int):
        """Exchange-3 groups of the in-library communicator (collective; lfds_set_comm_groups)."""
        _check(_lib.lfds_set_comm_groups(self._h, int(color_m), int(color_l)))

    def exchange_view(self, ws, nrhs: int, which: int):
        """float64 view of exchange `which` (1: interface residual, 2: plane projections) in ws."""
        torch = self._torch()
        off, n = ctypes.c_size_t(), ctypes.c_size_t()
        _check(_lib.lfds_exchange_layout(self._h, nrhs, which, ctypes.byref(off), ctypes.byref(n)))
        return ws[off.value:off.value + 8 * n.value].view(torch.float64)

    def solve_phase(self, phase: int, f, u, ws, stream=None):
        """One phase of a sharded solve (1, 2, 3; with the formation split 2 = 4 + 5);
        f, u: (nrhs, nz, ny, nx) device tensors."""
        torch = self._torch()
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _check(_lib.lfds_solve_phase(self._h, int(phase), _P(f.data_ptr()), _P(u.data_ptr()), f.shape[0],
                                     _P(ws.data_ptr()), ws.numel(), _P(st)))

    def residual(self, u, f=None, dd: bool = True, stream=None):
        """(r, norms): r = M f - A u (complex128), norms[r] = (||r||_2, ||M f||_2)."""
        torch = self._torch()
        single = u.dim() == 3
        U = u.unsqueeze(0) if single else u
        F = None if f is None else (f.unsqueeze(0) if single else f)
        nrhs = U.shape[0]
        r = torch.empty(U.shape, dtype=torch.complex128, device=U.device)
        norms = np.zeros(2 * nrhs, np.float64)
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _check(_lib.lfds_residual(self._h, _P(U.data_ptr()), None if F is None else _P(F.data_ptr()),
                                  _P(r.data_ptr()), nrhs, int(dd), norms.ctypes.data_as(_P), _P(st)))
        return (r[0] if single else r), norms.reshape(nrhs, 2)

    def residual_f(self, u, f, dd: bool = False, stream=None):
        """r = f - M^{-1} A u (f-units: the right side of the correction solve), complex128,
        stream-ordered (lfds_residual_f)."""
        torch = self._torch()
        U = u.unsqueeze(0) if u.dim() == 3 else u
        F = f.unsqueeze(0) if f.dim() == 3 else f
        if U.shape != F.shape or not (U.is_cuda and F.is_cuda and U.is_contiguous() and F.is_contiguous()):
            raise ValueError("u, f: contiguous device tensors of the same shape")
        r = torch.empty(U.shape, dtype=torch.complex128, device=U.device)
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _check(_lib.lfds_residual_f(self._h, _P(U.data_ptr()), _P(F.data_ptr()), _P(r.data_ptr()), U.shape[0],
                                    int(dd), _P(st)))
        return r if u.dim() == 4 else r[0]

    def axpy(self, delta, u, stream=None):
        """u += delta in place (lfds_axpy); delta complex128 of u's shape."""
        torch = self._torch()
        D = delta.unsqueeze(0) if delta.dim() == 3 else delta
        U = u.unsqueeze(0) if u.dim() == 3 else u
        if D.shape != U.shape or D.dtype != torch.complex128 or not (D.is_contiguous() and U.is_contiguous()):
            raise ValueError("delta: contiguous complex128 of u's shape")
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _check(_lib.lfds_axpy(self._h, _P(D.data_ptr()), _P(U.data_ptr()), U.shape[0], _P(st)))
        return u

    def close(self):
        if getattr(self, "_h", None):
            _lib.lfds_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fp64_peak(stream=None) -> float:
    """In-run FP64 tensor-pipe (DMMA) peak of the current device in TFLOP/s (lfds_fp64_peak)."""
    import torch
    st = (stream or torch.cuda.current_stream()).cuda_stream
    tf = ctypes.c_double()
    _check(_lib.lfds_fp64_peak(_P(st), ctypes.byref(tf)))
    return tf.value


def nccl_unique_id() -> bytes:
    """128-byte NCCL group id (lfds_nccl_unique_id) for Plan.set_comm."""
    buf = (ctypes.c_ubyte * 128)()
    _check(_lib.lfds_nccl_unique_id(ctypes.cast(buf, _P)))
    return bytes(buf)


def _ml_check(rc):
    if rc != 0:
        raise LfdsError(rc, _lib.lfds_ml_last_error().decode())


class MLPlan:
    """Multi-level (nested) partition, lfds_ml_setup: coarse interfaces
    (coarse_x, coarse_y) take the global step 5, every coarse block is solved by the two-level
    method of its own fine partition (fine_x, fine_y, a superset of the coarse ones)."""

    def __init__(self, hx, hy, hz, sigma_node, sigma_edge, lam, coarse_x=(), coarse_y=(), fine_x=(), fine_y=(), *,
                 device: int = 0, s5_modal: bool = True, plane_dst: bool = True, resonance_tol: float = 1e-13,
                 dst_tma: bool = True):
        opt = Options()
        _lib.lfds_default_options(ctypes.byref(opt))
        opt.dtype = LFDS_C128
        opt.device = int(device)
        opt.s5_modal, opt.plane_dst = int(bool(s5_modal)), int(bool(plane_dst))
        opt.resonance_tol, opt.dst_tma = float(resonance_tol), int(bool(dst_tma))
        self.device = int(device)
        hx_, px = _zarr(hx); hy_, py = _zarr(hy); hz_, pz = _zarr(hz)
        sn_, psn = _zarr(sigma_node); se_, pse = _zarr(sigma_edge)
        ints = [np.ascontiguousarray(np.asarray(list(v), dtype=np.int32)) for v in (coarse_x, coarse_y, fine_x, fine_y)]
        lam = complex(lam)
        h = _P()
        _ml_check(_lib.lfds_ml_setup(len(hx_) - 1, px, len(hy_) - 1, py, len(hz_) - 1, pz, psn, pse,
                                     _Z(lam.real, lam.imag), *[a for v in ints for a in (len(v), v.ctypes.data_as(_P))],
                                     ctypes.byref(opt), ctypes.byref(h)))
        self._h = h
        self.shape = (len(hz_) - 1, len(hy_) - 1, len(hx_) - 1)
        self._ws = None

    def n_coarse_blocks(self) -> int:
        n = ctypes.c_int()
        _ml_check(_lib.lfds_ml_get_plans(self._h, ctypes.byref(n)))
        return n.value

    def workspace(self):
        import torch
        nb = int(_lib.lfds_ml_workspace_bytes(self._h))
        if self._ws is None or self._ws.numel() < nb:
            self._ws = torch.empty(nb, dtype=torch.uint8, device=torch.device("cuda", self.device))
        return self._ws

    def solve(self, f, out=None, stream=None):
        """u = A^{-1} M f for one contiguous CUDA complex128 right-hand side (nz, ny, nx)."""
        import torch
        if not (f.is_cuda and f.is_contiguous() and f.dtype == torch.complex128) or tuple(f.shape) != self.shape:
            raise ValueError(f"f must be a contiguous CUDA complex128 tensor of shape {self.shape}")
        if out is not None and (tuple(out.shape) != self.shape or out.dtype != f.dtype or not out.is_contiguous()
                                or out.device != f.device):
            raise ValueError("out must match f")
        U = torch.empty_like(f) if out is None else out
        ws = self.workspace()
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _ml_check(_lib.lfds_ml_solve(self._h, _P(f.data_ptr()), _P(U.data_ptr()), _P(ws.data_ptr()), ws.numel(),
                                     _P(st)))
        return U

    def close(self):
        if getattr(self, "_h", None):
            _lib.lfds_ml_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _mw_check(rc):
    if rc != 0:
        raise LfdsError(rc, _lib.lfds_mw_last_error().decode())


class MWPlan:
    """Lebedev-grid Maxwell solve in a layered medium (lfds_mw_setup, §3): H = A_h^{-1} f
    with A_h = curl rho curl - i omega mu.  Fields are CUDA complex128 (3, N_z, N_y, N_x)."""

    def __init__(self, hx, hy, hz, c1, c2, c3, mu, omega: float, *, device: int = 0, profile: bool = False):
        hx_, px = _zarr(hx); hy_, py = _zarr(hy); hz_, pz = _zarr(hz)
        a1, p1 = _zarr(c1); a2, p2 = _zarr(c2); a3, p3 = _zarr(c3)
        mu = complex(mu)
        h = _P()
        _mw_check(_lib.lfds_mw_setup(len(hx_) + 1, px, len(hy_) + 1, py, len(hz_) + 1, pz, p1, p2, p3,
                                     _Z(mu.real, mu.imag), float(omega), int(device), int(bool(profile)),
                                     ctypes.byref(h)))
        self._h = h
        self.device = int(device)
        self.shape = (3, len(hz_) + 1, len(hy_) + 1, len(hx_) + 1)
        self._ws = None

    @classmethod
    def from_problem(cls, p, **kw):
        return cls(p.hx, p.hy, p.hz, p.c1, p.c2, p.c3, p.mu, p.omega, **kw)

    def workspace(self):
        import torch
        nb = int(_lib.lfds_mw_workspace_bytes(self._h))
        if self._ws is None or self._ws.numel() < nb:
            self._ws = torch.empty(nb, dtype=torch.uint8, device=torch.device("cuda", self.device))
        return self._ws

    def _chk(self, t, name):
        import torch
        if not (t.is_cuda and t.is_contiguous() and t.dtype == torch.complex128) or tuple(t.shape) != self.shape:
            raise ValueError(f"{name} must be a contiguous CUDA complex128 tensor of shape {self.shape}")

    def solve(self, f, out=None, stream=None):
        import torch
        self._chk(f, "f")
        H = torch.empty_like(f) if out is None else out
        self._chk(H, "out")
        ws = self.workspace()
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _mw_check(_lib.lfds_mw_solve(self._h, _P(f.data_ptr()), _P(H.data_ptr()), _P(ws.data_ptr()), ws.numel(),
                                     _P(st)))
        return H

    def residual(self, H, f, out=None, stream=None):
        """r = f - A_h H on the interior P nodes (lfds_mw_residual)."""
        import torch
        self._chk(H, "H")
        self._chk(f, "f")
        r = torch.empty_like(f) if out is None else out
        ws = self.workspace()
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _mw_check(_lib.lfds_mw_residual(self._h, _P(H.data_ptr()), _P(f.data_ptr()), _P(r.data_ptr()),
                                        _P(ws.data_ptr()), ws.numel(), _P(st)))
        return r

    def kernel_times(self) -> dict:
        n = _lib.lfds_mw_kernel_count()
        ms = np.zeros(n, np.float64)
        la = np.zeros(n, np.int32)
        _mw_check(_lib.lfds_mw_kernel_times(self._h, ms.ctypes.data_as(_P), la.ctypes.data_as(_P)))
        return {_lib.lfds_mw_kernel_name(i).decode(): (float(ms[i]), int(la[i])) for i in range(n)}

    def close(self):
        if getattr(self, "_h", None):
            _lib.lfds_mw_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MW2Plan(MWPlan):
    """Two-level (blocked) Maxwell solve, lfds_mw2_setup: x-interfaces ix and
    y-interfaces iy (even node indices) split the grid into blocks; H = H^1 + H^2."""

    def __init__(self, hx, hy, hz, c1, c2, c3, mu, omega: float, ix=(), iy=(), *, device: int = 0):
        hx_, px = _zarr(hx); hy_, py = _zarr(hy); hz_, pz = _zarr(hz)
        a1, p1 = _zarr(c1); a2, p2 = _zarr(c2); a3, p3 = _zarr(c3)
        ix_ = np.ascontiguousarray(np.asarray(list(ix), dtype=np.int32))
        iy_ = np.ascontiguousarray(np.asarray(list(iy), dtype=np.int32))
        mu = complex(mu)
        h = _P()
        _mw_check(_lib.lfds_mw2_setup(len(hx_) + 1, px, len(hy_) + 1, py, len(hz_) + 1, pz, p1, p2, p3,
                                      _Z(mu.real, mu.imag), float(omega), len(ix_), ix_.ctypes.data_as(_P),
                                      len(iy_), iy_.ctypes.data_as(_P), int(device), ctypes.byref(h)))
        self._h = h
        self.device = int(device)
        self.shape = (3, len(hz_) + 1, len(hy_) + 1, len(hx_) + 1)
        self._ws = None

    @classmethod
    def from_problem(cls, p, ix=(), iy=(), **kw):
        return cls(p.hx, p.hy, p.hz, p.c1, p.c2, p.c3, p.mu, p.omega, ix, iy, **kw)

    def n_blocks(self) -> int:
        n = ctypes.c_int()
        _mw_check(_lib.lfds_mw2_blocks(self._h, ctypes.byref(n)))
        return n.value

    def workspace(self):
        import torch
        nb = int(_lib.lfds_mw2_workspace_bytes(self._h))
        if self._ws is None or self._ws.numel() < nb:
            self._ws = torch.empty(nb, dtype=torch.uint8, device=torch.device("cuda", self.device))
        return self._ws

    def solve(self, f, out=None, stream=None):
        import torch
        self._chk(f, "f")
        H = torch.empty_like(f) if out is None else out
        self._chk(H, "out")
        ws = self.workspace()
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _mw_check(_lib.lfds_mw2_solve(self._h, _P(f.data_ptr()), _P(H.data_ptr()), _P(ws.data_ptr()), ws.numel(),
                                      _P(st)))
        return H

    def residual(self, H, f, out=None, stream=None):
        raise NotImplementedError("use an MWPlan of the same grid for residuals")

    def kernel_times(self) -> dict:
        return {}

    def close(self):
        if getattr(self, "_h", None):
            _lib.lfds_mw2_destroy(self._h)
            self._h = None


def setup_grid(hx, hy, hz, sigma_node, sigma_edge, lam, iface_x=(), iface_y=(), **kw) -> Plan:
    """Python name of lfds_setup_grid."""
    return Plan(hx, hy, hz, sigma_node, sigma_edge, lam, iface_x, iface_y, **kw)
