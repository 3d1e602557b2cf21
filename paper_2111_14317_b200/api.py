"""Thin Python surface over the C ABI (SURVEY §8(b) "Python surface").

torch is used only for device memory and streams: every tensor handed to a call is a
caller-owned CUDA buffer whose data_ptr() goes straight to the kernel; no arithmetic of the
method happens here.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import PhtError, check  # noqa: F401


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class System:
    """A loaded homotopy (pht_system_create).  Arguments as in include/pht.h."""

    def __init__(self, offsets, exponents, coeffs, lifting, device: int = 0, projective: bool = False):
        lib = _lib.load()
        self._lib = lib
        off = np.ascontiguousarray(offsets, np.int64)
        exps = np.ascontiguousarray(exponents, np.int32)
        c = np.ascontiguousarray(coeffs, np.complex128)
        w = np.ascontiguousarray(lifting, np.float64)
        n = int(exps.shape[1])
        h = ctypes.c_void_p()
        create = lib.pht_system_create_projective if projective else lib.pht_system_create
        rc = create(len(off) - 1, n, off.ctypes.data_as(ctypes.c_void_p),
                                   exps.ctypes.data_as(ctypes.c_void_p), c.ctypes.data_as(ctypes.c_void_p),
                                   w.ctypes.data_as(ctypes.c_void_p), int(device), ctypes.byref(h))
        check(rc, "pht_system_create")
        self._h = h
        self.device = int(device)
        nn, M, mt, dev = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        check(lib.pht_system_info(h, ctypes.byref(nn), ctypes.byref(M), ctypes.byref(mt), ctypes.byref(dev)),
              "pht_system_info")
        self.n, self.M, self.max_terms = nn.value, M.value, mt.value
        self.dense = bool(lib.pht_system_flags(h) & _lib.SYS_DENSE)  # FP64 tensor-core evaluation path

    def homogenize(self, x, log_input: bool = False):
        """pht_homogenize: affine points x [p, n_eq] (or z = log x) -> y [p, n_eq + 1] on ||y|| = 1."""
        if not (x.is_cuda and x.dtype == torch.complex128 and x.dim() == 2 and x.shape[1] == self.n - 1
                and x.is_contiguous()):
            raise PhtError("x must be a contiguous cuda complex128 tensor [p, n_eq]")
        y = torch.empty((x.shape[0], self.n), dtype=torch.complex128, device=self._dev())
        check(self._lib.pht_homogenize(self._h, x.shape[0], _ptr(x), int(bool(log_input)), _ptr(y),
                                       _stream(self._dev())), "pht_homogenize")
        return y

    def set_solver(self, solver: str = "lu"):
        """pht_system_set_solver: 'lu' (Gauss-Jordan, default) or 'qr' (Householder)."""
        code = {"lu": _lib.SOLVER_LU, "qr": _lib.SOLVER_QR}[solver]
        check(self._lib.pht_system_set_solver(self._h, code), "pht_system_set_solver")
        return self

    def set_kernels(self, family: str = "auto"):
        """pht_system_set_kernels: 'auto' (measured-best, default), 'tile', 'warp', 'dense' (FP64
        tensor-core evaluation) or 'specialized' (after specialize())."""
        check(self._lib.pht_system_set_kernels(self._h, _lib.KERNELS[family]), "pht_system_set_kernels")
        return self

    @property
    def kernels(self) -> str:
        code = int(self._lib.pht_system_kernels(self._h))
        return {v: k for k, v in _lib.KERNELS.items()}[code]

    def specialize(self, what: int = _lib.SPEC_ALL):
        """pht_system_specialize: compile and load the system-specialised kernels (NVRTC)."""
        check(self._lib.pht_system_specialize(self._h, int(what)), "pht_system_specialize")
        return self

    @property
    def specialized(self) -> bool:
        return bool(self._lib.pht_system_flags(self._h) & _lib.SYS_SPECIALIZED)

    @classmethod
    def from_workload(cls, system, device: int = 0, projective: bool = False):
        return cls(system.offsets, system.exps, system.coeffs, system.lifting, device, projective)

    @property
    def projective(self) -> bool:
        """Projective system (pht_system_create_projective): points are y in C^{n_eq + 1}."""
        return bool(self._lib.pht_system_flags(self._h) & _lib.SYS_PROJECTIVE)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.pht_system_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------
    def _dev(self):
        return torch.device("cuda", self.device)

    def _check_pts(self, x, t):
        if not (x.is_cuda and x.dtype == torch.complex128 and x.dim() == 2 and x.shape[1] == self.n
                and x.is_contiguous()):
            raise PhtError("x must be a contiguous cuda complex128 tensor [p, n]")
        if not (t.is_cuda and t.dtype == torch.float64 and t.shape == (x.shape[0],) and t.is_contiguous()):
            raise PhtError("t/tau must be a contiguous cuda float64 tensor [p]")

    def evaluate(self, x, t, scaled: bool = False, out=None):
        """H, Jx, Jt (+ row_exp2 if scaled), status at points x [p,n], t [p] (pht_evaluate).
        out: optional preallocated (H, Jx, Jt, status) device tensors (no allocation per call)."""
        self._check_pts(x, t)
        p, n = x.shape
        d = self._dev()
        if out is not None:
            H, Jx, Jt, st = out
            for a, shape, dt in ((H, (p, n), torch.complex128), (Jx, (p, n, n), torch.complex128),
                                 (Jt, (p, n), torch.complex128), (st, (p,), torch.uint8)):
                if not (a.is_cuda and a.dtype == dt and tuple(a.shape) == shape and a.is_contiguous()):
                    raise PhtError("out tensors must be contiguous cuda (H [p,n], Jx [p,n,n], Jt [p,n] c128, status [p] u8)")
        else:
            H = torch.empty((p, n), dtype=torch.complex128, device=d)
            Jx = torch.empty((p, n, n), dtype=torch.complex128, device=d)
            Jt = torch.empty((p, n), dtype=torch.complex128, device=d)
            st = torch.empty(p, dtype=torch.uint8, device=d)
        e2 = torch.empty((p, n), dtype=torch.int32, device=d) if scaled else None
        check(self._lib.pht_evaluate(self._h, p, _ptr(x), _ptr(t), _ptr(H), _ptr(Jx), _ptr(Jt), _ptr(e2),
                                     _ptr(st), _stream(d)), "pht_evaluate")
        return (H, Jx, Jt, e2, st) if scaled else (H, Jx, Jt, st)

    def evaluate_log(self, z, tau, scaled: bool = True):
        """H, Jz = dH/dz, Jtau = dH/dtau (+ row_exp2) at z = log x, tau = log t."""
        self._check_pts(z, tau)
        p, n = z.shape
        d = self._dev()
        H = torch.empty((p, n), dtype=torch.complex128, device=d)
        Jz = torch.empty((p, n, n), dtype=torch.complex128, device=d)
        Jtau = torch.empty((p, n), dtype=torch.complex128, device=d)
        e2 = torch.empty((p, n), dtype=torch.int32, device=d) if scaled else None
        st = torch.empty(p, dtype=torch.uint8, device=d)
        check(self._lib.pht_evaluate_log(self._h, p, _ptr(z), _ptr(tau), _ptr(H), _ptr(Jz), _ptr(Jtau),
                                         _ptr(e2), _ptr(st), _stream(d)), "pht_evaluate_log")
        return (H, Jz, Jtau, e2, st) if scaled else (H, Jz, Jtau, st)

    def euler_newton(self, x, t):
        """dE (Jx dE = -dH/dt), dN (Jx dN = -H), status (pht_euler_newton)."""
        self._check_pts(x, t)
        p, n = x.shape
        d = self._dev()
        dE = torch.empty((p, n), dtype=torch.complex128, device=d)
        dN = torch.empty((p, n), dtype=torch.complex128, device=d)
        st = torch.empty(p, dtype=torch.uint8, device=d)
        check(self._lib.pht_euler_newton(self._h, p, _ptr(x), _ptr(t), _ptr(dE), _ptr(dN), _ptr(st),
                                         _stream(d)), "pht_euler_newton")
        return dE, dN, st

    def pc_step(self, x, tau, dtau, newton_iters: int = 1, status=None, dn_norm=None):
        """In-place Euler-Newton step (pht_pc_step); returns (status, dn_norm)."""
        self._check_pts(x, tau)
        p = x.shape[0]
        d = self._dev()
        if not (dtau.is_cuda and dtau.dtype == torch.float64 and dtau.shape == (p,)):
            raise PhtError("dtau must be a cuda float64 tensor [p]")
        st = status if status is not None else torch.empty(p, dtype=torch.uint8, device=d)
        dn = dn_norm if dn_norm is not None else torch.empty(p, dtype=torch.float64, device=d)
        check(self._lib.pht_pc_step(self._h, p, _ptr(x), _ptr(tau), _ptr(dtau), int(newton_iters), _ptr(st),
                                    _ptr(dn), _stream(d)), "pht_pc_step")
        return st, dn

    def pc_step_host(self, x: np.ndarray, tau: np.ndarray, dtau: np.ndarray, newton_iters: int = 1,
                     status: np.ndarray = None, dn_norm: np.ndarray = None, asynchronous: bool = False):
        """pht_pc_step_host on host numpy buffers (x, tau updated in place; pass pinned buffers,
        including status/dn_norm, for copy/compute overlap).  asynchronous=True calls
        pht_pc_step_host_async: the buffers (pass status/dn_norm to own them) are in flight until
        host_wait(); consecutive calls overlap."""
        def host(a, dt, shape, what):
            if not (isinstance(a, np.ndarray) and a.dtype == dt and a.shape == shape and a.flags.c_contiguous):
                raise PhtError(f"{what} must be a C-contiguous numpy {np.dtype(dt).name} array of shape {shape}")
            return a
        if not isinstance(x, np.ndarray) or x.ndim != 2:
            raise PhtError("x must be a numpy complex128 array [p, n]")
        p = x.shape[0]
        host(x, np.complex128, (p, self.n), "x")
        host(tau, np.float64, (p,), "tau")
        host(dtau, np.float64, (p,), "dtau")
        st = host(status, np.uint8, (p,), "status") if status is not None else np.empty(p, np.uint8)
        dn = host(dn_norm, np.float64, (p,), "dn_norm") if dn_norm is not None else np.empty(p, np.float64)
        if not x.flags.writeable or not tau.flags.writeable:
            raise PhtError("x and tau are updated in place: they must be writeable")
        if asynchronous and (status is None or dn_norm is None):
            raise PhtError("asynchronous host steps need caller-owned status and dn_norm buffers")
        d = self._dev()
        fn = self._lib.pht_pc_step_host_async if asynchronous else self._lib.pht_pc_step_host
        check(fn(self._h, p, x.ctypes.data_as(ctypes.c_void_p), tau.ctypes.data_as(ctypes.c_void_p),
                 dtau.ctypes.data_as(ctypes.c_void_p), int(newton_iters), st.ctypes.data_as(ctypes.c_void_p),
                 dn.ctypes.data_as(ctypes.c_void_p), _stream(d)), "pht_pc_step_host")
        return st, dn

    def host_wait(self):
        """pht_host_wait: the current stream waits for (and synchronises with) every host step."""
        check(self._lib.pht_host_wait(self._h, _stream(self._dev())), "pht_host_wait")

    def track(self, x, tau, stats: bool = True, **opts):
        """Adaptive tracking tau0 -> 0 in place (pht_track).  x: complex128 [p, n] start points,
        tau: float64 [p] start parameters.  Keyword options = pht_track_opts fields.
        Returns (status uint8 [p], stats int64 [p, 4] or None)."""
        self._check_pts(x, tau)
        p = x.shape[0]
        d = self._dev()
        o = _lib.TrackOpts()
        self._lib.pht_track_opts_default(ctypes.byref(o))
        for k, v in opts.items():
            if not hasattr(o, k):
                raise PhtError(f"unknown tracker option {k}")
            setattr(o, k, v)
        st = torch.empty(p, dtype=torch.uint8, device=d)
        sv = torch.empty((p, 4), dtype=torch.int64, device=d) if stats else None
        check(self._lib.pht_track(self._h, p, _ptr(x), _ptr(tau), ctypes.byref(o), _ptr(sv), _ptr(st),
                                  _stream(d)), "pht_track")
        return st, sv

    def track_cells(self, w, tau, cell_lift, path_cell, stats: bool = True, **opts):
        """pht_track_cells: tracking in cell coordinates.  w: complex128 [p, n] start values log y,
        tau: float64 [p], cell_lift: float64 [ncells, M] cell-shifted liftings, path_cell: int32 [p]
        (all cuda).  w is replaced by z = log x at tau = 0.  Returns (status, stats)."""
        self._check_pts(w, tau)
        p = w.shape[0]
        d = self._dev()
        if not (cell_lift.is_cuda and cell_lift.dtype == torch.float64 and cell_lift.dim() == 2
                and cell_lift.shape[1] == self.M and cell_lift.is_contiguous()):
            raise PhtError("cell_lift must be a contiguous cuda float64 tensor [ncells, M]")
        if not (path_cell.is_cuda and path_cell.dtype == torch.int32 and path_cell.shape == (p,)):
            raise PhtError("path_cell must be a cuda int32 tensor [p]")
        o = _lib.TrackOpts()
        self._lib.pht_track_opts_default(ctypes.byref(o))
        for k, v in opts.items():
            if not hasattr(o, k):
                raise PhtError(f"unknown tracker option {k}")
            setattr(o, k, v)
        st = torch.empty(p, dtype=torch.uint8, device=d)
        sv = torch.empty((p, 4), dtype=torch.int64, device=d) if stats else None
        check(self._lib.pht_track_cells(self._h, p, _ptr(w), _ptr(tau), _ptr(cell_lift), cell_lift.shape[0],
                                        _ptr(path_cell), ctypes.byref(o), _ptr(sv), _ptr(st), _stream(d)),
              "pht_track_cells")
        return st, sv


def _host_tables(system):
    off = np.ascontiguousarray(system.offsets, np.int64)
    exps = np.ascontiguousarray(system.exps, np.int32)
    c = np.ascontiguousarray(system.coeffs, np.complex128)
    w = np.ascontiguousarray(system.lifting, np.float64)
    return off, exps, c, w


def specialize_source(system) -> str:
    """The generated CUDA source of the specialised kernels (pht_specialize_source; no GPU)."""
    lib = _lib.load()
    off, exps, c, w = _host_tables(system)
    args = (len(off) - 1, int(exps.shape[1]), off.ctypes.data_as(ctypes.c_void_p),
            exps.ctypes.data_as(ctypes.c_void_p), c.ctypes.data_as(ctypes.c_void_p), w.ctypes.data_as(ctypes.c_void_p))
    need = lib.pht_specialize_source(*args, None, 0)
    check(int(need) if need < 0 else 0, "pht_specialize_source")
    buf = ctypes.create_string_buffer(int(need))
    lib.pht_specialize_source(*args, buf, int(need))
    return buf.value.decode()


def specialize_compile(system, what: int = _lib.SPEC_ALL) -> int:
    """Generate + compile (NVRTC, sm_100a) the specialised kernels without loading them (no GPU);
    returns the cubin size in bytes."""
    lib = _lib.load()
    off, exps, c, w = _host_tables(system)
    nb = ctypes.c_int64()
    check(lib.pht_specialize_compile(len(off) - 1, int(exps.shape[1]), off.ctypes.data_as(ctypes.c_void_p),
                                     exps.ctypes.data_as(ctypes.c_void_p), c.ctypes.data_as(ctypes.c_void_p),
                                     w.ctypes.data_as(ctypes.c_void_p), int(what), ctypes.byref(nb)),
          "pht_specialize_compile")
    return int(nb.value)


def launch_count() -> int:
    return int(_lib.load().pht_launch_count())
