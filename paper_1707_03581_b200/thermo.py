"""Thin ctypes binding of libthermo.so (include/thermo.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels.  There is no CPU fallback:
if the library is missing or no GPU is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libthermo.so")

THERMO_OK, THERMO_EINVAL, THERMO_ENOMEM, THERMO_ECUDA, THERMO_ENOCONV, THERMO_EGEOM = 0, -1, -2, -3, -4, -5
_CODES = {-1: "EINVAL", -2: "ENOMEM", -3: "ECUDA", -4: "ENOCONV", -5: "EGEOM"}

# symbols declared in include/thermo.h
EXPORTS = ["thermo_create_mesh", "thermo_set_bc", "thermo_step", "thermo_get_T", "thermo_set_T",
           "thermo_set_solver", "thermo_get_stats", "thermo_get_step_iters", "thermo_last_error",
           "thermo_destroy", "thermo_set_timing", "thermo_set_method", "thermo_stationary",
           "thermo_get_T_async", "thermo_get_T_all_async", "thermo_sync", "thermo_set_guess", "thermo_get_interface"]


class ThermoError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"thermo {_CODES.get(code, code)}: {msg}")
        self.code = code


class _Mesh(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int64), ("xyz", ctypes.c_void_p), ("n_tets", ctypes.c_int64),
                ("tets", ctypes.c_void_p), ("n_bfaces", ctypes.c_int64), ("bfaces", ctypes.c_void_p),
                ("bface_tag", ctypes.c_void_p)]


class _Scenario(ctypes.Structure):
    _fields_ = [("s0", ctypes.c_double), ("amp", ctypes.c_double), ("period", ctypes.c_double),
                ("dir", ctypes.c_double * 3), ("eta0", ctypes.c_double), ("eta_amp", ctypes.c_double),
                ("eta_period", ctypes.c_double)]


class Stats(ctypes.Structure):
    _fields_ = [("n_fixed", ctypes.c_int64), ("n_moving", ctypes.c_int64), ("nnz_volume", ctypes.c_int64),
                ("nnz_volume_padded", ctypes.c_int64), ("n_scen", ctypes.c_int32),
                ("n_iface_rows", ctypes.c_int32), ("iface_capacity", ctypes.c_int32),
                ("last_nsteps", ctypes.c_int32), ("total_iters", ctypes.c_int64), ("max_iters", ctypes.c_int32),
                ("failed_step", ctypes.c_int32), ("failed_scen", ctypes.c_int32),
                ("failed_relres", ctypes.c_double), ("last_relres", ctypes.c_double),
                ("steps_done", ctypes.c_int64), ("iface_area", ctypes.c_double),
                ("ms_iface", ctypes.c_double), ("ms_solve", ctypes.c_double), ("solve_grid", ctypes.c_int32),
                ("solve_block", ctypes.c_int32), ("launches_per_step", ctypes.c_int32),
                ("reordered", ctypes.c_int32), ("order_max_runs", ctypes.c_int32),
                ("order_max_window", ctypes.c_int32), ("solve_variant", ctypes.c_int32),
                ("solve_kind", ctypes.c_int32), ("solve_max_runs", ctypes.c_int32),
                ("solve_window", ctypes.c_int32), ("latency_path", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load(path: str = LIB_PATH):
    """Load libthermo.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path)
    vp, i32, i64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    L.thermo_create_mesh.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(_Mesh), ctypes.POINTER(_Mesh), i32, i32,
                                     d, d, d, i32, ctypes.POINTER(_Scenario), d, vp]
    L.thermo_set_bc.argtypes = [vp, i32, i32, d, d, ctypes.POINTER(ctypes.c_double)]
    L.thermo_step.argtypes = [vp, d, d, i32]
    L.thermo_get_T.argtypes = [vp, i32, i32, vp, i64, i32]
    L.thermo_set_T.argtypes = [vp, i32, i32, vp, i64, i32]
    L.thermo_set_solver.argtypes = [vp, d, i32]
    L.thermo_set_guess.argtypes = [vp, i32]
    L.thermo_get_interface.argtypes = [vp, i32, d, d, vp, vp, vp, vp, vp]
    L.thermo_get_stats.argtypes = [vp, ctypes.POINTER(Stats)]
    L.thermo_get_step_iters.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), i64]
    L.thermo_last_error.argtypes = [vp]
    L.thermo_last_error.restype = ctypes.c_char_p
    L.thermo_destroy.argtypes = [vp]
    L.thermo_set_timing.argtypes = [vp, i32]
    L.thermo_set_method.argtypes = [vp, i32, i32, i32, i32]
    L.thermo_stationary.argtypes = [vp, ctypes.c_double, i32]
    L.thermo_get_T_async.argtypes = [vp, i32, i32, vp, ctypes.c_int64]
    L.thermo_get_T_all_async.argtypes = [vp, vp, ctypes.c_int64]
    L.thermo_sync.argtypes = [vp]
    _lib = L
    return L


def _mesh(m, keep):
    xyz = np.ascontiguousarray(m.xyz, dtype=np.float64)
    tets = np.ascontiguousarray(m.tets, dtype=np.int32)
    bf = np.ascontiguousarray(m.bfaces, dtype=np.int32)
    tg = np.ascontiguousarray(m.bface_tag, dtype=np.int32)
    keep += [xyz, tets, bf, tg]
    return _Mesh(xyz.shape[0], xyz.ctypes.data, tets.shape[0], tets.ctypes.data, bf.shape[0], bf.ctypes.data,
                 tg.ctypes.data)


class Thermo:
    """One library context: two meshes, S scenarios, state on the device."""

    def __init__(self, fixed, moving, nu: float, rho_cp: float, alpha_iface: float, scenarios: Sequence,
                 T_init: float, iface_tag=(4, 4), robin=(), stream: Optional[int] = None):
        L = load()
        keep = []
        mf, mm = _mesh(fixed, keep), _mesh(moving, keep)
        S = len(scenarios)
        sc = (_Scenario * S)()
        for k, s in enumerate(scenarios):
            sc[k].s0, sc[k].amp, sc[k].period = s.s0, s.amp, s.period
            for d in range(3):
                sc[k].dir[d] = s.dir[d]
            sc[k].eta0, sc[k].eta_amp, sc[k].eta_period = s.eta0, s.eta_amp, s.eta_period
        if stream is None:
            import torch
            stream = torch.cuda.current_stream().cuda_stream
        h = ctypes.c_void_p()
        rc = L.thermo_create_mesh(ctypes.byref(h), ctypes.byref(mf), ctypes.byref(mm), iface_tag[0], iface_tag[1],
                                  nu, rho_cp, alpha_iface, S, sc, T_init, ctypes.c_void_p(stream))
        if rc:
            raise ThermoError(rc, L.thermo_last_error(None).decode())
        self.h = h
        self.nf, self.nm, self.S = fixed.n_nodes, moving.n_nodes, S
        self.n = self.nf + self.nm
        for r in robin:
            self.set_bc(r.part, r.tag, r.alpha, r.T_ref, r.grad)

    @classmethod
    def from_config(cls, cfg, stream=None, scenarios=None):
        return cls(cfg.fixed, cfg.moving, cfg.nu, cfg.rho_cp, cfg.alpha_iface,
                   cfg.scenarios if scenarios is None else scenarios, cfg.T0,
                   (cfg.iface_tag, cfg.iface_tag), cfg.robin, stream)

    def _check(self, rc):
        if rc:
            raise ThermoError(rc, load().thermo_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            load().thermo_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_bc(self, part, tag, alpha, T_ref, grad=(0.0, 0.0, 0.0)):
        g = (ctypes.c_double * 3)(*grad)
        self._check(load().thermo_set_bc(self.h, part, tag, alpha, T_ref, g))

    def set_timing(self, enable=True):
        self._check(load().thermo_set_timing(self.h, 1 if enable else 0))

    def set_method(self, method: str = "ie", M: int = 3, P: int = 2, K: int = 1):
        """'ie' (implicit Euler, default), 'mrsdc' (MRSDC(M, P) with K sweeps) or
        'sdc' (single-rate SDC(M) with K sweeps, interface implicit)."""
        code = {"ie": 0, "mrsdc": 1, "sdc": 2}[method]
        self._check(load().thermo_set_method(self.h, code, M, P, K))

    def stationary(self, t: float = 0.0, with_interface: bool = False):
        """Replace T by the stationary state at rest; see thermo_stationary."""
        self._check(load().thermo_stationary(self.h, float(t), 1 if with_interface else 0))

    def set_solver(self, rtol=1e-12, maxit=0):
        self._check(load().thermo_set_solver(self.h, rtol, maxit))

    def get_interface(self, t: float, dt: float, scen: int = 0):
        """Interface rows of scenario `scen` at time t for step dt (thermo_get_interface):
        (rows[n_if], cnt[n_if], col[n_if, cap], val[n_if, cap] = -dt K_G entries, b[n_if])."""
        import numpy as np
        st = self.stats()
        n, cap = st["n_iface_rows"], st["iface_capacity"]
        rows, cnt = np.zeros(n, np.int32), np.zeros(n, np.int32)
        col, val, b = np.zeros((n, cap), np.int32), np.zeros((n, cap)), np.zeros(n)
        self._check(load().thermo_get_interface(self.h, int(scen), float(t), float(dt), rows.ctypes.data,
                                                cnt.ctypes.data, col.ctypes.data, val.ctypes.data, b.ctypes.data))
        return rows, cnt, col, val, b

    def set_guess(self, order: int):
        """CG initial guess: 0 = T^n, 1 / 2 = linear / quadratic extrapolation (thermo_set_guess)."""
        self._check(load().thermo_set_guess(self.h, int(order)))

    def step(self, t: float, dt: float, nsteps: int):
        self._check(load().thermo_step(self.h, t, dt, nsteps))

    def _count(self, part):
        return {0: self.nf, 1: self.nm, -1: self.n}[part]

    def get_T(self, scen: int = 0, part: int = -1, out=None) -> np.ndarray:
        """Host copy (numpy) of one scenario's temperature, or a device copy into `out`
        (a CUDA torch tensor of float64) when given."""
        n = self._count(part)
        if out is not None:
            assert out.is_cuda and out.dtype.is_floating_point and out.numel() == n and out.is_contiguous()
            self._check(load().thermo_get_T(self.h, scen, part, ctypes.c_void_p(out.data_ptr()), n, 1))
            return out
        a = np.empty(n, np.float64)
        self._check(load().thermo_get_T(self.h, scen, part, a.ctypes.data_as(ctypes.c_void_p), n, 0))
        return a

    def get_T_host_ptr(self, ptr: int, scen: int = 0, part: int = -1):
        """Copy into caller-owned host memory at address `ptr` (e.g. a pinned torch tensor);
        synchronises the context stream."""
        n = self._count(part)
        self._check(load().thermo_get_T(self.h, scen, part, ctypes.c_void_p(ptr), n, 0))

    def get_T_async(self, ptr: int, scen: int = 0, part: int = -1):
        """Enqueue a copy of the current state into caller-owned (pinned) host memory at `ptr`
        and return at once; valid after sync()."""
        n = self._count(part)
        self._check(load().thermo_get_T_async(self.h, scen, part, ctypes.c_void_p(ptr), n))

    def get_T_all_async(self, ptr: int):
        """Enqueue one copy of every scenario's field (scenario-major [S][N], caller numbering)
        into caller-owned (pinned) host memory at `ptr`; valid after sync()."""
        self._check(load().thermo_get_T_all_async(self.h, ctypes.c_void_p(ptr), self.n * self.S))

    def sync(self):
        self._check(load().thermo_sync(self.h))

    def set_T(self, T, scen: int = 0, part: int = -1):
        n = self._count(part)
        if hasattr(T, "is_cuda") and T.is_cuda:
            self._check(load().thermo_set_T(self.h, scen, part, ctypes.c_void_p(T.data_ptr()), n, 1))
        else:
            a = np.ascontiguousarray(T, dtype=np.float64)
            assert a.shape == (n,)
            self._check(load().thermo_set_T(self.h, scen, part, a.ctypes.data_as(ctypes.c_void_p), n, 0))

    def stats(self) -> dict:
        s = Stats()
        self._check(load().thermo_get_stats(self.h, ctypes.byref(s)))
        return s.as_dict()

    def step_iters(self) -> np.ndarray:
        st = self.stats()
        n = max(st["last_nsteps"], 0) * self.S
        a = np.zeros(max(n, 1), np.int32)
        self._check(load().thermo_get_step_iters(self.h, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), n))
        return a[:n].reshape(-1, self.S)
