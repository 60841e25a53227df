"""ctypes wrapper of the plain CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product path (paper_1707_03581_b200) never
imports this package.  See oracle/oracle.h for what is computed and the passages it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_d = ctypes.c_double
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_p = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (plain C99, -O2, OpenMP on the CG loops)."""
    hdr = os.path.join(_HERE, "oracle.h")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC), os.path.getmtime(hdr)):
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.or_create.restype = _p
        L.or_create.argtypes = [_i64, _p, _i64, _p, _i64, _p, _p, _i64, _p, _i64, _p, _i64, _p, _p,
                                _i32, _d, _d, _d]
        L.or_last_error.restype = ctypes.c_char_p
        L.or_threads.restype = ctypes.c_int
        L.or_destroy.argtypes = [_p]
        L.or_set_robin.argtypes = [_p, _i32, _i32, _d, _d, _d, _d, _d]
        L.or_n.restype = _i64
        L.or_n.argtypes = [_p]
        L.or_n_fixed.restype = _i64
        L.or_n_fixed.argtypes = [_p]
        L.or_vol_nnz.restype = _i64
        L.or_vol_nnz.argtypes = [_p]
        L.or_get_volume.argtypes = [_p, _p, _p, _p, _p, _p, _p]
        L.or_assemble_interface.argtypes = [_p, _d, _d, _d, _d]
        L.or_iface_nnz.restype = _i64
        L.or_iface_nnz.argtypes = [_p]
        L.or_get_interface.argtypes = [_p, _p, _p, _p, _p, _p]
        L.or_set_guess.argtypes = [_p, _i32]
        L.or_step.argtypes = [_p, _d, _d, _i32, _d, _d, _d, _d, _d, _d, _d, _d, _d, _p, _i32, _d, _i32, _p]
        L.or_ie_residual_rows.argtypes = [_p, _d, _d, _d, _d, _d, _p, _p, _i64, _p, _p, _p]
        L.or_apply_system.argtypes = [_p, _d, _p, _p]
        L.or_stationary.argtypes = [_p, _d, _i32, _d, _d, _d, _d, _d, _d, _d, _d, _d, _p, _i32, _d, _i32, _p]
        L.or_step_sdc.argtypes = [_p, _d, _d, _i32, _i32, _i32, _d, _d, _d, _d, _d, _d, _d, _d, _d, _p, _d, _p]
        L.or_mrsdc_weights.argtypes = [ctypes.c_int, ctypes.c_int, _d, _d, _p, _p, _p, _p, _p, _p]
        L.or_step_mrsdc.argtypes = [_p, _d, _d, _i32, _i32, _i32, _i32, _d, _d, _d, _d, _d, _d, _d, _d, _d, _p,
                                    _d, _p]
        _lib = L
    return _lib


def threads() -> int:
    """Host threads the oracle's CG loops run on (OMP_NUM_THREADS, default all cores)."""
    return int(lib().or_threads())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Oracle:
    """One coupled two-mesh system (fixed part rows first, then moving part)."""

    def __init__(self, fixed, moving, nu, rho_cp, alpha_iface, iface_tag=4, robin=(), guess=0):
        L = lib()
        self._keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return a
        xf, tf, ff, gf = (arr(fixed.xyz, np.float64), arr(fixed.tets, np.int32),
                          arr(fixed.bfaces, np.int32), arr(fixed.bface_tag, np.int32))
        xm, tm, fm, gm = (arr(moving.xyz, np.float64), arr(moving.tets, np.int32),
                          arr(moving.bfaces, np.int32), arr(moving.bface_tag, np.int32))
        h = L.or_create(xf.shape[0], _ptr(xf), tf.shape[0], _ptr(tf), ff.shape[0], _ptr(ff), _ptr(gf),
                        xm.shape[0], _ptr(xm), tm.shape[0], _ptr(tm), fm.shape[0], _ptr(fm), _ptr(gm),
                        iface_tag, nu, rho_cp, alpha_iface)
        self._keep = []
        if not h:
            raise ValueError("oracle: " + L.or_last_error().decode())
        self.h = h
        self.n = int(L.or_n(h))
        self.nf = int(L.or_n_fixed(h))
        for r in robin:
            self.set_robin(r.part, r.tag, r.alpha, r.T_ref, r.grad)
        if guess:
            self.set_guess(guess)

    @classmethod
    def from_config(cls, cfg, guess=0):
        return cls(cfg.fixed, cfg.moving, cfg.nu, cfg.rho_cp, cfg.alpha_iface, cfg.iface_tag, cfg.robin, guess)

    def set_guess(self, order: int):
        """CG start of step(): 0 = T^n, 1 / 2 = linear / quadratic extrapolation (or_set_guess)."""
        if lib().or_set_guess(self.h, int(order)):
            raise ValueError("oracle: " + lib().or_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_destroy(self.h)
            self.h = None

    def set_robin(self, part, tag, alpha, T_ref, grad=(0.0, 0.0, 0.0)):
        rc = lib().or_set_robin(self.h, part, tag, alpha, T_ref, *grad)
        if rc:
            raise ValueError("oracle: " + lib().or_last_error().decode())

    def volume(self):
        """(rowptr, col, A, B, ML, benv) of the fixed-pattern volume operator."""
        L = lib()
        nnz = int(L.or_vol_nnz(self.h))
        rowptr = np.zeros(self.n + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        A = np.zeros(nnz)
        B = np.zeros(nnz)
        ML = np.zeros(self.n)
        benv = np.zeros(self.n)
        L.or_get_volume(self.h, _ptr(rowptr), _ptr(col), _ptr(A), _ptr(B), _ptr(ML), _ptr(benv))
        return rowptr, col, A, B, ML, benv

    def interface(self, offset: Sequence[float], eta: float):
        """(rowptr, col, val, bG, area) of K_G = M_B + C_B at the given offset."""
        L = lib()
        rc = L.or_assemble_interface(self.h, float(offset[0]), float(offset[1]), float(offset[2]), float(eta))
        if rc:
            raise ValueError("oracle: " + L.or_last_error().decode())
        nnz = int(L.or_iface_nnz(self.h))
        rowptr = np.zeros(self.n + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        val = np.zeros(nnz)
        bG = np.zeros(self.n)
        area = ctypes.c_double(0.0)
        L.or_get_interface(self.h, _ptr(rowptr), _ptr(col), _ptr(val), _ptr(bG), ctypes.byref(area))
        return rowptr, col, val, bG, area.value

    def step(self, T: np.ndarray, t: float, dt: float, nsteps: int, scen, solver: str = "cg",
             rtol: float = 1e-12, maxit: int = 0):
        """Advance T (length n, modified copy returned) by nsteps implicit-Euler steps.
        Returns (T_new, stats[nsteps, 4] = iterations, rel. res, true rel. res, |Gamma_R|)."""
        T = np.array(T, dtype=np.float64, copy=True)
        stats = np.zeros((nsteps, 4))
        rc = lib().or_step(self.h, t, dt, nsteps, scen.s0, scen.amp, scen.period,
                           scen.dir[0], scen.dir[1], scen.dir[2], scen.eta0, scen.eta_amp,
                           scen.eta_period, _ptr(T), 1 if solver == "cholesky" else 0, rtol,
                           maxit, _ptr(stats))
        if rc:
            raise RuntimeError(f"oracle step failed rc={rc}: " + lib().or_last_error().decode())
        return T, stats

    def residual_rows(self, dt, offset, eta, T0, T1, rows):
        T0 = np.ascontiguousarray(T0, dtype=np.float64)
        T1 = np.ascontiguousarray(T1, dtype=np.float64)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        res = np.zeros(rows.shape[0])
        bnorm = ctypes.c_double(0.0)
        rc = lib().or_ie_residual_rows(self.h, dt, float(offset[0]), float(offset[1]), float(offset[2]),
                                       float(eta), _ptr(T0), _ptr(T1), rows.shape[0], _ptr(rows),
                                       _ptr(res), ctypes.byref(bnorm))
        if rc:
            raise RuntimeError("oracle residual failed: " + lib().or_last_error().decode())
        return res, bnorm.value

    def apply_system(self, dt, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        lib().or_apply_system(self.h, dt, _ptr(x), _ptr(y))
        return y


def mrsdc_weights(M: int, P: int, t0: float = 0.0, dt: float = 1.0):
    """(tau[M], taue[M,P], s[M,M], shat[M,P], stilde[M,P,M], semb[M,P,P]) of Table 1."""
    tau, taue = np.zeros(M), np.zeros((M, P))
    s, shat = np.zeros((M, M)), np.zeros((M, P))
    st, se = np.zeros((M, P, M)), np.zeros((M, P, P))
    rc = lib().or_mrsdc_weights(M, P, t0, dt, _ptr(tau), _ptr(taue), _ptr(s), _ptr(shat), _ptr(st), _ptr(se))
    if rc:
        raise ValueError("oracle: " + lib().or_last_error().decode())
    return tau, taue, s, shat, st, se


def _step_mrsdc(self, T, t, dt, nsteps, scen, M=3, P=2, K=1, rtol=1e-12):
    """MRSDC(M, P) with K sweeps (Algorithms 1-2).  Returns (T_new, stats[nsteps, 3])."""
    T = np.array(T, dtype=np.float64, copy=True)
    stats = np.zeros((nsteps, 3))
    rc = lib().or_step_mrsdc(self.h, t, dt, nsteps, M, P, K, scen.s0, scen.amp, scen.period, scen.dir[0],
                             scen.dir[1], scen.dir[2], scen.eta0, scen.eta_amp, scen.eta_period, _ptr(T), rtol,
                             _ptr(stats))
    if rc:
        raise RuntimeError(f"oracle mrsdc failed rc={rc}: " + lib().or_last_error().decode())
    return T, stats


Oracle.step_mrsdc = _step_mrsdc


def _stationary(self, T, t, scen, with_interface=False, solver="cg", rtol=1e-12, maxit=0):
    """Stationary state (reading R19/R28) from the initial guess T.
    Returns (T, stats[3] = iterations, rel. residual, true rel. residual)."""
    T = np.array(T, dtype=np.float64, copy=True)
    stats = np.zeros(3)
    rc = lib().or_stationary(self.h, t, 1 if with_interface else 0, scen.s0, scen.amp, scen.period,
                             scen.dir[0], scen.dir[1], scen.dir[2], scen.eta0, scen.eta_amp, scen.eta_period,
                             _ptr(T), 1 if solver == "cholesky" else 0, rtol, maxit, _ptr(stats))
    if rc:
        raise RuntimeError(f"oracle stationary failed rc={rc}: " + lib().or_last_error().decode())
    return T, stats


Oracle.stationary = _stationary


def _step_sdc(self, T, t, dt, nsteps, scen, M=3, K=1, rtol=1e-12):
    """Single-rate SDC(M) with K sweeps, interface implicit (reading R29).
    Returns (T_new, stats[nsteps, 3] = solves, CG iterations, SDC residual)."""
    T = np.array(T, dtype=np.float64, copy=True)
    stats = np.zeros((nsteps, 3))
    rc = lib().or_step_sdc(self.h, t, dt, nsteps, M, K, scen.s0, scen.amp, scen.period, scen.dir[0], scen.dir[1],
                           scen.dir[2], scen.eta0, scen.eta_amp, scen.eta_period, _ptr(T), rtol, _ptr(stats))
    if rc:
        raise RuntimeError(f"oracle sdc failed rc={rc}: " + lib().or_last_error().decode())
    return T, stats


Oracle.step_sdc = _step_sdc


def run_config(cfg, scen_index: int = 0, T_init: Optional[np.ndarray] = None, nsteps: Optional[int] = None,
               solver: str = "cg", t0: float = 0.0, guess: int = 0):
    """Oracle run of one scenario of a config from T0 (uniform) or T_init."""
    o = Oracle.from_config(cfg, guess)
    T = np.full(o.n, cfg.T0) if T_init is None else np.array(T_init, dtype=np.float64)
    return o.step(T, t0, cfg.dt, cfg.nsteps if nsteps is None else nsteps,
                  cfg.scenarios[scen_index], solver=solver)
