"""ctypes wrapper of oracle/libkfvm_oracle.so (TEST INFRASTRUCTURE ONLY).

The oracle consumes the same table bytes (kfvm_table) and configuration
(kfvm_config) as the GPU path; those are inputs, described by the public
header include/kfvm_b200.h.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2401_16543_b200 import _abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkfvm_oracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-C", os.path.dirname(_HERE), "oracle/libkfvm_oracle.so"],
                           check=True, capture_output=True)
        L = C.CDLL(LIB_PATH)
        P, D, I = C.c_void_p, C.POINTER(C.c_double), C.c_int
        # tables as plain pointers: ReconstructionSet and oracle.table_file
        # structs both pass (whatever module instance defined their class)
        T, CF = C.c_void_p, C.POINTER(_abi.KfvmConfig)
        sig = {
            "kfo_rhs": (I, [CF, T, P, P, I]),
            "kfo_states": (I, [CF, T, P, P, I]),
            "kfo_select_dt": (I, [CF, P, D]),
            "kfo_stage": (I, [CF, T, P, P, P, I, C.c_double, I]),
            "kfo_run": (I, [CF, T, P, I, P, I, I]),
            "kfo_sample_stage": (I, [CF, T, P, I, I, I, D]),
            "kfo_slab_rhs": (I, [CF, T, I, I, P, P, I]),
            "kfo_max_speed": (C.c_double, [CF, P, C.c_longlong]),
            "kfo_fill_ghost": (I, [CF, P, P]),
            "kfo_combine": (None, [I, C.c_longlong, P, P, P, C.c_double, P]),
            "kfo_pressure": (C.c_double, [I, P, C.c_double]),
            "kfo_sound_speed": (C.c_double, [I, P, C.c_double]),
            "kfo_transform": (None, [I, P, C.c_double, P, P]),
            "kfo_to_recon": (None, [I, P, C.c_double, P, P]),
            "kfo_from_recon": (None, [I, P, C.c_double, P, P]),
            "kfo_riemann": (None, [I, I, I, P, P, C.c_double, P]),
            "kfo_wavespeeds": (None, [I, I, P, P, C.c_double, P]),
            "kfo_exact_flux": (None, [I, I, P, C.c_double, P]),
            "kfo_weno": (None, [T, C.c_double, C.c_double, P, P, P, P]),
            "kfo_limit": (I, [I, I, P, P, C.c_double, C.c_double, C.c_double, P]),
            "kfo_kxrcf_flags": (I, [CF, T, P, P, I]),
            "kfo_advance43": (I, [CF, T, P, C.c_double, I, P, I, P, D, I]),
            "kfo_pow": (C.c_double, [C.c_double, C.c_double]),
            "kfo_viscous_face": (None, [CF, P, I, I, I, I, P]),
            "kfo_combine43": (None, [I, C.c_longlong, P, P, P, C.c_double, P, P]),
            "kfo_ic_generate": (I, [CF, C.POINTER(_abi.KfvmIcParams), I, I, I, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data


class Oracle:
    """Whole-grid oracle operations for one GridConfig + ReconstructionSet."""

    def __init__(self, grid, rset, nthreads: int | None = None):
        self.L = lib()
        self.grid, self.rset = grid, rset
        self.cfg = grid.c_config()
        self.nthreads = nthreads or min(32, os.cpu_count() or 1)

    def _chk(self, rc, what):
        if rc:
            raise RuntimeError(f"oracle {what} failed with code {rc}")

    def compute_rhs(self, U):
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        self._chk(self.L.kfo_rhs(C.byref(self.cfg), self.rset.c_table, _p(U), _p(out),
                                 self.nthreads), "rhs")
        return out

    def reconstruct_states(self, U):
        U = np.ascontiguousarray(U, dtype=np.float64)
        n = self.grid.ncells
        out = np.empty((n, self.rset.n_face_points(), self.grid.nvar))
        self._chk(self.L.kfo_states(C.byref(self.cfg), self.rset.c_table, _p(U), _p(out),
                                    self.nthreads), "states")
        return out

    def kxrcf_flags(self, U):
        """KXRCF flags (1 = WENO) of every cell, shape of the grid."""
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.zeros(self.grid.shape, dtype=np.uint8)
        self._chk(self.L.kfo_kxrcf_flags(C.byref(self.cfg), self.rset.c_table, _p(U), _p(out),
                                         self.nthreads), "kxrcf_flags")
        return out

    def viscous_face(self, U, i, j, k, d):
        """F^(v) of the face between global cells (i,j,k) - e_d and (i,j,k)."""
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.zeros(self.grid.nvar)
        self.L.kfo_viscous_face(C.byref(self.cfg), _p(U), int(i), int(j), int(k), int(d), _p(out))
        return out

    def select_dt(self, U):
        U = np.ascontiguousarray(U, dtype=np.float64)
        dt = C.c_double()
        self._chk(self.L.kfo_select_dt(C.byref(self.cfg), _p(U), C.byref(dt)), "select_dt")
        return dt.value

    def stage(self, U0, Uk, stage, dt):
        U0 = np.ascontiguousarray(U0, dtype=np.float64)
        Uk = np.ascontiguousarray(Uk, dtype=np.float64)
        out = np.empty_like(U0)
        self._chk(self.L.kfo_stage(C.byref(self.cfg), self.rset.c_table, _p(U0), _p(Uk), _p(out),
                                   int(stage), float(dt), self.nthreads), "stage")
        return out

    def run(self, U, nsteps, nslabs: int = 1):
        U = np.array(U, dtype=np.float64, copy=True, order="C")
        dts = np.empty(max(nsteps, 1))
        self._chk(self.L.kfo_run(C.byref(self.cfg), self.rset.c_table, _p(U), int(nsteps),
                                 _p(dts), int(nslabs), self.nthreads), "run")
        return U, dts[:nsteps]

    def advance43(self, U, t_final, max_attempts=1000, cap=4096):
        """SSP(4,3)+SSP(3,2) with the PI controller to t_final: returns
        (U, accepted dts, n_accepted, n_rejected, t_reached)."""
        U = np.array(U, dtype=np.float64, copy=True, order="C")
        dts = np.zeros(cap)
        st = np.zeros(2, dtype=np.int32)
        tr = C.c_double()
        self._chk(self.L.kfo_advance43(C.byref(self.cfg), self.rset.c_table, _p(U),
                                       float(t_final), int(max_attempts), _p(dts), int(cap),
                                       _p(st), C.byref(tr), self.nthreads), "advance43")
        return U, dts[:min(int(st[0]), cap)], int(st[0]), int(st[1]), tr.value

    def slab_rhs(self, U_local, p0, np_planes):
        """RHS of planes [p0, p0+np) from the slab's array incl. R+1 halo planes."""
        U_local = np.ascontiguousarray(U_local, dtype=np.float64)
        H = self.grid.radius + 1
        out = np.empty((np_planes,) + U_local.shape[1:])
        assert U_local.shape[0] == np_planes + 2 * H
        self._chk(self.L.kfo_slab_rhs(C.byref(self.cfg), self.rset.c_table, int(p0),
                                      int(np_planes), _p(U_local), _p(out), self.nthreads), "slab_rhs")
        return out

    def fill_ghost(self, U):
        """The domain padded with R+1 ghost cells per side (fill_ghost,
        S:553-561), shape (n_z+2H,) n_y+2H, n_x+2H, nvar."""
        g = self.grid
        H = g.radius + 1
        shape = tuple(n + 2 * H for n in g.shape) + (g.nvar,)
        out = np.zeros(shape)
        U = np.ascontiguousarray(U, dtype=np.float64)
        self._chk(lib().kfo_fill_ghost(C.byref(self.cfg), _p(U), _p(out)), "fill_ghost")
        return out

    def max_speed(self, U):
        U = np.ascontiguousarray(U, dtype=np.float64)
        return self.L.kfo_max_speed(C.byref(self.cfg), _p(U), U.size // self.grid.nvar)

    def combine(self, stage, U0, Uk, L, dt):
        U0, Uk, L = (np.ascontiguousarray(a, dtype=np.float64) for a in (U0, Uk, L))
        out = np.empty_like(U0)
        self.L.kfo_combine(int(stage), U0.size, _p(U0), _p(Uk), _p(L), float(dt), _p(out))
        return out

    def sample_stage_seconds(self, U, p0, np_planes):
        U = np.ascontiguousarray(U, dtype=np.float64)
        sec = C.c_double()
        self._chk(self.L.kfo_sample_stage(C.byref(self.cfg), self.rset.c_table, _p(U), int(p0),
                                          int(np_planes), self.nthreads, C.byref(sec)), "sample")
        return sec.value


def initial_condition(grid, ic, z0: int = 0, nz_local: int | None = None,
                      nthreads: int | None = None) -> np.ndarray:
    """The seeded BASELINE IC from the oracle's own restatement
    (kfvm_oracle_ic.cpp): same shape and bytes as
    paper_2401_16543_b200.initial_condition, without the product library."""
    nzl = grid.slab_extent - z0 if nz_local is None else nz_local
    plane = grid.nx * (grid.ny if grid.dim == 3 else 1)
    U = np.empty(plane * nzl * grid.nvar, dtype=np.float64)
    cfg = grid.c_config()
    p = ic.c_params()
    nt = nthreads or min(64, os.cpu_count() or 1)
    rc = lib().kfo_ic_generate(C.byref(cfg), C.byref(p), int(z0), int(nzl), int(nt), _p(U))
    if rc:
        raise ValueError(f"kfo_ic_generate failed with code {rc}")
    shp = ((nzl, grid.ny, grid.nx) if grid.dim == 3 else (nzl, grid.nx)) + (grid.nvar,)
    return U.reshape(shp)


class _PointAPI:
    """Single-point oracle functions (SPEC known-answer tests)."""

    def pressure(self, U, gamma=1.4):
        U = np.ascontiguousarray(U, dtype=np.float64)
        return lib().kfo_pressure(len(U) - 2, _p(U), gamma)

    def sound_speed(self, U, gamma=1.4):
        U = np.ascontiguousarray(U, dtype=np.float64)
        return lib().kfo_sound_speed(len(U) - 2, _p(U), gamma)

    def transform(self, Uref, gamma=1.4):
        Uref = np.ascontiguousarray(Uref, dtype=np.float64)
        n = len(Uref)
        phi, inv = np.zeros((n, n)), np.zeros((n, n))
        lib().kfo_transform(n - 2, _p(Uref), gamma, _p(phi), _p(inv))
        return phi, inv

    def to_recon(self, Uref, U, gamma=1.4):
        Uref = np.ascontiguousarray(Uref, dtype=np.float64)
        U = np.ascontiguousarray(U, dtype=np.float64)
        W = np.zeros_like(U)
        lib().kfo_to_recon(len(U) - 2, _p(Uref), gamma, _p(U), _p(W))
        return W

    def from_recon(self, Uref, W, gamma=1.4):
        Uref = np.ascontiguousarray(Uref, dtype=np.float64)
        W = np.ascontiguousarray(W, dtype=np.float64)
        U = np.zeros_like(W)
        lib().kfo_from_recon(len(W) - 2, _p(Uref), gamma, _p(W), _p(U))
        return U

    def riemann(self, UL, UR, axis=0, solver="hllc", gamma=1.4):
        UL = np.ascontiguousarray(UL, dtype=np.float64)
        UR = np.ascontiguousarray(UR, dtype=np.float64)
        F = np.zeros_like(UL)
        lib().kfo_riemann(len(UL) - 2, 0 if solver == "hllc" else 1, axis, _p(UL), _p(UR),
                          gamma, _p(F))
        return F

    def wavespeeds(self, UL, UR, axis=0, gamma=1.4):
        UL = np.ascontiguousarray(UL, dtype=np.float64)
        UR = np.ascontiguousarray(UR, dtype=np.float64)
        out = np.zeros(3)
        lib().kfo_wavespeeds(len(UL) - 2, axis, _p(UL), _p(UR), gamma, _p(out))
        return out

    def exact_flux(self, U, axis=0, gamma=1.4):
        U = np.ascontiguousarray(U, dtype=np.float64)
        F = np.zeros_like(U)
        lib().kfo_exact_flux(len(U) - 2, axis, _p(U), gamma, _p(F))
        return F

    def weno(self, rset, g, dx=1.0, eps=1e-40):
        g = np.ascontiguousarray(g, dtype=np.float64)
        beta = np.zeros(rset.n_stencils)
        omega = np.zeros(rset.n_stencils)
        vals = np.zeros(rset.n_face_points())
        lib().kfo_weno(rset.c_table, dx, eps, _p(g), _p(beta), _p(omega), _p(vals))
        return beta, omega, vals

    def limit(self, states, nbr, gamma=1.4, kappa=0.4, kf=0.33):
        st = np.array(states, dtype=np.float64, copy=True, order="C")
        nbr = np.ascontiguousarray(nbr, dtype=np.float64)
        info = np.zeros(6)
        rc = lib().kfo_limit(st.shape[1] - 2, st.shape[0], _p(st), _p(nbr), gamma, kappa, kf,
                             _p(info))
        return rc, st, dict(zip(("eta", "rho_min", "rho_max", "p_min", "theta_rho", "theta_p"),
                                info))


point_api = _PointAPI()
