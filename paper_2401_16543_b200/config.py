"""Run configuration and the BASELINE.json workloads.

GridConfig mirrors the solver subset of RunConfig and maps
onto ``kfvm_config`` in include/kfvm_b200.h.  BASELINE_CONFIGS pins the five
BASELINE.json configs; their IC recipes are completed by the pinned choices
documented in DESIGN.md §6 (seeds below, splitmix64, max|s| over every GL
point of the global grid, minimum-image sphere).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field, replace

import numpy as np

from . import _abi


_BC_KINDS = {"periodic": _abi.BC_PERIODIC, "outflow": _abi.BC_OUTFLOW,
             "reflecting": _abi.BC_REFLECTING, "dirichlet": _abi.BC_DIRICHLET,
             "slit": _abi.BC_SLIT}


@dataclass(frozen=True)
class GridConfig:
    dim: int = 2
    radius: int = 2
    nx: int = 64
    ny: int = 64
    nz: int = 1
    bc: str = "periodic"        # "periodic" | "outflow" | "reflecting": every side
    # per-side kinds (BoundaryKind S:534-537), order x-lo, x-hi, y-lo, y-hi
    # [, z-lo, z-hi]; each "periodic" | "outflow" | "reflecting" | "dirichlet"
    # | "slit".  None = `bc` on every side.
    sides: tuple | None = None
    side_states: tuple | None = None  # per side: conservative state (dirichlet, slit inflow) or None
    slits: tuple | None = None        # per side: (centre (tangential axes), radius) or None
    riemann: str = "hllc"       # "hllc" | "hll"   (riemann.solver)
    dx: float | None = None     # defaults to 1/nx (unit domain)
    gamma: float = 1.4
    cfl: float = 1.0            # S:728 default
    eps: float = 1e-40
    kappa: float = 0.4          # limiter.kappa
    flattener_kf: float = 0.33  # limiter.flattener_kf
    ell_over_delta: float = 5.0
    kxrcf: bool = False         # kxrcf.enabled: WENO only in flagged cells
    kxrcf_m: float = 1.5        # kxrcf.m
    integrator: str = "ssprk3"  # "ssprk3" (BASELINE) | "ssp43" (adaptive)
    atol: float = 1e-4
    rtol: float = 1e-4
    safety: float = 0.9
    dt_min: float = 0.0         # 0 = none
    dt_max: float = 0.0         # 0 = none
    viscous: bool = False       # Navier-Stokes fluxes
    reynolds: float = 1.0       # Re
    prandtl: float = 0.71       # Pr
    mach: float = 1.0           # Ma: T = gamma Ma^2 p / rho
    froude: float | None = None  # gravity source 1/Fr^2 along +y (P eq rtSource); None = off

    def __post_init__(self):
        if self.dim not in (2, 3):
            raise ValueError("dim must be 2 or 3")
        if self.radius not in (2, 3):
            raise ValueError("unsupported stencil radius (must be 2 or 3)")
        if self.bc not in ("periodic", "outflow", "reflecting"):
            raise ValueError("bc must be periodic, outflow or reflecting")
        if self.sides is not None:
            ns = 2 * self.dim
            if len(self.sides) != ns or any(k not in _BC_KINDS for k in self.sides):
                raise ValueError(f"sides needs {ns} kinds from {sorted(_BC_KINDS)}")
            for a in range(self.dim):
                if (self.sides[2 * a] == "periodic") != (self.sides[2 * a + 1] == "periodic"):
                    raise ValueError("periodic sides come in matching pairs (S:536)")
            for q, k in enumerate(self.sides):
                st = self.side_states[q] if self.side_states else None
                if k in ("dirichlet", "slit") and (st is None or len(st) != self.nvar):
                    raise ValueError(f"side {q} ({k}) needs a {self.nvar}-component state")
                if k == "slit" and not (self.slits and self.slits[q] and self.slits[q][1] > 0):
                    raise ValueError(f"side {q} needs a slit (centre, radius > 0)")
        if self.integrator not in ("ssprk3", "ssp43"):
            raise ValueError("integrator must be ssprk3 or ssp43")
        if self.riemann not in ("hllc", "hll"):
            raise ValueError("riemann must be hllc or hll")
        if self.viscous and not (self.reynolds > 0 and self.prandtl > 0 and self.mach > 0):
            raise ValueError("viscous terms need Re, Pr, Ma > 0")
        if self.froude is not None and not self.froude > 0:
            raise ValueError("froude must be positive")
        if min(self.nx, self.ny, self.nz) < 1:
            raise ValueError("grid extents must be positive")

    @property
    def nvar(self) -> int:
        return self.dim + 2

    @property
    def ncells(self) -> int:
        return self.nx * self.ny * (self.nz if self.dim == 3 else 1)

    @property
    def shape(self) -> tuple:
        return (self.nz, self.ny, self.nx) if self.dim == 3 else (self.ny, self.nx)

    @property
    def slab_extent(self) -> int:
        return self.nz if self.dim == 3 else self.ny

    def c_config(self) -> _abi.KfvmConfig:
        c = _abi.KfvmConfig()
        c.dim, c.radius = self.dim, self.radius
        c.nx, c.ny, c.nz = self.nx, self.ny, (self.nz if self.dim == 3 else 1)
        c.bc = _BC_KINDS[self.bc]
        if self.sides is not None:
            c.bc_per_side = 1
            for q, k in enumerate(self.sides):
                c.bc_side[q] = _BC_KINDS[k]
                st = self.side_states[q] if self.side_states else None
                if st is not None:
                    for v, x in enumerate(st):
                        c.bc_state[q][v] = float(x)
                sl = self.slits[q] if self.slits else None
                if sl is not None:
                    for m, x in enumerate(sl[0]):
                        c.slit_center[q][m] = float(x)
                    c.slit_radius[q] = float(sl[1])
        c.riemann = _abi.RIEMANN_HLLC if self.riemann == "hllc" else _abi.RIEMANN_HLL
        c.dx = float(self.dx if self.dx is not None else 1.0 / self.nx)
        c.gamma, c.cfl, c.eps = self.gamma, self.cfl, self.eps
        c.kappa, c.flattener_kf = self.kappa, self.flattener_kf
        c.kxrcf, c.kxrcf_m = int(bool(self.kxrcf)), float(self.kxrcf_m)
        c.integrator = 1 if self.integrator == "ssp43" else 0
        c.atol, c.rtol, c.safety = self.atol, self.rtol, self.safety
        c.dt_min, c.dt_max = self.dt_min, self.dt_max
        c.viscous = int(bool(self.viscous))
        c.reynolds, c.prandtl, c.mach = float(self.reynolds), float(self.prandtl), float(self.mach)
        c.inv_froude2 = 0.0 if self.froude is None else 1.0 / (float(self.froude) * float(self.froude))
        return c


@dataclass(frozen=True)
class ICSpec:
    kind: str                 # fourier | voronoi | fourier_sphere | uniform | vortex | density_wave
    seed: int = 0
    n_modes: int = 8
    n_regions: int = 16
    origin: tuple = (0.0, 0.0, 0.0)
    value: tuple = (1.0, 0.0, 0.0, 0.0, 1.0)

    def c_params(self) -> _abi.KfvmIcParams:
        kinds = {"fourier": _abi.IC_FOURIER, "voronoi": _abi.IC_VORONOI,
                 "fourier_sphere": _abi.IC_FOURIER_SPHERE, "uniform": _abi.IC_UNIFORM,
                 "vortex": _abi.IC_VORTEX, "density_wave": _abi.IC_DENSITY_WAVE}
        p = _abi.KfvmIcParams()
        p.kind = kinds[self.kind]
        p.n_modes, p.n_regions, p.seed = self.n_modes, self.n_regions, self.seed
        for i in range(3):
            p.origin[i] = float(self.origin[i])
        for i in range(5):
            p.value[i] = float(self.value[i])
        return p


@dataclass(frozen=True)
class Workload:
    index: int
    grid: GridConfig
    ic: ICSpec
    steps: int
    text: str = ""


def _wl(index, dim, n, bc, radius, cfl, steps, ic):
    g = GridConfig(dim=dim, radius=radius, nx=n, ny=n, nz=(n if dim == 3 else 1), bc=bc, cfl=cfl)
    return Workload(index, g, ic, steps)


# BASELINE.json "configs" (1-based index as in SURVEY.md §8(d))
BASELINE_CONFIGS = {
    1: _wl(1, 2, 256, "periodic", 2, 0.4, 20, ICSpec("fourier", seed=0x5EED0001, n_modes=8)),
    2: _wl(2, 2, 1024, "outflow", 2, 0.4, 50, ICSpec("voronoi", seed=0x5EED0002, n_regions=16)),
    3: _wl(3, 3, 256, "periodic", 2, 0.3, 10, ICSpec("fourier", seed=0x5EED0003, n_modes=12)),
    4: _wl(4, 3, 512, "outflow", 2, 0.3, 10, ICSpec("voronoi", seed=0x5EED0004, n_regions=64)),
    5: _wl(5, 3, 1024, "periodic", 3, 0.3, 5, ICSpec("fourier_sphere", seed=0x5EED0005, n_modes=12)),
}


def baseline_config(index: int, n: int | None = None, nz: int | None = None) -> Workload:
    """Config `index` of BASELINE.json, optionally at a reduced resolution n
    (same recipe, same seed; used for parity cases and CPU samples)."""
    w = BASELINE_CONFIGS[index]
    if n is None and nz is None:
        return w
    g = w.grid
    n = n or g.nx
    nzz = nz if nz is not None else (n if g.dim == 3 else 1)
    return replace(w, grid=replace(g, nx=n, ny=n, nz=nzz, dx=1.0 / n))


def initial_condition(grid: GridConfig, ic: ICSpec, z0: int = 0, nz_local: int | None = None,
                      nthreads: int | None = None) -> np.ndarray:
    """Cell averages (AoS, shape grid.shape + (nvar,)) of the seeded IC on the
    slab-axis planes [z0, z0+nz_local)."""
    L = _abi.lib()
    nzl = grid.slab_extent - z0 if nz_local is None else nz_local
    plane = grid.nx * (grid.ny if grid.dim == 3 else 1)
    U = np.empty(plane * nzl * grid.nvar, dtype=np.float64)
    cfg = grid.c_config()
    p = ic.c_params()
    nt = nthreads or min(32, os.cpu_count() or 1)
    rc = L.kfvm_ic_generate(C.byref(cfg), C.byref(p), z0, nzl, nt, U.ctypes.data)
    if rc:
        raise ValueError(f"kfvm_ic_generate failed with code {rc}")
    shp = ((nzl, grid.ny, grid.nx) if grid.dim == 3 else (nzl, grid.nx)) + (grid.nvar,)
    return U.reshape(shp)
