"""Initial/boundary condition catalog (SPEC module `problems`, S:647-708;
PAPER.md §6.2-§6.4, §6.6) on the per-side boundary kinds of GridConfig.

Each constructor returns a Problem: the GridConfig (domain, boundary kinds per
side, gamma, Riemann solver, integrator, viscous / source parameters) and the
initial cell averages, computed from the pointwise primitive IC by the tensor
R^d Gauss-Legendre rule (init_cell_averages).  The averaging is
host-side setup (not the hot path); the GPU solver and the oracle consume the
same bytes.

Domain coordinates: the grid's low corner is ``origin``; cell (i, j) has its
centre at origin + (i + 1/2, j + 1/2) * dx.  Slit centres (GridConfig.slits)
are measured from the low corner, as in include/kfvm_b200.h.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .config import GridConfig


@dataclass(frozen=True)
class Problem:
    name: str
    grid: GridConfig
    U0: np.ndarray          # cell averages, grid.shape + (nvar,)
    t_final: float
    origin: tuple = (0.0, 0.0, 0.0)


def cons(gamma: float, rho, vel, p) -> np.ndarray:
    """Conservative state(s) from primitives: (rho, rho u, E)."""
    rho = np.asarray(rho, dtype=np.float64)
    vel = [np.asarray(v, dtype=np.float64) for v in vel]
    ke = sum(0.5 * rho * v * v for v in vel)
    return np.stack([rho] + [rho * v for v in vel] + [p / (gamma - 1.0) + ke], axis=-1)


def cell_averages(grid: GridConfig, origin, prim) -> np.ndarray:
    """Tensor R^d Gauss-Legendre cell averages of the conservative state of
    ``prim(x, y[, z]) -> (rho, (u, v[, w]), p)`` (pointwise, vectorised)."""
    R, d = grid.radius, grid.dim
    dx = float(grid.dx if grid.dx is not None else 1.0 / grid.nx)
    xg, wg = np.polynomial.legendre.leggauss(R)
    xg, wg = 0.5 * xg, 0.5 * wg          # nodes on [-1/2, 1/2], weights sum to 1
    n = (grid.nx, grid.ny, grid.nz)[:d]
    centres = [origin[a] + (np.arange(n[a]) + 0.5) * dx for a in range(d)]
    out = np.zeros(grid.shape + (grid.nvar,))
    for idx in np.ndindex(*([R] * d)):
        w = float(np.prod([wg[i] for i in idx]))
        pts = [centres[a] + xg[idx[a]] * dx for a in range(d)]
        mesh = np.meshgrid(*pts[::-1], indexing="ij")[::-1]   # arrays shaped grid.shape
        rho, vel, p = prim(*mesh)
        U = cons(grid.gamma, rho, vel, p)
        if not (np.all(U[..., 0] > 0) and np.all(np.asarray(p) > 0)):
            raise ValueError("inadmissible IC point (S:545)")
        out += w * U
    return out


def _grid(**kw) -> GridConfig:
    return GridConfig(**kw)


def sod_aligned(n: int = 100, radius: int = 2, ny: int = 4) -> Problem:
    """Sod: Omega = [0,1] x [0, ny/n], outflow in x, periodic in y,
    left (1,0,0,1) for x < 0.5, right (0.125,0,0,0.1), t_final = 0.2."""
    g = _grid(dim=2, radius=radius, nx=n, ny=ny, dx=1.0 / n, cfl=1.25,
              sides=("outflow", "outflow", "periodic", "periodic"),
              integrator="ssp43", atol=1e-4, rtol=1e-4)
    def prim(x, y):
        left = x < 0.5
        return (np.where(left, 1.0, 0.125), (0 * x, 0 * x), np.where(left, 1.0, 0.1))
    return Problem("sod_aligned", g, cell_averages(g, (0, 0, 0), prim), 0.2)


def richtmyer_meshkov(n: int = 32, radius: int = 2, ma: float = 3.0, rho_d: float = 2.0,
                      gamma: float = 1.4) -> Problem:
    """Richtmyer-Meshkov (PAPER §6.3): Omega = [-1/2, 11/2] x [0, 1],
    dx = 1/n; fixed post-shock inflow (dirichlet) at x = -1/2, outflow at
    x = 11/2, reflecting in y.  Piecewise IC, conditions in listed order (first
    match wins): x < 0.2 shocked gas; x < y: rho = 1; else rho_D."""
    rho_s = 1.0 / (1.0 - (2.0 / (gamma + 1.0)) * (1.0 - 1.0 / (ma * ma)))
    p_s = 1.0 + (2.0 * gamma / (gamma + 1.0)) * (ma * ma - 1.0)
    u_s = ma * math.sqrt(gamma) * (1.0 - 1.0 / rho_s)
    inflow = tuple(cons(gamma, rho_s, (u_s, 0.0), p_s))
    g = _grid(dim=2, radius=radius, nx=6 * n, ny=n, dx=1.0 / n, gamma=gamma, cfl=1.0,
              sides=("dirichlet", "outflow", "reflecting", "reflecting"),
              side_states=(inflow, None, None, None),
              integrator="ssp43", atol=1e-3, rtol=1e-3)

    def prim(x, y):
        shocked = x < 0.2
        rho = np.where(shocked, rho_s, np.where(x < y, 1.0, rho_d))
        p = np.where(shocked, p_s, 1.0)
        u = np.where(shocked, u_s, 0.0)
        return rho, (u, 0 * x), p
    org = (-0.5, 0.0, 0.0)
    return Problem("richtmyer_meshkov", g, cell_averages(g, org, prim), 3.33, org)


def astro_jet(kind: str = "high", n: int = 64, radius: int = 3, gamma: float = 1.4) -> Problem:
    """Astrophysical jets (PAPER §6.4): Omega = [0,1/2] x [0,3/2],
    dx = 1/n; reflecting at x = 0, outflow at x = 1/2 and y = 3/2, slit inflow
    at y = 0 where x^2 < 0.05^2 (outflow elsewhere on that side).  Jet
    (rho, p) = (gamma, 1); high: v_jet = 800 into (gamma/10, 0, 0, 1),
    t_final = 0.002; low: v_jet = 100 into (10 gamma, 0, 0, 1), t_final = 0.04.
    HLL, SSP(4,3,2) with atol = rtol = 1e-2, CFL 1.0."""
    if kind not in ("high", "low"):
        raise ValueError("kind must be high or low")
    v_jet, rho_a, t_final = (800.0, gamma / 10.0, 0.002) if kind == "high" else (100.0, 10.0 * gamma, 0.04)
    jet = tuple(cons(gamma, gamma, (0.0, v_jet), 1.0))
    if n % 2:
        raise ValueError("n must be even (nx = n/2)")
    g = _grid(dim=2, radius=radius, nx=n // 2, ny=3 * n // 2, dx=1.0 / n, gamma=gamma,
              riemann="hll", cfl=1.0, integrator="ssp43", atol=1e-2, rtol=1e-2,
              sides=("reflecting", "outflow", "slit", "outflow"),
              side_states=(None, None, jet, None),
              slits=(None, None, ((0.0,), 0.05), None))

    def prim(x, y):
        return rho_a + 0 * x, (0 * x, 0 * x), 1.0 + 0 * x
    return Problem(f"astro_jet_{kind}", g, cell_averages(g, (0, 0, 0), prim), t_final)


def rayleigh_taylor(n: int = 64, radius: int = 3, gamma: float = 5.0 / 3.0, froude: float = 1.0,
                    reynolds: float = 20000.0, prandtl: float = 0.71, mach: float = 1.0) -> Problem:
    """Viscous Rayleigh-Taylor (PAPER §6.6): Omega = [0,1/4] x [0,1],
    dx = 1/n; rho = 2 below y = 1/2, 1 above; p per the piecewise hydrostatic
    profile; v = -0.025 sqrt(gamma p / rho) cos(8 pi x); reflecting in x;
    y boundaries held at the initial density and pressure with zero velocity
    (dirichlet); gravity +y with 1/Fr^2.  The temperature scale Ma (T = gamma
    Ma^2 p / rho) is not stated for this problem; Ma = 1 here."""
    if n % 4:
        raise ValueError("n must be a multiple of 4 (nx = n/4)")
    f2 = 1.0 / (froude * froude)
    rho_hi, rho_lo = 2.0, 1.0

    def pres(y):
        return np.where(y < 0.5, rho_hi * f2 * y + 1.0,
                        f2 * (y * rho_lo - (rho_hi - rho_lo) / 2.0) + 1.0)
    bottom = tuple(cons(gamma, rho_hi, (0.0, 0.0), float(pres(np.float64(0.0)))))
    top = tuple(cons(gamma, rho_lo, (0.0, 0.0), float(pres(np.float64(1.0)))))
    g = _grid(dim=2, radius=radius, nx=n // 4, ny=n, dx=1.0 / n, gamma=gamma, cfl=1.0,
              sides=("reflecting", "reflecting", "dirichlet", "dirichlet"),
              side_states=(None, None, bottom, top),
              viscous=True, reynolds=reynolds, prandtl=prandtl, mach=mach, froude=froude,
              integrator="ssp43", atol=1e-3, rtol=1e-3)

    def prim(x, y):
        rho = np.where(y < 0.5, rho_hi, rho_lo)
        p = pres(y)
        v = -0.025 * np.sqrt(gamma * p / rho) * np.cos(8.0 * math.pi * x)
        return rho, (0 * x, v), p
    return Problem("rayleigh_taylor", g, cell_averages(g, (0, 0, 0), prim), 2.5)


CATALOG = {
    "sod_aligned": sod_aligned,
    "richtmyer_meshkov": richtmyer_meshkov,
    "astro_jet_high": lambda **kw: astro_jet("high", **kw),
    "astro_jet_low": lambda **kw: astro_jet("low", **kw),
    "rayleigh_taylor": rayleigh_taylor,
}


def problem(name: str, **kw) -> Problem:
    """Problems addressable by name."""
    if name not in CATALOG:
        raise KeyError(f"unknown problem {name!r}; known: {sorted(CATALOG)}")
    return CATALOG[name](**kw)
