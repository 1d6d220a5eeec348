"""Navier-Stokes viscous fluxes and the gravity source (
S:571-588, PAPER.md eqs nsVisc/shearTensor/thermalFlux/rtSource).

CPU: the oracle against the SPEC's inline examples (uniform flow, linear
shear, constant temperature, gravity source values) and exact discrete
properties (shear-wave diffusion eigenvalue, conservation).  GPU: the C-ABI
path bit-identical to the oracle with the viscous fluxes and the source on.
"""
from dataclasses import replace

import numpy as np
import pytest

import paper_2401_16543_b200 as K
from paper_2401_16543_b200.config import GridConfig
from oracle import Oracle

GAMMA = 1.4


def cons(rho, u, v, p, w=None):
    """Conservative AoS state from primitive arrays (2-D, or 3-D with w)."""
    if w is None:
        E = p / (GAMMA - 1) + 0.5 * rho * (u * u + v * v)
        return np.stack([rho, rho * u, rho * v, E], axis=-1)
    E = p / (GAMMA - 1) + 0.5 * rho * (u * u + v * v + w * w)
    return np.stack([rho, rho * u, rho * v, rho * w, E], axis=-1)


def grid2(n=16, **kw):
    base = dict(dim=2, radius=2, nx=n, ny=n, bc="periodic", viscous=True, reynolds=10.0,
                prandtl=0.71, mach=0.5)
    base.update(kw)
    return GridConfig(**base)


def centres(n, L=1.0):
    return (np.arange(n) + 0.5) * (L / n)


# ------------------------------------------------------------------ CPU
def test_uniform_flow_has_no_viscous_flux():
    g = grid2()
    U = cons(*(np.full((16, 16), c) for c in (1.3, 0.4, -0.2, 2.0)))
    o = Oracle(g, K.precompute(2, dim=2))
    for d in (0, 1):
        assert np.array_equal(o.viscous_face(U, 5, 7, 0, d), np.zeros(4))


def test_linear_shear_stress_and_constant_temperature():
    # u = (y, 0), rho = p = 1 (T constant): sigma_xy = 1/Re, sigma_xx = 0,
    # q = 0 (S:574-576 examples); outflow so the linear field is not wrapped
    n, Re = 16, 20.0
    g = grid2(n, bc="outflow", reynolds=Re)
    y = centres(n)
    Y = np.repeat(y[:, None], n, axis=1)
    U = cons(np.ones((n, n)), Y, np.zeros((n, n)), np.ones((n, n)))
    o = Oracle(g, K.precompute(2, dim=2))
    Fx = o.viscous_face(U, 8, 6, 0, 0)   # x-face, interior
    assert Fx[0] == 0.0
    assert abs(Fx[1]) < 1e-14                       # sigma_xx
    assert abs(Fx[2] - 1.0 / Re) < 1e-12            # sigma_yx
    assert abs(Fx[3]) < 1e-14                       # q_x + sigma_xx u + sigma_xy v (v = 0)
    Fy = o.viscous_face(U, 8, 6, 0, 1)   # y-face between rows 5 and 6
    assert abs(Fy[1] - 1.0 / Re) < 1e-12            # sigma_xy
    assert abs(Fy[2]) < 1e-14                       # sigma_yy
    assert abs(Fy[3] - (1.0 / Re) * (0.5 * (y[5] + y[6]))) < 1e-12  # sigma_xy u_face, q_y = 0


def test_linear_temperature_heat_flux():
    # T = gamma Ma^2 p / rho linear in x through p: q_x = (dT/dx) / (Pr Re)
    n, Re, Pr, Ma = 16, 5.0, 0.71, 0.3
    g = grid2(n, bc="outflow", reynolds=Re, prandtl=Pr, mach=Ma)
    x = centres(n)
    P = np.repeat((1.0 + x)[None, :], n, axis=0)
    U = cons(np.ones((n, n)), np.zeros((n, n)), np.zeros((n, n)), P)
    Fx = Oracle(g, K.precompute(2, dim=2)).viscous_face(U, 7, 4, 0, 0)
    dTdx = GAMMA * Ma * Ma * 1.0
    assert abs(Fx[3] - dTdx / (Pr * Re)) < 1e-11
    assert np.abs(Fx[1:3]).max() < 1e-14


def test_shear_wave_diffusion_eigenvalue():
    # v = A sin(2 pi k x), u = 0, rho = p = 1: the inviscid RHS vanishes and
    # the viscous one is the exact second difference of the cell averages,
    # d(m_y)/dt = -(2 - 2 cos(k' Delta)) / (Delta^2 Re) m_y
    n, Re, A, kk = 32, 2.0, 1e-3, 1
    g = grid2(n, reynolds=Re)
    x = centres(n)
    V = np.repeat((A * np.sin(2 * np.pi * kk * x))[None, :], n, axis=0)
    U = cons(np.ones((n, n)), np.zeros((n, n)), V, np.ones((n, n)))
    rset = K.precompute(2, dim=2)
    L = Oracle(g, rset).compute_rhs(U)
    Li = Oracle(replace(g, viscous=False), rset).compute_rhs(U)
    dx = 1.0 / n
    lam = -(2 - 2 * np.cos(2 * np.pi * kk * dx)) / (dx * dx * Re)
    assert np.abs(Li[..., 2]).max() < 1e-12
    assert np.abs((L[..., 2] - Li[..., 2]) - lam * V).max() < 1e-10 * np.abs(lam * A)


def test_viscous_rhs_conserves_on_periodic_domain():
    w = K.baseline_config(1, n=24)
    g = replace(w.grid, viscous=True, reynolds=3.0, mach=0.4)
    U = K.initial_condition(g, w.ic)
    L = Oracle(g, K.precompute(2, dim=2)).compute_rhs(U)
    tot = np.abs(L).sum(axis=(0, 1))
    assert (np.abs(L.sum(axis=(0, 1))) <= 1e-12 * tot).all()


def test_gravity_source_values():
    # S = (0, 0, rho/Fr^2, rho v / Fr^2) from the averages (S:583-586 examples)
    n = 8
    rset = K.precompute(2, dim=2)
    g = grid2(n, viscous=False, froude=1.0)
    U = cons(np.full((n, n), 2.0), np.zeros((n, n)), np.zeros((n, n)), np.ones((n, n)))
    L = Oracle(g, rset).compute_rhs(U)
    assert np.allclose(L[..., 0], 0.0, atol=1e-13) and np.allclose(L[..., 1], 0.0, atol=1e-13)
    assert np.allclose(L[..., 2], 2.0, atol=1e-13) and np.allclose(L[..., 3], 0.0, atol=1e-13)
    g2 = grid2(n, viscous=False, froude=2.0)
    U2 = cons(np.full((n, n), 1.5), np.zeros((n, n)), np.full((n, n), 2.0), np.ones((n, n)))
    L2 = Oracle(g2, rset).compute_rhs(U2)
    assert np.allclose(L2[..., 3], 3.0 / 4.0, atol=1e-12)   # rho v = 3, Fr = 2
    assert np.allclose(L2[..., 2], 1.5 / 4.0, atol=1e-12)


def tgv(n, Ma=0.1):
    """Taylor-Green vortex on [-pi, pi]^3, point values at centres."""
    c = -np.pi + (np.arange(n) + 0.5) * (2 * np.pi / n)
    Z, Y, X = np.meshgrid(c, c, c, indexing="ij")
    s = (np.cos(2 * X) + np.cos(2 * Y)) * (np.cos(2 * Z) + 2)
    rho = 1 + GAMMA * Ma * Ma / 16 * s
    p = 1 / (GAMMA * Ma * Ma) + s / 16
    u = np.sin(X) * np.cos(Y) * np.cos(Z)
    v = -np.cos(X) * np.sin(Y) * np.cos(Z)
    return cons(rho, u, v, p, np.zeros_like(u))


def test_taylor_green_initial_dissipation_rate():
    # viscous part of d<E_k>/dt at t = 0 equals -3/(4 Re) up to the O(Delta^2)
    # of the second-order differences
    n, Re = 24, 1.0
    g = GridConfig(dim=3, radius=2, nx=n, ny=n, nz=n, bc="periodic", dx=2 * np.pi / n,
                   viscous=True, reynolds=Re, prandtl=0.71, mach=0.1)
    U = tgv(n)
    rset = K.precompute(2, dim=3)
    dL = Oracle(g, rset).compute_rhs(U) - Oracle(replace(g, viscous=False), rset).compute_rhs(U)
    rho = U[..., 0]
    vel = U[..., 1:4] / rho[..., None]
    dek = (vel * dL[..., 1:4]).sum(-1) - 0.5 * (vel * vel).sum(-1) * dL[..., 0]
    rate = dek.mean()
    assert abs(rate / (-3.0 / (4.0 * Re)) - 1.0) < 0.03, rate


# ------------------------------------------------------------------ GPU
VCASES = [
    ("2d_r2_periodic_visc", 1, 24, 3, dict(viscous=True, reynolds=50.0, mach=0.5)),
    ("2d_r2_outflow_visc_grav", 2, 24, 3, dict(viscous=True, reynolds=20.0, mach=0.3, froude=1.0)),
    ("2d_r3_periodic_visc_hll", 1, 20, 2, dict(radius=3, riemann="hll", viscous=True, reynolds=10.0)),
    ("3d_r2_periodic_visc_grav", 3, 12, 2, dict(viscous=True, reynolds=30.0, mach=0.2, froude=2.0)),
    ("3d_r2_outflow_visc", 4, 10, 2, dict(viscous=True, reynolds=8.0, mach=0.7)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,idx,n,steps,over", VCASES, ids=[c[0] for c in VCASES])
def test_viscous_gpu_parity(require_gpu, name, idx, n, steps, over):
    w = K.baseline_config(idx, n=n)
    g = replace(w.grid, **over)
    U = K.initial_condition(g, w.ic)
    rset = K.precompute(g.radius, dim=g.dim)
    o = Oracle(g, rset)
    with K.Solver(g, rset) as s:
        Lg = s.compute_rhs(U)
        s.set_state(U)
        dts = s.advance(steps)
        Ug = s.get_state()
    assert np.array_equal(Lg, o.compute_rhs(U))
    Uo, dto = o.run(U, steps)
    assert np.array_equal(dts, dto)
    assert np.array_equal(Ug, Uo)


@pytest.mark.gpu
@pytest.mark.parametrize("engine", [0, 1, 3, 4])
def test_viscous_gpu_engines_and_kxrcf(require_gpu, engine):
    w = K.baseline_config(2, n=24)
    g = replace(w.grid, viscous=True, reynolds=40.0, mach=0.4, froude=1.5)
    U = K.initial_condition(g, w.ic)
    rset = K.precompute(2, dim=2)
    Uo, dto = Oracle(g, rset).run(U, 2)
    with K.Solver(g, rset) as s:
        s.set_option("engine", engine)
        s.set_state(U)
        dts = s.advance(2)
        Ug = s.get_state()
    assert np.array_equal(dts, dto) and np.array_equal(Ug, Uo)
    gk = replace(g, kxrcf=True)
    Uk, dk = Oracle(gk, rset).run(U, 2)
    with K.Solver(gk, rset) as s:
        s.set_state(U)
        dg = s.advance(2)
        assert np.array_equal(dg, dk) and np.array_equal(s.get_state(), Uk)


@pytest.mark.gpu
def test_taylor_green_gpu_matches_oracle(require_gpu):
    n = 16
    g = GridConfig(dim=3, radius=2, nx=n, ny=n, nz=n, bc="periodic", dx=2 * np.pi / n, cfl=0.3,
                   viscous=True, reynolds=1600.0, prandtl=0.71, mach=0.1)
    U = tgv(n)
    rset = K.precompute(2, dim=3)
    Uo, dto = Oracle(g, rset).run(U, 2)
    with K.Solver(g, rset) as s:
        s.set_state(U)
        dts = s.advance(2)
        Ug = s.get_state()
    assert np.array_equal(dts, dto) and np.array_equal(Ug, Uo)
