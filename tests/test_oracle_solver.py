"""Whole-solver properties of the CPU oracle (SPEC solver invariants S:626-630,
acceptance criteria S:788-798, SURVEY §4 tiers i-iii)."""
import math

import numpy as np
import pytest

import paper_2401_16543_b200 as K
from paper_2401_16543_b200.config import GridConfig, ICSpec
from oracle import Oracle


def run(idx, n, steps, nslabs=1, over=None):
    from dataclasses import replace
    w = K.baseline_config(idx, n=n)
    g = replace(w.grid, **(over or {}))
    U = K.initial_condition(g, w.ic)
    o = Oracle(g, K.precompute(g.radius, dim=g.dim))
    return g, U, o, o.run(U, steps, nslabs)


@pytest.mark.parametrize("idx,n,steps", [(1, 24, 4), (3, 10, 2)])
def test_conservation_periodic(idx, n, steps):
    """totals of every conserved variable constant to 1e-12 relative."""
    g, U, o, (U2, _) = run(idx, n, steps)
    ax = tuple(range(U.ndim - 1))
    rel = np.abs(U2.sum(axis=ax) - U.sum(axis=ax)) / np.abs(U).sum(axis=ax)
    assert (rel < 1e-12).all(), rel


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("bc", ["periodic", "outflow"])
def test_free_stream_and_constant_rhs(dim, bc):
    """a uniform moving state is preserved exactly."""
    g = GridConfig(dim=dim, radius=2, nx=10, ny=10, nz=10 if dim == 3 else 1, bc=bc, cfl=0.3)
    U = K.initial_condition(g, ICSpec("uniform", value=(1.3, 0.7, -0.4, 0.2, 2.0)))
    o = Oracle(g, K.precompute(2, dim=dim))
    assert np.abs(o.compute_rhs(U)).max() == 0.0
    U2, _ = o.run(U, 3)
    assert np.array_equal(U2, U)


@pytest.mark.parametrize("idx,n,steps,nslabs", [(1, 20, 2, 3), (2, 20, 2, 2), (3, 10, 1, 3),
                                                (4, 10, 1, 2), (5, 10, 1, 2)])
def test_virtual_slabs_bitwise(idx, n, steps, nslabs):
    """P virtual slabs with in-memory halo copies == 1 slab."""
    g, U, o, (U1, d1) = run(idx, n, steps)
    U2, d2 = o.run(U, steps, nslabs)
    assert np.array_equal(d1, d2) and np.array_equal(U1, U2)


def test_baseline_workloads_stay_admissible():
    """Positivity stress: the discontinuous Voronoi configs (2 and 4) run their
    full step counts at reduced resolution without an inadmissible average."""
    for idx, n in ((2, 48), (4, 12)):
        w = K.baseline_config(idx, n=n)
        U = K.initial_condition(w.grid, w.ic)
        o = Oracle(w.grid, K.precompute(2, dim=w.grid.dim))
        U2, dts = o.run(U, w.steps)
        assert np.isfinite(U2).all() and (U2[..., 0] > 0).all() and (dts > 0).all()


def vortex_l1(n, R=2, cfl=0.4, t_end=20.0):
    ic = ICSpec("vortex", origin=(-10.0, -10.0, 0.0))
    g = GridConfig(dim=2, radius=R, nx=n, ny=n, bc="periodic", dx=20.0 / n, cfl=cfl)
    U0 = K.initial_condition(g, ic)
    o = Oracle(g, K.precompute(R, dim=2))
    U, t = U0.copy(), 0.0
    while t < t_end:
        dt = min(o.select_dt(U), t_end - t)
        U1 = o.stage(U, U, 1, dt)
        U2 = o.stage(U, U1, 2, dt)
        U = o.stage(U, U2, 3, dt)
        t += dt
    return np.abs(U[..., 0] - U0[..., 0]).sum() * g.dx ** 2


def test_isentropic_vortex_eoc_r2():
    """S:791 / PAPER Table 1: R=2 vortex 32^2 -> 64^2, EOC >= 2.4 (paper 2.68)."""
    e32, e64 = vortex_l1(32), vortex_l1(64)
    eoc = math.log(e32 / e64) / math.log(2)
    assert eoc >= 2.4, (e32, e64, eoc)
