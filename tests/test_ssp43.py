"""SSP(4,3) with the embedded SSP(3,2) and the PI step-size controller
(S:598-616): the stage formulas on linear ODEs (SPEC acceptance 8), the
controller contract on the Euler path, and — on the GPU — advance_to runs
bit-identical to the oracle (states, accepted dts, rejection counts)."""
import ctypes as C
from dataclasses import replace

import numpy as np
import pytest

import paper_2401_16543_b200 as K
from paper_2401_16543_b200.config import GridConfig, ICSpec
from oracle import kfvm_oracle as O


def _ode_step(lam, u, dt):
    """one SSP(4,3) step of u' = lam u through the oracle's stage combine;
    returns (u+, uhat)."""
    L_ = O.lib()
    n = u.size
    p = lambda a: a.ctypes.data  # noqa: E731
    y, uh = u.copy(), np.zeros(n)
    for st in (11, 12, 13, 14):
        Lv = lam * y
        out = np.empty(n)
        L_.kfo_combine43(st, n, p(u), p(y), p(Lv), dt, p(out), p(uh) if st == 13 else None)
        y = out
    return y, uh


def test_linear_ode_orders():
    """global error of order 3, embedded (local) estimate of order >= 2
    on u' = lam u (SPEC acceptance 8)."""
    lam = np.array([-1.0, -0.5 + 0.0, -2.0, 0.3])
    errs, ests = [], []
    for nsteps in (20, 40, 80):
        dt = 1.0 / nsteps
        u = np.ones(4)
        est = 0.0
        for _ in range(nsteps):
            u, uh = _ode_step(lam, u, dt)
            est = max(est, np.abs(u - uh).max())
        errs.append(np.abs(u - np.exp(lam)).max())
        ests.append(est)
    r1, r2 = np.log2(errs[0] / errs[1]), np.log2(errs[1] / errs[2])
    assert 2.9 < r1 < 3.1 and 2.9 < r2 < 3.1, (r1, r2)
    # the per-step difference u+ - uhat is O(dt^3) (a second-order embedded method)
    assert np.log2(ests[1] / ests[2]) > 2.8


def test_zero_rhs_identity():
    """L == 0 -> u+ = u and the embedded solution equals it (error 0)."""
    u = np.linspace(0.5, 2.0, 7)
    y, uh = _ode_step(0.0, u, 0.1)
    assert np.array_equal(y, u) and np.array_equal(uh, u)


def _grid(idx, n, **kw):
    w = K.baseline_config(idx, n=n)
    return w, replace(w.grid, integrator="ssp43", **kw)


def test_constant_field_no_rejections():
    g = GridConfig(dim=2, radius=2, nx=12, ny=12, integrator="ssp43", cfl=0.8)
    U = K.initial_condition(g, ICSpec("uniform", value=(1.0, 0.3, 0.2, 0.0, 1.0)))
    o = O.Oracle(g, K.precompute(2, dim=2))
    Un, dts, na, nr, t = o.advance43(U, 0.1)
    assert nr == 0 and t == 0.1 and na == len(dts)
    assert np.allclose(Un, U, rtol=0, atol=1e-13)
    assert abs(dts.sum() - 0.1) < 1e-15


def test_tolerances_control_the_step():
    """loose tolerances: CFL-limited steps; tight: the controller limits dt
    and rejects a few attempts; t_final is reached exactly."""
    w, g = _grid(1, 24, cfl=0.8)
    U = K.initial_condition(g, w.ic)
    rs = K.precompute(2, dim=2)
    _, d1, n1, r1, t1 = O.Oracle(g, rs).advance43(U, 0.02)
    _, d2, n2, r2, t2 = O.Oracle(replace(g, atol=1e-9, rtol=1e-9), rs).advance43(U, 0.02)
    assert t1 == 0.02 and t2 == 0.02 and r1 == 0
    assert n2 > 3 * n1 and d2.max() < d1.min()


@pytest.mark.gpu
@pytest.mark.parametrize("idx,n,tf,tol", [(1, 24, 0.02, 1e-4), (1, 24, 0.01, 1e-9),
                                          (2, 32, 0.01, 1e-6), (3, 10, 0.01, 1e-4),
                                          (4, 10, 0.005, 1e-7)])
def test_gpu_advance43_bitwise(require_gpu, idx, n, tf, tol):
    w, g = _grid(idx, n, atol=tol, rtol=tol)
    U = K.initial_condition(g, w.ic)
    rs = K.precompute(g.radius, dim=g.dim)
    Uo, dto, na, nr, to = O.Oracle(g, rs).advance43(U, tf)
    with K.Solver(g, rs) as s:
        s.set_state(U)
        steps, t = s.advance_to(tf, 10000)
        acc, rej = s.step_stats()
        dts = s.dt_sequence(acc)
        A = s.get_state()
    assert (acc, rej) == (na, nr) and steps == na
    assert t == to
    assert np.array_equal(dts, dto)
    assert np.array_equal(A, Uo), np.abs(A - Uo).max()
