"""CPU oracle point functions against the SPEC known answers and invariants
(weno S:241-300, euler_state S:302-384, limiters S:410-464, riemann
S:466-519, select_dt S:607-615)."""
import json
import math
import os

import numpy as np
import pytest

import paper_2401_16543_b200 as K
from paper_2401_16543_b200.config import GridConfig, ICSpec
from oracle import Oracle, point_api as P

HERE = os.path.dirname(os.path.abspath(__file__))
SPEC = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))
G = 1.4
rng = np.random.default_rng(1234)


def prim_to_cons(r, vel, p, g=G):
    vel = np.asarray(vel, dtype=float)
    return np.array([r, *(r * vel), p / (g - 1) + 0.5 * r * vel @ vel])


def rand_state(dim):
    r = rng.uniform(0.2, 3.0)
    return prim_to_cons(r, rng.uniform(-2, 2, dim), rng.uniform(0.2, 5.0))


# ------------------------------------------------------------ euler_state
def test_pressure_and_sound_speed():
    e = SPEC["euler"]
    # gamma - 1 is evaluated in FP64 (0.3999999999999999), hence approx
    assert P.pressure(e["pressure_unit"]["U"]) == pytest.approx(e["pressure_unit"]["p"], rel=1e-15)
    assert P.sound_speed(e["sound_unit"]["U"]) == pytest.approx(e["sound_unit"]["c"], rel=1e-15)
    U = prim_to_cons(G, [0, 0], 1.0)
    assert P.sound_speed(U) == pytest.approx(1.0, rel=1e-15)
    # Sod left state: E = 2.5; boost leaves p unchanged
    assert prim_to_cons(1.0, [0, 0], 1.0)[3] == pytest.approx(2.5, rel=1e-15)
    assert P.pressure(prim_to_cons(1.0, [0.7, 0], 1.0)) == pytest.approx(1.0, rel=1e-15)


def test_exact_flux():
    U = prim_to_cons(1.3, [0, 0], 2.0)
    assert P.exact_flux(U, 0).tolist() == pytest.approx([0, 2.0, 0, 0])
    U = rand_state(2)
    assert P.exact_flux(U, 0)[0] == U[1]
    assert P.exact_flux(U, 1)[0] == U[2]


def test_transform_known_answers_and_round_trip():
    e = SPEC["euler"]
    phi, inv = P.transform(np.array(e["phi_zero_velocity_energy_row"]["Uref"]))
    assert phi[3].tolist() == pytest.approx(e["phi_zero_velocity_energy_row"]["row"], abs=1e-15)
    phi, inv = P.transform(np.array(e["phi_inv_energy_row"]["Uref"]))
    assert inv[3].tolist() == pytest.approx(e["phi_inv_energy_row"]["row"], abs=1e-15)
    for dim in (2, 3):
        worst_i, worst_rt = 0.0, 0.0
        for _ in range(2000):
            Ur = rand_state(dim)
            phi, inv = P.transform(Ur)
            worst_i = max(worst_i, np.abs(phi @ inv - np.eye(dim + 2)).max())
            U = rand_state(dim)
            back = P.from_recon(Ur, P.to_recon(Ur, U))
            worst_rt = max(worst_rt, (np.abs(back - U) / np.abs(U).max()).max())
            # sparsity pattern of the Appendix matrices
            assert np.count_nonzero(phi[0]) == 1 and np.count_nonzero(inv[0]) == 1
        assert worst_i < 1e-12 and worst_rt < 1e-12


# ------------------------------------------------------------------- weno
def mavg_1d(c, k):
    return ((c + 0.5) ** (k + 1) - (c - 0.5) ** (k + 1)) / (k + 1)


@pytest.mark.parametrize("dim,R", [(2, 2), (2, 3), (3, 2)])
def test_weno_known_answers(dim, R):
    rs = K.precompute(R, dim=dim)
    n0 = rs.st[0].count
    beta, om, vals = P.weno(rs, np.full(n0, 3.25))
    # constant data -> beta = 0 up to the rounding of sum_h d_h (~1e-16 g)
    assert np.all(beta < 1e-25)
    assert np.allclose(vals, 3.25, rtol=0, atol=1e-13)
    # equal beta -> omega = gamma: exact when the betas are exactly equal
    _, om_eq, _ = P.weno(rs, np.zeros(n0))
    assert om_eq == pytest.approx(rs.gamma, rel=1e-14)
    g = rng.normal(size=n0)
    b1, o1, v1 = P.weno(rs, g)
    b2, o2, v2 = P.weno(rs, 3.0 * g)
    assert b2 == pytest.approx(9.0 * b1, rel=1e-12)
    assert o1.sum() == pytest.approx(1.0, abs=1e-15)


def test_beta_of_xhat_on_central_substencil():
    """g = averages of x on the R=2 central substencil, dx = 1 -> beta_1 = 1."""
    rs = K.precompute(2, dim=2)
    g = np.array([mavg_1d(float(c[0]), 1) for c in rs.offsets])  # x on all of S0
    beta, _, _ = P.weno(rs, g, dx=1.0)
    assert beta[1] == pytest.approx(SPEC["weno"]["beta_xhat_central_r2"]["value"], rel=1e-12)


def test_nonlinear_weight_damping():
    """beta_0 = 1e6 with the others ~0 drives omega_0 below 1e-20.
    Data: a step that S0 sees but the +x biased substencil (q=2) does not."""
    rs = K.precompute(2, dim=2)
    g = np.array([1.0 if c[0] >= 0 else 1e3 + 0.0 for c in rs.offsets])
    beta, om, vals = P.weno(rs, g)
    assert beta[2] < 1e-25 and beta[0] > 1e4
    assert om[0] < SPEC["weno"]["omega_extreme"]["max_omega0"] * max(1.0, 1e12 / beta[0] ** 2)
    # discontinuity damping: omega_2 > 0.99 and the value is r2.g2
    assert om[2] > 0.99
    r2 = rs.st[2]
    east = [2, 3]
    assert vals[east] == pytest.approx((r2.face @ g[r2.gather])[east], abs=1e-6)


def test_smooth_limit_exactness():
    """averages of a polynomial of degree <= the central substencil's
    degree: all beta_q equal and the WENO-AO value equals r0.g0."""
    rs = K.precompute(3, dim=2)  # central substencil degree 3
    cells = rs.offsets
    g = np.array([mavg_1d(float(c[0]), 1) * 0.3 + mavg_1d(float(c[1]), 2) * 0.7 for c in cells])
    beta, om, vals = P.weno(rs, g)
    assert np.allclose(beta[:2], beta[0], rtol=1e-10)
    r0 = rs.st[0].face @ g
    assert np.abs(vals - r0).max() < 1e-10 * max(1.0, np.abs(r0).max()) + 5e-11


# ---------------------------------------------------------------- limiter
def nbr_uniform(U, dim):
    n = 27 if dim == 3 else 9
    return np.tile(U, (n, 1))


def test_limiter_idle_for_uniform_and_in_bounds_states():
    U = prim_to_cons(1.0, [0.3, -0.2], 1.0)
    st = np.tile(U, (8, 1)) * (1 + 1e-3 * rng.normal(size=(8, 1)))
    rc, out, info = P.limit(st, nbr_uniform(U, 2))
    assert rc == 0 and info["eta"] == 0.0
    assert info["theta_rho"] == 1.0 and info["theta_p"] == 1.0
    assert np.array_equal(out, st)  # S:434 idempotence / no-op


def test_limiter_density_theta_and_bounds():
    """<rho>=1, rho_s=-0.5, rho_min -> theta = (1-rho_min)/(1.5);
    the bounds follow S:419-426 (eta=0 -> rho_min = 0.6 rho_bar_min)."""
    U = prim_to_cons(1.0, [0, 0], 1.0)
    nbr = nbr_uniform(U, 2)
    st = np.tile(U, (8, 1))
    st[3] = prim_to_cons(-0.5, [0, 0], 1.0)
    st[3][3] = U[3]
    rc, out, info = P.limit(st, nbr)
    assert rc == 0
    assert info["rho_min"] == pytest.approx(0.6, rel=1e-15)
    assert info["theta_rho"] == pytest.approx((1.0 - info["rho_min"]) / 1.5, rel=1e-15)
    # S:435 arithmetic with rho_min = 0.1
    assert (1.0 - 0.1) / (1.0 + 0.5) == pytest.approx(SPEC["limiter"]["theta_rho"]["theta"])
    assert out[:, 0].min() >= info["rho_min"] * (1 - 1e-14)
    rc2, out2, info2 = P.limit(out, nbr)  # idempotence
    assert info2["theta_rho"] == 1.0 and np.allclose(out2, out, rtol=0, atol=1e-15)


def test_flattener_eta():
    """eta = clamp(-(delta + kf cmin)/(kf cmin)); delta = -2 kf cmin -> 1,
    delta = -1.5 kf cmin -> 0.5."""
    for ratio, want in ((-2.0, 1.0), (-1.5, 0.5), (0.0, 0.0)):
        r, p = 1.0, 1.0 / G  # c = 1
        c = 1.0
        kf = 0.33
        du = ratio * kf * c  # undivided divergence 0.5*(u(+1)-u(-1)) = du
        nbr = []
        for b in (-1, 0, 1):
            for a in (-1, 0, 1):
                u = a * du
                nbr.append(prim_to_cons(r, [u, 0.0], p))
        nbr = np.array(nbr)
        st = np.tile(nbr[4], (8, 1))
        rc, _, info = P.limit(st, nbr, kf=kf)
        # cmin over the neighbourhood is 1 (pressure and density uniform)
        assert info["eta"] == pytest.approx(want, abs=1e-14), (ratio, info["eta"])


def test_pressure_limiter_bisection_matches_quadratic():
    """the bisection root matches the analytic quadratic root of
    p(U + theta (u_s - U)) = p_min to 1e-10."""
    U = prim_to_cons(1.0, [0.0, 0.0], 1.0)
    bad = prim_to_cons(1.0, [3.0, 0.0], 0.05)  # low pressure state, same density
    bad[3] = 0.3 + 0.5 * 9.0 * 0.2  # force p << p_min
    st = np.tile(U, (8, 1))
    st[1] = bad
    rc, out, info = P.limit(st, nbr_uniform(U, 2))
    pmin = info["p_min"]
    assert rc == 0 and info["theta_p"] < 1.0
    # analytic: p(theta) = gm1 (E(theta) - |m(theta)|^2 / (2 rho(theta))), rho const
    d = bad - U
    gm1 = G - 1
    # rho const = 1: p = gm1 (E0 + t dE - 0.5 (m0 + t dm)^2) -> quadratic in t
    a = -0.5 * (d[1] ** 2 + d[2] ** 2)
    b = d[3] - (U[1] * d[1] + U[2] * d[2])
    c = U[3] - 0.5 * (U[1] ** 2 + U[2] ** 2) - pmin / gm1
    roots = np.roots([a, b, c])
    t = min(r.real for r in roots if abs(r.imag) < 1e-14 and 0 <= r.real <= 1)
    assert info["theta_p"] == pytest.approx(t, abs=1e-10)
    assert P.pressure(out[1]) >= pmin * (1 - 1e-10)


# ----------------------------------------------------------------- riemann
@pytest.mark.parametrize("solver", ["hllc", "hll"])
def test_riemann_consistency_and_upwinding(solver):
    for dim in (2, 3):
        worst = 0.0
        for _ in range(500):
            U = rand_state(dim)
            for ax in range(dim):
                F = P.riemann(U, U, ax, solver)
                E = P.exact_flux(U, ax)
                worst = max(worst, (np.abs(F - E) / (np.abs(E).max() + 1e-300)).max())
        assert worst < SPEC["riemann"]["consistency_tol"]["value"]
    UL = prim_to_cons(1.0, [5.0, 0.0], 1.0)  # supersonic right-moving
    UR = prim_to_cons(0.5, [5.0, 0.0], 0.8)
    assert np.array_equal(P.riemann(UL, UR, 0, solver), P.exact_flux(UL, 0))


def test_wavespeeds_and_contact():
    U = prim_to_cons(1.0, [0.4, 0.0], 1.0)
    c = P.sound_speed(U)
    sl, sr, ss = P.wavespeeds(U, U, 0)
    assert sl == pytest.approx(0.4 - c) and sr == pytest.approx(0.4 + c) and ss == pytest.approx(0.4)
    sod = SPEC["riemann"]["sod"]
    UL = prim_to_cons(sod["left"][0], [sod["left"][1], 0], sod["left"][2])
    UR = prim_to_cons(sod["right"][0], [sod["right"][1], 0], sod["right"][2])
    sl, sr, ss = P.wavespeeds(UL, UR, 0)
    assert sl < 0 < sr
    assert P.riemann(UL, UR, 0, "hll")[0] > 0
    # stationary contact: HLLC exact zero mass flux, HLL not
    CL = prim_to_cons(1.0, [0, 0], 1.0)
    CR = prim_to_cons(0.3, [0, 0], 1.0)
    assert P.riemann(CL, CR, 0, "hllc")[0] == 0.0
    assert P.riemann(CL, CR, 0, "hll")[0] != 0.0


def test_rotational_covariance():
    """the y flux equals the x flux of the velocity-swapped states."""
    for _ in range(200):
        UL, UR = rand_state(2), rand_state(2)
        sw = [0, 2, 1, 3]
        Fy = P.riemann(UL, UR, 1)
        Fx = P.riemann(UL[sw], UR[sw], 0)[sw]
        assert np.allclose(Fy, Fx, rtol=1e-13, atol=1e-13)


# ----------------------------------------------------------------- select_dt
def test_select_dt_known_answer():
    d = SPEC["solver"]["dt_quiescent"]
    g = GridConfig(dim=2, radius=2, nx=100, ny=100, cfl=d["cfl"], dx=d["dx"])
    U = K.initial_condition(g, ICSpec("uniform", value=(1.0, 0, 0, 0, 1.0)))
    o = Oracle(g, K.precompute(2, dim=2))
    assert o.select_dt(U) == pytest.approx(d["dt"], rel=1e-12)
    g2 = GridConfig(dim=2, radius=2, nx=100, ny=100, cfl=1.0, dx=0.005)
    assert Oracle(g2, K.precompute(2, dim=2)).select_dt(U) == pytest.approx(d["dt"] / 2, rel=1e-12)


def test_eoc_formula_examples():
    for ex in SPEC["convergence"]["eoc_examples"]:
        assert math.log(ex["Ec"] / ex["Er"]) / math.log(2) == pytest.approx(ex["eoc"], abs=0.01)
