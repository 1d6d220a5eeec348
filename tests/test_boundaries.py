"""Boundary kinds and the problem catalog (SPEC S:534-561 fill_ghost,
S:647-708 problems).

CPU: the oracle's fill_ghost against the SPEC examples and the kinds'
definitions, the catalog's SPEC examples, and solver invariants of the new
kinds (a closed reflecting box at rest stays at rest and conserves mass; a
dirichlet inflow of the free stream preserves it; the multi-slab split is
bit-identical with reflecting / dirichlet slab ends).  GPU: bitwise parity of
the device ghost fill (k_ghost / k_halo_local) through whole runs."""
import math

import numpy as np
import pytest

import paper_2401_16543_b200 as K
from paper_2401_16543_b200 import problems as P
from paper_2401_16543_b200.config import GridConfig
from oracle import Oracle

GAM = 1.4


def _rand_state(shape, seed=0, dim=2):
    rng = np.random.default_rng(seed)
    rho = 1.0 + 0.3 * rng.random(shape)
    vel = [0.4 * (rng.random(shape) - 0.5) for _ in range(dim)]
    p = 1.0 + 0.3 * rng.random(shape)
    return P.cons(GAM, rho, vel, p)


def _oracle(g):
    return Oracle(g, K.precompute(g.radius, dim=g.dim))


# ------------------------------------------------------------ fill_ghost
def test_fill_ghost_spec_examples():
    """periodic ghost(-1) = interior(nx-1); reflecting in x:
    ghost m_x = -interior m_x, rho / m_y / E copied (mirror image);
    outflow copies the nearest interior cell; dirichlet writes its state."""
    n = 8
    wall = tuple(P.cons(GAM, 0.5, (0.25, -0.5), 0.75))
    g = GridConfig(dim=2, radius=2, nx=n, ny=n, dx=1.0 / n,
                   sides=("reflecting", "outflow", "periodic", "periodic"))
    U = _rand_state((n, n))
    V = _oracle(g).fill_ghost(U)
    H = 3
    inner = V[H:H + n, H:H + n]
    assert np.array_equal(inner, U)
    # periodic in y: ghost row -1 = row n-1, row n = row 0
    assert np.array_equal(V[H - 1, H:H + n], U[n - 1])
    assert np.array_equal(V[H + n, H:H + n], U[0])
    # reflecting at x = 0: ghost column -1-k mirrors column k, m_x negated
    for k in range(H):
        gcol, icol = V[H:H + n, H - 1 - k], U[:, k]
        assert np.array_equal(gcol[:, 1], -icol[:, 1])
        assert np.array_equal(gcol[:, [0, 2, 3]], icol[:, [0, 2, 3]])
    # outflow at x = 1: every ghost column is the last interior column
    for k in range(H):
        assert np.array_equal(V[H:H + n, H + n + k], U[:, n - 1])
    # dirichlet at y = 0 (periodic x here)
    g2 = GridConfig(dim=2, radius=2, nx=n, ny=n, dx=1.0 / n,
                    sides=("periodic", "periodic", "dirichlet", "outflow"),
                    side_states=(None, None, wall, None))
    V2 = _oracle(g2).fill_ghost(U)
    assert np.all(V2[:H] == np.array(wall))
    assert np.array_equal(V2[H + n + 1, H:H + n], U[n - 1])


def test_fill_ghost_slit_membership():
    """S:561 / S:689: the jet ghost state strictly inside x^2 < r^2 on the
    lower y side (x = 0.04 < 0.05 -> jet), outflow elsewhere; a cell centre
    exactly on the slit edge takes the outflow side."""
    n = 64
    dx = 1.0 / n
    jet = tuple(P.cons(GAM, GAM, (0.0, 800.0), 1.0))
    U = _rand_state((8, 16))
    r = 2.5 * dx  # = the centre of cell 2: on the edge, strict -> outflow
    g = GridConfig(dim=2, radius=2, nx=16, ny=8, dx=dx,
                   sides=("reflecting", "outflow", "slit", "outflow"),
                   side_states=(None, None, jet, None), slits=(None, None, ((0.0,), r), None))
    V = _oracle(g).fill_ghost(U)
    H = 3
    for i in range(16):
        x = (i + 0.5) * dx
        ghost = V[H - 1, H + i]
        if x * x < r * r:
            assert np.array_equal(ghost, np.array(jet)), i
        else:
            assert np.array_equal(ghost, U[0, i]), i
    assert not np.array_equal(V[H - 1, H + 2], np.array(jet))
    # the SPEC example with the paper's slit: x = 0.04 < 0.05 -> jet
    g5 = GridConfig(dim=2, radius=2, nx=16, ny=8, dx=0.02,
                    sides=("reflecting", "outflow", "slit", "outflow"),
                    side_states=(None, None, jet, None), slits=(None, None, ((0.0,), 0.05), None))
    V5 = _oracle(g5).fill_ghost(U)
    assert np.array_equal(V5[H - 1, H + 1], np.array(jet))   # centre x = 0.03
    assert np.array_equal(V5[H - 1, H + 3], U[0, 3])          # centre x = 0.07


def test_fill_ghost_corner_composition():
    """Corner ghosts compose the axis rules in order x, y(, z): the
    (reflecting x, reflecting y) corner is the point mirror with both
    momenta negated; a dirichlet x side under a reflecting y side keeps the
    dirichlet state with m_y negated."""
    n = 6
    U = _rand_state((n, n), seed=3)
    g = GridConfig(dim=2, radius=2, nx=n, ny=n, dx=1.0 / n, bc="reflecting")
    V = _oracle(g).fill_ghost(U)
    H = 3
    c = V[H - 1, H - 2]   # (x=-2, y=-1) <- (x=1, y=0)
    assert np.array_equal(c, U[0, 1] * np.array([1, -1, -1, 1]))
    st = tuple(P.cons(GAM, 1.2, (0.3, 0.2), 0.9))
    g2 = GridConfig(dim=2, radius=2, nx=n, ny=n, dx=1.0 / n,
                    sides=("dirichlet", "outflow", "reflecting", "reflecting"),
                    side_states=(st, None, None, None))
    V2 = _oracle(g2).fill_ghost(U)
    assert np.array_equal(V2[H - 1, H - 1], np.array(st) * np.array([1, 1, -1, 1]))


def test_config_validation():
    with pytest.raises(ValueError):
        GridConfig(dim=2, nx=8, ny=8, sides=("periodic", "outflow", "periodic", "periodic"))
    with pytest.raises(ValueError):
        GridConfig(dim=2, nx=8, ny=8, sides=("dirichlet", "outflow", "periodic", "periodic"))
    with pytest.raises(ValueError):
        GridConfig(dim=2, nx=8, ny=8, sides=("outflow",) * 3)


# ------------------------------------------------------------ solver invariants
@pytest.mark.parametrize("dim", [2, 3])
def test_reflecting_box_at_rest(dim):
    """A uniform gas at rest in a closed reflecting box: dU/dt = 0 to rounding."""
    n = 8
    g = GridConfig(dim=dim, radius=2, nx=n, ny=n, nz=n if dim == 3 else 1, bc="reflecting")
    U = np.broadcast_to(P.cons(GAM, 1.3, (0.0,) * dim, 0.8), g.shape + (g.nvar,)).copy()
    L = _oracle(g).compute_rhs(U)
    assert np.abs(L).max() < 1e-12


def test_reflecting_box_conserves_mass_and_energy():
    """Closed reflecting box: the wall mass / energy fluxes vanish (the
    ghost's reconstruction mirrors the interior one), so sum dU/dt of rho and
    E is ~0; momentum changes only through the wall pressure."""
    n = 12
    g = GridConfig(dim=2, radius=2, nx=n, ny=n, bc="reflecting")
    U = _rand_state((n, n), seed=5)
    L = _oracle(g).compute_rhs(U)
    for v in (0, 3):
        assert abs(L[..., v].sum()) <= 1e-10 * np.abs(L[..., v]).sum()


def test_dirichlet_inflow_preserves_free_stream():
    n = 10
    st = P.cons(GAM, 1.1, (0.8, 0.3), 1.2)
    g = GridConfig(dim=2, radius=2, nx=n, ny=n,
                   sides=("dirichlet", "outflow", "periodic", "periodic"),
                   side_states=(tuple(st), None, None, None))
    U = np.broadcast_to(st, g.shape + (4,)).copy()
    L = _oracle(g).compute_rhs(U)
    assert np.abs(L).max() < 1e-12


@pytest.mark.parametrize("sides", [
    ("outflow", "outflow", "reflecting", "dirichlet"),
    ("reflecting", "dirichlet", "reflecting", "reflecting"),
])
def test_slab_split_bitwise_with_walls(sides):
    """P virtual slabs along y (the slab axis) with reflecting / dirichlet
    slab ends == one domain, bit for bit (the multi-GPU invariant)."""
    n = 16
    st = tuple(P.cons(GAM, 0.9, (0.1, -0.2), 1.1))
    g = GridConfig(dim=2, radius=2, nx=n, ny=n, cfl=0.4, sides=sides,
                   side_states=tuple(st if k == "dirichlet" else None for k in sides))
    U = _rand_state((n, n), seed=7)
    o = _oracle(g)
    U1, d1 = o.run(U, 2, nslabs=1)
    U3, d3 = o.run(U, 2, nslabs=3)
    assert np.array_equal(d1, d3) and np.array_equal(U1, U3)


# ------------------------------------------------------------ catalog
def test_rmi_spec_examples():
    pr = P.richtmyer_meshkov(n=8)
    g = pr.grid
    assert (g.nx, g.ny) == (48, 8) and g.sides[0] == "dirichlet"
    rho_s = 1.0 / (1.0 - (2.0 / 2.4) * (1.0 - 1.0 / 9.0))
    p_s = 1.0 + (2.8 / 2.4) * 8.0
    assert abs(p_s - 10.333333333333334) < 1e-12
    assert np.allclose(g.side_states[0], P.cons(GAM, rho_s, (3.0 * math.sqrt(GAM) * (1 - 1 / rho_s), 0.0), p_s))
    # x >= 0.2, x >= y -> (rho_D, 0, 0, p=1): cell centred at (0.9375 + ..) far right
    U = pr.U0
    far = U[0, -1]
    assert np.allclose(far, P.cons(GAM, 2.0, (0.0, 0.0), 1.0))
    # x < 0.2 (leftmost cells): the shocked state
    assert np.allclose(U[3, 0], np.array(g.side_states[0]))


def test_jet_spec_examples():
    pr = P.astro_jet("high", n=16)
    g = pr.grid
    jet = np.array(g.side_states[2])
    assert np.allclose(jet, [GAM, 0.0, 800.0 * GAM, 1.0 / (GAM - 1) + 0.5 * GAM * 800.0 ** 2])
    assert np.allclose(pr.U0[..., 0], GAM / 10)
    assert g.riemann == "hll" and g.slits[2] == ((0.0,), 0.05)
    assert np.allclose(P.astro_jet("low", n=16).U0[..., 0], 10 * GAM)


def test_rt_spec_examples():
    pr = P.rayleigh_taylor(n=16)
    g = pr.grid
    assert g.gamma == 5.0 / 3.0 and g.viscous and g.froude == 1.0
    # dirichlet y states: (rho, p) = (2, 1) at y = 0 and (1, 1.5) at y = 1, at rest
    gm = 5.0 / 3.0
    assert np.allclose(g.side_states[2], [2.0, 0, 0, 1.0 / (gm - 1)])
    assert np.allclose(g.side_states[3], [1.0, 0, 0, 1.5 / (gm - 1)])
    # pressure profile: y = 0.25 -> 1.5; y = 0.75 -> 1.25; continuous at y = 1/2 (= 2)
    lo = 2.0 * 0.25 + 1.0
    hi = (0.75 * 1.0 - 0.5) + 1.0
    assert lo == 1.5 and hi == 1.25 and 2.0 * 0.5 + 1.0 == (0.5 - 0.5) + 1.0 + 1.0


def test_catalog_admissible():
    for name in P.CATALOG:
        kw = {"n": 16} if name != "sod_aligned" else {"n": 20}
        pr = P.problem(name, **kw)
        U = pr.U0
        d = pr.grid.dim
        q = (U[..., 1:1 + d] ** 2).sum(-1)
        p = (pr.grid.gamma - 1) * (U[..., -1] - 0.5 * q / U[..., 0])
        assert (U[..., 0] > 0).all() and (p > 0).all(), name


# ------------------------------------------------------------ GPU parity
GPU_CASES = [
    # (name, problem, t_final, overrides): the problems' own SSP(4,3,2) +
    # PI controller, a few accepted steps each
    ("rmi_r2", lambda: P.richtmyer_meshkov(n=8), 0.02, {}),
    ("jet_high_r3", lambda: P.astro_jet("high", n=32), 1e-4, {}),
    ("jet_low_r2_kxrcf", lambda: P.astro_jet("low", n=32, radius=2), 1e-3, {"kxrcf": True}),
    ("rt_r3_viscous", lambda: P.rayleigh_taylor(n=32), 0.02, {}),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,mk,tf,over", GPU_CASES, ids=[c[0] for c in GPU_CASES])
def test_gpu_catalog_parity(require_gpu, name, mk, tf, over):
    from dataclasses import replace
    pr = mk()
    g = replace(pr.grid, **over)
    rset = K.precompute(g.radius, dim=g.dim)
    Uo, dto, na, nr, to = Oracle(g, rset).advance43(pr.U0, tf)
    with K.Solver(g, rset) as s:
        s.set_state(pr.U0)
        steps, t = s.advance_to(tf, 10000)
        acc, rej = s.step_stats()
        dts = s.dt_sequence(acc)
        Ug = s.get_state()
    assert (acc, rej) == (na, nr) and t == to
    assert np.array_equal(dts, dto), (dts, dto)
    assert np.array_equal(Ug, Uo)


@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 3])
def test_gpu_3d_mixed_walls_parity(require_gpu, R):
    """3-D: reflecting x, dirichlet/outflow y, slit z-low (round slit in
    the x-y plane) / reflecting z-high — every kind on the tensor engine,
    including corner composition and the slab-axis (z) halo planes."""
    n = 10
    st = tuple(P.cons(GAM, 1.4, (0.0, 0.0, 2.0), 1.0))
    amb = tuple(P.cons(GAM, 1.0, (0.1, 0.2, -0.1), 1.0))
    g = GridConfig(dim=3, radius=R, nx=n, ny=n, nz=n, cfl=0.4,
                   sides=("reflecting", "reflecting", "dirichlet", "outflow", "slit", "reflecting"),
                   side_states=(None, None, amb, None, st, None),
                   slits=(None, None, None, None, ((0.5, 0.5), 0.25), None))
    rng = np.random.default_rng(11)
    U = P.cons(GAM, 1.0 + 0.2 * rng.random(g.shape), [0.2 * (rng.random(g.shape) - 0.5) for _ in range(3)],
               1.0 + 0.2 * rng.random(g.shape))
    rset = K.precompute(R, dim=3)
    with K.Solver(g, rset) as s:
        s.set_state(U)
        dts = s.advance(2)
        Ug = s.get_state()
        Lg = s.compute_rhs(U)
    o = Oracle(g, rset)
    Uo, dto = o.run(U, 2)
    assert np.array_equal(dts, dto)
    assert np.array_equal(Ug, Uo)
    assert np.array_equal(Lg, o.compute_rhs(U))


@pytest.mark.gpu
def test_gpu_2d_engines_with_walls(require_gpu):
    """Every 2-D reconstruction engine on a reflecting / dirichlet box."""
    n = 24
    st = tuple(P.cons(GAM, 1.2, (0.5, 0.0), 1.0))
    g = GridConfig(dim=2, radius=2, nx=n, ny=n, cfl=0.4,
                   sides=("dirichlet", "outflow", "reflecting", "reflecting"),
                   side_states=(st, None, None, None))
    U = _rand_state((n, n), seed=13)
    rset = K.precompute(2, dim=2)
    Uo, dto = Oracle(g, rset).run(U, 2)
    for eng in (0, 1, 2, 3, 4):
        with K.Solver(g, rset) as s:
            s.set_option("engine", eng)
            s.set_state(U)
            dts = s.advance(2)
            assert np.array_equal(dts, dto), eng
            assert np.array_equal(s.get_state(), Uo), eng


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("opts", [{"chunk_planes": 4}, {"overlap": 1}, {"overlap": 1, "chunk_planes": 4}])
def test_gpu_walls_chunked_and_overlapped(require_gpu, dim, opts):
    """Wall / inflow slab ends through the multi-chunk stage and the
    overlapped (halo-split) schedule == the oracle, bit for bit."""
    n = 12
    nv = dim + 2
    st = tuple(P.cons(GAM, 1.3, (0.2,) + (0.0,) * (dim - 1), 1.1))
    sides = ("reflecting", "outflow") + (("periodic", "periodic") if dim == 3 else ()) + ("dirichlet", "reflecting")
    g = GridConfig(dim=dim, radius=2, nx=n, ny=n, nz=n if dim == 3 else 1, cfl=0.4, sides=sides,
                   side_states=tuple(st if k == "dirichlet" else None for k in sides))
    rng = np.random.default_rng(17)
    U = P.cons(GAM, 1.0 + 0.2 * rng.random(g.shape), [0.2 * (rng.random(g.shape) - 0.5) for _ in range(dim)],
               1.0 + 0.2 * rng.random(g.shape))
    assert U.shape[-1] == nv
    rset = K.precompute(2, dim=dim)
    Uo, dto = Oracle(g, rset).run(U, 2)
    with K.Solver(g, rset) as s:
        for k, v in opts.items():
            s.set_option(k, v)
        s.set_state(U)
        dts = s.advance(2)
        assert np.array_equal(dts, dto)
        assert np.array_equal(s.get_state(), Uo)


@pytest.mark.gpu
def test_gpu_walls_ring_split(require_gpu):
    """nx = 32 (ring split: ring columns by the DFMA engine) with reflecting /
    dirichlet x sides, 3-D tensor engine, both settings of the split."""
    st = tuple(P.cons(GAM, 1.2, (0.4, 0.0, 0.0), 1.0))
    g = GridConfig(dim=3, radius=2, nx=32, ny=6, nz=6, cfl=0.4,
                   sides=("dirichlet", "reflecting", "periodic", "periodic", "outflow", "outflow"),
                   side_states=(st, None, None, None, None, None))
    rng = np.random.default_rng(23)
    U = P.cons(GAM, 1.0 + 0.2 * rng.random(g.shape), [0.2 * (rng.random(g.shape) - 0.5) for _ in range(3)],
               1.0 + 0.2 * rng.random(g.shape))
    rset = K.precompute(2, dim=3)
    Uo, dto = Oracle(g, rset).run(U, 2)
    for split in (0, 1):
        with K.Solver(g, rset) as s:
            s.set_option("ring_split", split)
            s.set_state(U)
            assert np.array_equal(s.advance(2), dto)
            assert np.array_equal(s.get_state(), Uo)


@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 3])
def test_gpu_3d_kxrcf_walls(require_gpu, R):
    """KXRCF mode (pass-1 states, flags with wall faces exempt, WENO on
    flagged cells) with reflecting / dirichlet / outflow sides in 3-D."""
    n = 12
    st = tuple(P.cons(GAM, 2.0, (0.5, 0.0, 0.0), 3.0))
    g = GridConfig(dim=3, radius=R, nx=n, ny=n, nz=n, cfl=0.3, kxrcf=True,
                   sides=("dirichlet", "outflow", "reflecting", "reflecting", "reflecting", "outflow"),
                   side_states=(st, None, None, None, None, None))
    rng = np.random.default_rng(29)
    # a density / pressure jump so that some cells are flagged
    x = (np.arange(n) + 0.5) / n
    jump = np.broadcast_to(x > 0.5, g.shape)
    rho = np.where(jump, 0.5, 1.5) + 1e-4 * rng.random(g.shape)
    p = np.where(jump, 0.4, 1.2)
    U = P.cons(GAM, rho, [1e-4 * (rng.random(g.shape) - 0.5) for _ in range(3)], p)
    rset = K.precompute(R, dim=3)
    o = Oracle(g, rset)
    Uo, dto = o.run(U, 2)
    with K.Solver(g, rset) as s:
        fl = s.kxrcf_flags(U)
        assert np.array_equal(fl, o.kxrcf_flags(U)) and 0 < fl.sum() < fl.size
        s.set_state(U)
        assert np.array_equal(s.advance(2), dto)
        assert np.array_equal(s.get_state(), Uo)
