"""KXRCF troubled-cell indicator: the
oracle's pinned power function, the SPEC examples for the flags, and — on the
GPU — flags and whole runs bit-identical to the oracle with the indicator on."""
from dataclasses import replace

import numpy as np
import pytest

import paper_2401_16543_b200 as K
from paper_2401_16543_b200.config import GridConfig, ICSpec
from oracle import kfvm_oracle as O


def test_pinned_pow_accuracy():
    L = O.lib()
    rng = np.random.default_rng(7)
    x = np.exp(rng.uniform(-30, 30, 4000))
    y = rng.uniform(0.2, 3.0, 4000)
    got = np.array([L.kfo_pow(float(a), float(b)) for a, b in zip(x, y)])
    assert np.max(np.abs(got / x ** y - 1)) < 1e-14
    assert L.kfo_pow(1.0, 1.4) == 1.0
    assert L.kfo_pow(4.0, 0.5) == 2.0


def _flags(g, U):
    return O.Oracle(g, K.precompute(g.radius, dim=g.dim)).kxrcf_flags(U)


def test_constant_field_not_flagged():
    """globally constant field -> zero cells flagged."""
    g = GridConfig(dim=2, radius=2, nx=16, ny=16, kxrcf=True)
    U = K.initial_condition(g, ICSpec("uniform", value=(1.3, 0.7, -0.4, 0.0, 2.0)))
    assert _flags(g, U).sum() == 0
    g3 = GridConfig(dim=3, radius=2, nx=8, ny=8, nz=8, kxrcf=True, bc="outflow")
    U3 = K.initial_condition(g3, ICSpec("uniform", value=(0.5, 0.1, 0.2, 0.3, 0.7)))
    assert _flags(g3, U3).sum() == 0


def test_smooth_vortex_flag_fraction():
    """smooth isentropic vortex 64^2 -> flagged fraction < 1%."""
    g = GridConfig(dim=2, radius=2, nx=64, ny=64, dx=20.0 / 64, kxrcf=True)
    U = K.initial_condition(g, ICSpec("vortex", origin=(-10.0, -10.0, 0.0)))
    assert _flags(g, U).mean() < 0.01


def test_step_flags_cells_at_the_jump():
    """Sod-like step: the cells next to the jump are flagged, far cells not
    (S:566)."""
    g = GridConfig(dim=2, radius=2, nx=32, ny=8, bc="outflow", kxrcf=True)
    U = np.zeros(g.shape + (4,))
    left = np.arange(g.nx) < g.nx // 2
    rho = np.where(left, 1.0, 0.125)
    p = np.where(left, 1.0, 0.1)
    U[..., 0] = rho[None, :]
    U[..., 3] = (p / 0.4)[None, :]
    f = _flags(g, U)
    assert f[:, 15].all() and f[:, 16].all()
    assert not f[:, :10].any() and not f[:, 22:].any()


def test_kxrcf_states_are_pass1_away_from_flags():
    """with no cell flagged, every face state is the unlimited full-stencil
    r_0 reconstruction of the conservative averages (S:565 pass 1; the limiter
    is inactive on this smooth periodic field) — checked against an
    independent numpy evaluation of r_0 . U over S_0."""
    w = K.baseline_config(1, n=24)
    g = replace(w.grid, kxrcf=True)
    U = K.initial_condition(g, w.ic)
    rs = K.precompute(2, dim=2)
    orc = O.Oracle(g, rs)
    assert orc.kxrcf_flags(U).sum() == 0
    a = orc.reconstruct_states(U).reshape(g.ny, g.nx, -1, 4)
    r0 = rs.st[0].face                       # [points][N0]
    offs = rs.cells(0)                       # [N0][3] (x, y, .)
    yy, xx = np.meshgrid(np.arange(g.ny), np.arange(g.nx), indexing="ij")
    G = np.stack([U[(yy + o[1]) % g.ny, (xx + o[0]) % g.nx] for o in offs], axis=2)
    ref = np.einsum("sh,yxhv->yxsv", r0, G)
    assert np.max(np.abs(a - ref)) < 1e-13
    b = O.Oracle(w.grid, rs).reconstruct_states(U).reshape(a.shape)
    assert not np.array_equal(a, b)  # WENO-AO everywhere gives different states


@pytest.mark.gpu
@pytest.mark.parametrize("idx,n,over", [(1, 24, {}), (2, 32, {}), (2, 24, {"bc": "periodic"}),
                                        (3, 10, {}), (4, 10, {}), (5, 12, {})])
def test_gpu_flags_match_oracle(require_gpu, idx, n, over):
    w = K.baseline_config(idx, n=n)
    g = replace(w.grid, kxrcf=True, **over)
    U = K.initial_condition(g, w.ic)
    rs = K.precompute(g.radius, dim=g.dim)
    with K.Solver(g, rs) as s:
        fg = s.kxrcf_flags(U)
    fo = O.Oracle(g, rs).kxrcf_flags(U)
    assert np.array_equal(fg, fo), (fg != fo).sum()


@pytest.mark.gpu
@pytest.mark.parametrize("idx,n,steps", [(1, 24, 3), (2, 32, 3), (3, 10, 2), (4, 10, 2),
                                         (5, 12, 1)])
def test_gpu_kxrcf_run_bitwise(require_gpu, idx, n, steps):
    w = K.baseline_config(idx, n=n)
    g = replace(w.grid, kxrcf=True)
    U = K.initial_condition(g, w.ic)
    rs = K.precompute(g.radius, dim=g.dim)
    ref, dto = O.Oracle(g, rs).run(U, steps)
    for eng in ((0, 4) if g.dim == 2 else (0, 2)):
        with K.Solver(g, rs) as s:
            s.set_option("engine", eng)
            s.set_state(U)
            d = s.advance(steps)
            A = s.get_state()
        assert np.array_equal(d, dto), eng
        assert np.array_equal(A, ref), (eng, np.abs(A - ref).max())
