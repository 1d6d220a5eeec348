"""GPU parity against the CPU oracle through the C-ABI (BASELINE.json
north_star gate: relative L1 <= 1e-11 per conserved variable after the stated
steps, identical dt sequence).  The implementation targets bit-identity
(pinned FP contract); the max ulp difference is asserted == 0
where the contract guarantees it."""
import numpy as np
import pytest

import paper_2401_16543_b200 as K
from paper_2401_16543_b200.config import ICSpec
from oracle import Oracle

pytestmark = pytest.mark.gpu

TOL = 1e-11  # relative L1 per conserved variable (north_star)


def rel_l1(a, b):
    ax = tuple(range(a.ndim - 1))
    return np.abs(a - b).sum(axis=ax) / np.maximum(np.abs(b).sum(axis=ax), 1e-300)


def max_ulp(a, b):
    d = np.abs(a.view(np.int64) - b.view(np.int64))
    return int(d.max()) if a.size else 0


CASES = [
    # (name, config index, n, steps, overrides)
    ("cfg1_2d_r2_periodic_fourier", 1, 32, 3, {}),
    ("cfg2_2d_r2_outflow_voronoi", 2, 40, 3, {}),
    ("cfg1_2d_r3_periodic_hll", 1, 24, 2, {"radius": 3, "riemann": "hll"}),
    ("cfg3_3d_r2_periodic_fourier", 3, 16, 2, {}),
    ("cfg4_3d_r2_outflow_voronoi", 4, 14, 2, {}),
    ("cfg5_3d_r3_periodic_sphere", 5, 12, 1, {}),
    # nx = 32: the segment engine covers interior x, the ring columns come
    # from k_states_fast (3-D ring split)
    ("cfg3_3d_r2_ring_split", 3, 32, 1, {}),
]


def _setup(idx, n, over):
    from dataclasses import replace
    w = K.baseline_config(idx, n=n)
    g = replace(w.grid, **over) if over else w.grid
    U = K.initial_condition(g, w.ic)
    rset = K.precompute(g.radius, dim=g.dim)
    return g, w.ic, U, rset


@pytest.mark.parametrize("name,idx,n,steps,over", CASES, ids=[c[0] for c in CASES])
def test_run_parity(require_gpu, name, idx, n, steps, over):
    g, ic, U, rset = _setup(idx, n, over)
    with K.Solver(g, rset) as s:
        s.set_state(U)
        dts = s.advance(steps)
        Ug = s.get_state()
    Uo, dto = Oracle(g, rset).run(U, steps)
    assert np.array_equal(dts, dto), (dts, dto)
    err = rel_l1(Ug, Uo)
    assert (err <= TOL).all(), err
    assert np.array_equal(Ug, Uo), f"max ulp {max_ulp(Ug, Uo)}"


@pytest.mark.parametrize("idx,n", [(1, 24), (3, 10), (4, 10)])
def test_rhs_and_states_parity(require_gpu, idx, n):
    g, ic, U, rset = _setup(idx, n, {})
    o = Oracle(g, rset)
    with K.Solver(g, rset) as s:
        Lg = s.compute_rhs(U)
        Sg = s.reconstruct_states(U)
        dtg = s.select_dt(U)
    assert np.array_equal(Lg, o.compute_rhs(U))
    assert np.array_equal(Sg, o.reconstruct_states(U))
    assert dtg == o.select_dt(U)


def test_stage_api_matches_run(require_gpu):
    g, ic, U, rset = _setup(1, 20, {})
    with K.Solver(g, rset) as s:
        s.set_state(U)
        dt = s.select_dt()
        for st in (1, 2, 3):
            s.ssp_rk3_stage(st, dt)
        U1 = s.get_state()
    Uo, dto = Oracle(g, rset).run(U, 1)
    assert dt == dto[0]
    assert np.array_equal(U1, Uo)


def test_chunked_equals_unchunked(require_gpu):
    g, ic, U, rset = _setup(3, 12, {})
    with K.Solver(g, rset) as s:
        s.set_state(U)
        d1 = s.advance(2)
        A = s.get_state()
    with K.Solver(g, rset) as s:
        s.set_option("engine", 2)  # the face-state engines run in chunks
        s.set_option("chunk_planes", 5)
        s.set_state(U)
        d2 = s.advance(2)
        B = s.get_state()
    assert np.array_equal(d1, d2) and np.array_equal(A, B)


def test_device_ic_matches_host(require_gpu):
    for idx, n in ((1, 32), (2, 32), (3, 12), (4, 12), (5, 10)):
        w = K.baseline_config(idx, n=n)
        U = K.initial_condition(w.grid, w.ic)
        with K.Solver(w.grid) as s:
            s.generate_ic(w.ic)
            Ud = s.get_state()
        assert np.array_equal(U, Ud), idx


def test_free_stream_preserved(require_gpu):
    g = K.GridConfig(dim=3, radius=2, nx=12, ny=12, nz=12, cfl=0.3)
    U = K.initial_condition(g, ICSpec("uniform", value=(1.3, 0.7, -0.4, 0.2, 2.0)))
    with K.Solver(g) as s:
        s.set_state(U)
        s.advance(3)
        assert np.array_equal(s.get_state(), U)


def test_runtime_error_on_inadmissible_state(require_gpu):
    g = K.GridConfig(dim=2, radius=2, nx=16, ny=16, cfl=0.4)
    U = K.initial_condition(g, ICSpec("uniform", value=(1.0, 0.0, 0.0, 0.0, 1.0)))
    U[5, 5, 0] = -1.0
    with K.Solver(g) as s:
        s.set_state(U)
        with pytest.raises(K.KfvmRuntimeError):
            s.advance(1)


@pytest.mark.parametrize("idx,n", [(1, 20), (2, 24), (3, 10), (4, 10), (5, 10)])
def test_engines_bitwise_identical(require_gpu, idx, n):
    """generic / unrolled-DFMA / DMMA / row-marching DFMA reconstruction engines and
    the fused 3-D stage engine agree bit for bit."""
    g, ic, U, rset = _setup(idx, n, {})
    outs = []
    engines = (0, 1, 2, 3, 4) if g.dim == 2 else ((0, 1, 2, 5) if g.radius == 2 else (0, 1, 2))
    for eng in engines:
        with K.Solver(g, rset) as s:
            s.set_option("engine", eng)
            s.set_state(U)
            d = s.advance(2)
            outs.append((d, s.get_state()))
    for d, A in outs[1:]:
        assert np.array_equal(d, outs[0][0]) and np.array_equal(A, outs[0][1])


def test_advance_to_matches_oracle(require_gpu):
    """advance_to: fixed-CFL steps, last one clipped onto t_final."""
    from paper_2401_16543_b200.config import GridConfig
    g = GridConfig(dim=2, radius=2, nx=24, ny=24, bc="periodic", dx=20.0 / 24, cfl=0.4)
    ic = ICSpec("vortex", origin=(-10.0, -10.0, 0.0))
    U0 = K.initial_condition(g, ic)
    rset = K.precompute(2, dim=2)
    o = Oracle(g, rset)
    U, t, n = U0.copy(), 0.0, 0
    while t < 1.0:
        dt = min(o.select_dt(U), 1.0 - t)
        U1 = o.stage(U, U, 1, dt)
        U2 = o.stage(U, U1, 2, dt)
        U = o.stage(U, U2, 3, dt)
        t += dt
        n += 1
    with K.Solver(g, rset) as s:
        s.set_state(U0)
        steps, tg = s.advance_to(1.0)
        Ug = s.get_state()
    assert tg == t and steps >= n
    assert np.array_equal(Ug, U)


def test_isentropic_vortex_eoc_gpu(require_gpu):
    """S:791 acceptance / PAPER Table 1 on the GPU: R=2 64^2 -> 128^2 EOC >= 3.5
    (paper 3.95); R=3 32^2 -> 64^2 EOC >= 3.0 (paper 3.32)."""
    import math
    from paper_2401_16543_b200.config import GridConfig
    ic = ICSpec("vortex", origin=(-10.0, -10.0, 0.0))

    def l1(n, R):
        g = GridConfig(dim=2, radius=R, nx=n, ny=n, bc="periodic", dx=20.0 / n, cfl=0.4)
        U0 = K.initial_condition(g, ic)
        with K.Solver(g) as s:
            s.set_state(U0)
            s.advance_to(20.0)
            U = s.get_state()
        return np.abs(U[..., 0] - U0[..., 0]).sum() * g.dx ** 2

    e = {n: l1(n, 2) for n in (64, 128)}
    assert math.log(e[64] / e[128]) / math.log(2) >= 3.5, e
    e3 = {n: l1(n, 3) for n in (32, 64)}
    assert math.log(e3[32] / e3[64]) / math.log(2) >= 3.0, e3


@pytest.mark.parametrize("chunk", [None, 5])
@pytest.mark.parametrize("idx,n", [(1, 24), (2, 24), (3, 12), (4, 12), (5, 14)])
def test_overlapped_stage_bitwise(require_gpu, idx, n, chunk):
    """The overlapped stage schedule (halo exchange on a side stream while the
    halo-independent states compute, then the rest) gives the same bits as the
    serial schedule; forced on one GPU with the local halo copy, for the
    one-chunk (plane-range split) and multi-chunk (chunk order) variants."""
    g, ic, U, rset = _setup(idx, n, {})
    outs = []
    for ov in (0, 1):
        with K.Solver(g, rset) as s:
            s.set_option("overlap", ov)
            if chunk:
                s.set_option("chunk_planes", chunk)  # several chunks, interior ones first
            s.set_state(U)
            d = s.advance(2)
            outs.append((d, s.get_state()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


def test_async_two_handles_pipeline(require_gpu):
    """set_state_async / run_async / get_state_async on two handles (the
    bench's e2e ensemble pipeline) == the synchronous path, bit for bit."""
    g, ic, U, rset = _setup(1, 32, {})
    with K.Solver(g, rset) as s:
        s.set_state(U)
        s.advance(1)
        ref1 = s.get_state()
        s.advance(1)
        ref2 = s.get_state()
    bufs = [U.copy(), U.copy()]
    with K.Solver(g, rset) as a, K.Solver(g, rset) as b:
        for _ in range(2):
            for sv, hb in ((a, bufs[0]), (b, bufs[1])):
                sv.set_state_async(hb)
                sv.run_async(1)
                sv.get_state_async(hb)
        a.sync()
        b.sync()
    assert np.array_equal(bufs[0], ref2) and np.array_equal(bufs[1], ref2)
    assert not np.array_equal(ref1, ref2)


@pytest.mark.parametrize("idx", [3, 4])
def test_tma_ring_bitwise(require_gpu, idx):
    """3-D R=2 with nx = 64 (ring split): the tensor engine's ring planes
    arrive by TMA (cp.async.bulk.tensor + mbarrier); with option tma=0 by
    cp.async.  Both, in one chunk and in several (chunk_planes), give the
    oracle's bits."""
    from dataclasses import replace
    w = K.baseline_config(idx, n=8)
    g = replace(w.grid, nx=64, ny=12, nz=14, dx=1.0 / 64)
    U = K.initial_condition(g, w.ic)
    rset = K.precompute(2, dim=3)
    Uo, do = Oracle(g, rset).run(U, 2)
    for opts in ((("tma", 1),), (("tma", 0),), (("tma", 1), ("chunk_planes", 4))):
        with K.Solver(g, rset) as s:
            for k, v in opts:
                s.set_option(k, v)
            s.set_state(U)
            d = s.advance(2)
            assert np.array_equal(d, do), opts
            assert np.array_equal(s.get_state(), Uo), opts


@pytest.mark.parametrize("R", [2, 3])
def test_periodic_ring_copy_bitwise(require_gpu, R):
    """Periodic x: the extended box's ring columns are copied from their
    periodic images (k_ring_copy) instead of recomputed; with the option
    ring_split=0 every column is computed.  Both equal the oracle."""
    from dataclasses import replace
    w = K.baseline_config(3 if R == 2 else 5, n=8)
    g = replace(w.grid, nx=32, ny=9, nz=10, dx=1.0 / 32)
    U = K.initial_condition(g, w.ic)
    rset = K.precompute(R, dim=3)
    Uo, do = Oracle(g, rset).run(U, 2)
    for split in (1, 0):
        with K.Solver(g, rset) as s:
            s.set_option("ring_split", split)
            s.set_state(U)
            d = s.advance(2)
            assert np.array_equal(d, do) and np.array_equal(s.get_state(), Uo), split


@pytest.mark.parametrize("bc", ["outflow", "reflecting"])
def test_ring_column_tiles_bitwise(require_gpu, bc):
    """Non-periodic x with nx = 32 (ring split): the extended box's two ring
    columns run on the tensor engine as transposed column tiles (32 cells
    along the mid axis, region [36 rows][5 columns]); with the option
    ring_tiles=0 the DFMA ring engine computes them.  Both give the oracle's
    bits, including a mid extent that leaves a partial last column tile."""
    from dataclasses import replace
    w = K.baseline_config(4, n=8)
    g = replace(w.grid, nx=32, ny=37, nz=9, dx=1.0 / 32, bc=bc)
    U = K.initial_condition(g, w.ic)
    rset = K.precompute(2, dim=3)
    Uo, do = Oracle(g, rset).run(U, 2)
    for tiles in (1, 0):
        with K.Solver(g, rset) as s:
            s.set_option("ring_tiles", tiles)
            s.set_state(U)
            d = s.advance(2)
            assert np.array_equal(d, do) and np.array_equal(s.get_state(), Uo), tiles
