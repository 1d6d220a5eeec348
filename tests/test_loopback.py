"""The library's multi-rank slab path with nranks = 2 and 3 on one GPU, through
the in-process loopback transport (kfvm_loopback_id): one Solver handle per
rank, each driven by its own host thread like an MPI rank, exchanging halo
planes / KXRCF edge flags / the dt maximum / the SSP(4,3) error planes by
device copies with NCCL's semantics.  This runs halo(), k_halo_local, the
rank-offset boundary code, the overlapped stage schedule and the collectives
with real peers; the gathered slabs must be the oracle's bits on the whole
grid (BASELINE north_star (4); the reference's Kokkos+MPI decomposition,
PAPER.md:463)."""
import threading
from dataclasses import replace

import numpy as np
import pytest

import paper_2401_16543_b200 as K
from paper_2401_16543_b200 import problems as P
from paper_2401_16543_b200.config import GridConfig
from paper_2401_16543_b200.solver import loopback_id
from oracle import Oracle

pytestmark = pytest.mark.gpu

GAM = 1.4


def run_ranks(g, rset, U, nranks, body, options=()):
    """Create nranks loopback handles, give each its slab of U, run body(s) on
    one thread per rank; returns the per-rank results and the gathered state."""
    lid = loopback_id()
    solvers = [K.Solver(g, rset, rank=r, nranks=nranks, nccl_id=lid) for r in range(nranks)]
    out, err = [None] * nranks, []
    try:
        for s in solvers:
            for k, v in options:
                s.set_option(k, v)
            s.set_state(np.ascontiguousarray(U[s.p0:s.p0 + s.np_local]))

        def work(r):
            try:
                out[r] = body(solvers[r])
            except Exception as e:  # noqa: BLE001
                err.append((r, e))

        th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
        assert not any(t.is_alive() for t in th), "a rank hung"
        assert not err, err
        Ug = np.concatenate([s.get_state() for s in solvers], axis=0)
    finally:
        for s in solvers:
            s.close()
    return out, Ug


CASES = [
    ("cfg1_2d_periodic", lambda: K.baseline_config(1, n=24), 2),
    ("cfg2_2d_outflow", lambda: K.baseline_config(2, n=24), 2),
    ("cfg3_3d_periodic", lambda: K.baseline_config(3, n=16), 2),
    ("cfg4_3d_outflow", lambda: K.baseline_config(4, n=14), 2),
    ("cfg5_3d_r3", lambda: K.baseline_config(5, n=12), 1),
]


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("name,mk,steps", CASES, ids=[c[0] for c in CASES])
def test_loopback_run(require_gpu, name, mk, steps, nranks):
    w = mk()
    g = w.grid
    U = K.initial_condition(g, w.ic)
    rset = K.precompute(g.radius, dim=g.dim)
    Uo, dto = Oracle(g, rset).run(U, steps)
    dts, Ug = run_ranks(g, rset, U, nranks, lambda s: s.advance(steps))
    for d in dts:
        assert np.array_equal(d, dto)
    assert np.array_equal(Ug, Uo)


@pytest.mark.parametrize("overlap", [0, 1])
def test_loopback_schedules(require_gpu, overlap):
    """Serial and overlapped (halo on a second stream) stage schedules, and a
    chunked slab (halo-dependent chunks after the exchange)."""
    w = K.baseline_config(4, n=14)
    g = w.grid
    U = K.initial_condition(g, w.ic)
    rset = K.precompute(2, dim=3)
    Uo, dto = Oracle(g, rset).run(U, 2)
    for opts in ((("overlap", overlap),), (("overlap", overlap), ("chunk_planes", 2))):
        dts, Ug = run_ranks(g, rset, U, 2, lambda s: s.advance(2), opts)
        assert np.array_equal(dts[0], dto) and np.array_equal(Ug, Uo)


def _walls3():
    st = tuple(P.cons(GAM, 1.4, (0.0, 0.0, 2.0), 1.0))
    return GridConfig(dim=3, radius=2, nx=12, ny=12, nz=12, cfl=0.4,
                      sides=("reflecting", "outflow", "periodic", "periodic", "slit", "reflecting"),
                      side_states=(None, None, None, None, st, None),
                      slits=(None, None, None, None, ((0.5, 0.5), 0.25), None))


@pytest.mark.parametrize("nranks", [2, 3])
def test_loopback_walls_kxrcf_ssp43(require_gpu, nranks):
    """Slit inflow / reflecting slab ends, the KXRCF edge-flag exchange and
    SSP(4,3) with the error-norm allgather and the PI controller."""
    g = _walls3()
    rng = np.random.default_rng(31)
    U = P.cons(GAM, 1.0 + 0.2 * rng.random(g.shape),
               [0.2 * (rng.random(g.shape) - 0.5) for _ in range(3)],
               1.0 + 0.2 * rng.random(g.shape))
    rset = K.precompute(2, dim=3)
    for gg in (g, replace(g, kxrcf=True)):
        Uo, dto = Oracle(gg, rset).run(U, 2)
        dts, Ug = run_ranks(gg, rset, U, nranks, lambda s: s.advance(2))
        assert all(np.array_equal(d, dto) for d in dts)
        assert np.array_equal(Ug, Uo)
    g43 = replace(g, integrator="ssp43", atol=1e-5, rtol=1e-5)
    Uo, dto, na, nr, to = Oracle(g43, rset).advance43(U, 0.01)

    def body(s):
        steps, t = s.advance_to(0.01, 10000)
        return s.step_stats(), t, s.dt_sequence(na)

    res, Ug = run_ranks(g43, rset, U, nranks, body)
    for stats, t, d in res:
        assert stats == (na, nr) and t == to
        assert np.array_equal(d, dto)
    assert np.array_equal(Ug, Uo)


def test_loopback_group_mismatch(require_gpu):
    """A handle whose rank count differs from its group's is refused."""
    w = K.baseline_config(1, n=16)
    lid = loopback_id()
    with K.Solver(w.grid, rank=0, nranks=2, nccl_id=lid):
        with pytest.raises(ValueError):
            K.Solver(w.grid, rank=1, nranks=4, nccl_id=lid)


@pytest.mark.parametrize("cfg,n", [(2, 24), (4, 14), (5, 12)])
def test_loopback_rank_offset_ic(require_gpu, cfg, n):
    """The device IC generator on each rank's slab (rank-offset planes) equals
    the host generator's global field."""
    w = K.baseline_config(cfg, n=n)
    g = w.grid
    U = K.initial_condition(g, w.ic)
    lid = loopback_id()
    solvers = [K.Solver(g, rank=r, nranks=3, nccl_id=lid) for r in range(3)]
    try:
        for s in solvers:
            s.generate_ic(w.ic)
        Ug = np.concatenate([s.get_state() for s in solvers], axis=0)
    finally:
        for s in solvers:
            s.close()
    assert np.array_equal(Ug, U)
