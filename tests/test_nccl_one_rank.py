"""The multi-GPU (NCCL) slab path on one GPU: KFVM_FORCE_NCCL=1 makes a
one-rank handle take every multi-rank branch — a one-rank communicator, the
halo planes by ncclSend/ncclRecv to itself (periodic) or k_halo_local at the
global ends, the overlapped stage schedule, ncclAllReduce(max) for dt, the
KXRCF flag exchange and the SSP(4,3) error-norm ncclAllGather — and must give
the oracle's bits.  (Only one GPU is available in this run; the N-rank
decomposition itself is covered by tests/test_dist_gloo.py.)"""
import numpy as np
import pytest

import paper_2401_16543_b200 as K
from paper_2401_16543_b200 import problems as P
from paper_2401_16543_b200.config import GridConfig
from oracle import Oracle

pytestmark = pytest.mark.gpu

GAM = 1.4


def _walls3():
    st = tuple(P.cons(GAM, 1.4, (0.0, 0.0, 2.0), 1.0))
    return GridConfig(dim=3, radius=2, nx=12, ny=12, nz=12, cfl=0.4,
                      sides=("reflecting", "outflow", "periodic", "periodic", "slit", "reflecting"),
                      side_states=(None, None, None, None, st, None),
                      slits=(None, None, None, None, ((0.5, 0.5), 0.25), None))


CASES = [
    ("cfg1_2d_periodic", lambda: K.baseline_config(1, n=24), 2),
    ("cfg2_2d_outflow", lambda: K.baseline_config(2, n=24), 2),
    ("cfg3_3d_periodic", lambda: K.baseline_config(3, n=16), 2),
    ("cfg4_3d_outflow", lambda: K.baseline_config(4, n=14), 2),
    ("cfg5_3d_r3", lambda: K.baseline_config(5, n=12), 1),
]


@pytest.mark.parametrize("name,mk,steps", CASES, ids=[c[0] for c in CASES])
def test_forced_nccl_run(require_gpu, monkeypatch, name, mk, steps):
    monkeypatch.setenv("KFVM_FORCE_NCCL", "1")
    w = mk()
    g = w.grid
    U = K.initial_condition(g, w.ic)
    rset = K.precompute(g.radius, dim=g.dim)
    Uo, dto = Oracle(g, rset).run(U, steps)
    with K.Solver(g, rset) as s:
        s.set_state(U)
        dts = s.advance(steps)
        assert np.array_equal(dts, dto)
        assert np.array_equal(s.get_state(), Uo)


def test_forced_nccl_walls_kxrcf_ssp43(require_gpu, monkeypatch):
    monkeypatch.setenv("KFVM_FORCE_NCCL", "1")
    from dataclasses import replace
    g = _walls3()
    rng = np.random.default_rng(31)
    U = P.cons(GAM, 1.0 + 0.2 * rng.random(g.shape), [0.2 * (rng.random(g.shape) - 0.5) for _ in range(3)],
               1.0 + 0.2 * rng.random(g.shape))
    rset = K.precompute(2, dim=3)
    for gg in (g, replace(g, kxrcf=True)):
        Uo, dto = Oracle(gg, rset).run(U, 2)
        with K.Solver(gg, rset) as s:
            s.set_state(U)
            assert np.array_equal(s.advance(2), dto)
            assert np.array_equal(s.get_state(), Uo)
    g43 = replace(g, integrator="ssp43", atol=1e-5, rtol=1e-5)
    Uo, dto, na, nr, to = Oracle(g43, rset).advance43(U, 0.01)
    with K.Solver(g43, rset) as s:
        s.set_state(U)
        steps, t = s.advance_to(0.01, 10000)
        assert s.step_stats() == (na, nr) and t == to
        assert np.array_equal(s.dt_sequence(na), dto)
        assert np.array_equal(s.get_state(), Uo)
