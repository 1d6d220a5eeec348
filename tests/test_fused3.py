"""The fused 3-D stage engine (k_fused3 + k_edges3, engine 5: reconstruction,
Riemann solves and face quadrature in one kernel; face states only on tile
edges) against the CPU oracle, bit for bit, on shapes that exercise every
edge class: partial 8x4 tiles, x/y tile edges, z-block edges (small KZ), the
overlapped three-range schedule, periodic and outflow boundaries, HLL."""
import numpy as np
import pytest
from dataclasses import replace

import paper_2401_16543_b200 as K
from oracle import Oracle

pytestmark = pytest.mark.gpu

SHAPES = [(10, 7, 9), (17, 13, 6), (16, 8, 12), (9, 21, 5)]


def _case(idx, shape, **over):
    w = K.baseline_config(idx, n=8)
    nx, ny, nz = shape
    g = replace(w.grid, nx=nx, ny=ny, nz=nz, dx=1.0 / nx, **over)
    return g, w.ic, K.initial_condition(g, w.ic), K.precompute(2, dim=3)


@pytest.mark.parametrize("shape", SHAPES, ids=["x".join(map(str, s)) for s in SHAPES])
@pytest.mark.parametrize("idx", [3, 4], ids=["periodic", "outflow"])
@pytest.mark.parametrize("kz", [32, 2])
def test_fused3_run_bitwise(require_gpu, idx, shape, kz):
    g, ic, U, rset = _case(idx, shape)
    with K.Solver(g, rset) as s:
        s.set_option("engine", 5)
        s.set_option("kz", kz)
        s.set_state(U)
        d = s.advance(2)
        Ug = s.get_state()
    Uo, do = Oracle(g, rset).run(U, 2)
    assert np.array_equal(d, do)
    assert np.array_equal(Ug, Uo)


@pytest.mark.parametrize("idx", [3, 4])
def test_fused3_rhs_and_hll(require_gpu, idx):
    g, ic, U, rset = _case(idx, (12, 11, 10), riemann="hll")
    with K.Solver(g, rset) as s:
        s.set_option("engine", 5)
        L = s.compute_rhs(U)
    assert np.array_equal(L, Oracle(g, rset).compute_rhs(U))


@pytest.mark.parametrize("kz", [32, 3])
def test_fused3_overlapped_ranges(require_gpu, kz):
    """The overlapped schedule splits each stage into three plane ranges
    (halo-independent planes first): their z-edges go through the edge
    buffers, the bits stay the oracle's."""
    g, ic, U, rset = _case(4, (12, 10, 14))
    outs = []
    for ov in (0, 1):
        with K.Solver(g, rset) as s:
            s.set_option("engine", 5)
            s.set_option("kz", kz)
            s.set_option("overlap", ov)
            s.set_state(U)
            outs.append((s.advance(2), s.get_state()))
    Uo, do = Oracle(g, rset).run(U, 2)
    for d, A in outs:
        assert np.array_equal(d, do) and np.array_equal(A, Uo)


def test_fused3_equals_tensor_engine_and_states_api(require_gpu):
    """engine 5 == engine 2 (face states through HBM) on config 3's recipe;
    reconstruct_states on a fused handle runs the states engine (same bits)."""
    g, ic, U, rset = _case(3, (14, 14, 14))
    outs = []
    for eng in (5, 2):
        with K.Solver(g, rset) as s:
            s.set_option("engine", eng)
            s.set_state(U)
            outs.append((s.advance(3), s.get_state(), s.reconstruct_states(U)))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])
    assert np.array_equal(outs[0][2], outs[1][2])
