"""The 16-warp W-cache engine (k_states_w, kfvm_recon_w.cuh) against the CPU
oracle and against k_states_u (option wide=0), bit for bit: row counts that
leave a partial 4-row block (rows past the box are zero-filled by the TMA
unit and never stored), periodic and outflow/wall sides, several z blocks
(kz), the chunked stage schedule, and runs of several steps.  The engine
applies to every 3-D R=2 grid: ring-split segments (nx = 32 k or 32 k - 1,
periodic x) start on an even x, the others one column earlier."""
from dataclasses import replace

import numpy as np
import pytest

import paper_2401_16543_b200 as K
from paper_2401_16543_b200.config import GridConfig
from oracle import Oracle

pytestmark = pytest.mark.gpu

GRIDS = [
    # (nx, ny, nz, bc): ny + 2 = 4 m + {0, 1, 2, 3} rows of extended cells
    (32, 10, 9, "periodic"),
    (32, 11, 8, "outflow"),
    (64, 13, 7, "outflow"),
    (32, 12, 8, "reflecting"),
    (40, 9, 8, "periodic"),   # periodic x: ring copy, interior segments (last one partial)
    (40, 10, 8, "outflow"),   # no ring split: segments start at x = -1 (odd: shifted TMA box)
    (100, 9, 7, "outflow"),
]


def _case(nx, ny, nz, bc):
    w = K.baseline_config(4 if bc != "periodic" else 3, n=16)
    g = replace(w.grid, nx=nx, ny=ny, nz=nz, dx=1.0 / nx, bc=bc)
    U = K.initial_condition(g, w.ic)
    return g, U, K.precompute(2, dim=3)


@pytest.mark.parametrize("nx,ny,nz,bc", GRIDS, ids=[f"{a}x{b}x{c}_{d}" for a, b, c, d in GRIDS])
def test_wide_states_and_run_bitwise(require_gpu, nx, ny, nz, bc):
    g, U, rset = _case(nx, ny, nz, bc)
    o = Oracle(g, rset)
    So = o.reconstruct_states(U)
    Uo, dto = o.run(U, 2)
    for wide in (1, 0):
        with K.Solver(g, rset) as s:
            s.set_option("wide", wide)
            assert np.array_equal(s.reconstruct_states(U), So), f"states, wide={wide}"
            s.set_state(U)
            dts = s.advance(2)
            assert np.array_equal(dts, dto), (wide, dts, dto)
            assert np.array_equal(s.get_state(), Uo), f"run, wide={wide}"


@pytest.mark.parametrize("kz,chunk", [(3, 0), (5, 4), (32, 3)])
def test_wide_z_blocks_and_chunks(require_gpu, kz, chunk):
    g, U, rset = _case(32, 14, 11, "outflow")
    Uo, dto = Oracle(g, rset).run(U, 2)
    with K.Solver(g, rset) as s:
        s.set_option("kz", kz)
        if chunk:
            s.set_option("chunk_planes", chunk)
        s.set_state(U)
        dts = s.advance(2)
        assert np.array_equal(dts, dto)
        assert np.array_equal(s.get_state(), Uo)
