"""compute_rhs of the C++ oracle against a second, independent
straightforward implementation (oracle/rhs_numpy.py: numpy, formulas as the
SPEC/PAPER write them, no shared code or arithmetic order) to 1e-12."""
import numpy as np
import pytest

import paper_2401_16543_b200 as K
from oracle import Oracle
from oracle.rhs_numpy import compute_rhs as rhs_numpy
from paper_2401_16543_b200.config import GridConfig, ICSpec

TOL = 1e-12


def rel_l1(a, b):
    ax = tuple(range(a.ndim - 1))
    return np.abs(a - b).sum(axis=ax) / np.abs(b).sum(axis=ax)


CASES = {
    # S:597's own case: the isentropic vortex on 64^2 (PAPER §6.1 domain [-10,10]^2)
    "vortex_2d_r2_64": (GridConfig(dim=2, radius=2, nx=64, ny=64, dx=20.0 / 64, cfl=0.4),
                        ICSpec("vortex", origin=(-10.0, -10.0, 0.0))),
    "vortex_2d_r3_64": (GridConfig(dim=2, radius=3, nx=64, ny=64, dx=20.0 / 64, cfl=0.4),
                        ICSpec("vortex", origin=(-10.0, -10.0, 0.0))),
    "cfg3_3d_r2_16": (K.baseline_config(3, n=16).grid, K.baseline_config(3).ic),
    "cfg4_3d_r2_outflow_12": (K.baseline_config(4, n=12).grid, K.baseline_config(4).ic),
    "cfg5_3d_r3_12": (K.baseline_config(5, n=12).grid, K.baseline_config(5).ic),
}


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_rhs_matches_independent_numpy(name):
    g, ic = CASES[name]
    U = K.initial_condition(g, ic)
    rset = K.precompute(g.radius, dim=g.dim)
    a = Oracle(g, rset).compute_rhs(U)
    b = rhs_numpy(U, g, rset)
    err = rel_l1(a, b)
    assert (err <= TOL).all(), (name, err)
