"""Small runs covering every kernel family (2-D/3-D engines, ring split,
boundary kinds incl. slit and dirichlet, KXRCF, SSP(4,3), viscous): a quick
all-families check on a GPU (`python tools/all_kernels_run.py`)."""
import os
import sys
from dataclasses import replace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_16543_b200 as K  # noqa: E402
from paper_2401_16543_b200 import problems as P  # noqa: E402
from paper_2401_16543_b200.config import GridConfig  # noqa: E402

GAM = 1.4


def rand_state(g, seed):
    rng = np.random.default_rng(seed)
    return P.cons(GAM, 1.0 + 0.2 * rng.random(g.shape),
                  [0.2 * (rng.random(g.shape) - 0.5) for _ in range(g.dim)],
                  1.0 + 0.2 * rng.random(g.shape))


def run(g, U, steps=1, opts=None, to=None):
    with K.Solver(g, K.precompute(g.radius, dim=g.dim)) as s:
        for k, v in (opts or {}).items():
            s.set_option(k, v)
        s.set_state(U)
        if to is None:
            s.advance(steps)
        else:
            s.advance_to(to, 1000)
        s.get_state()


st3 = tuple(P.cons(GAM, 1.4, (0.0, 0.0, 2.0), 1.0))
g3 = GridConfig(dim=3, radius=2, nx=32, ny=8, nz=8, cfl=0.4,
                sides=("reflecting", "dirichlet", "periodic", "periodic", "slit", "outflow"),
                side_states=(None, st3, None, None, st3, None),
                slits=(None, None, None, None, ((0.25, 0.1), 0.1), None))
U3 = rand_state(g3, 1)
run(g3, U3)                                   # tensor engine + ring split + walls
run(replace(g3, kxrcf=True), U3)              # KXRCF 3-D
run(replace(g3, radius=3), U3)                # R=3 tensor engine + k_limit_states
run(replace(g3, viscous=True, reynolds=100.0), U3)
g2 = GridConfig(dim=2, radius=2, nx=40, ny=24, cfl=0.4,
                sides=("reflecting", "outflow", "slit", "outflow"),
                side_states=(None, None, tuple(P.cons(GAM, GAM, (0.0, 10.0), 1.0)), None),
                slits=(None, None, ((0.0,), 0.2), None))
U2 = rand_state(g2, 2)
for eng in (0, 1, 2, 3, 4):
    run(g2, U2, opts={"engine": eng})
run(replace(g2, kxrcf=True), U2)
run(replace(g2, integrator="ssp43", atol=1e-4, rtol=1e-4), U2, to=0.01)
w = K.baseline_config(3, n=16)
run(w.grid, K.initial_condition(w.grid, w.ic), opts={"chunk_planes": 5, "overlap": 1})
print("all kernel families ran")
