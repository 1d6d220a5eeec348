"""Run a few SSP-RK3 steps of a BASELINE workload on cuda:0 (for ncu/compute-sanitizer)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_16543_b200 as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--engine", type=int, default=-1, help="-1: the solver default")
a = ap.parse_args()
w = K.baseline_config(a.config, n=a.n)
with K.Solver(w.grid) as s:
    if a.engine >= 0:
        s.set_option("engine", a.engine)
    s.generate_ic(w.ic)
    d = s.advance(a.steps)
    print("ok", w.grid.shape, d)
