"""Run the SPEC problem catalog (paper_2401_16543_b200/problems.py) to each
problem's final time on the GPU with its own integrator (SSP(4,3)+SSP(3,2),
PI controller) and record run statistics: accepted / rejected steps, the
final time, min density / pressure, total mass change (mass enters and leaves
only through inflow / outflow sides), wall time.  Output: one JSON document
(argv[1], default gpurun_out/catalog.json)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_16543_b200 as K  # noqa: E402
from paper_2401_16543_b200 import problems as P  # noqa: E402

RUNS = [
    # (name, constructor kwargs) — resolutions below the paper's 1/512 so
    # the whole catalog runs in a few minutes on one GPU
    ("sod_aligned", {"n": 200, "radius": 2}),
    ("richtmyer_meshkov", {"n": 64, "radius": 2}),
    ("astro_jet_high", {"n": 128, "radius": 3}),
    ("astro_jet_low", {"n": 128, "radius": 3}),
    ("rayleigh_taylor", {"n": 128, "radius": 3}),
]


def pressure(U, gamma, dim):
    q = (U[..., 1:1 + dim] ** 2).sum(-1)
    return (gamma - 1.0) * (U[..., -1] - 0.5 * q / U[..., 0])


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "catalog.json")
    res = []
    for name, kw in RUNS:
        pr = P.problem(name, **kw)
        g = pr.grid
        cell = (g.dx if g.dx else 1.0 / g.nx) ** g.dim
        with K.Solver(g, K.precompute(g.radius, dim=g.dim)) as s:
            s.set_state(pr.U0)
            t0 = time.perf_counter()
            try:
                steps, t = s.advance_to(pr.t_final, 2_000_000)
                err = None
            except Exception as e:  # record the failure, keep going
                steps, t, err = -1, float("nan"), str(e)
            wall = time.perf_counter() - t0
            acc, rej = s.step_stats()
            U = s.get_state()
        p = pressure(U, g.gamma, g.dim)
        res.append({
            "problem": name, "grid": list(g.shape), "radius": g.radius, "sides": list(g.sides),
            "riemann": g.riemann, "t_final": pr.t_final, "t_reached": t, "accepted": acc,
            "rejected": rej, "error": err, "wall_s": round(wall, 3),
            "min_rho": float(U[..., 0].min()), "min_p": float(p.min()),
            "max_rho": float(U[..., 0].max()),
            "mass_initial": float(pr.U0[..., 0].sum() * cell), "mass_final": float(U[..., 0].sum() * cell),
            "finite": bool(np.isfinite(U).all()),
        })
        print(json.dumps(res[-1]))
    with open(out, "w") as f:
        json.dump({"note": __doc__.split("\n\n")[0], "runs": res}, f, indent=1)


if __name__ == "__main__":
    main()
