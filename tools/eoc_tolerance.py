"""R = 3 vortex EOC 64^2 -> 128^2 with SSP(4,3) at decreasing atol = rtol: separates the
temporal error of the adaptive third-order integrator from the spatial order."""
import sys, math, json
sys.path.insert(0,'.')
import numpy as np
import paper_2401_16543_b200 as K
from paper_2401_16543_b200.config import GridConfig, ICSpec
V = ICSpec("vortex", origin=(-10.0, -10.0, 0.0))
def l1(n, tol):
    g = GridConfig(dim=2, radius=3, nx=n, ny=n, dx=20.0/n, integrator="ssp43", atol=tol, rtol=tol, cfl=1.0)
    U0 = K.initial_condition(g, V)
    with K.Solver(g) as s:
        s.set_state(U0); s.advance_to(20.0, 10_000_000); U = s.get_state(); st = s.step_stats()
    return float(np.abs(U[...,0]-U0[...,0]).sum()*g.dx**2), st
out = {}
for tol in (1e-6, 1e-8, 1e-10):
    e = {n: l1(n, tol) for n in (64, 128)}
    out[str(tol)] = {"l1": {k: v[0] for k, v in e.items()}, "steps": {k: v[1] for k, v in e.items()},
                     "eoc_128": math.log(e[64][0]/e[128][0])/math.log(2)}
    print(tol, out[str(tol)], flush=True)
print(json.dumps(out))
