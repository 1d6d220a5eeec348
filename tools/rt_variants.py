"""RT mirror-symmetry growth under variants (diagnosis for the SPEC item-9 check):
asymmetry of the x-momentum (max |m_x(x) + m_x(1/4 - x)|) at checkpoints."""
import json
import sys
from dataclasses import replace

import numpy as np

sys.path.insert(0, '.')
import paper_2401_16543_b200 as K  # noqa: E402
from paper_2401_16543_b200 import problems as P  # noqa: E402


def asym(U):
    M = U[:, ::-1, :].copy()
    M[..., 1] *= -1.0
    return [float(x) for x in np.abs(U - M).max(axis=(0, 1))]


VARIANTS = [
    ("full", {}, 3),
    ("xper", {"sides": ("periodic", "periodic", "dirichlet", "dirichlet")}, 3),
    ("ywall", {"sides": ("reflecting", "reflecting", "reflecting", "reflecting"), "side_states": None}, 3),
    ("xper_ywall", {"sides": ("periodic", "periodic", "reflecting", "reflecting"), "side_states": None}, 3),
    ("r2", {}, 2),
    ("kappa0", {"kappa": 0.0}, 3),
]
for name, kw, R in VARIANTS:
    pr = P.rayleigh_taylor(n=128, radius=R)
    g = replace(pr.grid, **kw)
    ic = pr.U0
    Mi = ic[:, ::-1, :].copy()
    Mi[..., 1] *= -1.0
    U0 = 0.5 * (ic + Mi)
    h = []
    with K.Solver(g) as s:
        s.set_state(U0)
        for tc in (0.05, 0.1, 0.15, 0.2, 0.25, 0.3):
            s.advance_to(tc, 10_000_000)
            U = s.get_state()
            a = asym(U)
            # where: the row (y) and column (x) of the largest x-momentum asymmetry
            M = U[:, ::-1, 1]
            d = np.abs(U[..., 1] + M)
            j, i = np.unravel_index(np.argmax(d), d.shape)
            h.append((tc, a[1], int(j), int(i)))
    print(name, json.dumps(h), flush=True)
