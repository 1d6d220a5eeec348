#!/usr/bin/env python
"""Generate tests/golden/recon_golden.npz: reconstruction vectors computed by the
independent mpmath restatement (oracle/recon_ref.py, 40 digits, rounded once
to FP64).  These pin the product's binary128 table.
3-D R=3 covers the substencils only (the 123-cell full stencil takes tens of
minutes in mpmath without factor reuse)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.recon_ref import recon_vectors, stencils  # noqa: E402

CASES = [(2, 2, range(6)), (2, 3, range(6)), (3, 2, range(8)), (3, 3, [1, 2, 5])]
out = {}
for dim, R, qs in CASES:
    for q in qs:
        t = time.time()
        F, D, p = recon_vectors(dim, R, q, dps=40)
        out[f"d{dim}r{R}q{q}_face"] = F
        out[f"d{dim}r{R}q{q}_deriv"] = D
        out[f"d{dim}r{R}q{q}_degree"] = np.array(p)
        full, members = stencils(dim, R)
        out[f"d{dim}r{R}q{q}_cells"] = np.array([full[h] for h in members[q]])
        print(dim, R, q, "deg", p, f"{time.time() - t:.1f}s", flush=True)
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "recon_golden.npz"), **out)
print("wrote tests/golden/recon_golden.npz")
