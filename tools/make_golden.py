#!/usr/bin/env python
"""Generate tests/golden/recon_golden.npz: reconstruction vectors computed by the
independent mpmath restatement (oracle/recon_ref.py, 40 digits, rounded once
to FP64).  These pin the product's binary128 table.
3-D R=3 covers the full stencil (the worst-conditioned system, cond ~7e17)
and three substencils."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.recon_ref import recon_vectors, stencils  # noqa: E402

CASES = [(2, 2, range(6)), (2, 3, range(6)), (3, 2, range(8)), (3, 3, [0, 1, 2, 5])]
# `make_golden.py d r q [q ...]`: (re)compute only those cases and merge them
# into the existing file (the 3-D R=3 full stencil, N = 123 + 56 monomials,
# takes a few minutes with the factor reused for its 73 right-hand sides)
PATH = os.path.join(ROOT, "tests", "golden", "recon_golden.npz")
out = {}
if len(sys.argv) > 3:
    CASES = [(int(sys.argv[1]), int(sys.argv[2]), [int(x) for x in sys.argv[3:]])]
    out = dict(np.load(PATH))
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
np.savez_compressed(PATH, **out)
print("wrote tests/golden/recon_golden.npz")
