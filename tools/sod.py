"""Sod shock tube (PAPER §6.2, SPEC acceptance 3) on the GPU: L1 density error
against the exact Riemann solution for R=2 and R=3 at Delta = 1/100 and 1/400
with SSP(4,3)+SSP(3,2) (atol = rtol = 1e-4, CFL 1.25).

    python tools/sod.py [--out profiles/r01/sod.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_problems import sod_aligned_metrics  # noqa: E402

rows = [sod_aligned_metrics(R, n) for R in (2, 3) for n in (100, 200, 400)]
for r in rows:
    print(r, flush=True)
if "--out" in sys.argv:
    with open(sys.argv[sys.argv.index("--out") + 1], "w") as f:
        json.dump(rows, f, indent=1)
