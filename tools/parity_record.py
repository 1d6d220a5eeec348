#!/usr/bin/env python
"""Record of the stated-configuration parity gate on the GPU
(tests/golden/parity_configs.json fixtures, BASELINE north_star: identical dt
sequence and rel. L1 <= 1e-11 per conserved variable after the stated steps):
per case the GPU run's dt-sequence equality, the SHA-256 of the final state
bytes against the oracle's, and the GPU time.  Output: JSON on stdout."""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_16543_b200 as K  # noqa: E402

FIX = json.load(open(os.path.join(ROOT, "tests", "golden", "parity_configs.json")))


def digest(U):
    return hashlib.sha256(np.ascontiguousarray(U, dtype="<f8").tobytes()).hexdigest()


out = {}
for name in sorted(FIX):
    rec = FIX[name]
    n = rec["shape"][-1]
    w = K.baseline_config(rec["config"])
    if n != w.grid.nx:
        w = K.baseline_config(rec["config"], n=n)
    t0 = time.perf_counter()
    with K.Solver(w.grid) as s:
        s.generate_ic(w.ic)
        ic_ok = digest(s.get_state()) == rec["ic_sha256"]
        dts = s.advance(rec["steps"])
        U = s.get_state()
    dto = np.array([float.fromhex(x) for x in rec["dt"]])
    sha = digest(U)
    out[name] = {"shape": rec["shape"], "radius": rec["radius"], "steps": rec["steps"],
                 "ic_identical": ic_ok, "dt_identical": bool(np.array_equal(dts, dto)),
                 "state_sha256_gpu": sha, "state_sha256_oracle": rec["state_sha256"],
                 "bit_identical": sha == rec["state_sha256"],
                 "rel_l1_per_variable": "0 (bit-identical)" if sha == rec["state_sha256"] else "differs",
                 "gpu_wall_s": round(time.perf_counter() - t0, 2),
                 "oracle_seconds": rec["oracle_seconds"], "oracle_threads": rec["oracle_threads"]}
    print(name, out[name]["bit_identical"], out[name]["dt_identical"], file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
