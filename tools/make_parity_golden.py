#!/usr/bin/env python
"""Oracle fixtures for the stated-configuration parity gate
(tests/test_gpu_parity_configs.py; BASELINE.json north_star: rel. L1 <= 1e-11
per conserved variable after the stated steps, identical dt sequence).

For each case the CPU oracle (oracle/libkfvm_oracle.so, all host threads)
runs the BASELINE recipe from the oracle's own IC restatement and the
hash-pinned table file, and tests/golden/parity_configs.json records:
the dt sequence (exact, float.hex), the SHA-256 of the final AoS state
bytes, per-variable L1 norms and the run time.  The GPU test compares the
device result's bytes against the hash (bit-identity => every per-variable
rel. L1 is 0) and, on a mismatch, re-runs the oracle live to report the
actual rel. L1 / max-ulp.

    python tools/make_parity_golden.py [case ...]     (default: every case)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2401_16543_b200 as K  # noqa: E402  (configs only: no library load)
from oracle import Oracle  # noqa: E402
from oracle.kfvm_oracle import initial_condition  # noqa: E402
from oracle.table_file import load_table  # noqa: E402

PATH = os.path.join(ROOT, "tests", "golden", "parity_configs.json")

# name: (config index, n (None = stated size), steps (None = stated))
CASES = {
    "cfg1_full_256sq_20steps": (1, None, None),
    "cfg2_full_1024sq_50steps": (2, None, None),
    "cfg3_128cube_10steps": (3, 128, None),
    "cfg4_recipe_128cube_10steps": (4, 128, None),
    "cfg5_recipe_128cube_r3_5steps": (5, 128, None),
    "cfg3_full_256cube_10steps": (3, None, None),
}


def case_workload(name):
    idx, n, steps = CASES[name]
    w = K.baseline_config(idx, n=n)
    return w, (steps or w.steps)


def state_digest(U: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(U, dtype="<f8").tobytes()).hexdigest()


def main(names):
    data = json.load(open(PATH)) if os.path.exists(PATH) else {}
    nt = os.cpu_count() or 1
    for name in names:
        w, steps = case_workload(name)
        g = w.grid
        t0 = time.time()
        U = initial_condition(g, w.ic, nthreads=nt)
        Uo, dts = Oracle(g, load_table(g.dim, g.radius), nthreads=nt).run(U, steps)
        dt_run = time.time() - t0
        ax = tuple(range(Uo.ndim - 1))
        data[name] = {
            "config": w.index, "shape": list(g.shape), "radius": g.radius, "bc": g.bc,
            "steps": steps, "ic_sha256": state_digest(U), "state_sha256": state_digest(Uo),
            "dt": [float(x).hex() for x in dts],
            "l1": np.abs(Uo).sum(axis=ax).tolist(),
            "oracle_seconds": round(dt_run, 1), "oracle_threads": nt,
            "generator": "tools/make_parity_golden.py",
        }
        print(f"{name}: {dt_run:.0f} s, dt[0] {dts[0]:.6e}, sha {data[name]['state_sha256'][:16]}",
              flush=True)
        with open(PATH, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
