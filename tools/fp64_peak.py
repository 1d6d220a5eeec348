"""Measure the FP64 roofline denominators on the current B200 (DFMA pipe and
DMMA) with the microbenchmarks in libkfvm_b200.so; prints one JSON line and,
with --write, stores it as profiles/fp64_peak.json."""
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_16543_b200 import _abi  # noqa: E402

L = _abi.lib()
best = {"dfma_tflops": 0.0, "dmma_tflops": 0.0}
for _ in range(5):
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    rc = L.kfvm_fp64_peak(C.byref(a), C.byref(b), C.byref(c))
    assert rc == 0, rc
    best["dfma_tflops"] = max(best["dfma_tflops"], a.value)
    best["dmma_tflops"] = max(best["dmma_tflops"], b.value)
    best["sm_clock_ghz_attr"] = c.value
try:
    best["gpu"] = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.sm,clocks.max.sm",
                                  "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
except Exception:
    pass
best["how"] = ("k_dfma_peak: 8 independent fma chains/thread, 4 CTAs x 512 thr per SM; "
               "k_dmma_peak: 4 independent mma.sync.m8n8k4.f64 chains/warp; best of 5, CUDA events")
print(json.dumps(best))
if "--write" in sys.argv:
    with open(os.path.join(ROOT, "profiles", "fp64_peak.json"), "w") as f:
        json.dump(best, f, indent=1)
