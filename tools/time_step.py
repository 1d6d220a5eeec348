"""Device time per SSP-RK3 step of a BASELINE workload (CUDA events on the
solver stream), tolerating device-reported runtime errors — for timing
ablation builds whose results are deliberately wrong (KFVM_LIB=...)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2401_16543_b200 as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--opt", action="append", default=[])
a = ap.parse_args()
w = K.baseline_config(a.config, n=a.n)
s = K.Solver(w.grid)
for o in a.opt:
    k, v = o.split("=")
    s.set_option(k, int(v))
st = torch.cuda.ExternalStream(s.stream)
s.generate_ic(w.ic)
s.run_async(1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
s.run_async(a.steps)
e1.record(st)
torch.cuda.synchronize()
try:
    s.sync()
    ok = "ok"
except Exception as ex:  # noqa: BLE001
    ok = f"device error ({type(ex).__name__})"
print(f"{os.environ.get('KFVM_LIB', 'default')}: {e0.elapsed_time(e1) / a.steps:.2f} ms/step [{ok}]")
