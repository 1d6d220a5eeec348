"""Per-phase cycle breakdown of the reconstruction kernel (needs a library
built with EXTRA=-DKFVM_PHASE_TIMING)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_16543_b200 as K  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
eng = int(sys.argv[3]) if len(sys.argv) > 3 else 5
w = K.baseline_config(cfg, n=n)
L = K._lib()
buf = (C.c_ulonglong * 8)()
with K.Solver(w.grid) as s:
    s.set_option("engine", eng)
    s.generate_ic(w.ic)
    s.advance(1)
    L.kfvm_phase_cycles(buf, 1)
    s.advance(2)
    L.kfvm_phase_cycles(buf, 0)
if eng == 5:
    names = ["plane-setup", "pass1", "omega", "pass2", "phiinv+limiter", "exchange+edges+sync",
             "riemann+quadrature+F", "wait+sync"]
else:
    names = ["plane-setup", "pass1", "omega", "pass2", "phiinv+limiter+store", "wait+sync", "-", "-"]
tot = sum(buf) or 1
for i in range(8):
    print(f"{names[i]:12s} {buf[i]:16d}  {100.0 * buf[i] / tot:5.1f}%")
