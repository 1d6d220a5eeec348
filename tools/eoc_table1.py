"""PAPER Table 1 (isentropic vortex EOC) on the GPU.

The vortex of [-10,10]^2 (periodic) is advanced one period (t = 20) and the
L1 density error sum|rho - rho0| dx^2 against the initial state is reported
with the EOC, next to the paper's numbers.  Integrator: the reference's
SSP(4,3)+SSP(3,2) with the PI controller at atol = rtol = 1e-6 and a maximal
CFL of 1.0 (the paper used the [4S]* pair at the same tolerances), and,
for comparison, BASELINE's fixed-CFL SSP-RK3 at CFL 0.4.

    python tools/eoc_table1.py [--max-n 128] [--out profiles/r01/eoc_table1.json]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_16543_b200 as K  # noqa: E402
from paper_2401_16543_b200.config import GridConfig, ICSpec  # noqa: E402

PAPER = {2: {32: 1.45e-3, 64: 2.27e-4, 128: 1.47e-5, 256: 5.39e-7},
         3: {32: 7.51e-4, 64: 7.50e-5, 128: 1.46e-6, 256: 1.76e-8}}


def l1_error(n, R, integrator):
    kw = dict(integrator="ssp43", atol=1e-6, rtol=1e-6, cfl=1.0) if integrator == "ssp43" \
        else dict(cfl=0.4)
    g = GridConfig(dim=2, radius=R, nx=n, ny=n, bc="periodic", dx=20.0 / n, **kw)
    U0 = K.initial_condition(g, ICSpec("vortex", origin=(-10.0, -10.0, 0.0)))
    t0 = time.perf_counter()
    with K.Solver(g) as s:
        s.set_state(U0)
        steps, t = s.advance_to(20.0, 200000)
        stats = s.step_stats() if integrator == "ssp43" else (steps, 0)
        U = s.get_state()
    return (float((abs(U[..., 0] - U0[..., 0])).sum() * g.dx ** 2), stats,
            time.perf_counter() - t0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-n", type=int, default=128)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for integ in ("ssp43", "ssprk3"):
        for R in (2, 3):
            prev = None
            for n in (32, 64, 128, 256):
                if n > a.max_n:
                    break
                e, (acc, rej), sec = l1_error(n, R, integ)
                eoc = math.log(prev / e) / math.log(2) if prev else None
                pe = PAPER[R][n]
                pprev = PAPER[R].get(n // 2)
                peoc = math.log(pprev / pe) / math.log(2) if prev and pprev else None
                rows.append({"integrator": integ, "R": R, "n": n, "l1": e, "eoc": eoc,
                             "paper_l1": pe, "paper_eoc": peoc, "accepted": acc,
                             "rejected": rej, "seconds": round(sec, 3)})
                print(f"{integ:7s} R={R} {n:4d}^2  L1 {e:.3e}  EOC "
                      f"{'   -' if eoc is None else f'{eoc:5.2f}'}   paper {pe:.2e} "
                      f"{'   -' if peoc is None else f'{peoc:5.2f}'}   steps {acc} rej {rej}",
                      flush=True)
                prev = e
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
