#!/usr/bin/env python
"""SPEC acceptance checks for the §8(f) rows, run on the GPU path
(/root/reference/SPEC.md "ACCEPTANCE CRITERIA"):

  conservation  item 4: periodic isentropic vortex (and a 3-D periodic case),
                200 accepted steps; totals of every conserved variable change
                by <= 1e-12 relative
  kxrcf_rmi     item 6: Richtmyer-Meshkov at dx = 1/128 to t = 1.0 with the
                KXRCF indicator: flagged fraction over the last 50 steps
                < 15 %; final density L1 difference against the run without
                the indicator < 1e-3
  rt_mirror     item 9: viscous Rayleigh-Taylor at dx = 1/128 to t = 1.0
                (the cos(8 pi x) perturbation is mirror-symmetric about
                x = 1/8 on [0, 1/4]): reflection symmetry to 1e-11
  vortex_eoc    item 2: R = 3 vortex EOC 64^2 -> 128^2 (>= 5.0), with
                SSP(4,3) at atol = rtol = 1e-6 and with SSP-RK3 at CFL 0.4

Each function returns a dict of measured values; `python tools/acceptance.py
[name ...] > out.json` runs them (tests/test_acceptance.py asserts the
thresholds)."""
import json
import math
import os
import sys
import time
from dataclasses import replace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_16543_b200 as K  # noqa: E402
from paper_2401_16543_b200 import problems as P  # noqa: E402
from paper_2401_16543_b200.config import GridConfig, ICSpec  # noqa: E402

VORTEX = ICSpec("vortex", origin=(-10.0, -10.0, 0.0))


def _totals(U):
    ax = tuple(range(U.ndim - 1))
    return U.sum(axis=ax), np.abs(U).sum(axis=ax)


def conservation(steps=200):
    out = {}
    cases = [
        ("vortex_2d_r2_64", GridConfig(dim=2, radius=2, nx=64, ny=64, dx=20.0 / 64, cfl=0.4), VORTEX),
        ("vortex_2d_r3_64", GridConfig(dim=2, radius=3, nx=64, ny=64, dx=20.0 / 64, cfl=0.4), VORTEX),
        ("cfg3_3d_r2_32", None, None),
    ]
    for name, g, ic in cases:
        if g is None:
            w = K.baseline_config(3, n=32)
            g, ic = w.grid, w.ic
        U0 = K.initial_condition(g, ic)
        with K.Solver(g) as s:
            s.set_state(U0)
            s.advance(steps)
            U = s.get_state()
        t0, a0 = _totals(U0)
        t1, _ = _totals(U)
        # relative to the total (the scale of |U| where a total is ~0)
        rel = np.abs(t1 - t0) / np.maximum(np.abs(t0), a0 * 1e-3)
        out[name] = {"steps": steps, "rel_change": rel.tolist(), "max": float(rel.max())}
    # SSP(4,3): 200 accepted steps of the adaptive integrator
    g = GridConfig(dim=2, radius=2, nx=64, ny=64, dx=20.0 / 64, cfl=1.0, integrator="ssp43",
                   atol=1e-6, rtol=1e-6)
    U0 = K.initial_condition(g, VORTEX)
    with K.Solver(g) as s:
        s.set_state(U0)
        s.advance_to(1e9, max_steps=steps)  # attempts; stops at max_steps attempts
        acc, rej = s.step_stats()
        U = s.get_state()
    t0, a0 = _totals(U0)
    t1, _ = _totals(U)
    rel = np.abs(t1 - t0) / np.maximum(np.abs(t0), a0 * 1e-3)
    out["vortex_2d_r2_ssp43"] = {"accepted": acc, "rejected": rej, "rel_change": rel.tolist(),
                                 "max": float(rel.max())}
    return out


def kxrcf_rmi(n=128, t_final=1.0, last=50):
    pr = P.richtmyer_meshkov(n=n, radius=2)
    # fixed-CFL SSP-RK3 steps so the trajectory can be replayed step by step
    g = replace(pr.grid, integrator="ssprk3", cfl=0.4)
    gk = replace(g, kxrcf=True)
    rset = K.precompute(2)
    t0 = time.perf_counter()
    with K.Solver(gk, rset) as s:
        s.set_state(pr.U0)
        nsteps, t = s.advance_to(t_final)
        Uk = s.get_state()
        fl_final = s.kxrcf_flags().astype(bool)
    with K.Solver(gk, rset) as s:  # replay: flags at the start of each of the last steps
        s.set_state(pr.U0)
        s.advance(nsteps - last)
        frac = []
        for _ in range(last):
            frac.append(float(s.kxrcf_flags().mean()))
            s.advance(1)
    with K.Solver(g, rset) as s:
        s.set_state(pr.U0)
        n_plain, t_plain = s.advance_to(t_final)
        Up = s.get_state()
    dx = g.dx
    d = np.abs(Uk[..., 0] - Up[..., 0])
    l1 = float(d.sum() * dx * dx)
    # smooth region: cells more than 2 cells away from any cell flagged at the end
    near = fl_final.copy()
    for ax in (0, 1):
        for sh in (-2, -1, 1, 2):
            near |= np.roll(fl_final, sh, axis=ax)
    l1_smooth = float(d[~near].sum() * dx * dx)
    area = g.nx * g.ny * dx * dx
    # the catalog's own integrator (SSP(4,3), atol = rtol = 1e-3, CFL 1.0)
    fin = []
    for gg in (pr.grid, replace(pr.grid, kxrcf=True)):
        with K.Solver(gg, rset) as s:
            s.set_state(pr.U0)
            s.advance_to(t_final, 10_000_000)
            fin.append(s.get_state()[..., 0])
    l1_43 = float(np.abs(fin[0] - fin[1]).sum() * dx * dx)
    return {"grid": list(g.shape), "steps": int(nsteps), "t": t, "steps_plain": int(n_plain),
            "rho_l1_diff_ssp43": l1_43,
            "flagged_last50_mean": float(np.mean(frac)), "flagged_last50_max": float(np.max(frac)),
            "rho_l1_diff": l1, "rho_l1_diff_per_area": l1 / area,
            "rho_l1_diff_smooth": l1_smooth, "smooth_fraction": float((~near).mean()),
            "rho_linf_diff": float(d.max()), "wall_s": time.perf_counter() - t0}


def rt_mirror(n=128, t_final=1.0, radius=3):
    pr = P.rayleigh_taylor(n=n, radius=radius)
    g = pr.grid
    # the symmetric variant: the IC averaged with its mirror image (exactly
    # mirror-symmetric in floating point: 0.5 (a + b) is commutative)
    ic = pr.U0
    Mi = ic[:, ::-1, :].copy()
    Mi[..., 1] *= -1.0
    U0 = 0.5 * (ic + Mi)
    def asym(U):
        M = U[:, ::-1, :].copy()
        M[..., 1] *= -1.0
        return float((np.abs(U - M).max(axis=(0, 1)) / np.abs(U).max(axis=(0, 1))).max())

    t0 = time.perf_counter()
    hist = []
    with K.Solver(g) as s:  # the history: one advance_to per checkpoint
        s.set_state(U0)
        for tc in np.linspace(0.1, t_final, 10):
            s.advance_to(float(tc), 10_000_000)
            hist.append((round(float(tc), 3), asym(s.get_state())))
    with K.Solver(g) as s:
        s.set_state(U0)
        steps, t = s.advance_to(t_final, 10_000_000)
        acc, rej = s.step_stats()
        U = s.get_state()
        s.set_state(U0)
        s.advance(1)
        one_step = asym(s.get_state())
    M = U[:, ::-1, :].copy()  # x-mirror about x = 1/8: reverse x, negate x-momentum
    M[..., 1] *= -1.0
    d = np.abs(U - M)
    scale = np.abs(U).max(axis=(0, 1))
    M0 = U0[:, ::-1, :].copy()
    M0[..., 1] *= -1.0
    return {"grid": list(g.shape), "t": t, "accepted": acc, "rejected": rej,
            "ic_mirror_max_abs_raw": float(np.abs(ic - Mi).max()),
            "ic_mirror_max_abs": float(np.abs(U0 - M0).max()),
            "mirror_max_abs": d.max(axis=(0, 1)).tolist(),
            "mirror_max_rel": float((d.max(axis=(0, 1)) / scale).max()),
            "finite": bool(np.isfinite(U).all()), "min_rho": float(U[..., 0].min()),
            "radius": radius, "one_step_mirror_rel": one_step, "history": hist,
            "wall_s": time.perf_counter() - t0}


def _vortex_l1(n, R, integrator):
    kw = dict(integrator="ssp43", atol=1e-6, rtol=1e-6, cfl=1.0) if integrator == "ssp43" \
        else dict(cfl=0.4)
    g = GridConfig(dim=2, radius=R, nx=n, ny=n, dx=20.0 / n, **kw)
    U0 = K.initial_condition(g, VORTEX)
    with K.Solver(g) as s:
        s.set_state(U0)
        s.advance_to(20.0, 10_000_000)
        U = s.get_state()
    return float(np.abs(U[..., 0] - U0[..., 0]).sum() * g.dx ** 2)


def vortex_eoc():
    out = {}
    for integ in ("ssp43", "ssprk3"):
        e = {n: _vortex_l1(n, 3, integ) for n in (32, 64, 128)}
        out[integ] = {"l1": e, "eoc_64": math.log(e[32] / e[64]) / math.log(2),
                      "eoc_128": math.log(e[64] / e[128]) / math.log(2)}
    return out


CHECKS = {"conservation": conservation, "kxrcf_rmi": kxrcf_rmi, "rt_mirror": rt_mirror,
          "rt_mirror_r2": lambda: rt_mirror(radius=2), "vortex_eoc": vortex_eoc}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CHECKS)
    res = {}
    for nm in names:
        t = time.perf_counter()
        res[nm] = CHECKS[nm]()
        res[nm]["_seconds"] = round(time.perf_counter() - t, 1)
        print(nm, json.dumps(res[nm]), file=sys.stderr, flush=True)
    print(json.dumps(res, indent=1))
