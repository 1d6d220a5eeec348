"""Exact Riemann solver for the 1-D Euler equations (ideal gas), the test
oracle of the Sod problems (SPEC exact_riemann): the classic
pressure-function Newton iteration for the star state (tol 1e-12, <= 100
iterations) and full wave-fan sampling.  Test infrastructure only."""
import math

import numpy as np


def _f(p, rho, pk, c, g):
    """pressure function and derivative of one side."""
    if p > pk:  # shock
        A = 2.0 / ((g + 1.0) * rho)
        B = (g - 1.0) / (g + 1.0) * pk
        q = math.sqrt(A / (p + B))
        return (p - pk) * q, q * (1.0 - 0.5 * (p - pk) / (B + p))
    # rarefaction
    pr = p / pk
    return (2.0 * c / (g - 1.0)) * (pr ** ((g - 1.0) / (2.0 * g)) - 1.0), \
        (1.0 / (rho * c)) * pr ** (-(g + 1.0) / (2.0 * g))


def star_state(L, R, g=1.4):
    """(p*, u*) for primitive states L, R = (rho, u, p)."""
    rl, ul, pl = L
    rr, ur, pr = R
    cl, cr = math.sqrt(g * pl / rl), math.sqrt(g * pr / rr)
    if 2.0 * (cl + cr) / (g - 1.0) <= ur - ul:
        raise ValueError("vacuum")
    p = max(1e-8, 0.5 * (pl + pr))
    for _ in range(100):
        fl, dl = _f(p, rl, pl, cl, g)
        fr, dr = _f(p, rr, pr, cr, g)
        pn = p - (fl + fr + ur - ul) / (dl + dr)
        pn = max(pn, 1e-12)
        if abs(pn - p) <= 1e-12 * 0.5 * (pn + p):
            p = pn
            break
        p = pn
    else:
        raise RuntimeError("exact Riemann: no convergence")
    fl, _ = _f(p, rl, pl, cl, g)
    fr, _ = _f(p, rr, pr, cr, g)
    return p, 0.5 * (ul + ur) + 0.5 * (fr - fl)


def sample(L, R, xi, g=1.4):
    """primitive state (rho, u, p) at x/t = xi of the Riemann problem L|R."""
    rl, ul, pl = L
    rr, ur, pr = R
    ps, us = star_state(L, R, g)
    gm = (g - 1.0) / (g + 1.0)
    if xi <= us:  # left of the contact
        cl = math.sqrt(g * pl / rl)
        if ps > pl:  # left shock
            sl = ul - cl * math.sqrt((g + 1.0) / (2 * g) * ps / pl + (g - 1.0) / (2 * g))
            if xi <= sl:
                return rl, ul, pl
            return rl * (ps / pl + gm) / (gm * ps / pl + 1.0), us, ps
        cs = cl * (ps / pl) ** ((g - 1.0) / (2 * g))
        if xi <= ul - cl:
            return rl, ul, pl
        if xi >= us - cs:
            return rl * (ps / pl) ** (1.0 / g), us, ps
        u = 2.0 / (g + 1.0) * (cl + 0.5 * (g - 1.0) * ul + xi)
        c = 2.0 / (g + 1.0) * (cl + 0.5 * (g - 1.0) * (ul - xi))
        rho = rl * (c / cl) ** (2.0 / (g - 1.0))
        return rho, u, pl * (c / cl) ** (2.0 * g / (g - 1.0))
    cr = math.sqrt(g * pr / rr)
    if ps > pr:  # right shock
        sr = ur + cr * math.sqrt((g + 1.0) / (2 * g) * ps / pr + (g - 1.0) / (2 * g))
        if xi >= sr:
            return rr, ur, pr
        return rr * (ps / pr + gm) / (gm * ps / pr + 1.0), us, ps
    cs = cr * (ps / pr) ** ((g - 1.0) / (2 * g))
    if xi >= ur + cr:
        return rr, ur, pr
    if xi <= us + cs:
        return rr * (ps / pr) ** (1.0 / g), us, ps
    u = 2.0 / (g + 1.0) * (-cr + 0.5 * (g - 1.0) * ur + xi)
    c = 2.0 / (g + 1.0) * (cr - 0.5 * (g - 1.0) * (ur - xi))
    rho = rr * (c / cr) ** (2.0 / (g - 1.0))
    return rho, u, pr * (c / cr) ** (2.0 * g / (g - 1.0))


def cell_average_density(L, R, x_edges, x0, t, g=1.4, sub=32):
    """cell averages of the exact density on the cells [x_edges[i], x_edges[i+1])."""
    out = np.empty(len(x_edges) - 1)
    for i in range(len(out)):
        xs = x_edges[i] + (np.arange(sub) + 0.5) / sub * (x_edges[i + 1] - x_edges[i])
        out[i] = np.mean([sample(L, R, (x - x0) / t, g)[0] for x in xs])
    return out
