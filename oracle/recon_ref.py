"""Independent restatement of the reconstruction-vector precompute in mpmath.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates, in arbitrary
precision and without sharing code with the product's binary128 builder
(paper_2401_16543_b200/csrc/kfvm_table.cpp):

* stencil geometry and substencils — proj/core/src/geometry.cpp:10-34
  (2-D) and PAPER.md §3.1 (3-D);
* graded monomial basis — proj/core/include/kfvm/monomials.hpp:21-47;
* SE-kernel cell averages (erf closed form), point/derivative sample vectors
  and the transposed block solve [[Q^T,P],[P^T,0]](r;w) = (T;S) —
  proj/core/include/kfvm/kernel_recon.hpp:30-62.

The degree of every (sub)stencil follows the reference rank test
(geometry.cpp:39-65, sigma_min > 1e-10 sigma_max) evaluated with numpy SVD.
"""
from __future__ import annotations

import numpy as np

try:
    import mpmath as mp
except ImportError:  # pragma: no cover
    mp = None


def full_stencil(dim: int, R: int):
    kr = R if dim == 3 else 0
    return [(i, j, k) for k in range(-kr, kr + 1) for j in range(-R, R + 1)
            for i in range(-R, R + 1) if i * i + j * j + k * k <= R * R]


def in_substencil(dim: int, R: int, q: int, o) -> bool:
    if q == 1:
        return sum(c * c for c in o) <= (R - 1) ** 2
    axis, sgn = (q - 2) // 2, (-1 if (q - 2) % 2 else 1)
    a = sgn * o[axis]
    return all(abs(o[t]) <= a for t in range(dim) if t != axis)


def graded(dim: int, lo: int, hi: int):
    out = []
    for n in range(lo, hi + 1):
        if dim == 2:
            out += [(n - k, k, 0) for k in range(n + 1)]
        else:
            out += [(a, b, n - a - b) for a in range(n, -1, -1) for b in range(n - a, -1, -1)]
    return out


def mavg_1d(c, k):
    return ((c + 0.5) ** (k + 1) - (c - 0.5) ** (k + 1)) / (k + 1)


def degree(dim: int, R: int, cells) -> int:
    deg = 0
    for p in range(1, 2 * R):
        mono = graded(dim, 0, p)
        if len(mono) > len(cells):
            break
        P = np.array([[np.prod([mavg_1d(float(c[a]), m[a]) for a in range(dim)]) for m in mono]
                      for c in cells])
        sv = np.linalg.svd(P, compute_uv=False)
        if not sv[-1] > 1e-10 * sv[0]:
            break
        deg = p
    return deg


def stencils(dim: int, R: int):
    full = full_stencil(dim, R)
    ns = 2 * dim + 2
    members = [list(range(len(full)))]
    for q in range(1, ns):
        members.append([h for h, o in enumerate(full) if in_substencil(dim, R, q, o)])
    return full, members


def gl_nodes(n: int):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * x, 0.5 * w


def face_points(dim: int, R: int, dps: int = 50):
    """Face GL points, face order W,E,S,N(,B,T), R^(d-1) per face (first
    tangential axis fastest), from the closed-form Gauss-Legendre nodes."""
    mp.mp.dps = dps
    if R == 2:
        nodes = [-1 / (2 * mp.sqrt(3)), 1 / (2 * mp.sqrt(3))]
    elif R == 3:
        nodes = [-mp.sqrt(mp.mpf(3) / 5) / 2, mp.mpf(0), mp.sqrt(mp.mpf(3) / 5) / 2]
    else:
        raise ValueError("R must be 2 or 3")
    pts = []
    for f in range(2 * dim):
        axis, side = f // 2, (mp.mpf(0.5) if f % 2 else mp.mpf(-0.5))
        tan = [a for a in range(dim) if a != axis]
        for m in range(R ** (dim - 1)):
            x = [mp.mpf(0)] * 3
            x[axis] = side
            x[tan[0]] = nodes[m % R]
            if dim == 3:
                x[tan[1]] = nodes[m // R]
            pts.append(x)
    return pts


def recon_vectors(dim: int, R: int, q: int, ell: float = 5.0, dps: int = 50,
                  points=None, alphas=None):
    """Face-point and derivative vectors of (sub)stencil q, in mpmath at `dps`
    digits, returned as float64 arrays (rounded once)."""
    mp.mp.dps = dps
    full, members = stencils(dim, R)
    cells = [full[h] for h in members[q]]
    p = degree(dim, R, cells)
    mono = graded(dim, 0, p)
    N, D = len(cells), len(mono)
    el = mp.mpf(ell)
    s2 = el * mp.sqrt(2)

    def avgk(c):
        return el * mp.sqrt(mp.pi / 2) * (mp.erf((c + mp.mpf(0.5)) / s2) - mp.erf((c - mp.mpf(0.5)) / s2))

    def mavg(c, k):
        c = mp.mpf(c)
        return ((c + mp.mpf(0.5)) ** (k + 1) - (c - mp.mpf(0.5)) ** (k + 1)) / (k + 1)

    M = mp.matrix(N + D, N + D)
    for h in range(N):
        for l in range(N):
            v = mp.mpf(1)
            for a in range(dim):
                v *= avgk(mp.mpf(cells[h][a] - cells[l][a]))
            M[l, h] = v  # Q^T
    for h in range(N):
        for v_ in range(D):
            pv = mp.mpf(1)
            for a in range(dim):
                pv *= mavg(cells[h][a], mono[v_][a])
            M[h, N + v_] = pv
            M[N + v_, h] = pv
    # factor once per stencil and reuse it for every right-hand side: the
    # operations of mp.lu_solve (10 guard bits, LU_decomp, L_solve, U_solve)
    with mp.extraprec(10):
        LU, piv = mp.mp.LU_decomp(M.copy())

    def solve(rhs):
        with mp.extraprec(10):
            return mp.mp.U_solve(LU, mp.mp.L_solve(LU, rhs.copy(), piv))

    pts = points if points is not None else face_points(dim, R, dps)
    als = alphas if alphas is not None else graded(dim, 1, R)
    F = np.zeros((len(pts), N))
    for s, x in enumerate(pts):
        rhs = mp.matrix(N + D, 1)
        for l in range(N):
            v = mp.mpf(1)
            for a in range(dim):
                d = x[a] - cells[l][a]
                v *= mp.exp(-d * d / (2 * el * el))
            rhs[l] = v
        for v_ in range(D):
            m = mp.mpf(1)
            for a in range(dim):
                m *= x[a] ** mono[v_][a]
            rhs[N + v_] = m
        z = solve(rhs)
        F[s] = [float(z[l]) for l in range(N)]
    Dv = np.zeros((len(als), N))
    for ia, al in enumerate(als):
        rhs = mp.matrix(N + D, 1)
        for l in range(N):
            v = mp.mpf(1)
            for a in range(dim):
                u = -mp.mpf(cells[l][a]) / s2
                n = al[a]
                h0, h1 = mp.mpf(1), 2 * u
                hn = h0 if n == 0 else h1
                for k in range(1, n):
                    h0, h1 = h1, 2 * u * h1 - 2 * k * h0
                    hn = h1
                v *= (-1 / s2) ** n * hn * mp.exp(-u * u)
            rhs[l] = v
        for v_ in range(D):
            fac = 0
            if tuple(mono[v_]) == tuple(al):
                fac = 1
                for a in range(3):
                    fac *= mp.factorial(al[a])
            rhs[N + v_] = fac
        z = solve(rhs)
        Dv[ia] = [float(z[l]) for l in range(N)]
    return F, Dv, p
