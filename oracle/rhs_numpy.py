"""A second, independent code path for compute_rhs (TEST INFRASTRUCTURE ONLY).

SPEC.md S:597 names "a one-step reference computed by an independent
straightforward implementation ... to 1e-12" as the oracle of compute_rhs.
This is that implementation: plain numpy, written directly from the formulas
of the reference, sharing no code and no arithmetic order with the C++
oracle (oracle/kfvm_oracle.cpp) or the GPU engines:

* fill_ghost: np.pad, 'wrap' (periodic) / 'edge' (outflow);
* Phi = dV/dU at the central average (PAPER.md eq. consToLPMat),
  W = Phi U over S0 with the constant part dropped, and
  Phi^-1 = dU/dV (eq. lpToConsMat, written as the exact inverse:
  the energy row carries rho~ u~_d);
* beta_q = sum_alpha Delta^(2|alpha|) (d_alpha . g_q)^2,
  omega~ = gamma_q / (beta^2 + eps), omega = omega~ / sum,
  value = (omega_0/gamma_0) r_0.g_0 + sum_q>=1 (omega_q - omega_0 gamma_q/gamma_0) r_q.g_q
   — every dot product an np.einsum (pairwise / BLAS order), the
  combination per stencil as the SPEC writes it;
* positivity limiter: flattener eta from the undivided velocity
  divergence and c_min over the 3^d neighbourhood, bounds
  rho_max (1 + kappa (1 - eta)), rho_min / p_min (1 - kappa (1 - eta)),
  theta_rho, theta_p by bisection (rel. tol 1e-12, <= 100 iterations);
* Batten / Roe wavespeeds and HLLC / HLL in their textbook form
  (divisions as written, no reciprocals);
* face Gauss-Legendre quadrature and RHS = -(1/Delta) sum_d (F_d+ - F_d-)
  (S:589-592).

Agreement with the C++ oracle to ~1e-12 relative therefore checks the oracle's
pinned arithmetic order against the reference formulas themselves.
"""
from __future__ import annotations

import numpy as np


def _prim(U, gamma):
    d = U.shape[-1] - 2
    rho = U[..., 0]
    vel = U[..., 1:1 + d] / rho[..., None]
    p = (gamma - 1.0) * (U[..., -1] - 0.5 * rho * (vel ** 2).sum(-1))
    return rho, vel, p


def _flux(U, axis, gamma):
    rho, vel, p = _prim(U, gamma)
    un = vel[..., axis]
    F = U * un[..., None]
    F[..., 1 + axis] += p
    F[..., -1] += p * un
    return F


def _hllc(UL, UR, axis, gamma, solver="hllc"):
    rL, vL, pL = _prim(UL, gamma)
    rR, vR, pR = _prim(UR, gamma)
    cL, cR = np.sqrt(gamma * pL / rL), np.sqrt(gamma * pR / rR)
    HL, HR = (UL[..., -1] + pL) / rL, (UR[..., -1] + pR) / rR
    sl, sr = np.sqrt(rL), np.sqrt(rR)
    vroe = (sl[..., None] * vL + sr[..., None] * vR) / (sl + sr)[..., None]
    Hroe = (sl * HL + sr * HR) / (sl + sr)
    croe = np.sqrt(np.maximum((gamma - 1.0) * (Hroe - 0.5 * (vroe ** 2).sum(-1)), 0.0))
    uL, uR, uroe = vL[..., axis], vR[..., axis], vroe[..., axis]
    SL = np.minimum(uL - cL, uroe - croe)
    SR = np.maximum(uR + cR, uroe + croe)
    FL, FR = _flux(UL, axis, gamma), _flux(UR, axis, gamma)
    if solver == "hll":
        Fs = (SR[..., None] * FL - SL[..., None] * FR
              + (SL * SR)[..., None] * (UR - UL)) / (SR - SL)[..., None]
    else:
        sstar = ((pR - pL + rL * uL * (SL - uL) - rR * uR * (SR - uR))
                 / (rL * (SL - uL) - rR * (SR - uR)))

        def star(U, r, v, p, S):
            u = v[..., axis]
            fac = r * (S - u) / (S - sstar)
            Us = np.empty_like(U)
            Us[..., 0] = fac
            for m in range(v.shape[-1]):
                Us[..., 1 + m] = fac * (sstar if m == axis else v[..., m])
            Us[..., -1] = fac * (U[..., -1] / r + (sstar - u) * (sstar + p / (r * (S - u))))
            return Us

        FsL = FL + SL[..., None] * (star(UL, rL, vL, pL, SL) - UL)
        FsR = FR + SR[..., None] * (star(UR, rR, vR, pR, SR) - UR)
        Fs = np.where((sstar >= 0.0)[..., None], FsL, FsR)
    out = np.where((SL >= 0.0)[..., None], FL, Fs)
    return np.where((SR <= 0.0)[..., None], FR, out)


def compute_rhs(U, grid, table, riemann="hllc"):
    """dU/dt of the interior cells (AoS, grid.shape + (nvar,)) with the
    ReconstructionSet `table` (paper_2401_16543_b200.ReconstructionSet)."""
    dim, R, gamma = grid.dim, grid.radius, grid.gamma
    dx = grid.dx if grid.dx else 1.0 / grid.nx
    nv = dim + 2
    eps, kappa, kf = grid.eps, grid.kappa, grid.flattener_kf
    H = R + 1
    mode = "wrap" if grid.bc == "periodic" else "edge"
    Up = np.pad(U, [(H, H)] * dim + [(0, 0)], mode=mode)  # axes (z,) y, x
    n = U.shape[:dim]                      # (nz,) ny, nx
    ext = tuple(m + 2 for m in n)          # interior + one ring: the face states' owners
    lo = H - 1                             # first extended cell in padded coordinates

    def shifted(o):  # padded values at extended cell + o (o in x, y, z order)
        sl = tuple(slice(lo + o[dim - 1 - a], lo + o[dim - 1 - a] + ext[a]) for a in range(dim))
        return Up[sl]

    # reference state, Phi and Phi^-1 per extended cell
    Uc = shifted((0, 0, 0))
    rt, vt, _ = _prim(Uc, gamma)
    Phi = np.zeros(ext + (nv, nv))
    Phi[..., 0, 0] = 1.0
    for d in range(dim):
        Phi[..., 1 + d, 0] = -vt[..., d] / rt
        Phi[..., 1 + d, 1 + d] = 1.0 / rt
        Phi[..., nv - 1, 1 + d] = (1.0 - gamma) * vt[..., d]
    Phi[..., nv - 1, 0] = (gamma - 1.0) * 0.5 * (vt ** 2).sum(-1)
    Phi[..., nv - 1, nv - 1] = gamma - 1.0
    Pinv = np.zeros(ext + (nv, nv))
    Pinv[..., 0, 0] = 1.0
    for d in range(dim):
        Pinv[..., 1 + d, 0] = vt[..., d]
        Pinv[..., 1 + d, 1 + d] = rt
        Pinv[..., nv - 1, 1 + d] = rt * vt[..., d]
    Pinv[..., nv - 1, 0] = 0.5 * (vt ** 2).sum(-1)
    Pinv[..., nv - 1, nv - 1] = 1.0 / (gamma - 1.0)

    offs = table.offsets
    G = np.stack([shifted(tuple(o)) for o in offs], axis=dim)      # ext + (N0, nv)
    W = np.einsum("...vu,...hu->...hv", Phi, G)                    # W = Phi U per stencil cell
    alphas = table.alphas
    scale = np.array([dx ** (2 * int(a.sum())) for a in alphas])
    gam = table.gamma
    NS = table.n_stencils
    beta = []
    pvals = []
    for q in range(NS):
        st = table.st[q]
        g = W[..., st.gather, :]                                       # ext + (N_q, nv)
        dq = np.einsum("ah,...hv->...av", st.deriv, g)
        beta.append(np.einsum("a,...av->...v", scale, dq ** 2))
        pvals.append(np.einsum("sh,...hv->...sv", st.face, g))
    beta = np.stack(beta, axis=dim)                                    # ext + (NS, nv)
    wt = gam[:, None] / (beta ** 2 + eps)
    om = wt / wt.sum(axis=dim, keepdims=True)
    w0 = om[..., 0, :] / gam[0]
    w = w0[..., None, :] * pvals[0]
    for q in range(1, NS):
        w = w + (om[..., q, :] - om[..., 0, :] * gam[q] / gam[0])[..., None, :] * pvals[q]
    S = np.einsum("...uv,...sv->...su", Pinv, w)                      # ext + (NP, nv)

    # positivity limiter
    rho_n, vel_n, p_n = _prim(Up, gamma)
    c_n = np.sqrt(gamma * p_n / rho_n)
    import itertools
    nb = list(itertools.product((-1, 0, 1), repeat=dim))

    def sh(a, o):
        sl = tuple(slice(lo + o[a_], lo + o[a_] + ext[a_]) for a_ in range(dim))
        return a[sl]

    rmax = np.max([sh(rho_n, o) for o in nb], axis=0)
    rmin = np.min([sh(rho_n, o) for o in nb], axis=0)
    pmin = np.min([sh(p_n, o) for o in nb], axis=0)
    cmin = np.min([sh(c_n, o) for o in nb], axis=0)
    delta = np.zeros(ext)
    for d in range(dim):            # physical axis d is array axis dim-1-d
        e = [0] * dim
        e[dim - 1 - d] = 1
        delta += 0.5 * (sh(vel_n[..., d], e) - sh(vel_n[..., d], [-x for x in e]))
    eta = np.clip(-(delta + kf * cmin) / (kf * cmin), 0.0, 1.0)
    # 1 + kappa - kappa eta grouped as 1 + kappa (1 - eta): exactly 1 at eta = 1
    # (the literal left-to-right form rounds to 1 - 1 ulp there and puts the
    # bound inside the average, theta_rho = -inf)
    rho_hi = rmax * (1.0 + kappa * (1.0 - eta))
    rho_lo = rmin * (1.0 - kappa * (1.0 - eta))
    p_lo = pmin * (1.0 - kappa * (1.0 - eta))
    rs = S[..., 0]
    rbar = Uc[..., 0][..., None]
    with np.errstate(divide="ignore", invalid="ignore"):
        th = np.ones_like(rs)
        th = np.where(rs < rho_lo[..., None], (rbar - rho_lo[..., None]) / (rbar - rs), th)
        th = np.where(rs > rho_hi[..., None], (rho_hi[..., None] - rbar) / (rs - rbar), th)
    theta = np.minimum(th.min(axis=-1), 1.0)
    S = Uc[..., None, :] + theta[..., None, None] * (S - Uc[..., None, :])

    def pressure(X):
        return _prim(X, gamma)[2]

    bad = pressure(S) < p_lo[..., None]
    if bad.any():
        thp = np.ones(ext)
        for idx in zip(*np.nonzero(bad)):
            c, s = idx[:-1], idx[-1]
            a, b = 0.0, 1.0
            for _ in range(100):
                m = 0.5 * (a + b)
                X = Uc[c] + m * (S[c + (s,)] - Uc[c])
                if pressure(X) < p_lo[c]:
                    b = m
                else:
                    a = m
                if b - a <= 1e-12 * b:
                    break
            thp[c] = min(thp[c], a)
        S = Uc[..., None, :] + thp[..., None, None] * (S - Uc[..., None, :])

    # Riemann solves at the face points and face quadrature
    rp = table.n_face_points() // (2 * dim)
    fw = table.face_weights
    L = np.zeros(n + (nv,))
    for d in range(dim):
        ax = dim - 1 - d
        lo_sl = [slice(1, 1 + m) for m in n]
        hi_sl = list(lo_sl)
        lo_sl[ax] = slice(0, n[ax] + 1)      # left cells of the faces 0..n
        hi_sl[ax] = slice(1, n[ax] + 2)      # right cells
        Fsum = 0.0
        for m in range(rp):
            sm, sp = (2 * d) * rp + m, (2 * d + 1) * rp + m
            UL = S[tuple(lo_sl)][..., sp, :]
            UR = S[tuple(hi_sl)][..., sm, :]
            Fsum = Fsum + fw[sm] * _hllc(UL, UR, d, gamma, riemann)
        a = [slice(None)] * dim
        b = [slice(None)] * dim
        a[ax] = slice(1, None)
        b[ax] = slice(0, -1)
        L -= (Fsum[tuple(a)] - Fsum[tuple(b)]) / dx
    return L
