// kfvm_oracle.cpp — CPU oracle of the KFVM-WENO FP64 stage update.
//
// TEST INFRASTRUCTURE ONLY (see kfvm_oracle.h).  Compiled with
// -ffp-contract=off: every fused multiply-add below is an explicit std::fma,
// so the arithmetic sequence is the pinned FP contract of DESIGN.md §4 that
// the CUDA path follows operation for operation.
//
// Reference anchors (S: = SPEC.md, P: = PAPER.md):
//   pressure / sound speed / exact flux ........ S:321-349
//   Phi, Phi^-1 (linearised primitives) ........ S:350-367
//   smoothness indicator, weights, WENO-AO ..... S:256-282
//   flattener, bounds, density/pressure limit .. S:410-446
//   Roe/Batten speeds, HLL, HLLC ............... S:477-503
//   fill_ghost (periodic/outflow) .............. S:553-561 (outflow = index clamp)
//   KXRCF pass 1 / flags / flagged-only WENO ...... S:401-409
//   reconstruct_states (KXRCF off) ............. S:562-570
//   compute_rhs ................................ S:589-597
//   SSP-RK3 (BASELINE.json; replaces S:598) .... Shu-Osher form
//   select_dt .................................. S:607-615 (+|w|+c in 3-D)
#include "kfvm_oracle.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

namespace {

using std::fma;

struct Consts {
  int dim, nv, R, riemann, bc;
  int n[3];
  double gamma, gm1, inv_gm1, dx, cfl, eps, kappa, kf, onepk, onemk;
  double scale[32];  // Delta^(2|alpha|)
  int kx;            // KXRCF on
  double dm;         // Delta^m (host std::pow, the same double the GPU handle uses)
  double atol, rtol, safety, dt_min, dt_max;  // SSP(4,3) controller
  int visc;                                    // Navier-Stokes terms
  double inv_re, inv_prre, gmm, g2;            // 1/Re, 1/(Pr Re), gamma Ma^2, 1/Fr^2
  int side[6], per[3];  // boundary kind per side 2a+s, periodic axes
  double bst[6][5];     // dirichlet / slit inflow states
  double slc[6][2];     // slit centres in the side's tangential axes
  double slr2[6];       // slit radius^2
};

Consts make_consts(const kfvm_config* c, const kfvm_table* t) {
  Consts k{};
  k.dim = c->dim;
  k.nv = c->dim + 2;
  k.R = c->radius;
  k.riemann = c->riemann;
  k.bc = c->bc;
  k.n[0] = c->nx;
  k.n[1] = c->ny;
  k.n[2] = c->dim == 3 ? c->nz : 1;
  k.gamma = c->gamma;
  k.gm1 = c->gamma - 1.0;
  k.inv_gm1 = 1.0 / (c->gamma - 1.0);
  k.dx = c->dx;
  k.cfl = c->cfl;
  k.eps = c->eps;
  k.kappa = c->kappa;
  k.kf = c->flattener_kf;
  k.onepk = 1.0 + c->kappa;
  k.onemk = 1.0 - c->kappa;
  k.kx = c->kxrcf;
  k.dm = std::pow(c->dx, c->kxrcf_m);
  k.atol = c->atol;
  k.rtol = c->rtol;
  k.safety = c->safety;
  k.dt_min = c->dt_min;
  k.dt_max = c->dt_max > 0.0 ? c->dt_max : INFINITY;
  k.visc = c->viscous;
  k.inv_re = 1.0 / c->reynolds;
  k.inv_prre = 1.0 / (c->prandtl * c->reynolds);
  k.gmm = c->gamma * (c->mach * c->mach);
  k.g2 = c->inv_froude2;
  for (int a = 0; a < 3; ++a) {
    for (int sd = 0; sd < 2; ++sd) {
      const int q = 2 * a + sd;
      k.side[q] = a >= c->dim ? KFVM_BC_PERIODIC : (c->bc_per_side ? c->bc_side[q] : c->bc);
      for (int v = 0; v < 5; ++v) k.bst[q][v] = c->bc_state[q][v];
      k.slc[q][0] = c->slit_center[q][0];
      k.slc[q][1] = c->slit_center[q][1];
      k.slr2[q] = c->slit_radius[q] * c->slit_radius[q];
    }
    k.per[a] = k.side[2 * a] == KFVM_BC_PERIODIC ? 1 : 0;
  }
  if (t) {
    for (int a = 0; a < t->n_alpha; ++a) {
      const int ord = t->alpha[3 * a] + t->alpha[3 * a + 1] + t->alpha[3 * a + 2];
      double s = 1.0;
      for (int e = 0; e < 2 * ord; ++e) s *= c->dx;  // Delta^(2|alpha|)
      k.scale[a] = s;
    }
  }
  return k;
}

// ---------------------------------------------------------------- state algebra
inline double pressure(int dim, const double* U, double gm1) {
  double q = U[1] * U[1];
  q = fma(U[2], U[2], q);
  if (dim == 3) q = fma(U[3], U[3], q);
  return gm1 * (U[dim + 1] - 0.5 * (q / U[0]));
}

// p(U) < pmin for a state with rho > 0, written without the division:
// gm1 (E rho - |m|^2 / 2) < pmin rho  (used by the limiter)
inline bool p_below(int dim, const double* U, double gm1, double pmin) {
  double q = U[1] * U[1];
  q = fma(U[2], U[2], q);
  if (dim == 3) q = fma(U[3], U[3], q);
  return gm1 * fma(U[dim + 1], U[0], -0.5 * q) < pmin * U[0];
}

inline double sound(double gamma, double p, double rho) {
  return std::sqrt((gamma * p) / rho);
}

struct Transform {  // Phi / Phi^-1 at the central average
  double rt, inv_r, ut[3], mt[3], ke;
};

inline Transform make_transform(int dim, const double* Ur) {
  Transform T;
  T.rt = Ur[0];
  T.inv_r = 1.0 / Ur[0];
  T.ut[2] = 0.0;
  T.mt[2] = 0.0;
  for (int d = 0; d < dim; ++d) {
    T.ut[d] = Ur[1 + d] / Ur[0];
    T.mt[d] = Ur[1 + d];
  }
  double ke = T.ut[0] * T.ut[0];
  ke = fma(T.ut[1], T.ut[1], ke);
  if (dim == 3) ke = fma(T.ut[2], T.ut[2], ke);
  T.ke = 0.5 * ke;
  return T;
}

// W = Phi U, one component v (constant part dropped)
inline double to_recon(int dim, const Transform& T, double gm1, const double* U, int v) {
  if (v == 0) return U[0];
  if (v <= dim) return fma(-T.ut[v - 1], U[0], U[v]) * T.inv_r;
  double t = fma(T.ke, U[0], U[dim + 1]);
  t = fma(-T.ut[0], U[1], t);
  t = fma(-T.ut[1], U[2], t);
  if (dim == 3) t = fma(-T.ut[2], U[3], t);
  return gm1 * t;
}

// U = Phi^-1 W.  Phi^-1 = dU/dV: its energy row is
// (|u|^2/2, rho u_1, rho u_2, rho u_3, 1/(gamma-1)); PAPER.md's appendix
// prints u_d in place of rho u_d, which is the inverse only for rho = 1 — the
// SPEC's invariant Phi Phi^-1 = I requires the exact inverse, written
// with the central momentum m_d = rho u_d.
inline void from_recon(int dim, const Transform& T, double inv_gm1, const double* W, double* U) {
  U[0] = W[0];
  for (int d = 0; d < dim; ++d) U[1 + d] = fma(T.ut[d], W[0], T.rt * W[1 + d]);
  double t = W[dim + 1] * inv_gm1;
  t = fma(T.mt[0], W[1], t);
  t = fma(T.mt[1], W[2], t);
  if (dim == 3) t = fma(T.mt[2], W[3], t);
  U[dim + 1] = fma(T.ke, W[0], t);
}

// ------------------------------------------------------------------- WENO-AO
// First derivative index evaluated as four slot chains (3-D only; 2-D keeps
// every derivative a single stencil-order chain).
inline int kfo_alpha_tail(int dim, int n_alpha) { return dim == 3 ? 8 * (n_alpha / 8) : n_alpha; }

// beta_q, omega_q and the WENO-AO values at every face point for one scalar
// field g on S0.  Dot products accumulate in stencil order.
void weno_field(const kfvm_table* t, const Consts& k, const double* g, double* beta_out,
                double* omega_out, double* vals) {
  const int NS = t->n_stencils;
  double wt[KFVM_MAX_STENCILS], c[KFVM_MAX_STENCILS];
  for (int q = 0; q < NS; ++q) {
    const int N = t->size[q];
    const int* gat = t->gather + t->cell_offset[q];
    const double* D = t->deriv + (size_t)t->cell_offset[q] * t->n_alpha;
    // beta_q = sum_alpha Delta^(2|alpha|) d_alpha^2 summed in four
    // interleaved partial chains — alpha = 8n + 2j + e goes to partial j, in
    // (n, e) order — combined as (p0 + p1) + (p2 + p3).  This is the order in
    // which the tensor-core engine's quads hold the derivative columns
    // (DESIGN.md §4), so no cross-lane sequential chain is needed.
    // d_alpha = d_alpha . g as the stencil-order fma chain, except in 3-D for
    // the tail alphas >= 8 floor(n_alpha / 8) (the columns that would fill
    // only part of an 8-wide tensor-core tile): those are four slot chains —
    // entry h goes to slot (h + pad_q) mod 4, pad_q = (-N_q) mod 4, each slot
    // chain in stencil order — combined as (s0 + s1) + (s2 + s3).  That is the
    // order in which the lanes of a quad hold the 4-entry DMMA chunks (front
    // padded), so the tensor-core engine computes them with per-lane DFMA
    // instead of a mostly-empty DMMA tile.
    const int a_tail = kfo_alpha_tail(t->dim, t->n_alpha);
    const int pad = (4 - N % 4) % 4;
    double d[32];
    for (int a = 0; a < t->n_alpha; ++a) {
      if (a < a_tail) {
        d[a] = 0.0;
        for (int h = 0; h < N; ++h) d[a] = fma(D[a * N + h], g[gat[h]], d[a]);
      } else {
        double sl[4] = {0.0, 0.0, 0.0, 0.0};
        for (int h = 0; h < N; ++h) {
          const int j = (h + pad) % 4;
          sl[j] = fma(D[a * N + h], g[gat[h]], sl[j]);
        }
        d[a] = (sl[0] + sl[1]) + (sl[2] + sl[3]);
      }
    }
    double part[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = 0; j < 4; ++j)
      for (int n = 0; 8 * n < t->n_alpha; ++n)
        for (int e = 0; e < 2; ++e) {
          const int a = 8 * n + 2 * j + e;
          if (a < t->n_alpha) part[j] = fma(k.scale[a], d[a] * d[a], part[j]);
        }
    const double beta = (part[0] + part[1]) + (part[2] + part[3]);
    if (beta_out) beta_out[q] = beta;
    // P eq. nlinWts: gamma_q / (beta_q^2 + eps), evaluated as gamma_q * (1 / d)
    wt[q] = t->gamma_lin[q] * (1.0 / fma(beta, beta, k.eps));
  }
  double sum = wt[0];
  for (int q = 1; q < NS; ++q) sum = sum + wt[q];
  const double inv_sum = 1.0 / sum;
  double om[KFVM_MAX_STENCILS] = {0};
  for (int q = 0; q < NS; ++q) om[q] = wt[q] * inv_sum;
  if (omega_out)
    for (int q = 0; q < NS; ++q) omega_out[q] = om[q];
  c[0] = om[0] * (1.0 / t->gamma_lin[0]);
  for (int q = 1; q < NS; ++q) c[q] = fma(-c[0], t->gamma_lin[q], om[q]);
  // WENO-AO value at point s: sum_q c_q (r_qs . g_q), evaluated
  // as ONE stencil-order fma chain over every stencil entry with the entry
  // scaled by its stencil's coefficient first: v = fma(r_qsh, c_q * g_h, v),
  // q = 0..NS-1, h in stencil order (this is the order in which
  // the FP64 tensor-core engine accumulates, with no per-stencil partials).
  for (int s = 0; s < t->n_points; ++s) {
    double v = 0.0;
    for (int q = 0; q < NS; ++q) {
      const int N = t->size[q];
      const int* gat = t->gather + t->cell_offset[q];
      const double* r = t->face + (size_t)t->cell_offset[q] * t->n_points + (size_t)s * N;
      for (int h = 0; h < N; ++h) v = fma(r[h], c[q] * g[gat[h]], v);
    }
    vals[s] = v;
  }
}

// ------------------------------------------------------- positivity limiter
// nbr: 3^dim averages (i fastest), centre at index (3^dim)/2.  Returns 0 ok,
// 2 if the cell average itself is inadmissible.
int limit_cell(const Consts& k, int npts, double* st, const double* nbr, double* info) {
  const int dim = k.dim, nv = k.nv;
  const int nn = dim == 3 ? 27 : 9;
  const double* Uc = nbr + (size_t)(nn / 2) * nv;
  double rbmax = Uc[0], rbmin = Uc[0];
  double pbmin = pressure(dim, Uc, k.gm1);
  double cmin = sound(k.gamma, pbmin, Uc[0]);
  for (int m = 0; m < nn; ++m) {
    const double* U = nbr + (size_t)m * nv;
    const double p = pressure(dim, U, k.gm1);
    rbmax = std::fmax(rbmax, U[0]);
    rbmin = std::fmin(rbmin, U[0]);
    pbmin = std::fmin(pbmin, p);
    cmin = std::fmin(cmin, sound(k.gamma, p, U[0]));
  }
  // undivided velocity divergence
  auto vel = [&](int m, int d) { return nbr[(size_t)m * nv + 1 + d] / nbr[(size_t)m * nv]; };
  const int c0 = nn / 2;
  double delta = 0.5 * (vel(c0 + 1, 0) - vel(c0 - 1, 0));
  delta = fma(0.5, vel(c0 + 3, 1) - vel(c0 - 3, 1), delta);
  if (dim == 3) delta = fma(0.5, vel(c0 + 9, 2) - vel(c0 - 9, 2), delta);
  const double kc = k.kf * cmin;
  double eta = -(delta + kc) / kc;
  eta = std::fmin(1.0, std::fmax(0.0, eta));
  // bounds
  // (1 + kappa - kappa eta) written as 1 + kappa (1 - eta) so the factor is
  // exactly 1 at eta = 1 and the bounds always bracket the cell average
  const double fup = fma(k.kappa, 1.0 - eta, 1.0);
  const double flo = fma(-k.kappa, 1.0 - eta, 1.0);
  const double rmax = rbmax * fup;
  const double rmin = rbmin * flo;
  const double pmin = pbmin * flo;
  const double rt = Uc[0];
  const double pt = pressure(dim, Uc, k.gm1);
  if (!(rt > 0.0) || !(pt > 0.0) || !(rmin > 0.0) || !(pmin > 0.0)) return 2;
  // density (P eq. ppThetaRho)
  double th = 1.0;
  for (int s = 0; s < npts; ++s) {
    const double r = st[s * nv];
    if (r < rmin)
      th = std::fmin(th, (rt - rmin) / (rt - r));
    else if (r > rmax)
      th = std::fmin(th, (rmax - rt) / (r - rt));
  }
  if (th < 1.0)
    for (int s = 0; s < npts; ++s)
      for (int v = 0; v < nv; ++v) st[s * nv + v] = fma(th, st[s * nv + v] - Uc[v], Uc[v]);
  // pressure by bisection (P eqs. thetapRoot/thetaP)
  double thp = 1.0;
  for (int s = 0; s < npts; ++s) {
    if (p_below(dim, st + s * nv, k.gm1, pmin)) {
      double lo = 0.0, hi = 1.0, x[5];
      for (int it = 0; it < 100 && (hi - lo) > 1e-12 * hi; ++it) {
        const double mid = 0.5 * (lo + hi);
        for (int v = 0; v < nv; ++v) x[v] = fma(mid, st[s * nv + v] - Uc[v], Uc[v]);
        if (!p_below(dim, x, k.gm1, pmin))
          lo = mid;
        else
          hi = mid;
      }
      thp = std::fmin(thp, lo);
    }
  }
  if (thp < 1.0)
    for (int s = 0; s < npts; ++s)
      for (int v = 0; v < nv; ++v) st[s * nv + v] = fma(thp, st[s * nv + v] - Uc[v], Uc[v]);
  if (info) {
    info[0] = eta;
    info[1] = rmin;
    info[2] = rmax;
    info[3] = pmin;
    info[4] = th;
    info[5] = thp;
  }
  return 0;
}

// ----------------------------------------------------------------- Riemann
inline void exact_flux(int dim, int d, const double* U, double un, double p, double* F) {
  const int nv = dim + 2;
  F[0] = U[1 + d];
  for (int m = 0; m < dim; ++m) F[1 + m] = U[1 + m] * un;
  F[1 + d] = F[1 + d] + p;
  F[nv - 1] = (U[nv - 1] + p) * un;
}

// Batten/Roe speeds + HLL/HLLC.  Pinned form: one reciprocal
// per side (1/rho) and per Roe denominator, so a solve costs 6 IEEE
// divisions (HLLC; 4 for HLL) instead of ~16.
void riemann(const Consts& k, int d, const double* UL, const double* UR, double* F,
             double* speeds = nullptr) {
  const int dim = k.dim, nv = k.nv;
  const double irL = 1.0 / UL[0], irR = 1.0 / UR[0];
  double uL[3] = {0, 0, 0}, uR[3] = {0, 0, 0};
  for (int m = 0; m < dim; ++m) {
    uL[m] = UL[1 + m] * irL;
    uR[m] = UR[1 + m] * irR;
  }
  double qL = UL[1] * UL[1], qR = UR[1] * UR[1];
  qL = fma(UL[2], UL[2], qL);
  qR = fma(UR[2], UR[2], qR);
  if (dim == 3) {
    qL = fma(UL[3], UL[3], qL);
    qR = fma(UR[3], UR[3], qR);
  }
  const double pL = k.gm1 * (UL[nv - 1] - 0.5 * (qL * irL));
  const double pR = k.gm1 * (UR[nv - 1] - 0.5 * (qR * irR));
  const double cL = std::sqrt((k.gamma * pL) * irL), cR = std::sqrt((k.gamma * pR) * irR);
  const double HL = (UL[nv - 1] + pL) * irL, HR = (UR[nv - 1] + pR) * irR;
  const double sl = std::sqrt(UL[0]), sr = std::sqrt(UR[0]);
  const double iden = 1.0 / (sl + sr);
  double roe[3] = {0, 0, 0};
  for (int m = 0; m < dim; ++m) roe[m] = fma(sl, uL[m], sr * uR[m]) * iden;
  const double Hroe = fma(sl, HL, sr * HR) * iden;
  double q2 = roe[0] * roe[0];
  q2 = fma(roe[1], roe[1], q2);
  if (dim == 3) q2 = fma(roe[2], roe[2], q2);
  const double croe = std::sqrt(std::fmax(k.gm1 * (Hroe - 0.5 * q2), 0.0));
  const double SL = std::fmin(uL[d] - cL, roe[d] - croe);
  const double SR = std::fmax(uR[d] + cR, roe[d] + croe);
  double FL[5], FR[5];
  exact_flux(dim, d, UL, uL[d], pL, FL);
  exact_flux(dim, d, UR, uR[d], pR, FR);
  const double aL = UL[0] * (SL - uL[d]);
  const double aR = UR[0] * (SR - uR[d]);
  double num = fma(aL, uL[d], pR - pL);
  num = fma(-aR, uR[d], num);
  const double sstar = num / (aL - aR);
  if (speeds) {
    speeds[0] = SL;
    speeds[1] = SR;
    speeds[2] = sstar;
  }
  if (SL >= 0.0) {
    for (int v = 0; v < nv; ++v) F[v] = FL[v];
    return;
  }
  if (SR <= 0.0) {
    for (int v = 0; v < nv; ++v) F[v] = FR[v];
    return;
  }
  if (k.riemann == KFVM_RIEMANN_HLL) {
    const double ssr = SL * SR;
    const double iw = 1.0 / (SR - SL);
    for (int v = 0; v < nv; ++v) {
      double t = SR * FL[v];
      t = fma(-SL, FR[v], t);
      t = fma(ssr, UR[v] - UL[v], t);
      F[v] = t * iw;
    }
    return;
  }
  // HLLC
  const bool left = sstar >= 0.0;
  const double* UK = left ? UL : UR;
  const double* FK = left ? FL : FR;
  const double* uK = left ? uL : uR;
  const double SK = left ? SL : SR;
  const double aK = left ? aL : aR;
  const double pK = left ? pL : pR;
  const double irK = left ? irL : irR;
  const double fac = aK / (SK - sstar);
  double Us[5];
  Us[0] = fac;
  for (int m = 0; m < dim; ++m) Us[1 + m] = fac * (m == d ? sstar : uK[m]);
  const double e = fma(sstar - uK[d], sstar + pK / aK, UK[nv - 1] * irK);
  Us[nv - 1] = fac * e;
  for (int v = 0; v < nv; ++v) F[v] = fma(SK, Us[v] - UK[v], FK[v]);
}

// ------------------------------------------------------------- grid / slab
// periodic wrap, or the nearest interior cell (the flag / index rule of the
// one-cell ring around a box)
inline int wrap(int i, int n, int periodic) {
  if (periodic) return ((i % n) + n) % n;
  return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

// fill_ghost: index map of one axis for a side's kind — periodic
// wrap, reflecting mirror image, otherwise the nearest interior cell.
inline int ghost_src(int i, int n, int kind) {
  if (i >= 0 && i < n) return i;
  if (kind == KFVM_BC_PERIODIC) return ((i % n) + n) % n;
  if (kind == KFVM_BC_REFLECTING) return i < 0 ? -1 - i : 2 * n - 1 - i;
  return i < 0 ? 0 : n - 1;
}

// fill_ghost value rule of one crossed side q = 2a+s for the ghost cell at
// global coords c: reflecting flips the wall-normal momentum,
// dirichlet writes the fixed state, the slit writes the inflow state where
// r^2 < radius^2 strictly over the tangential axes' cell-centre offsets
// (S:561), and outflow / periodic keep the source value.
void ghost_rule(const Consts& k, int a, int sd, const int* c, double* u) {
  const int q = 2 * a + sd;
  switch (k.side[q]) {
    case KFVM_BC_REFLECTING:
      u[1 + a] = -u[1 + a];
      break;
    case KFVM_BC_DIRICHLET:
      for (int v = 0; v < k.nv; ++v) u[v] = k.bst[q][v];
      break;
    case KFVM_BC_SLIT: {
      double r2 = 0.0;
      int m = 0;
      for (int b = 0; b < k.dim; ++b) {
        if (b == a) continue;
        const double off = ((double)c[b] + 0.5) * k.dx - k.slc[q][m];
        r2 = m == 0 ? off * off : r2 + off * off;
        ++m;
      }
      if (r2 < k.slr2[q])
        for (int v = 0; v < k.nv; ++v) u[v] = k.bst[q][v];
      break;
    }
    default:
      break;
  }
}

// A slab of planes [p0, p0+np) along the slab axis sa = dim-1, stored with H
// halo planes on each side and H ghost cells on each side of the other axes:
// every cell of the padded box holds its value (interior copy or fill_ghost
// rule), so at() is a plain offset.
struct Slab {
  const Consts* k;
  int sa, p0, np, H;
  int ext[3];  // padded local extents
  std::vector<double> U;

  void init(const Consts& kk, int p0_, int np_) {
    k = &kk;
    sa = kk.dim - 1;
    p0 = p0_;
    np = np_;
    H = kk.R + 1;
    for (int a = 0; a < 3; ++a) ext[a] = a < kk.dim ? kk.n[a] + 2 * H : 1;
    ext[sa] = np + 2 * H;
    U.assign((size_t)ext[0] * ext[1] * ext[2] * kk.nv, 0.0);
  }
  // global coords (i,j,k) within the padded box
  inline const double* at(int i, int j, int kk) const {
    int c[3] = {i, j, kk};
    for (int a = 0; a < k->dim; ++a) c[a] += a == sa ? H - p0 : H;
    return U.data() + (((size_t)c[2] * ext[1] + c[1]) * ext[0] + c[0]) * k->nv;
  }
  // every padded cell from src(sc), sc the composed ghost index map of its
  // global coords, then the value rules of the crossed sides in axis order
  // x, y, z.  A periodic slab axis is not remapped here (src resolves it:
  // the global array wraps, a rank's halo planes hold the neighbour's data).
  template <class Src>
  void fill(Src&& src) {
    const int nv = k->nv;
    for (int l2 = 0; l2 < ext[2]; ++l2)
      for (int l1 = 0; l1 < ext[1]; ++l1)
        for (int l0 = 0; l0 < ext[0]; ++l0) {
          const int l[3] = {l0, l1, l2};
          int c[3] = {0, 0, 0}, sc[3] = {0, 0, 0};
          for (int a = 0; a < k->dim; ++a) {
            c[a] = l[a] - H + (a == sa ? p0 : 0);
            const int q = 2 * a + (c[a] >= k->n[a]);
            sc[a] = (a == sa && k->per[a]) ? c[a] : ghost_src(c[a], k->n[a], k->side[q]);
          }
          double u[5];
          std::memcpy(u, src(sc), nv * sizeof(double));
          for (int a = 0; a < k->dim; ++a)
            if (c[a] < 0 || c[a] >= k->n[a]) ghost_rule(*k, a, c[a] >= k->n[a], c, u);
          std::memcpy(U.data() + (((size_t)l2 * ext[1] + l1) * ext[0] + l0) * nv, u,
                      nv * sizeof(double));
        }
  }
  // from a global AoS array (the in-memory halo exchange)
  void load(const double* G) {
    const Consts& kk = *k;
    fill([&](const int* sc) {
      const int g = wrap(sc[sa], kk.n[sa], 1);
      int c[3] = {sc[0], sc[1], sc[2]};
      c[sa] = g;
      return G + (((size_t)c[2] * kk.n[1] + c[1]) * kk.n[0] + c[0]) * kk.nv;
    });
  }
  // from the slab's local AoS array with its H halo planes (interior extents
  // in the other axes), as exchanged by the caller; planes beyond a
  // non-periodic global end are rebuilt from the slab's own planes.
  void load_local(const double* L) {
    const Consts& kk = *k;
    const size_t plane = (size_t)kk.nv * kk.n[0] * (sa == 2 ? kk.n[1] : 1);
    fill([&](const int* sc) {
      const int lp = sc[sa] - (p0 - H);
      const size_t in = sa == 2 ? (size_t)sc[1] * kk.n[0] + sc[0] : (size_t)sc[0];
      return L + (size_t)lp * plane + in * kk.nv;
    });
  }
};

// Contiguous slab split: the first n % P slabs get one extra plane.
void slab_range(int n, int P, int r, int* p0, int* np) {
  const int base = n / P, rem = n % P;
  *np = base + (r < rem ? 1 : 0);
  *p0 = r * base + (r < rem ? r : rem);
}

template <class F>
void parallel_for(int n, int nthreads, F&& f) {
  if (nthreads <= 1 || n < 2) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<int> next(0);
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back([&]() {
      for (int i; (i = next.fetch_add(1)) < n;) f(i);
    });
  for (auto& x : th) x.join();
}

size_t ncells(const Consts& k);

// ------------------------------------------------------------------ KXRCF
// Troubled-cell indicator: entropy q = p / rho^gamma.
// rho^gamma is evaluated with a pinned exp/log built from IEEE +,*,fma, rint
// and exponent bit manipulation only (no libm), so the CPU and the GPU get
// the same bits; the result only feeds the threshold test.
inline double kf_log(double x) {  // x > 0, finite, normal
  uint64_t b;
  std::memcpy(&b, &x, 8);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  b = (b & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL;
  double m;
  std::memcpy(&m, &b, 8);  // [1, 2)
  if (m > 0x1.6a09e667f3bcdp+0) {  // sqrt(2)
    m = m * 0.5;
    e += 1;
  }
  const double f = m - 1.0;
  const double sv = f / (2.0 + f);
  const double z = sv * sv;
  // log m = 2 atanh(s) = 2 s sum_k z^k / (2k+1), k = 0..9
  double P = 0x1.af286bca1af28p-5;  // 1/19
  P = fma(P, z, 0x1.e1e1e1e1e1e1ep-5);
  P = fma(P, z, 0x1.1111111111111p-4);
  P = fma(P, z, 0x1.3b13b13b13b14p-4);
  P = fma(P, z, 0x1.745d1745d1746p-4);
  P = fma(P, z, 0x1.c71c71c71c71cp-4);
  P = fma(P, z, 0x1.2492492492492p-3);
  P = fma(P, z, 0x1.999999999999ap-3);
  P = fma(P, z, 0x1.5555555555555p-2);
  P = fma(P, z, 1.0);
  const double lm = (2.0 * sv) * P;
  const double de = (double)e;
  return fma(de, 0x1.62e4200000000p-1, fma(de, 0x1.fdf473de6af28p-22, lm));
}
inline double kf_exp(double y) {  // |y| < 700
  const double n = std::rint(y * 0x1.71547652b82fep+0);
  double r = fma(-n, 0x1.62e4200000000p-1, y);
  r = fma(-n, 0x1.fdf473de6af28p-22, r);
  double p = 0x1.6124613a86d09p-33;  // 1/13!
  p = fma(p, r, 0x1.1eed8eff8d898p-29);
  p = fma(p, r, 0x1.ae64567f544e4p-26);
  p = fma(p, r, 0x1.27e4fb7789f5cp-22);
  p = fma(p, r, 0x1.71de3a556c734p-19);
  p = fma(p, r, 0x1.a01a01a01a01ap-16);
  p = fma(p, r, 0x1.a01a01a01a01ap-13);
  p = fma(p, r, 0x1.6c16c16c16c17p-10);
  p = fma(p, r, 0x1.1111111111111p-7);
  p = fma(p, r, 0x1.5555555555555p-5);
  p = fma(p, r, 0x1.5555555555555p-3);
  p = fma(p, r, 0x1.0000000000000p-1);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  return std::ldexp(p, (int)n);
}
inline double kf_pow(double x, double y) { return kf_exp(y * kf_log(x)); }

// entropy p / rho^gamma of a pointwise state; NaN for rho <= 0 (flags the cell)
inline double entropy(const Consts& k, const double* U) {
  if (!(U[0] > 0.0)) return NAN;
  return pressure(k.dim, U, k.gm1) / kf_pow(U[0], k.gamma);
}

// Unlimited full-stencil states (pass 1): conservative variables,
// r_0 vectors, stencil-order fma chains.
void pass1_cell(const kfvm_table* t, const Consts& k, const Slab& S, int i, int j, int kk,
                double* st) {
  const int nv = k.nv, N0 = t->n_full, np = t->n_points;
  for (int s = 0; s < np; ++s) {
    const double* r = t->face + (size_t)s * N0;  // stencil 0 is first in the table
    for (int v = 0; v < nv; ++v) {
      double acc = 0.0;
      for (int h = 0; h < N0; ++h)
        acc = fma(r[h], S.at(i + t->offsets[3 * h], j + t->offsets[3 * h + 1],
                             kk + t->offsets[3 * h + 2])[v],
                  acc);
      st[s * nv + v] = acc;
    }
  }
}

// Flags of every global cell (pass 2): flagged iff
// max_s |q_s(+) - q_s(-)| / <Q> >= Delta^m, <Q> = p(Ubar) / rhobar^gamma, over
// the points of every face with a neighbour (physical-boundary faces of
// outflow domains are exempt); a NaN jump or <Q> flags the cell.
std::vector<uint8_t> global_flags(const kfvm_table* t, const Consts& k, const double* U,
                                  int nthreads) {
  const int dim = k.dim, nv = k.nv, np = t->n_points, rp = np / (2 * dim);
  Slab S;
  S.init(k, 0, k.n[dim - 1]);
  S.load(U);
  const size_t nc = ncells(k), cs = (size_t)np * nv;
  std::vector<double> st(nc * cs);
  const int nrows = k.n[1] * k.n[2];
  parallel_for(nrows, nthreads, [&](int row) {
    const int j = row % k.n[1], kk = row / k.n[1];
    for (int i = 0; i < k.n[0]; ++i)
      pass1_cell(t, k, S, i, j, kk, st.data() + (((size_t)kk * k.n[1] + j) * k.n[0] + i) * cs);
  });
  std::vector<uint8_t> fl(nc, 0);
  parallel_for(nrows, nthreads, [&](int row) {
    const int j = row % k.n[1], kk = row / k.n[1];
    for (int i = 0; i < k.n[0]; ++i) {
      const int c[3] = {i, j, kk};
      const size_t id = ((size_t)kk * k.n[1] + j) * k.n[0] + i;
      const double* Uc = U + id * nv;
      const double Q = Uc[0] > 0.0 ? pressure(dim, Uc, k.gm1) / kf_pow(Uc[0], k.gamma) : NAN;
      double jmax = 0.0;
      bool nan = !(Q == Q);
      for (int d = 0; d < dim; ++d)
        for (int side = 0; side < 2; ++side) {
          int nb[3] = {c[0], c[1], c[2]};
          nb[d] += side ? 1 : -1;
          if (nb[d] < 0 || nb[d] >= k.n[d]) {
            if (!k.per[d]) continue;  // physical boundary face: exempt
            nb[d] = (nb[d] + k.n[d]) % k.n[d];
          }
          const size_t nid = ((size_t)nb[2] * k.n[1] + nb[1]) * k.n[0] + nb[0];
          for (int m = 0; m < rp; ++m) {
            const int so = (2 * d + side) * rp + m, sn = (2 * d + 1 - side) * rp + m;
            const double jq = std::fabs(entropy(k, st.data() + nid * cs + sn * nv) -
                                        entropy(k, st.data() + id * cs + so * nv));
            if (!(jq == jq)) nan = true;
            jmax = std::fmax(jmax, jq);
          }
        }
      fl[id] = (nan || jmax / Q >= k.dm) ? 1 : 0;
    }
  });
  return fl;
}

// flag of any cell of an extended box: global cells are their own, ghost
// cells take the flag of the periodic image, else of the nearest interior
// cell (with one ghost layer that is also the reflecting mirror image)
inline int flag_of(const Consts& k, const uint8_t* fl, int i, int j, int kk) {
  const int c[3] = {wrap(i, k.n[0], k.per[0]), wrap(j, k.n[1], k.per[1]),
                    k.dim == 3 ? wrap(kk, k.n[2], k.per[2]) : 0};
  return fl[((size_t)c[2] * k.n[1] + c[1]) * k.n[0] + c[0]];
}

// Face states of one cell (global coords), after WENO-AO + positivity.
int cell_states(const kfvm_table* t, const Consts& k, const Slab& S, int i, int j, int kk,
                double* st /* [npts][nv] */) {
  const int dim = k.dim, nv = k.nv, N0 = t->n_full, np = t->n_points;
  const double* Uc = S.at(i, j, kk);
  const Transform T = make_transform(dim, Uc);
  std::vector<const double*> cells(N0);
  for (int h = 0; h < N0; ++h)
    cells[h] = S.at(i + t->offsets[3 * h], j + t->offsets[3 * h + 1], kk + t->offsets[3 * h + 2]);
  double g[128], vals[64];
  double W[64 * 5];
  for (int v = 0; v < nv; ++v) {  // W = Phi U cell by cell, then WENO-AO per variable
    for (int h = 0; h < N0; ++h) g[h] = to_recon(dim, T, k.gm1, cells[h], v);
    weno_field(t, k, g, nullptr, nullptr, vals);
    for (int s = 0; s < np; ++s) W[s * nv + v] = vals[s];
  }
  for (int s = 0; s < np; ++s) from_recon(dim, T, k.inv_gm1, W + s * nv, st + s * nv);
  double nbr[27 * 5];
  const int kr = dim == 3 ? 1 : 0;
  int m = 0;
  for (int c = -kr; c <= kr; ++c)
    for (int b = -1; b <= 1; ++b)
      for (int a = -1; a <= 1; ++a, ++m) std::memcpy(nbr + m * nv, S.at(i + a, j + b, kk + c), nv * sizeof(double));
  return limit_cell(k, np, st, nbr, nullptr);
}

// KXRCF face states of one cell: WENO-AO (cell_states) when flagged, else the
// pass-1 states; positivity limiting in both cases.
int cell_states_kx(const kfvm_table* t, const Consts& k, const Slab& S, const uint8_t* fl,
                   int i, int j, int kk, double* st) {
  if (flag_of(k, fl, i, j, kk)) return cell_states(t, k, S, i, j, kk, st);
  const int dim = k.dim, nv = k.nv;
  pass1_cell(t, k, S, i, j, kk, st);
  double nbr[27 * 5];
  const int kr = dim == 3 ? 1 : 0;
  int m = 0;
  for (int c = -kr; c <= kr; ++c)
    for (int b = -1; b <= 1; ++b)
      for (int a = -1; a <= 1; ++a, ++m) std::memcpy(nbr + m * nv, S.at(i + a, j + b, kk + c), nv * sizeof(double));
  return limit_cell(k, t->n_points, st, nbr, nullptr);
}

// Viscous face flux F^(v) (P eqs nsVisc/shearTensor/thermalFlux,
// P:615-633) of the face between cell (i,j,kk) - e_d (L) and (i,j,kk) (R):
// second-order differences of the cell-average primitives (u_1..u_dim,
// T = gamma Ma^2 p / rho), normal = (R - L) / Delta, tangential = the
// four-cell average ((L+ - L-) + (R+ - R-)) / (4 Delta); sigma and q at the
// face centre; face velocity (L + R) / 2; midpoint rule.  Pinned operation
// order, identical on the device (k_visc).
inline void prim_vt(const Consts& k, const double* U, double* out) {  // u_1..u_dim, T
  const double p = pressure(k.dim, U, k.gm1);
  const double inv_r = 1.0 / U[0];
  for (int a = 0; a < k.dim; ++a) out[a] = U[1 + a] / U[0];
  out[k.dim] = k.gmm * (p * inv_r);
}

void viscous_flux(const Consts& k, const Slab& S, int d, int i, int j, int kk, double* Fv) {
  const int dim = k.dim, nv = k.nv;
  int cR[3] = {i, j, kk}, cL[3] = {i, j, kk};
  cL[d] -= 1;
  double L[4], R[4];
  prim_vt(k, S.at(cL[0], cL[1], cL[2]), L);
  prim_vt(k, S.at(cR[0], cR[1], cR[2]), R);
  double g[4][3];  // g[f][a] = d phi_f / d x_a, phi = (u_1..u_dim, T)
  for (int f = 0; f <= dim; ++f) g[f][d] = (R[f] - L[f]) / k.dx;
  for (int a = 0; a < dim; ++a) {
    if (a == d) continue;
    double Lp[4], Lm[4], Rp[4], Rm[4];
    int o[3] = {0, 0, 0};
    o[a] = 1;
    prim_vt(k, S.at(cL[0] + o[0], cL[1] + o[1], cL[2] + o[2]), Lp);
    prim_vt(k, S.at(cL[0] - o[0], cL[1] - o[1], cL[2] - o[2]), Lm);
    prim_vt(k, S.at(cR[0] + o[0], cR[1] + o[1], cR[2] + o[2]), Rp);
    prim_vt(k, S.at(cR[0] - o[0], cR[1] - o[1], cR[2] - o[2]), Rm);
    for (int f = 0; f <= dim; ++f) g[f][a] = ((Lp[f] - Lm[f]) + (Rp[f] - Rm[f])) / (4.0 * k.dx);
  }
  double div = g[0][0];
  for (int a = 1; a < dim; ++a) div = div + g[a][a];
  double sig[3];
  for (int a = 0; a < dim; ++a) {
    double t = g[a][d] + g[d][a];
    if (a == d) t = fma(-2.0 / 3.0, div, t);
    sig[a] = t * k.inv_re;
  }
  double e = g[dim][d] * k.inv_prre;
  for (int a = 0; a < dim; ++a) e = fma(sig[a], 0.5 * (L[a] + R[a]), e);
  Fv[0] = 0.0;
  for (int a = 0; a < dim; ++a) Fv[1 + a] = sig[a];
  Fv[nv - 1] = e;
}

// RHS over the slab's interior planes.  out: AoS [np planes]
int slab_rhs(const kfvm_table* t, const Consts& k, const Slab& S, double* out, int nthreads,
             double* states_out = nullptr, const uint8_t* flags = nullptr) {
  const int dim = k.dim, nv = k.nv, npts = t->n_points;
  const int rp = npts / (2 * dim);
  // extended-cell box: [-1, n] in every axis, slab axis [p0-1, p0+np]
  int lo[3], cnt[3];
  for (int a = 0; a < 3; ++a) {
    if (a >= dim) {
      lo[a] = 0;
      cnt[a] = 1;
    } else if (a == S.sa) {
      lo[a] = S.p0 - 1;
      cnt[a] = S.np + 2;
    } else {
      lo[a] = -1;
      cnt[a] = k.n[a] + 2;
    }
  }
  const size_t ncell = (size_t)cnt[0] * cnt[1] * cnt[2];
  const size_t cs = (size_t)npts * nv;
  std::vector<double> st(ncell * cs);
  std::atomic<int> err(0);
  const int nrows = cnt[1] * cnt[2];
  parallel_for(nrows, nthreads, [&](int row) {
    const int b = row % cnt[1], c = row / cnt[1];
    for (int a = 0; a < cnt[0]; ++a) {
      const size_t id = ((size_t)c * cnt[1] + b) * cnt[0] + a;
      const int e = flags ? cell_states_kx(t, k, S, flags, lo[0] + a, lo[1] + b, lo[2] + c,
                                           st.data() + id * cs)
                          : cell_states(t, k, S, lo[0] + a, lo[1] + b, lo[2] + c, st.data() + id * cs);
      if (e) err.store(e);
    }
  });
  if (err.load()) return err.load();
  auto sid = [&](int i, int j, int kk) {
    return (((size_t)(kk - lo[2]) * cnt[1] + (j - lo[1])) * cnt[0] + (i - lo[0])) * cs;
  };
  if (states_out) {  // interior cells of the slab, [cell][point][var]
    size_t o = 0;
    const int kn = dim == 3 ? k.n[2] : 1;
    for (int c = 0; c < kn; ++c)
      for (int b = 0; b < k.n[1]; ++b)
        for (int a = 0; a < k.n[0]; ++a) {
          const int cc[3] = {a, b, c};
          if (cc[S.sa] < S.p0 || cc[S.sa] >= S.p0 + S.np) continue;
          std::memcpy(states_out + o, st.data() + sid(a, b, c), cs * sizeof(double));
          o += cs;
        }
  }
  // face-averaged fluxes and the divergence
  int ilo[3] = {0, 0, 0}, icnt[3] = {k.n[0], k.n[1], dim == 3 ? k.n[2] : 1};
  ilo[S.sa] = S.p0;
  icnt[S.sa] = S.np;
  const double* fw = t->face_weights;
  auto face_flux = [&](int d, int i, int j, int kk, double* Fbar) {
    // face between cell (i,j,kk)-e_d (left) and (i,j,kk) (right)
    int li = i, lj = j, lk = kk;
    if (d == 0) li--;
    if (d == 1) lj--;
    if (d == 2) lk--;
    const double* SL = st.data() + sid(li, lj, lk);
    const double* SR = st.data() + sid(i, j, kk);
    for (int v = 0; v < nv; ++v) Fbar[v] = 0.0;
    double F[5];
    for (int m = 0; m < rp; ++m) {
      const int sL = (2 * d + 1) * rp + m;  // +d face of the left cell
      const int sR = (2 * d) * rp + m;      // -d face of the right cell
      riemann(k, d, SL + sL * nv, SR + sR * nv, F);
      for (int v = 0; v < nv; ++v) Fbar[v] = fma(fw[sR], F[v], Fbar[v]);
    }
    if (k.visc) {
      double Fv[5];
      viscous_flux(k, S, d, i, j, kk, Fv);
      for (int v = 0; v < nv; ++v) Fbar[v] = Fbar[v] - Fv[v];
    }
  };
  const int irows = icnt[1] * icnt[2];
  parallel_for(irows, nthreads, [&](int row) {
    const int j = ilo[1] + row % icnt[1], kk = ilo[2] + row / icnt[1];
    double Flo[3][5], Fhi[3][5];
    for (int i = 0; i < icnt[0]; ++i) {
      for (int d = 0; d < dim; ++d) {
        face_flux(d, i, j, kk, Flo[d]);
        face_flux(d, i + (d == 0), j + (d == 1), kk + (d == 2), Fhi[d]);
      }
      double* o = out + ((((size_t)(kk - ilo[2]) * icnt[1] + (j - ilo[1])) * icnt[0]) + i) * nv;
      for (int v = 0; v < nv; ++v) {
        double acc = Fhi[0][v] - Flo[0][v];
        acc = acc + (Fhi[1][v] - Flo[1][v]);
        if (dim == 3) acc = acc + (Fhi[2][v] - Flo[2][v]);
        o[v] = -(acc / k.dx);
      }
      if (k.g2 != 0.0) {  // gravity source from the cell average (P eq rtSource)
        const double* U = S.at(i, j, kk);
        o[2] = o[2] + k.g2 * U[0];
        o[nv - 1] = o[nv - 1] + k.g2 * U[2];
      }
    }
  });
  return 0;
}

double cell_speed(const Consts& k, const double* U) {  // S:610 (+|w|+c in 3-D)
  const double p = pressure(k.dim, U, k.gm1);
  const double c = sound(k.gamma, p, U[0]);
  double s = std::fabs(U[1] / U[0]) + c;
  s = s + (std::fabs(U[2] / U[0]) + c);
  if (k.dim == 3) s = s + (std::fabs(U[3] / U[0]) + c);
  return s;
}

bool admissible(const Consts& k, const double* U) {
  return U[0] > 0.0 && pressure(k.dim, U, k.gm1) > 0.0 && std::isfinite(U[k.nv - 1]);
}

size_t ncells(const Consts& k) { return (size_t)k.n[0] * k.n[1] * k.n[2]; }

// stage combine (pinned)
inline double combine(int stage, double u0, double uk, double L, double dt) {
  // Shu-Osher SSP-RK3 in increment form: u_{k+1} = u0 + b_k (w - u0) with
  // w = u_k + dt L(u_k), b = 1, 1/4, 2/3 (exact free-stream preservation)
  const double w = fma(dt, L, uk);
  if (stage == 1) return w;
  if (stage == 2) return fma(0.25, w - u0, u0);
  return fma(2.0 / 3.0, w - u0, u0);
}

// SSP(4,3) with the embedded SSP(3,2), increment form like the
// SSP-RK3 combine: h = dt/2;
//   Y2 = u + h L(u);  Y3 = Y2 + h L(Y2);  w = Y3 + h L(Y3);
//   Y4 = u + (1/3)(w - u);  uhat = u + (2/3)(w - u)  [= u + dt/3 (L1+L2+L3)];
//   u+ = Y4 + h L(Y4).
// Stage codes 11..14; stage 13 also returns uhat.
inline double combine43(int stage, double u0, double uk, double L, double hdt, double* uhat) {
  const double w = fma(hdt, L, uk);
  if (stage == 13) {
    *uhat = fma(2.0 / 3.0, w - u0, u0);
    return fma(1.0 / 3.0, w - u0, u0);
  }
  return w;
}

// Error norm of the embedded pair: sqrt(sum / N) of
// ((u+ - uhat) / (atol + rtol |u+|))^2, summed in a pinned three-level order
// that any slab decomposition reproduces: per row (x, then variables)
// sequential fma, per plane sequential over its rows, then sequential over
// the planes of the slab axis.
double error_norm(const Consts& k, const double* Up, const double* Uh) {
  const int nv = k.nv;
  const int nrow = k.dim == 3 ? k.n[1] : 1, npl = k.n[k.dim - 1];
  const int nx = k.n[0];
  double s = 0.0;
  for (int p = 0; p < npl; ++p) {
    double pl = 0.0;
    for (int j = 0; j < nrow; ++j) {
      const size_t o = ((size_t)p * nrow + j) * nx * nv;
      double r = 0.0;
      for (int i = 0; i < nx * nv; ++i) {
        const double q = (Up[o + i] - Uh[o + i]) / fma(k.rtol, std::fabs(Up[o + i]), k.atol);
        r = fma(q, q, r);
      }
      pl = pl + r;
    }
    s = s + pl;
  }
  return std::sqrt(s / ((double)ncells(k) * nv));
}

// PI step-size controller (orders 3/2): on acceptance
// fac = clamp(safety * e^(-0.7/3) * e_prev^(0.4/3), 0.2, 5) with
// e = max(err, 1e-10) (a zero estimate saturates at 5x); on rejection
// fac = max(0.2, safety * err^(-1/3)) (0.2 for a NaN estimate).  Powers by the
// pinned kf_pow.
inline double pi_factor(const Consts& k, bool accept, double err, double err_prev) {
  if (accept) {
    const double e = std::fmax(err, 1e-10);
    const double f = k.safety * kf_pow(e, -0.7 / 3.0) * kf_pow(err_prev, 0.4 / 3.0);
    return std::fmin(5.0, std::fmax(0.2, f));
  }
  if (!(err == err)) return 0.2;
  return std::fmax(0.2, k.safety * kf_pow(err, -1.0 / 3.0));
}

int full_rhs(const kfvm_table* t, const Consts& k, const double* U, double* out, int nslabs,
             int nthreads) {
  const int sa = k.dim - 1;
  const size_t plane = ncells(k) / k.n[sa] * k.nv;
  std::vector<uint8_t> fl;
  if (k.kx) fl = global_flags(t, k, U, nthreads);
  for (int r = 0; r < nslabs; ++r) {
    int p0, np;
    slab_range(k.n[sa], nslabs, r, &p0, &np);
    Slab S;
    S.init(k, p0, np);
    S.load(U);
    const int e = slab_rhs(t, k, S, out + (size_t)p0 * plane, nthreads, nullptr,
                           k.kx ? fl.data() : nullptr);
    if (e) return e;
  }
  return 0;
}

}  // namespace

extern "C" {

int kfo_rhs(const kfvm_config* cfg, const kfvm_table* t, const double* U, double* dUdt,
            int nthreads) {
  const Consts k = make_consts(cfg, t);
  return full_rhs(t, k, U, dUdt, 1, nthreads);
}

int kfo_states(const kfvm_config* cfg, const kfvm_table* t, const double* U, double* states,
               int nthreads) {
  const Consts k = make_consts(cfg, t);
  Slab S;
  S.init(k, 0, k.n[k.dim - 1]);
  S.load(U);
  std::vector<double> tmp(ncells(k) * k.nv);
  std::vector<uint8_t> fl;
  if (k.kx) fl = global_flags(t, k, U, nthreads);
  return slab_rhs(t, k, S, tmp.data(), nthreads, states, k.kx ? fl.data() : nullptr);
}

// Viscous flux F^(v) of one face (S:571-580 examples): the face between the
// global cells (i,j,k) - e_d and (i,j,k) of the global AoS state U.
void kfo_viscous_face(const kfvm_config* cfg, const double* U, int i, int j, int kk, int d,
                      double* Fv) {
  const Consts k = make_consts(cfg, nullptr);
  Slab S;
  S.init(k, 0, k.n[k.dim - 1]);
  S.load(U);
  viscous_flux(k, S, d, i, j, kk, Fv);
}

// KXRCF flags of every cell (1 = WENO), global AoS cell order
int kfo_kxrcf_flags(const kfvm_config* cfg, const kfvm_table* t, const double* U,
                    unsigned char* flags, int nthreads) {
  const Consts k = make_consts(cfg, t);
  const std::vector<uint8_t> fl = global_flags(t, k, U, nthreads);
  std::memcpy(flags, fl.data(), fl.size());
  return 0;
}

double kfo_pow(double x, double y) { return kf_pow(x, y); }

void kfo_combine43(int stage, long long n, const double* U0, const double* Uk, const double* L,
                   double dt, double* out, double* uhat) {
  const double hdt = 0.5 * dt;
  double dummy;
  for (long long i = 0; i < n; ++i)
    out[i] = combine43(stage, U0[i], Uk[i], L[i], hdt, uhat ? uhat + i : &dummy);
}

int kfo_select_dt(const kfvm_config* cfg, const double* U, double* dt) {
  const Consts k = make_consts(cfg, nullptr);
  double smax = 0.0;
  for (size_t c = 0; c < ncells(k); ++c) smax = std::fmax(smax, cell_speed(k, U + c * k.nv));
  *dt = (k.cfl * k.dx) / smax;
  return std::isfinite(*dt) && *dt > 0 ? 0 : 2;
}

int kfo_stage(const kfvm_config* cfg, const kfvm_table* t, const double* U0, const double* Uk,
              double* Uout, int stage, double dt, int nthreads) {
  const Consts k = make_consts(cfg, t);
  const size_t n = ncells(k) * k.nv;
  std::vector<double> L(n);
  const int e = full_rhs(t, k, Uk, L.data(), 1, nthreads);
  if (e) return e;
  for (size_t i = 0; i < n; ++i) Uout[i] = combine(stage, U0[i], Uk[i], L[i], dt);
  for (size_t c = 0; c < ncells(k); ++c)
    if (!admissible(k, Uout + c * k.nv)) return 2;
  return 0;
}

int kfo_run(const kfvm_config* cfg, const kfvm_table* t, double* U, int nsteps, double* dt_seq,
            int nslabs, int nthreads) {
  const Consts k = make_consts(cfg, t);
  const size_t n = ncells(k) * k.nv;
  std::vector<double> U0(n), Uk(n), L(n);
  for (int step = 0; step < nsteps; ++step) {
    double dt;
    if (kfo_select_dt(cfg, U, &dt)) return 2;
    if (dt_seq) dt_seq[step] = dt;
    std::memcpy(U0.data(), U, n * sizeof(double));
    for (int stage = 1; stage <= 3; ++stage) {
      const double* src = stage == 1 ? U0.data() : U;
      const int e = full_rhs(t, k, src, L.data(), nslabs, nthreads);
      if (e) return e;
      for (size_t i = 0; i < n; ++i) Uk[i] = combine(stage, U0[i], src[i], L[i], dt);
      std::memcpy(U, Uk.data(), n * sizeof(double));
      for (size_t c = 0; c < ncells(k); ++c)
        if (!admissible(k, U + c * k.nv)) return 2;
    }
  }
  return 0;
}

// advance_to with SSP(4,3)+SSP(3,2) and the PI controller:
// attempts until t_final (the last step lands exactly on it) or max_attempts.
// dt = min(dt_cfl, dt_err) (dt_err = inf before the first estimate), clamped
// above by dt_max; below dt_min aborts (code 2).  An attempt is accepted when
// every stage stayed admissible and err <= 1; a rejected attempt leaves u
// unchanged.  dt_seq receives the accepted steps' dt (up to cap).
int kfo_advance43(const kfvm_config* cfg, const kfvm_table* t, double* U, double t_final,
                  int max_attempts, double* dt_seq, int cap, int* stats, double* t_reached,
                  int nthreads) {
  const Consts k = make_consts(cfg, t);
  const size_t n = ncells(k) * k.nv;
  std::vector<double> Y(n), Z(n), Uh(n), L(n);
  double tt = 0.0, dt_err = INFINITY, err_prev = 1.0;
  int nacc = 0, nrej = 0;
  for (int at = 0; at < max_attempts && tt < t_final; ++at) {
    double dt;
    if (kfo_select_dt(cfg, U, &dt)) return 2;
    dt = std::fmin(dt, dt_err);
    if (dt < k.dt_min) return 2;  // unstable setup
    dt = std::fmin(dt, k.dt_max);
    const double rem = t_final - tt;
    if (rem < dt) dt = rem;
    const double hdt = 0.5 * dt;
    bool ok = true;
    const double* src = U;
    double* dst[4] = {Y.data(), Z.data(), Y.data(), Z.data()};
    for (int st = 0; st < 4 && ok; ++st) {
      if (full_rhs(t, k, src, L.data(), 1, nthreads)) {
        ok = false;
        break;
      }
      for (size_t i = 0; i < n; ++i)
        dst[st][i] = combine43(11 + st, U[i], src[i], L[i], hdt, &Uh[i]);
      for (size_t c = 0; c < ncells(k) && ok; ++c)
        if (!admissible(k, dst[st] + c * k.nv)) ok = false;
      src = dst[st];
    }
    const double err = ok ? error_norm(k, Z.data(), Uh.data()) : NAN;
    const bool accept = ok && err <= 1.0;
    dt_err = dt * pi_factor(k, accept, err, err_prev);
    if (accept) {
      err_prev = std::fmax(err, 1e-10);
      tt = tt + dt;
      std::memcpy(U, Z.data(), n * sizeof(double));
      if (dt_seq && nacc < cap) dt_seq[nacc] = dt;
      ++nacc;
    } else {
      ++nrej;
    }
  }
  if (stats) {
    stats[0] = nacc;
    stats[1] = nrej;
  }
  if (t_reached) *t_reached = tt;
  return 0;
}

int kfo_sample_stage(const kfvm_config* cfg, const kfvm_table* t, const double* U, int p0, int np,
                     int nthreads, double* seconds) {
  const Consts k = make_consts(cfg, t);
  Slab S;
  S.init(k, p0, np);
  S.load(U);
  std::vector<double> out(ncells(k) / k.n[k.dim - 1] * np * k.nv), un(out.size());
  const auto t0 = std::chrono::steady_clock::now();
  const int e = slab_rhs(t, k, S, out.data(), nthreads);
  // the stage-1 combine u1 = u + dt L(u) is part of the unit of work
  const size_t plane = out.size() / np;
  const double* Ui = U + (size_t)p0 * plane;
  for (size_t i = 0; i < out.size(); ++i) un[i] = combine(1, Ui[i], Ui[i], out[i], 1e-3);
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return e;
}

// RHS of the slab [p0, p0+np) of the slab axis, given the slab's local array
// WITH its H = R+1 halo planes on each side (AoS, planes of the slab axis);
// used by the multi-process (gloo) decomposition test.
int kfo_slab_rhs(const kfvm_config* cfg, const kfvm_table* t, int p0, int np,
                 const double* U_local, double* out, int nthreads) {
  const Consts k = make_consts(cfg, t);
  Slab S;
  S.init(k, p0, np);
  S.load_local(U_local);
  return slab_rhs(t, k, S, out, nthreads);
}

// fill_ghost of the whole domain: out = the padded box with
// R+1 ghost cells on every side (AoS, x fastest) — the boundary-kind hook of
// the tests.
int kfo_fill_ghost(const kfvm_config* cfg, const double* U, double* out) {
  const Consts k = make_consts(cfg, nullptr);
  Slab S;
  S.init(k, 0, k.n[k.dim - 1]);
  S.load(U);
  std::memcpy(out, S.U.data(), S.U.size() * sizeof(double));
  return 0;
}

// max over ncells AoS cells of sum_d (|u_d| + c) (the select_dt reduction)
double kfo_max_speed(const kfvm_config* cfg, const double* U, long long ncells) {
  const Consts k = make_consts(cfg, nullptr);
  double smax = 0.0;
  for (long long c = 0; c < ncells; ++c) smax = std::fmax(smax, cell_speed(k, U + c * k.nv));
  return smax;
}

// one SSP-RK3 stage combine over n values (the pinned increment form)
void kfo_combine(int stage, long long n, const double* U0, const double* Uk, const double* L,
                 double dt, double* out) {
  for (long long i = 0; i < n; ++i) out[i] = combine(stage, U0[i], Uk[i], L[i], dt);
}

double kfo_pressure(int dim, const double* U, double gamma) { return pressure(dim, U, gamma - 1.0); }

double kfo_sound_speed(int dim, const double* U, double gamma) {
  return sound(gamma, pressure(dim, U, gamma - 1.0), U[0]);
}

void kfo_transform(int dim, const double* Uref, double gamma, double* phi, double* phi_inv) {
  const int nv = dim + 2;
  const Transform T = make_transform(dim, Uref);
  const double gm1 = gamma - 1.0, inv_gm1 = 1.0 / gm1;
  for (int c = 0; c < nv; ++c) {
    double e[5] = {0, 0, 0, 0, 0}, w[5], u[5];
    e[c] = 1.0;
    for (int v = 0; v < nv; ++v) w[v] = to_recon(dim, T, gm1, e, v);
    // column c of Phi (resp. Phi^-1) is the image of the unit vector e_c
    for (int v = 0; v < nv; ++v) phi[v * nv + c] = w[v];
    from_recon(dim, T, inv_gm1, e, u);
    for (int v = 0; v < nv; ++v) phi_inv[v * nv + c] = u[v];
  }
}

void kfo_to_recon(int dim, const double* Uref, double gamma, const double* U, double* W) {
  const Transform T = make_transform(dim, Uref);
  for (int v = 0; v < dim + 2; ++v) W[v] = to_recon(dim, T, gamma - 1.0, U, v);
}

void kfo_from_recon(int dim, const double* Uref, double gamma, const double* W, double* U) {
  const Transform T = make_transform(dim, Uref);
  from_recon(dim, T, 1.0 / (gamma - 1.0), W, U);
}

void kfo_riemann(int dim, int solver, int axis, const double* UL, const double* UR, double gamma,
                 double* F) {
  kfvm_config c{};
  c.dim = dim;
  c.gamma = gamma;
  c.riemann = solver;
  c.dx = 1.0;
  c.nx = c.ny = c.nz = 1;
  Consts k = make_consts(&c, nullptr);
  riemann(k, axis, UL, UR, F);
}

void kfo_wavespeeds(int dim, int axis, const double* UL, const double* UR, double gamma,
                    double* out) {
  kfvm_config c{};
  c.dim = dim;
  c.gamma = gamma;
  c.dx = 1.0;
  c.nx = c.ny = c.nz = 1;
  Consts k = make_consts(&c, nullptr);
  double F[5];
  riemann(k, axis, UL, UR, F, out);
}

void kfo_exact_flux(int dim, int axis, const double* U, double gamma, double* F) {
  const double p = pressure(dim, U, gamma - 1.0);
  exact_flux(dim, axis, U, U[1 + axis] / U[0], p, F);
}

void kfo_weno(const kfvm_table* t, double dx, double eps, const double* g, double* beta,
              double* omega, double* values) {
  kfvm_config c{};
  c.dim = t->dim;
  c.radius = t->radius;
  c.dx = dx;
  c.eps = eps;
  c.gamma = 1.4;
  c.nx = c.ny = c.nz = 1;
  const Consts k = make_consts(&c, t);
  weno_field(t, k, g, beta, omega, values);
}

int kfo_limit(int dim, int n, double* states, const double* nbr, double gamma, double kappa,
              double kf, double* info) {
  kfvm_config c{};
  c.dim = dim;
  c.gamma = gamma;
  c.kappa = kappa;
  c.flattener_kf = kf;
  c.dx = 1.0;
  c.nx = c.ny = c.nz = 1;
  const Consts k = make_consts(&c, nullptr);
  return limit_cell(k, n, states, nbr, info);
}

}  // extern "C"
