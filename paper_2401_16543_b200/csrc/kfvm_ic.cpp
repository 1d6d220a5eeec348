// kfvm_ic.cpp — seeded synthetic initial conditions (host, multithreaded).
//
// BASELINE.json configs 1-5 define the workloads; their recipes leave the
// RNG, mode form and normalisation open, so they are pinned here (DESIGN.md
// §6): splitmix64 with a fixed seed per config; U[0,1) = (x >> 11) * 2^-53;
// per Fourier mode the draws are k_x..k_d in {1..4}, a in [-1,1],
// phi in [0, 2 pi); s = sum_m a_m sin(2 pi k_m.x + phi_m) / max|s| with the
// max over every cell-average GL point of the global grid; Voronoi seeds
// uniform in the box with Euclidean nearest seed (ties -> lowest index);
// log-uniform draws exp(U[ln a, ln b]); the sphere uses the minimum-image
// distance.  Cell averages by the tensor R^d GL rule.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/kfvm_b200.h"
#include "kfvm_ic_eval.h"
#include "kfvm_ic_host.h"

namespace kfvm_b200 {

namespace {
struct SplitMix {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
};

template <class F>
void par_for(int n, int nthreads, F&& f) {
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

const double kPi = 3.14159265358979323846;

// GL nodes/weights on [-1/2, 1/2] (standard values, as in the reference's
// gauss_legendre_rule, geometry.cpp:74-101)
void gl_rule(int R, double* x, double* w) {
  if (R == 2) {
    const double a = 0.5773502691896257645;
    x[0] = -0.5 * a;
    x[1] = 0.5 * a;
    w[0] = w[1] = 0.5;
  } else {
    const double a = 0.7745966692414833770;
    x[0] = -0.5 * a;
    x[1] = 0.0;
    x[2] = 0.5 * a;
    w[0] = w[2] = 0.5 * 0.5555555555555555556;
    w[1] = 0.5 * 0.8888888888888888889;
  }
}
}  // namespace

int ic_plan_build(const kfvm_config* cfg, const kfvm_ic_params* ic, ICHostPlan* hp) {
  ICPlan& P = hp->plan;
  std::memset(&P, 0, sizeof(P));
  P.kind = ic->kind;
  P.dim = cfg->dim;
  P.R = cfg->radius;
  P.n[0] = cfg->nx;
  P.n[1] = cfg->ny;
  P.n[2] = cfg->dim == 3 ? cfg->nz : 1;
  P.dx = cfg->dx;
  for (int a = 0; a < 3; ++a) P.origin[a] = ic->origin[a];
  P.gamma = cfg->gamma;
  P.inv_gm1 = 1.0 / (cfg->gamma - 1.0);
  gl_rule(P.R, P.node, P.w);
  SplitMix rng{ic->seed};
  if (ic->kind == KFVM_IC_FOURIER || ic->kind == KFVM_IC_FOURIER_SPHERE) {
    if (ic->n_modes < 1 || ic->n_modes > KFVM_IC_MAX_MODES) return KFVM_ERR_CONFIG;
    for (int a = 0; a < P.dim; ++a) {
      const int len = 4 * P.n[a] * P.R;
      hp->fc[a].resize(len);
      hp->fs[a].resize(len);
      for (int k = 1; k <= 4; ++k)
        for (int i = 0; i < P.n[a]; ++i)
          for (int q = 0; q < P.R; ++q) {
            const double x = P.origin[a] + P.dx * (((double)i + 0.5) + P.node[q]);
            const double th = 2.0 * kPi * (double)k * x;
            hp->fc[a][(k - 1) * P.n[a] * P.R + i * P.R + q] = std::cos(th);
            hp->fs[a][(k - 1) * P.n[a] * P.R + i * P.R + q] = std::sin(th);
          }
      P.fc[a] = hp->fc[a].data();
      P.fs[a] = hp->fs[a].data();
    }
    for (int f = 0; f < 1 + P.dim; ++f) {
      FourierField& F = P.f[f];
      F.nm = ic->n_modes;
      for (int m = 0; m < F.nm; ++m) {
        for (int a = 0; a < 3; ++a) F.k[m][a] = 1;
        for (int a = 0; a < P.dim; ++a) F.k[m][a] = 1 + std::min(3, (int)(rng.uniform() * 4.0));
        F.a[m] = 2.0 * rng.uniform() - 1.0;
        const double phi = 2.0 * kPi * rng.uniform();
        F.cphi[m] = std::cos(phi);
        F.sphi[m] = std::sin(phi);
      }
      F.norm = 1.0;
    }
    if (ic->kind == KFVM_IC_FOURIER_SPHERE) {
      for (int a = 0; a < P.dim; ++a) P.sph_c[a] = rng.uniform();
      P.sph_r2 = 0.2 * 0.2;
    }
    hp->needs_norm = true;
  } else if (ic->kind == KFVM_IC_VORONOI) {
    if (ic->n_regions < 1 || ic->n_regions > KFVM_IC_MAX_REGIONS) return KFVM_ERR_CONFIG;
    P.nreg = ic->n_regions;
    for (int r = 0; r < P.nreg; ++r)
      for (int a = 0; a < P.dim; ++a)
        P.seeds[r][a] = P.origin[a] + (double)P.n[a] * P.dx * rng.uniform();
    const double lr0 = std::log(0.1), lr1 = std::log(2.0), lp0 = std::log(0.1), lp1 = std::log(10.0);
    for (int r = 0; r < P.nreg; ++r) {
      const double rho = std::exp(lr0 + rng.uniform() * (lr1 - lr0));
      const double p = std::exp(lp0 + rng.uniform() * (lp1 - lp0));
      double vel[3] = {0, 0, 0};
      for (int a = 0; a < P.dim; ++a) vel[a] = 2.0 * rng.uniform() - 1.0;
      double ke = vel[0] * vel[0] + vel[1] * vel[1];
      if (P.dim == 3) ke = ke + vel[2] * vel[2];
      P.reg[r][0] = rho;
      for (int a = 0; a < P.dim; ++a) P.reg[r][1 + a] = rho * vel[a];
      P.reg[r][P.dim + 1] = p * P.inv_gm1 + 0.5 * (rho * ke);
    }
    hp->needs_norm = false;
  } else if (ic->kind == KFVM_IC_UNIFORM) {
    for (int v = 0; v < 5; ++v) P.value[v] = ic->value[v];
    hp->needs_norm = false;
  } else if (ic->kind == KFVM_IC_VORTEX || ic->kind == KFVM_IC_DENSITY_WAVE) {
    for (int v = 0; v < 5; ++v) P.value[v] = ic->value[v];
    hp->needs_norm = false;  // evaluated directly on the host
  } else {
    return KFVM_ERR_CONFIG;
  }
  return KFVM_OK;
}

// analytic ICs used by the convergence tests (host only: exp/pow/sin)
static void analytic_point(const ICPlan& P, const double x[3], double* U) {
  const int nv = P.dim + 2;
  double rho, vel[3] = {0, 0, 0}, p;
  const double g = P.gamma;
  if (P.kind == KFVM_IC_VORTEX) {  // PAPER.md §6.1
    const double om = 5.0 * std::sqrt(2.0 * std::exp(1.0)) / (4.0 * kPi) *
                      std::exp(-0.5 * (x[0] * x[0] + x[1] * x[1]));
    const double base = 1.0 + 0.5 * (1.0 - g) * om * om;
    rho = std::pow(base, 1.0 / (g - 1.0));
    vel[0] = 1.0 - x[1] * om;
    vel[1] = 1.0 + x[0] * om;
    p = std::pow(base, g / (g - 1.0)) / g;
  } else {  // density wave: value = (amp, u, v, w, kmode)
    double ph = 0.0;
    for (int a = 0; a < P.dim; ++a) ph += x[a];
    rho = 1.0 + P.value[0] * std::sin(2.0 * kPi * P.value[4] * ph);
    for (int a = 0; a < P.dim; ++a) vel[a] = P.value[1 + a];
    p = 1.0;
  }
  double ke = vel[0] * vel[0] + vel[1] * vel[1] + vel[2] * vel[2];
  U[0] = rho;
  for (int a = 0; a < P.dim; ++a) U[1 + a] = rho * vel[a];
  U[nv - 1] = p * P.inv_gm1 + 0.5 * (rho * ke);
}

int ic_generate_host(const kfvm_config* cfg, const kfvm_ic_params* ic, int z0, int nzl,
                     int nthreads, double* U) {
  ICHostPlan hp;
  int rc = ic_plan_build(cfg, ic, &hp);
  if (rc) return rc;
  ICPlan& P = hp.plan;
  const int sa = P.dim - 1;
  const int nv = P.dim + 2;
  if (z0 < 0 || nzl < 0 || z0 + nzl > P.n[sa]) return KFVM_ERR_CONFIG;
  if (nthreads < 1) nthreads = 1;
  const int nplanes_g = P.n[sa];
  if (hp.needs_norm) {
    for (int f = 0; f < 1 + P.dim; ++f) {
      std::vector<double> pm(nplanes_g, 0.0);
      par_for(nplanes_g, nthreads, [&](int pl) {
        double m = 0.0;
        if (P.dim == 3) {
          for (int j = 0; j < P.n[1]; ++j)
            for (int i = 0; i < P.n[0]; ++i) m = std::fmax(m, cell_field_max(P, P.f[f], i, j, pl));
        } else {
          for (int i = 0; i < P.n[0]; ++i) m = std::fmax(m, cell_field_max(P, P.f[f], i, pl, 0));
        }
        pm[pl] = m;
      });
      double m = 0.0;
      for (double x : pm) m = std::fmax(m, x);
      P.f[f].norm = m;
    }
  }
  const size_t plane = (size_t)P.n[0] * (P.dim == 3 ? P.n[1] : 1);
  par_for(nzl, nthreads, [&](int lp) {
    const int pl = z0 + lp;
    for (size_t c = 0; c < plane; ++c) {
      const int i = (int)(c % P.n[0]);
      const int j = P.dim == 3 ? (int)(c / P.n[0]) : pl;
      const int k = P.dim == 3 ? pl : 0;
      double* out = U + ((size_t)lp * plane + c) * nv;
      if (P.kind == KFVM_IC_VORTEX || P.kind == KFVM_IC_DENSITY_WAVE) {
        for (int v = 0; v < nv; ++v) out[v] = 0.0;
        const int R = P.R, rz = P.dim == 3 ? R : 1;
        const int ci[3] = {i, j, k};
        for (int cc = 0; cc < rz; ++cc)
          for (int b = 0; b < R; ++b)
            for (int a = 0; a < R; ++a) {
              const int qi[3] = {a, b, cc};
              double x[3] = {0, 0, 0};
              for (int d = 0; d < P.dim; ++d) x[d] = coord(P, d, ci[d], qi[d]);
              double Up[5];
              analytic_point(P, x, Up);
              double wgt = P.w[a] * P.w[b];
              if (P.dim == 3) wgt = wgt * P.w[cc];
              for (int v = 0; v < nv; ++v) out[v] = out[v] + wgt * Up[v];
            }
      } else {
        cell_average(P, i, j, k, out);
      }
    }
  });
  return KFVM_OK;
}

}  // namespace kfvm_b200

extern "C" int kfvm_ic_generate(const kfvm_config* cfg, const kfvm_ic_params* ic, int z0,
                                int nz_local, int nthreads, double* U_host) {
  if (!cfg || !ic || !U_host) return KFVM_ERR_CONFIG;
  return kfvm_b200::ic_generate_host(cfg, ic, z0, nz_local, nthreads, U_host);
}

extern "C" void kfvm_config_defaults(kfvm_config* c, int dim, int radius, int nx, int ny, int nz,
                                     int bc) {
  std::memset(c, 0, sizeof(*c));
  c->dim = dim;
  c->radius = radius;
  c->nx = nx;
  c->ny = ny;
  c->nz = dim == 3 ? nz : 1;
  c->bc = bc;
  c->riemann = KFVM_RIEMANN_HLLC;
  c->dx = 1.0 / (double)nx;
  c->gamma = 1.4;
  c->cfl = 1.0;  // S:728 default; BASELINE configs override
  c->eps = 1e-40;
  c->kappa = 0.4;
  c->flattener_kf = 0.33;
  c->kxrcf = 0;
  c->kxrcf_m = 1.5;
  c->integrator = KFVM_SSPRK3;
  c->atol = 1e-4;
  c->rtol = 1e-4;
  c->safety = 0.9;
  c->dt_min = 0.0;
  c->dt_max = 0.0;
  c->viscous = 0;
  c->reynolds = 1.0;
  c->prandtl = 0.71;
  c->mach = 1.0;
  c->inv_froude2 = 0.0;
}

extern "C" void kfvm_slab_range(int n_global, int nranks, int rank, int* p0, int* np) {
  const int base = n_global / nranks, rem = n_global % nranks;
  *np = base + (rank < rem ? 1 : 0);
  *p0 = rank * base + (rank < rem ? rank : rem);
}
