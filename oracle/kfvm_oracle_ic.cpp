// kfvm_oracle_ic.cpp — CPU oracle restatement of the seeded synthetic initial
// conditions of BASELINE.json configs 1-5 (TEST INFRASTRUCTURE ONLY).
//
// This lets the CPU reference arm of bench.py and the tests build the
// workload's cell averages without mapping the product library.  It restates
// the recipe pinned in DESIGN.md §6 independently of
// paper_2401_16543_b200/csrc/kfvm_ic*.{h,cpp}; tests/test_ic.py checks the two
// bit for bit.  Recipe:
//   * splitmix64 stream per config seed; U[0,1) = (x >> 11) 2^-53;
//   * Fourier field s = sum_m a_m sin(2 pi k_m.x + phi_m) / max|s| — the sine
//     is the imaginary part of e^{i phi} prod_a e^{i 2 pi k_a x_a}, multiplied
//     in axis order from per-axis cos/sin tables, the max over every
//     cell-average GL point of the global grid; draws per mode: k_a in
//     {1..4} (a < dim), a in [-1,1], phi in [0, 2 pi);
//   * rho = 1 + 0.2 s_rho, u_a = (1, 0.5, 0.25)_a + 0.05 s_{u_a}, p = 1;
//   * sphere (config 5): centre U[0,1)^d drawn after the fields, radius 0.2,
//     minimum-image distance d - rint(d), rho x4 and p x10 inside;
//   * Voronoi: seeds uniform in the box (all seeds first), then per region
//     rho = exp(U[ln .1, ln 2]), p = exp(U[ln .1, ln 10]), u_a = U[-1, 1];
//     Euclidean nearest seed, ties to the lowest index;
//   * cell averages by the tensor R^d Gauss-Legendre rule,
//     point states accumulated as out += w_a w_b (w_c) U in (c, b, a) order.
// Compiled with -ffp-contract=off like the product's host generator.
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "kfvm_oracle.h"

namespace {

constexpr double kTwoPi = 2.0 * 3.14159265358979323846;

uint64_t mix_next(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
double mix_uniform(uint64_t* s) { return (double)(mix_next(s) >> 11) * 0x1.0p-53; }

struct Mode {
  int k[3];
  double amp, c, s;
};

struct Recipe {
  int kind, dim, R, nv;
  int n[3];
  double dx, org[3], inv_gm1;
  double x[3], w[3];                       // GL nodes / weights on [-1/2, 1/2]
  std::vector<double> cs[3], sn[3];        // [k-1][i][q] per axis
  std::vector<Mode> field[4];              // rho, u, v, w
  double norm[4] = {1, 1, 1, 1};
  std::vector<std::array<double, 3>> seed;
  std::vector<std::array<double, 5>> reg;
  double centre[3] = {0, 0, 0};
  double value[5] = {0, 0, 0, 0, 0};

  double pos(int a, int i, int q) const { return org[a] + dx * (((double)i + 0.5) + x[q]); }

  double raw(int f, const int* gi) const {  // unnormalised Fourier sum at a GL point
    double acc = 0.0;
    for (const Mode& m : field[f]) {
      double re = m.c, im = m.s;
      for (int a = 0; a < dim; ++a) {
        const size_t o = ((size_t)(m.k[a] - 1) * n[a]) * R + gi[a];
        const double c = cs[a][o], s = sn[a][o];
        const double r2 = re * c - im * s;
        const double i2 = re * s + im * c;
        re = r2;
        im = i2;
      }
      acc = acc + m.amp * im;
    }
    return acc;
  }

  void point(const int* ci, const int* qi, double* U) const {
    if (kind == KFVM_IC_VORONOI) {
      int best = 0;
      double bd = 0.0;
      for (size_t r = 0; r < seed.size(); ++r) {
        double d = 0.0;
        for (int a = 0; a < dim; ++a) {
          const double t = pos(a, ci[a], qi[a]) - seed[r][a];
          d = a == 0 ? t * t : d + t * t;
        }
        if (r == 0 || d < bd) {
          bd = d;
          best = (int)r;
        }
      }
      for (int v = 0; v < nv; ++v) U[v] = reg[best][v];
      return;
    }
    double rho, u[3] = {0.0, 0.0, 0.0}, p;
    if (kind == KFVM_IC_UNIFORM) {
      rho = value[0];
      u[0] = value[1];
      u[1] = value[2];
      u[2] = value[3];
      p = value[4];
    } else {
      int gi[3];
      for (int a = 0; a < 3; ++a) gi[a] = ci[a] * R + qi[a];
      static const double base[3] = {1.0, 0.5, 0.25};
      rho = 1.0 + 0.2 * (raw(0, gi) / norm[0]);
      for (int a = 0; a < dim; ++a) u[a] = base[a] + 0.05 * (raw(1 + a, gi) / norm[1 + a]);
      p = 1.0;
      if (kind == KFVM_IC_FOURIER_SPHERE) {
        double d2 = 0.0;
        for (int a = 0; a < dim; ++a) {
          double d = pos(a, ci[a], qi[a]) - centre[a];
          d = d - std::rint(d);
          d2 = d2 + d * d;
        }
        if (d2 < 0.2 * 0.2) {
          rho = rho * 4.0;
          p = p * 10.0;
        }
      }
    }
    double ke = u[0] * u[0] + u[1] * u[1];
    if (dim == 3) ke = ke + u[2] * u[2];
    U[0] = rho;
    for (int a = 0; a < dim; ++a) U[1 + a] = rho * u[a];
    U[nv - 1] = p * inv_gm1 + 0.5 * (rho * ke);
  }

  void average(const int* ci, double* out) const {
    for (int v = 0; v < nv; ++v) out[v] = 0.0;
    const int rz = dim == 3 ? R : 1;
    for (int c = 0; c < rz; ++c)
      for (int b = 0; b < R; ++b)
        for (int a = 0; a < R; ++a) {
          const int qi[3] = {a, b, c};
          double U[5];
          point(ci, qi, U);
          double wt = w[a] * w[b];
          if (dim == 3) wt = wt * w[c];
          for (int v = 0; v < nv; ++v) out[v] = out[v] + wt * U[v];
        }
  }

  double cell_max(int f, const int* ci) const {
    const int rz = dim == 3 ? R : 1;
    double m = 0.0;
    for (int c = 0; c < rz; ++c)
      for (int b = 0; b < R; ++b)
        for (int a = 0; a < R; ++a) {
          const int gi[3] = {ci[0] * R + a, ci[1] * R + b, ci[2] * R + c};
          m = std::fmax(m, std::fabs(raw(f, gi)));
        }
    return m;
  }
};

template <class F>
void parallel(int n, int nthreads, F&& f) {
  std::atomic<int> next(0);
  auto work = [&]() {
    for (int i; (i = next.fetch_add(1)) < n;) f(i);
  };
  std::vector<std::thread> th;
  for (int t = 1; t < std::min(nthreads, n); ++t) th.emplace_back(work);
  work();
  for (auto& x : th) x.join();
}

int build(const kfvm_config* cfg, const kfvm_ic_params* ic, Recipe* P) {
  P->kind = ic->kind;
  P->dim = cfg->dim;
  P->R = cfg->radius;
  P->nv = cfg->dim + 2;
  P->n[0] = cfg->nx;
  P->n[1] = cfg->ny;
  P->n[2] = cfg->dim == 3 ? cfg->nz : 1;
  P->dx = cfg->dx;
  for (int a = 0; a < 3; ++a) P->org[a] = ic->origin[a];
  P->inv_gm1 = 1.0 / (cfg->gamma - 1.0);
  if (P->R == 2) {
    const double r = 0.5773502691896257645;  // 1/sqrt(3)
    P->x[0] = -0.5 * r;
    P->x[1] = 0.5 * r;
    P->w[0] = P->w[1] = 0.5;
  } else if (P->R == 3) {
    const double r = 0.7745966692414833770;  // sqrt(3/5)
    P->x[0] = -0.5 * r;
    P->x[1] = 0.0;
    P->x[2] = 0.5 * r;
    P->w[0] = P->w[2] = 0.5 * 0.5555555555555555556;
    P->w[1] = 0.5 * 0.8888888888888888889;
  } else {
    return KFVM_ERR_CONFIG;
  }
  uint64_t st = ic->seed;
  if (ic->kind == KFVM_IC_FOURIER || ic->kind == KFVM_IC_FOURIER_SPHERE) {
    if (ic->n_modes < 1 || ic->n_modes > 16) return KFVM_ERR_CONFIG;
    for (int a = 0; a < P->dim; ++a) {
      const size_t len = (size_t)4 * P->n[a] * P->R;
      P->cs[a].assign(len, 0.0);
      P->sn[a].assign(len, 0.0);
      for (int k = 1; k <= 4; ++k)
        for (int i = 0; i < P->n[a]; ++i)
          for (int q = 0; q < P->R; ++q) {
            const double th = kTwoPi * (double)k * P->pos(a, i, q);
            const size_t o = ((size_t)(k - 1) * P->n[a] + i) * P->R + q;
            P->cs[a][o] = std::cos(th);
            P->sn[a][o] = std::sin(th);
          }
    }
    for (int f = 0; f <= P->dim; ++f) {
      for (int m = 0; m < ic->n_modes; ++m) {
        Mode md{{1, 1, 1}, 0, 0, 0};
        for (int a = 0; a < P->dim; ++a)
          md.k[a] = 1 + std::min(3, (int)(mix_uniform(&st) * 4.0));
        md.amp = 2.0 * mix_uniform(&st) - 1.0;
        const double ph = kTwoPi * mix_uniform(&st);
        md.c = std::cos(ph);
        md.s = std::sin(ph);
        P->field[f].push_back(md);
      }
    }
    if (ic->kind == KFVM_IC_FOURIER_SPHERE)
      for (int a = 0; a < P->dim; ++a) P->centre[a] = mix_uniform(&st);
  } else if (ic->kind == KFVM_IC_VORONOI) {
    if (ic->n_regions < 1 || ic->n_regions > 128) return KFVM_ERR_CONFIG;
    P->seed.assign(ic->n_regions, {0.0, 0.0, 0.0});
    for (auto& s : P->seed)
      for (int a = 0; a < P->dim; ++a) s[a] = P->org[a] + (double)P->n[a] * P->dx * mix_uniform(&st);
    const double r0 = std::log(0.1), r1 = std::log(2.0), p0 = std::log(0.1), p1 = std::log(10.0);
    for (int r = 0; r < ic->n_regions; ++r) {
      const double rho = std::exp(r0 + mix_uniform(&st) * (r1 - r0));
      const double p = std::exp(p0 + mix_uniform(&st) * (p1 - p0));
      double u[3] = {0.0, 0.0, 0.0};
      for (int a = 0; a < P->dim; ++a) u[a] = 2.0 * mix_uniform(&st) - 1.0;
      double ke = u[0] * u[0] + u[1] * u[1];
      if (P->dim == 3) ke = ke + u[2] * u[2];
      std::array<double, 5> s{0, 0, 0, 0, 0};
      s[0] = rho;
      for (int a = 0; a < P->dim; ++a) s[1 + a] = rho * u[a];
      s[P->dim + 1] = p * P->inv_gm1 + 0.5 * (rho * ke);
      P->reg.push_back(s);
    }
  } else if (ic->kind == KFVM_IC_UNIFORM) {
    for (int v = 0; v < 5; ++v) P->value[v] = ic->value[v];
  } else {
    return KFVM_ERR_CONFIG;  // the analytic ICs are not needed by the bench arm
  }
  return KFVM_OK;
}

}  // namespace

extern "C" int kfo_ic_generate(const kfvm_config* cfg, const kfvm_ic_params* ic, int z0, int nzl,
                               int nthreads, double* U) {
  if (!cfg || !ic || !U) return KFVM_ERR_CONFIG;
  Recipe P;
  const int rc = build(cfg, ic, &P);
  if (rc) return rc;
  const int sa = P.dim - 1, ng = P.n[sa];
  if (z0 < 0 || nzl < 0 || z0 + nzl > ng) return KFVM_ERR_CONFIG;
  nthreads = std::max(1, nthreads);
  const int nm = P.dim == 3 ? P.n[1] : 1;
  auto cell = [&](int i, int j, int pl, int* ci) {
    ci[0] = i;
    ci[1] = P.dim == 3 ? j : pl;
    ci[2] = P.dim == 3 ? pl : 0;
  };
  if (P.kind == KFVM_IC_FOURIER || P.kind == KFVM_IC_FOURIER_SPHERE) {
    std::vector<double> pm((size_t)ng);
    for (int f = 0; f <= P.dim; ++f) {
      parallel(ng, nthreads, [&](int pl) {
        double m = 0.0;
        int ci[3];
        for (int j = 0; j < nm; ++j)
          for (int i = 0; i < P.n[0]; ++i) {
            cell(i, j, pl, ci);
            m = std::fmax(m, P.cell_max(f, ci));
          }
        pm[pl] = m;
      });
      double m = 0.0;
      for (double x : pm) m = std::fmax(m, x);
      P.norm[f] = m;
    }
  }
  const size_t plane = (size_t)P.n[0] * nm;
  parallel(nzl, nthreads, [&](int lp) {
    int ci[3];
    for (size_t c = 0; c < plane; ++c) {
      cell((int)(c % P.n[0]), (int)(c / P.n[0]), z0 + lp, ci);
      P.average(ci, U + ((size_t)lp * plane + c) * P.nv);
    }
  });
  return KFVM_OK;
}
