// kfvm_ic_eval.h — pointwise evaluation of the seeded synthetic initial
// conditions of BASELINE.json configs 1-5 (product code, host + device).
//
// All transcendental work (cos/sin of the per-axis Fourier factors, exp/log of
// the Voronoi region states) is done once on the host into small tables;
// the per-point work below is IEEE add/mul/div only, so the host generator
// (compiled with -ffp-contract=off) and the device generator (nvcc
// -fmad=false) produce bit-identical cell averages.  Cell averages use the
// tensor R^d Gauss-Legendre rule from pointwise primitives (SPEC.md S:544-552,
// PAPER.md §5.2).
#ifndef KFVM_IC_EVAL_H_
#define KFVM_IC_EVAL_H_

#include <math.h>

#ifdef __CUDACC__
#define KFVM_HD __host__ __device__ __forceinline__
#else
#define KFVM_HD inline
#endif

namespace kfvm_b200 {

#define KFVM_IC_MAX_MODES 16
#define KFVM_IC_MAX_REGIONS 128

struct FourierField {
  int nm;
  int k[KFVM_IC_MAX_MODES][3];
  double a[KFVM_IC_MAX_MODES];
  double cphi[KFVM_IC_MAX_MODES], sphi[KFVM_IC_MAX_MODES];
  double norm;  // max |s_raw| over every GL point of the global grid
};

struct ICPlan {
  int kind, dim, R;
  int n[3];
  double dx, origin[3], gamma, inv_gm1;
  double node[3], w[3];
  // per-axis Fourier factors: fc[a][(k-1)*n[a]*R + i*R + q] = cos(2 pi k x)
  const double* fc[3];
  const double* fs[3];
  FourierField f[4];  // rho, u, v, w perturbation fields
  int nreg;
  double seeds[KFVM_IC_MAX_REGIONS][3];
  double reg[KFVM_IC_MAX_REGIONS][5];  // conservative state per region
  double sph_c[3], sph_r2;
  double value[5];
};

// raw Fourier sum at GL point (gi = i*R+q per axis)
KFVM_HD double fourier_raw(const ICPlan& P, const FourierField& F, const int gi[3]) {
  double acc = 0.0;
  for (int m = 0; m < F.nm; ++m) {
    double re = F.cphi[m], im = F.sphi[m];
    for (int a = 0; a < P.dim; ++a) {
      const int off = (F.k[m][a] - 1) * P.n[a] * P.R + gi[a];
      const double c = P.fc[a][off], s = P.fs[a][off];
      const double nre = re * c - im * s;
      const double nim = re * s + im * c;
      re = nre;
      im = nim;
    }
    acc = acc + F.a[m] * im;
  }
  return acc;
}

KFVM_HD double coord(const ICPlan& P, int a, int i, int q) {
  return P.origin[a] + P.dx * (((double)i + 0.5) + P.node[q]);
}

// conservative state at one GL point (2-D: z components ignored)
KFVM_HD void point_state(const ICPlan& P, const int gi[3], const int ci[3], const int qi[3],
                         double* U) {
  const int nv = P.dim + 2;
  if (P.kind == 1) {  // Voronoi: Euclidean nearest seed, no periodic images
    double x[3];
    for (int a = 0; a < P.dim; ++a) x[a] = coord(P, a, ci[a], qi[a]);
    int best = 0;
    double bd = 0.0;
    for (int r = 0; r < P.nreg; ++r) {
      double t = x[0] - P.seeds[r][0];
      double d = t * t;
      t = x[1] - P.seeds[r][1];
      d = d + t * t;
      if (P.dim == 3) {
        t = x[2] - P.seeds[r][2];
        d = d + t * t;
      }
      if (r == 0 || d < bd) {
        bd = d;
        best = r;
      }
    }
    for (int v = 0; v < nv; ++v) U[v] = P.reg[best][v];
    return;
  }
  double rho, vel[3] = {0.0, 0.0, 0.0}, p;
  if (P.kind == 3) {
    rho = P.value[0];
    vel[0] = P.value[1];
    vel[1] = P.value[2];
    vel[2] = P.value[3];
    p = P.value[4];
  } else {  // Fourier (0) / Fourier + sphere (2)
    const double base[3] = {1.0, 0.5, 0.25};
    rho = 1.0 + 0.2 * (fourier_raw(P, P.f[0], gi) / P.f[0].norm);
    for (int a = 0; a < P.dim; ++a)
      vel[a] = base[a] + 0.05 * (fourier_raw(P, P.f[1 + a], gi) / P.f[1 + a].norm);
    p = 1.0;
    if (P.kind == 2) {  // sphere, minimum-image distance on the unit cube
      double d2 = 0.0;
      for (int a = 0; a < P.dim; ++a) {
        double d = coord(P, a, ci[a], qi[a]) - P.sph_c[a];
        d = d - rint(d);
        d2 = d2 + d * d;
      }
      if (d2 < P.sph_r2) {
        rho = rho * 4.0;
        p = p * 10.0;
      }
    }
  }
  double ke = vel[0] * vel[0] + vel[1] * vel[1];
  if (P.dim == 3) ke = ke + vel[2] * vel[2];
  U[0] = rho;
  for (int a = 0; a < P.dim; ++a) U[1 + a] = rho * vel[a];
  U[nv - 1] = p * P.inv_gm1 + 0.5 * (rho * ke);
}

// cell average of cell (i,j,k) by the tensor GL rule
KFVM_HD void cell_average(const ICPlan& P, int i, int j, int k, double* out) {
  const int nv = P.dim + 2;
  for (int v = 0; v < nv; ++v) out[v] = 0.0;
  const int R = P.R;
  const int rz = P.dim == 3 ? R : 1;
  const int ci[3] = {i, j, k};
  for (int c = 0; c < rz; ++c)
    for (int b = 0; b < R; ++b)
      for (int a = 0; a < R; ++a) {
        const int qi[3] = {a, b, c};
        const int gi[3] = {i * R + a, j * R + b, k * R + c};
        double U[5];
        point_state(P, gi, ci, qi, U);
        double wgt = P.w[a] * P.w[b];
        if (P.dim == 3) wgt = wgt * P.w[c];
        for (int v = 0; v < nv; ++v) out[v] = out[v] + wgt * U[v];
      }
}

// max |s_raw| of field f over the GL points of cell (i,j,k)
KFVM_HD double cell_field_max(const ICPlan& P, const FourierField& F, int i, int j, int k) {
  const int R = P.R, rz = P.dim == 3 ? R : 1;
  double m = 0.0;
  for (int c = 0; c < rz; ++c)
    for (int b = 0; b < R; ++b)
      for (int a = 0; a < R; ++a) {
        const int gi[3] = {i * R + a, j * R + b, k * R + c};
        m = fmax(m, fabs(fourier_raw(P, F, gi)));
      }
  return m;
}

}  // namespace kfvm_b200

#endif
