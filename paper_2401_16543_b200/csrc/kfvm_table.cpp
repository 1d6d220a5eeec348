// kfvm_table.cpp — one-time reconstruction-table precompute (host, binary128).
//
// Restates, generalised to 3-D, the reference's stencil geometry
// (proj/core/src/geometry.cpp:10-124), monomial basis
// (proj/core/include/kfvm/monomials.hpp:21-53) and the declared
// reconstruction-vector precompute (proj/core/include/kfvm/kernel_recon.hpp:
// 29-110; PAPER.md eqs. recVec1-recVec3, smoothIndic).
//
// Every block system [[Q^T, P],[P^T, 0]] (r; w) = (T; S) is factored once per
// (sub)stencil by partial-pivoting LU in IEEE binary128 and refined; r is then
// rounded to FP64.  FP64 solves of these systems are solver-dependent at the
// 1e-6..O(1) level for R=3 and 3-D, so this table *defines*
// the reconstruction vectors shared byte-for-byte by the GPU and the CPU
// oracle; its FNV-1a hash is recorded in the table.
#include <quadmath.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/kfvm_b200.h"

namespace kfvm_b200 {
namespace {

typedef __float128 qf;

struct Off {
  int c[3];
};

// Graded multi-indices of total degree lo..hi; in 2-D (n-k, k) for k=0..n as
// monomials.hpp:21-27, in 3-D (a, b, n-a-b) for a=n..0, b=n-a..0.
std::vector<std::array<int, 3>> graded(int dim, int lo, int hi) {
  std::vector<std::array<int, 3>> out;
  for (int n = lo; n <= hi; ++n) {
    if (dim == 2) {
      for (int k = 0; k <= n; ++k) out.push_back({n - k, k, 0});
    } else {
      for (int a = n; a >= 0; --a)
        for (int b = n - a; b >= 0; --b) out.push_back({a, b, n - a - b});
    }
  }
  return out;
}

// Full spherical stencil, lexicographic by (k, j, i) (geometry.cpp:10-20,
// PAPER.md §3.1).
std::vector<Off> full_stencil(int dim, int R) {
  std::vector<Off> s;
  const int kr = dim == 3 ? R : 0;
  for (int k = -kr; k <= kr; ++k)
    for (int j = -R; j <= R; ++j)
      for (int i = -R; i <= R; ++i)
        if (i * i + j * j + k * k <= R * R) s.push_back({{i, j, k}});
  return s;
}

// Substencil membership (geometry.cpp:22-34 in 2-D; §3.1 in 3-D).
// q = 1 central; q = 2 + 2*axis + neg is biased toward (neg ? -:+) axis.
bool in_substencil(int dim, int R, int q, const Off& o) {
  const int i = o.c[0], j = o.c[1], k = o.c[2];
  if (q == 1) return i * i + j * j + k * k <= (R - 1) * (R - 1);
  const int axis = (q - 2) / 2;
  const int sgn = ((q - 2) % 2) ? -1 : 1;
  const int a = sgn * o.c[axis];
  for (int t = 0; t < dim; ++t) {
    if (t == axis) continue;
    if (std::abs(o.c[t]) > a) return false;
  }
  return true;
}

qf mavg_1d(qf c, int k) {  // monomials.hpp:40-42
  qf hi = 1, lo = 1;
  for (int t = 0; t <= k; ++t) {
    hi *= (c + 0.5Q);
    lo *= (c - 0.5Q);
  }
  return (hi - lo) / (qf)(k + 1);
}

qf mavg_cell(int dim, const Off& o, const std::array<int, 3>& m) {  // monomials.hpp:45-47
  qf v = 1;
  for (int t = 0; t < dim; ++t) v *= mavg_1d((qf)o.c[t], m[t]);
  return v;
}

// Symmetric Jacobi eigenvalues of a small SPD matrix (binary128).
std::vector<qf> jacobi_eigs(std::vector<qf> a, int n) {
  for (int sweep = 0; sweep < 100; ++sweep) {
    qf off = 0, tot = 0;
    for (int p = 0; p < n; ++p)
      for (int q = 0; q < n; ++q) {
        tot += a[p * n + q] * a[p * n + q];
        if (p != q) off += a[p * n + q] * a[p * n + q];
      }
    if (off <= 1e-60Q * tot) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const qf apq = a[p * n + q];
        if (apq == 0) continue;
        const qf app = a[p * n + p], aqq = a[q * n + q];
        const qf theta = (aqq - app) / (2 * apq);
        const qf t = (theta >= 0 ? 1 : -1) / (fabsq(theta) + sqrtq(theta * theta + 1));
        const qf c = 1 / sqrtq(t * t + 1), s = t * c;
        for (int k = 0; k < n; ++k) {
          const qf akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = c * akp - s * akq;
          a[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const qf apk = a[p * n + k], aqk = a[q * n + k];
          a[p * n + k] = c * apk - s * aqk;
          a[q * n + k] = s * apk + c * aqk;
        }
      }
  }
  std::vector<qf> e(n);
  for (int i = 0; i < n; ++i) e[i] = a[i * n + i];
  return e;
}

// Full-column-rank test of the monomial cell-average matrix at degree p with
// the reference tolerance sigma_min > 1e-10 sigma_max (geometry.cpp:39-51),
// evaluated as lambda_min(P^T P) > 1e-20 lambda_max in binary128.
bool unisolvent(int dim, const std::vector<Off>& cells, int p) {
  const auto mono = graded(dim, 0, p);
  const int n = (int)cells.size(), d = (int)mono.size();
  if (d > n) return false;
  std::vector<qf> P((size_t)n * d), G((size_t)d * d, 0);
  for (int h = 0; h < n; ++h)
    for (int v = 0; v < d; ++v) P[h * d + v] = mavg_cell(dim, cells[h], mono[v]);
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      qf s = 0;
      for (int h = 0; h < n; ++h) s += P[h * d + a] * P[h * d + b];
      G[a * d + b] = s;
    }
  auto e = jacobi_eigs(G, d);
  qf mn = e[0], mx = e[0];
  for (qf x : e) {
    mn = x < mn ? x : mn;
    mx = x > mx ? x : mx;
  }
  return mn > 1e-20Q * mx;
}

// Gauss-Legendre rule with n points mapped to [-1/2,1/2] (geometry.cpp:74-101),
// computed by Newton iteration on P_n in binary128.
void gauss_legendre(int n, std::vector<qf>& x, std::vector<qf>& w) {
  x.assign(n, 0);
  w.assign(n, 0);
  for (int i = 0; i < n; ++i) {
    qf z = cosq(M_PIq * (i + 0.75Q) / (n + 0.5Q)), dp = 1;
    for (int it = 0; it < 200; ++it) {
      qf p0 = 1, p1 = z;  // P_0, P_1; recurrence up to P_n
      for (int k = 2; k <= n; ++k) {
        const qf p2 = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1);
      const qf dz = p1 / dp;
      z -= dz;
      if (fabsq(dz) < 1e-32Q) break;
    }
    x[n - 1 - i] = 0.5Q * z;  // ascending nodes on [-1/2, 1/2]
    w[n - 1 - i] = 0.5Q * (2 / ((1 - z * z) * dp * dp));
  }
}

// 1-D factor of the cell-averaged SE kernel (kernel_recon.hpp:32-35).
qf avg_kernel_1d(qf c, qf ell) {
  const qf s = ell * sqrtq(2.0Q);
  return ell * sqrtq(M_PIq / 2) * (erfq((c + 0.5Q) / s) - erfq((c - 0.5Q) / s));
}

// n-th derivative at x=0 of exp(-(x-c)^2/(2 ell^2)) via physicists' Hermite
// polynomials (kernel_recon.hpp:49-54).
qf gauss_deriv(int n, qf c, qf ell) {
  const qf s = ell * sqrtq(2.0Q);
  const qf u = -c / s;
  qf h0 = 1, h1 = 2 * u, hn = n == 0 ? h0 : h1;
  for (int k = 1; k < n; ++k) {
    const qf h2 = 2 * u * h1 - 2 * k * h0;
    h0 = h1;
    h1 = h2;
    hn = h2;
  }
  qf f = 1;
  for (int k = 0; k < n; ++k) f *= -1 / s;
  return f * hn * expq(-u * u);
}

struct LU {
  int n;
  std::vector<qf> a;
  std::vector<int> piv;
};

LU lu_factor(const std::vector<qf>& m, int n) {
  LU f{n, m, std::vector<int>(n)};
  auto& a = f.a;
  for (int k = 0; k < n; ++k) {
    int p = k;
    qf best = fabsq(a[k * n + k]);
    for (int i = k + 1; i < n; ++i)
      if (fabsq(a[i * n + k]) > best) {
        best = fabsq(a[i * n + k]);
        p = i;
      }
    if (best == 0) throw std::runtime_error("singular block system");
    f.piv[k] = p;
    if (p != k)
      for (int j = 0; j < n; ++j) std::swap(a[k * n + j], a[p * n + j]);
    for (int i = k + 1; i < n; ++i) {
      const qf l = a[i * n + k] / a[k * n + k];
      a[i * n + k] = l;
      if (l != 0)
        for (int j = k + 1; j < n; ++j) a[i * n + j] -= l * a[k * n + j];
    }
  }
  return f;
}

void lu_solve(const LU& f, std::vector<qf>& b) {
  const int n = f.n;
  const auto& a = f.a;
  for (int k = 0; k < n; ++k)
    if (f.piv[k] != k) std::swap(b[k], b[f.piv[k]]);
  for (int i = 1; i < n; ++i) {
    qf s = b[i];
    for (int j = 0; j < i; ++j) s -= a[i * n + j] * b[j];
    b[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    qf s = b[i];
    for (int j = i + 1; j < n; ++j) s -= a[i * n + j] * b[j];
    b[i] = s / a[i * n + i];
  }
}

// Solve M z = rhs with two refinement sweeps; returns max residual.
qf solve_refined(const std::vector<qf>& M, const LU& f, const std::vector<qf>& rhs,
                 std::vector<qf>& z) {
  const int n = f.n;
  z = rhs;
  lu_solve(f, z);
  qf res = 0;
  for (int sweep = 0; sweep < 3; ++sweep) {
    std::vector<qf> r(n);
    res = 0;
    for (int i = 0; i < n; ++i) {
      qf s = rhs[i];
      for (int j = 0; j < n; ++j) s -= M[i * n + j] * z[j];
      r[i] = s;
      res = fabsq(s) > res ? fabsq(s) : res;
    }
    if (sweep == 2) break;
    lu_solve(f, r);
    for (int i = 0; i < n; ++i) z[i] += r[i];
  }
  return res;
}

uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = (const unsigned char*)p;
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ULL;
  }
  return h;
}

// Exact symmetry of the table (kernel_recon.hpp:105-106: "symmetric vectors
// are exact permutations").  The cube's symmetry group G (signed axis
// permutations g(x)_b = s_b x_pi(b); 8 elements in 2-D, 48 in 3-D) maps every
// (sub)stencil onto a (sub)stencil, every face point onto a face point and
// every derivative d^alpha onto +-d^alpha' (alpha'_b = alpha_pi(b), sign
// prod_b s_b^alpha'_b).  The SE kernel is G-invariant, so in exact arithmetic
// r_{gS, gx}[g h] = r_{S, x}[h] and d_{gS, alpha'}[g h] = sign d_{S, alpha}[h].
// The binary128 solves satisfy this to ~1e-34; rounding a near-tie to FP64
// could still split an orbit by one ulp.  So every orbit of entries is
// replaced by its group average in binary128 (sum over g in G in a fixed
// order, divided by |G|), and the images are assigned sign * average before
// the one rounding to FP64: every mirror / rotation image is then bitwise
// equal (entries whose stabiliser flips the sign average to exactly 0).
void symmetrize(int dim, const kfvm_table& t, const std::vector<Off>& full,
                const std::vector<std::vector<int>>& members,
                const std::vector<std::array<qf, 3>>& pts,
                const std::vector<std::array<int, 3>>& alphas, std::vector<qf>& faceq,
                std::vector<qf>& derivq) {
  struct Elem {
    int perm[3], sgn[3];
  };
  std::vector<Elem> G;
  int p[3] = {0, 1, 2};
  do {
    if (dim == 2 && p[2] != 2) continue;
    for (int m = 0; m < (1 << dim); ++m) {
      Elem e{};
      for (int b = 0; b < 3; ++b) {
        e.perm[b] = p[b];
        e.sgn[b] = (b < dim && ((m >> b) & 1)) ? -1 : 1;
      }
      G.push_back(e);
    }
  } while (std::next_permutation(p, p + 3));
  const int NF = t.n_full, NS = t.n_stencils, NP = t.n_points, NA = t.n_alpha;
  auto apply = [&](const Elem& g, const Off& o) {
    Off r{{0, 0, 0}};
    for (int b = 0; b < 3; ++b) r.c[b] = g.sgn[b] * o.c[g.perm[b]];
    return r;
  };
  auto full_index = [&](const Off& o) {
    for (int h = 0; h < NF; ++h)
      if (full[h].c[0] == o.c[0] && full[h].c[1] == o.c[1] && full[h].c[2] == o.c[2]) return h;
    throw std::runtime_error("symmetry maps a stencil cell outside S0");
  };
  // per element: full-stencil cell map, stencil map, local position maps,
  // point map, derivative map and sign
  const int nG = (int)G.size();
  std::vector<int> cmap((size_t)nG * NF), qmap((size_t)nG * NS), smap((size_t)nG * NP),
      amap((size_t)nG * NA), asgn((size_t)nG * NA);
  std::vector<std::vector<int>> local(NS, std::vector<int>(NF, -1));  // S0 index -> position in S_q
  for (int q = 0; q < NS; ++q)
    for (int l = 0; l < (int)members[q].size(); ++l) local[q][members[q][l]] = l;
  for (int gi = 0; gi < nG; ++gi) {
    const Elem& g = G[gi];
    for (int h = 0; h < NF; ++h) cmap[(size_t)gi * NF + h] = full_index(apply(g, full[h]));
    for (int q = 0; q < NS; ++q) {
      std::vector<int> img;
      for (int h : members[q]) img.push_back(cmap[(size_t)gi * NF + h]);
      std::sort(img.begin(), img.end());
      int found = -1;
      for (int q2 = 0; q2 < NS && found < 0; ++q2) {
        std::vector<int> m2 = members[q2];
        std::sort(m2.begin(), m2.end());
        if (m2 == img) found = q2;
      }
      if (found < 0) throw std::runtime_error("symmetry does not map substencils onto substencils");
      qmap[(size_t)gi * NS + q] = found;
    }
    for (int s = 0; s < NP; ++s) {
      std::array<qf, 3> x{0, 0, 0};
      for (int b = 0; b < 3; ++b) x[b] = (qf)g.sgn[b] * pts[s][g.perm[b]];
      int found = -1;
      for (int s2 = 0; s2 < NP && found < 0; ++s2) {
        bool eq = true;
        for (int b = 0; b < 3; ++b) eq = eq && fabsq(pts[s2][b] - x[b]) < 1e-30Q;
        if (eq) found = s2;
      }
      if (found < 0) throw std::runtime_error("symmetry does not map face points onto face points");
      smap[(size_t)gi * NP + s] = found;
    }
    for (int a = 0; a < NA; ++a) {
      std::array<int, 3> al2{0, 0, 0};
      int sg = 1;
      for (int b = 0; b < 3; ++b) {
        al2[b] = alphas[a][g.perm[b]];
        if (g.sgn[b] < 0 && (al2[b] & 1)) sg = -sg;
      }
      int found = -1;
      for (int a2 = 0; a2 < NA && found < 0; ++a2)
        if (alphas[a2] == al2) found = a2;
      if (found < 0) throw std::runtime_error("symmetry does not map derivative indices");
      amap[(size_t)gi * NA + a] = found;
      asgn[(size_t)gi * NA + a] = sg;
    }
  }
  // orbit averages: rows of kind 0 (face points) and 1 (derivatives)
  for (int kind = 0; kind < 2; ++kind) {
    const int nr = kind ? NA : NP;
    std::vector<qf>& val = kind ? derivq : faceq;
    std::vector<char> done(val.size(), 0);
    auto at = [&](int q, int r, int l) {
      return (size_t)t.cell_offset[q] * nr + (size_t)r * t.size[q] + l;
    };
    for (int q = 0; q < NS; ++q)
      for (int r = 0; r < nr; ++r)
        for (int l = 0; l < t.size[q]; ++l) {
          if (done[at(q, r, l)]) continue;
          const int h = members[q][l];
          qf sum = 0;
          std::vector<std::pair<size_t, int>> img(nG);
          for (int gi = 0; gi < nG; ++gi) {
            const int q2 = qmap[(size_t)gi * NS + q];
            const int r2 = kind ? amap[(size_t)gi * NA + r] : smap[(size_t)gi * NP + r];
            const int sg = kind ? asgn[(size_t)gi * NA + r] : 1;
            const int l2 = local[q2][cmap[(size_t)gi * NF + h]];
            img[gi] = {at(q2, r2, l2), sg};
            sum += (qf)sg * val[img[gi].first];
          }
          // an entry its own stabiliser maps to minus itself is exactly 0
          bool odd = false;
          for (int gi = 0; gi < nG; ++gi) odd = odd || (img[gi].first == img[0].first && img[gi].second != img[0].second);
          const qf avg = odd ? (qf)0 : sum / (qf)nG;
          for (const auto& [e, sg] : img) {
            val[e] = (qf)sg * avg;
            done[e] = 1;
          }
        }
  }
}

struct TableStore {
  kfvm_table t;
  std::vector<int> offsets, gather, alpha;
  std::vector<double> face, deriv, gamma_lin, face_weights, points, gl_nodes,
      gl_weights;
};

}  // namespace

kfvm_table* build_table(int dim, int R, double ell_over_delta) {
  if ((dim != 2 && dim != 3) || (R != 2 && R != 3))
    throw std::invalid_argument("unsupported stencil radius/dimension");
  if (!(ell_over_delta > 0)) throw std::invalid_argument("ell_over_delta must be > 0");
  auto* st = new TableStore();
  kfvm_table& t = st->t;
  std::memset(&t, 0, sizeof(t));
  t.dim = dim;
  t.radius = R;
  t.n_stencils = 2 * dim + 2;
  int rp = 1;
  for (int k = 1; k < dim; ++k) rp *= R;
  t.n_points = 2 * dim * rp;
  const auto alphas = graded(dim, 1, R);  // derivative_indices (monomials.hpp:32-37)
  t.n_alpha = (int)alphas.size();
  t.ell_over_delta = ell_over_delta;
  const qf ell = (qf)ell_over_delta;

  const auto full = full_stencil(dim, R);
  t.n_full = (int)full.size();
  std::vector<std::vector<int>> members(t.n_stencils);
  for (int h = 0; h < t.n_full; ++h) members[0].push_back(h);
  for (int q = 1; q < t.n_stencils; ++q)
    for (int h = 0; h < t.n_full; ++h)
      if (in_substencil(dim, R, q, full[h])) members[q].push_back(h);

  // degrees by the rank test (geometry.cpp:55-65)
  for (int q = 0; q < t.n_stencils; ++q) {
    std::vector<Off> cells;
    for (int h : members[q]) cells.push_back(full[h]);
    int deg = 0;
    for (int p = 1; p <= 2 * R - 1; ++p) {
      if (!unisolvent(dim, cells, p)) break;
      deg = p;
    }
    t.degree[q] = deg;
    t.size[q] = (int)cells.size();
  }
  int acc = 0;
  for (int q = 0; q < t.n_stencils; ++q) {
    t.cell_offset[q] = acc;
    acc += t.size[q];
  }
  t.total_cells = acc;

  // quadrature and face points (geometry.cpp:103-115, generalised)
  std::vector<qf> gx, gw;
  gauss_legendre(R, gx, gw);
  std::vector<std::array<qf, 3>> pts;
  for (int f = 0; f < 2 * dim; ++f) {
    const int axis = f / 2;
    const qf side = (f % 2) ? 0.5Q : -0.5Q;
    int tan[2] = {-1, -1}, nt = 0;
    for (int a = 0; a < dim; ++a)
      if (a != axis) tan[nt++] = a;
    for (int m = 0; m < rp; ++m) {
      std::array<qf, 3> x = {0, 0, 0};
      x[axis] = side;
      x[tan[0]] = gx[m % R];
      if (dim == 3) x[tan[1]] = gx[m / R];
      pts.push_back(x);
      double w = (double)gw[m % R];
      if (dim == 3) w = w * (double)gw[m / R];
      st->face_weights.push_back(w);
    }
  }
  for (auto& x : pts)
    for (int a = 0; a < 3; ++a) st->points.push_back((double)x[a]);
  for (int k = 0; k < R; ++k) {
    st->gl_nodes.push_back((double)gx[k]);
    st->gl_weights.push_back((double)gw[k]);
  }

  for (const auto& o : full)
    for (int a = 0; a < 3; ++a) st->offsets.push_back(o.c[a]);
  for (int q = 0; q < t.n_stencils; ++q)
    for (int h : members[q]) st->gather.push_back(h);
  for (const auto& a : alphas)
    for (int k = 0; k < 3; ++k) st->alpha.push_back(a[k]);

  st->face.assign((size_t)t.total_cells * t.n_points, 0.0);
  st->deriv.assign((size_t)t.total_cells * t.n_alpha, 0.0);
  // binary128 solutions; rounded to FP64 after the orbit symmetrisation
  std::vector<qf> faceq((size_t)t.total_cells * t.n_points, 0), derivq((size_t)t.total_cells * t.n_alpha, 0);

  for (int q = 0; q < t.n_stencils; ++q) {
    std::vector<Off> cells;
    for (int h : members[q]) cells.push_back(full[h]);
    const int N = (int)cells.size();
    const auto mono = graded(dim, 0, t.degree[q]);
    const int D = (int)mono.size();
    const int n = N + D;
    // M = [[Q^T, P],[P^T, 0]] (kernel_recon.hpp:56-62)
    std::vector<qf> M((size_t)n * n, 0);
    for (int h = 0; h < N; ++h)
      for (int l = 0; l < N; ++l) {
        qf v = 1;  // Q_hl = prod_d avg_kernel_1d(x_h - x_l)
        for (int a = 0; a < dim; ++a)
          v *= avg_kernel_1d((qf)(cells[h].c[a] - cells[l].c[a]), ell);
        M[(size_t)l * n + h] = v;  // transposed
      }
    for (int h = 0; h < N; ++h)
      for (int v = 0; v < D; ++v) {
        const qf pv = mavg_cell(dim, cells[h], mono[v]);
        M[(size_t)h * n + N + v] = pv;
        M[(size_t)(N + v) * n + h] = pv;
      }
    const LU f = lu_factor(M, n);
    std::vector<qf> rhs(n), z;
    // point-value vectors at the face points (kernel_recon.hpp:45-47)
    for (int s = 0; s < t.n_points; ++s) {
      for (int l = 0; l < N; ++l) {
        qf v = 1;
        for (int a = 0; a < dim; ++a) {
          const qf d = pts[s][a] - (qf)cells[l].c[a];
          v *= expq(-d * d / (2 * ell * ell));
        }
        rhs[l] = v;
      }
      for (int v = 0; v < D; ++v) {
        qf m = 1;
        for (int a = 0; a < dim; ++a)
          for (int e = 0; e < mono[v][a]; ++e) m *= pts[s][a];
        rhs[N + v] = m;
      }
      const qf res = solve_refined(M, f, rhs, z);
      if (!(res < 1e-9Q)) throw std::runtime_error("block solve residual > 1e-9");
      qf* dst = faceq.data() + (size_t)t.cell_offset[q] * t.n_points + (size_t)s * N;
      for (int l = 0; l < N; ++l) dst[l] = z[l];
    }
    // derivative vectors at the cell centre (kernel_recon.hpp:49-54)
    for (int ia = 0; ia < t.n_alpha; ++ia) {
      const auto& al = alphas[ia];
      for (int l = 0; l < N; ++l) {
        qf v = 1;
        for (int a = 0; a < dim; ++a) v *= gauss_deriv(al[a], (qf)cells[l].c[a], ell);
        rhs[l] = v;
      }
      for (int v = 0; v < D; ++v) {
        qf fac = 0;
        if (mono[v] == al) {
          fac = 1;
          for (int a = 0; a < 3; ++a)
            for (int e = 2; e <= al[a]; ++e) fac *= e;
        }
        rhs[N + v] = fac;
      }
      const qf res = solve_refined(M, f, rhs, z);
      if (!(res < 1e-9Q)) throw std::runtime_error("block solve residual > 1e-9");
      qf* dst = derivq.data() + (size_t)t.cell_offset[q] * t.n_alpha + (size_t)ia * N;
      for (int l = 0; l < N; ++l) dst[l] = z[l];
    }
  }

  symmetrize(dim, t, full, members, pts, alphas, faceq, derivq);
  for (size_t i = 0; i < faceq.size(); ++i) st->face[i] = (double)faceq[i];
  for (size_t i = 0; i < derivq.size(); ++i) st->deriv[i] = (double)derivq[i];

  // WENO-AO linear weights (§3.2), evaluated in FP64 in
  // the order written there.
  const double ghi = 0.8, glo = 0.8;
  st->gamma_lin.push_back(ghi);
  st->gamma_lin.push_back((1.0 - ghi) * glo);
  for (int q = 2; q < t.n_stencils; ++q)
    st->gamma_lin.push_back((1.0 - ghi) * (1.0 - glo) / (double)(2 * dim));

  t.offsets = st->offsets.data();
  t.gather = st->gather.data();
  t.alpha = st->alpha.data();
  t.face = st->face.data();
  t.deriv = st->deriv.data();
  t.gamma_lin = st->gamma_lin.data();
  t.face_weights = st->face_weights.data();
  t.points = st->points.data();
  t.gl_nodes = st->gl_nodes.data();
  t.gl_weights = st->gl_weights.data();

  uint64_t h = 1469598103934665603ULL;
  int hdr[5] = {dim, R, t.n_full, t.n_points, t.n_alpha};
  h = fnv1a(h, hdr, sizeof(hdr));
  h = fnv1a(h, t.size, sizeof(t.size));
  h = fnv1a(h, t.degree, sizeof(t.degree));
  h = fnv1a(h, st->offsets.data(), st->offsets.size() * sizeof(int));
  h = fnv1a(h, st->gather.data(), st->gather.size() * sizeof(int));
  h = fnv1a(h, st->alpha.data(), st->alpha.size() * sizeof(int));
  h = fnv1a(h, st->face.data(), st->face.size() * sizeof(double));
  h = fnv1a(h, st->deriv.data(), st->deriv.size() * sizeof(double));
  h = fnv1a(h, st->gamma_lin.data(), st->gamma_lin.size() * sizeof(double));
  h = fnv1a(h, st->face_weights.data(), st->face_weights.size() * sizeof(double));
  h = fnv1a(h, &ell_over_delta, sizeof(double));
  t.hash = h;
  return &st->t;
}

void free_table(kfvm_table* t) {
  // kfvm_table is the first member of TableStore
  delete reinterpret_cast<TableStore*>(t);
}

}  // namespace kfvm_b200

extern "C" int kfvm_table_build(int dim, int radius, double ell_over_delta, kfvm_table** out) {
  if (!out) return KFVM_ERR_CONFIG;
  *out = nullptr;
  try {
    *out = kfvm_b200::build_table(dim, radius, ell_over_delta);
    return KFVM_OK;
  } catch (const std::invalid_argument&) {
    return KFVM_ERR_CONFIG;
  } catch (...) {
    return KFVM_ERR_RUNTIME;
  }
}

extern "C" void kfvm_table_free(kfvm_table* t) {
  if (t) kfvm_b200::free_table(t);
}
