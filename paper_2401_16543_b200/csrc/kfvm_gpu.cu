// kfvm_gpu.cu — B200 (sm_100a) FP64 KFVM-WENO stage update + C-ABI handle.
//
// Hot path (BASELINE.json north_star):
//   k_states  : per extended cell — stencil gather, Phi, beta_q, omega_q,
//               WENO-AO face values at every face GL point, Phi^-1,
//               positivity limiter (reconstruct_states)
//   k_flux    : per face — Riemann solve at the R^(d-1) face GL points and the
//               face quadrature
//   k_update  : per cell — flux divergence, SSP-RK3 combine, admissibility
//               check, max-wavespeed reduction for the next dt
// plus the slab-axis halo fill (fill_ghost S:553-561 / NCCL send-recv) and the
// device-resident dt.  The translation unit is compiled with -fmad=false:
// every fma below is explicit, matching the oracle's FP contract.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/kfvm_b200.h"
#include "kfvm_device.cuh"
#include "kfvm_gen.cuh"
#include "kfvm_ic_eval.h"
#include "kfvm_ic_host.h"

namespace kfvm_b200 {

#ifndef KFVM_FAST_MINB
#define KFVM_FAST_MINB 1
#endif
#ifndef KFVM_MMA_MINB
#define KFVM_MMA_MINB 3
#endif
// k_update CTAs per SM (2-D): 3 measured 0.130 vs 0.161 ms/step at 1 (config 2;
// 4: 0.128 with spills);
// 3-D keeps 1 (2.15 vs 2.97 ms/step at 4, config 3)
#ifndef KFVM_UPD_MINB2
#define KFVM_UPD_MINB2 3
#endif
#ifndef KFVM_FLUX_MINB2
#define KFVM_FLUX_MINB2 8
#endif
#ifndef KFVM_FLUX_MINB3
#define KFVM_FLUX_MINB3 4
#endif
__constant__ DevConsts c_k;
__constant__ DevTable c_t;
__constant__ int c_gather[512];

// Storage: [var][plane][mid][x] with ghost cells: H halo planes on the slab
// axis, G = H ghost columns in x and Gm (= H in 3-D, 0 in 2-D) ghost rows in
// the mid axis, filled every stage (k_ghost per boundary kind, then the
// slab-axis halo exchange of whole padded planes), so every gather is affine.
struct Geo {
  int nx, nm, np_loc, H;  // x extent, mid extent (1 in 2-D), local slab planes, halo
  int G, Gm, nxp;         // ghost columns, ghost rows, padded row length
  int xo;                 // offset of cell x = 0 in a row (>= G, 128-byte aligned)
  long long pstride;      // elements per slab-axis plane: nxp (nm + 2Gm)
  long long vstride;      // elements per variable
};

struct Chunk {
  int c0, C;              // first local plane and number of planes
  int ex, em, ep;         // extended box extents (x, mid, planes)
  long long next;         // extended cells
  int fx, fm, fp;         // face box extents
  long long nfb;          // face-box cells
  int e0, e1;             // extended planes whose states a states launch computes
};

__device__ __forceinline__ int remap(int i, int n, int periodic) {
  if (periodic) {
    // stencil offsets are at most R+1 cells beyond an edge: one conditional
    // wrap covers every grid with n >= R+1; the modulo is the rare fallback
    i = i < 0 ? i + n : (i >= n ? i - n : i);
    if ((unsigned)i >= (unsigned)n) {
      i %= n;
      i = i < 0 ? i + n : i;
    }
    return i;
  }
  return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

// Ghost-cell index map of one axis for the side's boundary kind (fill_ghost,
// S:553-561): periodic wrap, reflecting mirror image, otherwise the nearest
// interior cell (outflow; dirichlet/slit cells that take the fixed state
// ignore the source).
__device__ __forceinline__ int bc_src(int i, int n, int kind) {
  if (i >= 0 && i < n) return i;
  if (kind == KFVM_BC_PERIODIC) return remap(i, n, 1);
  if (kind == KFVM_BC_REFLECTING) return i < 0 ? -1 - i : 2 * n - 1 - i;
  return i < 0 ? 0 : n - 1;
}

// Value transform of one crossed side (physical axis a, side s) for variable
// v of the ghost cell at physical coordinates c: reflecting negates the
// wall-normal momentum, dirichlet writes the fixed state, a slit writes the
// inflow state strictly inside r^2 < radius^2.
__device__ __forceinline__ double bc_value(double u, int a, int s, int v, const int* c) {
  const int side = 2 * a + s, kind = c_k.bcs[side];
  if (kind == KFVM_BC_REFLECTING) return v == 1 + a ? -u : u;
  if (kind == KFVM_BC_DIRICHLET) return c_k.bst[side][v];
  if (kind == KFVM_BC_SLIT) {
    double r2 = 0.0;
    int m = 0;
    for (int t = 0; t < c_k.dim; ++t) {
      if (t == a) continue;
      const double d = ((double)c[t] + 0.5) * c_k.dx - c_k.slc[side][m];
      r2 = m == 0 ? d * d : r2 + d * d;
      ++m;
    }
    if (r2 < c_k.slr2[side]) return c_k.bst[side][v];
  }
  return u;
}

// value of variable v at ghost cell c (physical coordinates, extents n) from
// its source value u: the per-axis transforms composed in axis order x, y, z
__device__ __forceinline__ double bc_compose(double u, int v, const int* c, const int* n) {
  for (int a = 0; a < c_k.dim; ++a)
    if (c[a] < 0 || c[a] >= n[a]) u = bc_value(u, a, c[a] >= n[a], v, c);
  return u;
}

// padded-storage offsets of x, mid row j, local plane p (ghosts included)
__device__ __forceinline__ int xoff(const Geo& g, int x) { return x + g.xo; }
__device__ __forceinline__ long long moff(const Geo& g, int j) { return (long long)(j + g.Gm) * g.nxp; }
template <int DIM>
__device__ __forceinline__ long long uidx(const Geo& g, int x, int j, int p) {
  long long o = (long long)(p + g.H) * g.pstride + xoff(g, x);
  if (DIM == 3) o += moff(g, j);
  return o;
}

constexpr int full_size(int dim, int R) {
  return dim == 2 ? (R == 2 ? 13 : 29) : (R == 2 ? 33 : 123);
}
constexpr int npoints(int dim, int R) { return dim == 2 ? 4 * R : 6 * R * R; }

#include "kfvm_recon.cuh"
#include "kfvm_recon_u.cuh"
#include "kfvm_recon_row.cuh"
constexpr int kWideRows = 4;  // rows of cells per k_states_w CTA
#include "kfvm_recon_w.cuh"
#include "kfvm_fused3.cuh"

// ------------------------------------------------------------------ k_flux
template <int DIM>
__device__ __forceinline__ long long sidx(const Chunk& ch, int x, int j, int p) {
  // extended-cell index; p relative to the chunk's first plane
  return ((long long)(p + 1) * ch.em + (DIM == 3 ? j + 1 : 0)) * ch.ex + (x + 1);
}

// Flux of one face (Riemann solve at its R^(d-1) GL points, quadrature in
// point order): direction d, face box position (a, b, c), F index f.
template <int DIM, int R, int d>
__device__ __forceinline__ void face_flux(const double* __restrict__ St, double* __restrict__ F,
                                          const Chunk& ch, int a, int b, int c, long long f) {
  constexpr int nv = DIM + 2;
  constexpr int NP = npoints(DIM, R);
  constexpr int RP = NP / (2 * DIM);
  const bool slab = d == DIM - 1;
  const bool mid = DIM == 3 && d == 1;
  const int x = a, j = DIM == 3 ? b : 0, p = c;
  const int lx = x - (d == 0), lj = j - (mid ? 1 : 0), lp = p - (slab ? 1 : 0);
  const long long iL = sidx<DIM>(ch, lx, lj, lp);
  const long long iR = sidx<DIM>(ch, x, j, p);
  double Fb[nv];
#pragma unroll
  for (int v = 0; v < nv; ++v) Fb[v] = 0.0;
  // software-pipelined: the next point's states are in flight during this
  // point's Riemann solve (quadrature order unchanged)
  double UL[nv], UR[nv];
#pragma unroll
  for (int v = 0; v < nv; ++v) {
    UL[v] = St[(long long)(((2 * d + 1) * RP) * nv + v) * ch.next + iL];
    UR[v] = St[(long long)(((2 * d) * RP) * nv + v) * ch.next + iR];
  }
#pragma unroll
  for (int m = 0; m < RP; ++m) {
    double NL[nv], NR[nv], Fp[nv];
    if (m + 1 < RP) {
#pragma unroll
      for (int v = 0; v < nv; ++v) {
        NL[v] = St[(long long)(((2 * d + 1) * RP + m + 1) * nv + v) * ch.next + iL];
        NR[v] = St[(long long)(((2 * d) * RP + m + 1) * nv + v) * ch.next + iR];
      }
    }
    d_riemann_dir<DIM, d>(c_k, UL, UR, Fp);
#pragma unroll
    for (int v = 0; v < nv; ++v) Fb[v] = fma(c_t.face_w[(2 * d) * RP + m], Fp[v], Fb[v]);
    if (m + 1 < RP) {
#pragma unroll
      for (int v = 0; v < nv; ++v) {
        UL[v] = NL[v];
        UR[v] = NR[v];
      }
    }
  }
#pragma unroll
  for (int v = 0; v < nv; ++v) F[(long long)(d * nv + v) * ch.nfb + f] = Fb[v];
}

// one thread per face of direction d = blockIdx.y; min blocks per SM: 3-D 4
// (116-118 registers, no spills; 5 spilled 336 B at the same speed, 6 was
// slower); 2-D 8: 64 registers with 368 B (R=2) / 776 B (R=3) of spills —
// the HLLC solve alone needs more than 64 registers, and the 0-spill build
// (94 registers, 5 CTAs/SM) was slower on config 2 (1.36 vs 1.34 ms/step;
// profiles/r02/README.md)
template <int DIM, int R>
__global__ void __launch_bounds__(128, DIM == 2 ? KFVM_FLUX_MINB2 : KFVM_FLUX_MINB3) k_flux(const double* __restrict__ St,
                                                              double* __restrict__ F, Geo g,
                                                              Chunk ch) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= ch.nfb) return;
  const int d = blockIdx.y;
  const int a = (int)(tid % ch.fx);
  const long long r1 = tid / ch.fx;
  const int b = (int)(r1 % ch.fm);
  const int c = (int)(r1 / ch.fm);
  const int nm = DIM == 3 ? g.nm : 1;
  const bool slab = d == DIM - 1;
  const bool mid = DIM == 3 && d == 1;
  const bool valid = (d == 0 ? true : a < g.nx) && (mid ? true : (DIM == 3 ? b < nm : true)) &&
                     (slab ? true : c < ch.C);
  if (!valid) return;
  if (d == 0)
    face_flux<DIM, R, 0>(St, F, ch, a, b, c, tid);
  else if (d == 1)
    face_flux<DIM, R, 1>(St, F, ch, a, b, c, tid);
  else
    face_flux<DIM, R, DIM == 3 ? 2 : 1>(St, F, ch, a, b, c, tid);
}

// Fluxes of the faces on the tile edges of the fused 2-D stage kernel
// (k_stage_row): x-faces a = 32k+31 (between two x-segments) and y-faces
// c = KZ k + KZ-1 (between two row blocks); their states were stored in St.
template <int R>
__global__ void __launch_bounds__(128) k_flux_edges(const double* __restrict__ St,
                                                    double* __restrict__ F, Geo g, Chunk ch,
                                                    int KZ) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int nxb = g.nx >= 31 ? (g.nx - 31) / 32 + 1 : 0;
  const int nyb = ch.C >= KZ - 1 ? (ch.C - (KZ - 1)) / KZ + 1 : 0;
  const long long nx_faces = (long long)nxb * ch.C;
  if (tid < nx_faces) {
    const int a = 32 * (int)(tid % nxb) + 31, c = (int)(tid / nxb);
    face_flux<2, R, 0>(St, F, ch, a, 0, c, (long long)c * ch.fx + a);
  } else if (tid < nx_faces + (long long)nyb * g.nx) {
    const long long t = tid - nx_faces;
    const int a = (int)(t % g.nx), c = KZ * (int)(t / g.nx) + KZ - 1;
    face_flux<2, R, 1>(St, F, ch, a, 0, c, (long long)c * ch.fx + a);
  }
}

// ---------------------------------------------------------------- k_visc
// Viscous face flux (PAPER.md eqs nsVisc/shearTensor/thermalFlux,
// P:615-633), one thread per (face, direction) over k_flux's face box:
// F -= F^(v) with F^(v) from second-order differences of the cell-average
// primitives (k_prims' u_d, and T = gamma Ma^2 p (1/rho)), the same
// operations as the oracle's viscous_flux.
template <int DIM>
__device__ __forceinline__ void visc_prim(const double* __restrict__ Pr, long long vs, long long i,
                                          double* o) {
#pragma unroll
  for (int a = 0; a < DIM; ++a) o[a] = Pr[(3 + a) * vs + i];
  o[DIM] = c_k.gmm * (Pr[i] * Pr[2 * vs + i]);
}

template <int DIM>
__global__ void __launch_bounds__(128) k_visc(const double* __restrict__ Pr, double* __restrict__ F,
                                              Geo g, Chunk ch) {
  constexpr int nv = DIM + 2;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= ch.nfb) return;
  const int d = blockIdx.y;
  const int a = (int)(tid % ch.fx);
  const long long r1 = tid / ch.fx;
  const int b = (int)(r1 % ch.fm);
  const int c = (int)(r1 / ch.fm);
  const int nm = DIM == 3 ? g.nm : 1;
  const bool slab = d == DIM - 1;
  const bool mid = DIM == 3 && d == 1;
  const bool valid = (d == 0 ? true : a < g.nx) && (mid ? true : (DIM == 3 ? b < nm : true)) &&
                     (slab ? true : c < ch.C);
  if (!valid) return;
  // right cell (x, j, p) in local coordinates; left = right - e_d
  int cR[3] = {a, DIM == 3 ? b : 0, ch.c0 + c};
  int cL[3] = {cR[0], cR[1], cR[2]};
  const int ax = d == 0 ? 0 : (slab ? 2 : 1);  // storage axis of the normal
  cL[ax] -= 1;
  const long long vs = g.vstride;
  double L[4], R[4];
  visc_prim<DIM>(Pr, vs, uidx<DIM>(g, cL[0], cL[1], cL[2]), L);
  visc_prim<DIM>(Pr, vs, uidx<DIM>(g, cR[0], cR[1], cR[2]), R);
  double gr[4][3];  // gr[f][t]: d phi_f / d x_t (t = physical axis)
#pragma unroll
  for (int f = 0; f <= DIM; ++f) gr[f][d] = (R[f] - L[f]) / c_k.dx;
#pragma unroll
  for (int t = 0; t < DIM; ++t) {
    if (t == d) continue;
    const int tx = t == 0 ? 0 : (t == DIM - 1 ? 2 : 1);
    int o[3] = {0, 0, 0};
    o[tx] = 1;
    double Lp[4], Lm[4], Rp[4], Rm[4];
    visc_prim<DIM>(Pr, vs, uidx<DIM>(g, cL[0] + o[0], cL[1] + o[1], cL[2] + o[2]), Lp);
    visc_prim<DIM>(Pr, vs, uidx<DIM>(g, cL[0] - o[0], cL[1] - o[1], cL[2] - o[2]), Lm);
    visc_prim<DIM>(Pr, vs, uidx<DIM>(g, cR[0] + o[0], cR[1] + o[1], cR[2] + o[2]), Rp);
    visc_prim<DIM>(Pr, vs, uidx<DIM>(g, cR[0] - o[0], cR[1] - o[1], cR[2] - o[2]), Rm);
#pragma unroll
    for (int f = 0; f <= DIM; ++f) gr[f][t] = ((Lp[f] - Lm[f]) + (Rp[f] - Rm[f])) / (4.0 * c_k.dx);
  }
  double div = gr[0][0];
#pragma unroll
  for (int t = 1; t < DIM; ++t) div = div + gr[t][t];
  double sig[3];
#pragma unroll
  for (int t = 0; t < DIM; ++t) {
    double s = gr[t][d] + gr[d][t];
    if (t == d) s = fma(-2.0 / 3.0, div, s);
    sig[t] = s * c_k.inv_re;
  }
  double e = gr[DIM][d] * c_k.inv_prre;
#pragma unroll
  for (int t = 0; t < DIM; ++t) e = fma(sig[t], 0.5 * (L[t] + R[t]), e);
#pragma unroll
  for (int t = 0; t < DIM; ++t) {
    double* q = F + (long long)(d * nv + 1 + t) * ch.nfb + tid;
    *q = *q - sig[t];
  }
  double* q = F + (long long)(d * nv + nv - 1) * ch.nfb + tid;
  *q = *q - e;
}

#include "kfvm_kxrcf.cuh"

// max of non-negative doubles through their bit patterns (exact, order-free)
// over a whole block (blockDim a multiple of 32, <= 1024): one
// atomic per block instead of one per warp.  Every thread of the block must
// call it.
__device__ __forceinline__ void block_max_atomic(unsigned long long* dst, double s) {
  __shared__ unsigned long long wmax[32];
  unsigned long long v = s > 0.0 ? (unsigned long long)__double_as_longlong(s) : 0ULL;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? wmax[threadIdx.x] : 0ULL;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
      v = w > v ? w : v;
    }
    if (threadIdx.x == 0 && v) atomicMax(dst, v);
  }
}

// ---------------------------------------------------------------- k_update
// mode 0: write L(u) into Uout; mode 1..3: SSP-RK3 stage combine.
template <int DIM, bool GRAV = false>
__global__ void __launch_bounds__(256, DIM == 2 ? KFVM_UPD_MINB2 : 1) k_update(const double* __restrict__ F,
                                                const double* __restrict__ U0,
                                                const double* __restrict__ Uk,
                                                double* __restrict__ Uout, Geo g, Chunk ch,
                                                int stage, const double* __restrict__ dtp,
                                                unsigned long long* __restrict__ smax,
                                                int* __restrict__ err,
                                                double* __restrict__ Uhat = nullptr) {
  constexpr int nv = DIM + 2;
  const int nm = DIM == 3 ? g.nm : 1;
  const long long ncell = (long long)g.nx * nm * ch.C;
  const long long tid0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = tid0 < ncell;
  const long long tid = valid ? tid0 : ncell - 1;
  const int a = (int)(tid % g.nx);
  const long long r1 = tid / g.nx;
  const int b = (int)(r1 % nm);
  const int c = (int)(r1 / nm);
  const long long f0 = ((long long)c * ch.fm + (DIM == 3 ? b : 0)) * ch.fx + a;
  long long fh[3];
  fh[0] = f0 + 1;
  if (DIM == 3) {
    fh[1] = f0 + ch.fx;
    fh[2] = f0 + (long long)ch.fm * ch.fx;
  } else {
    fh[1] = f0 + (long long)ch.fm * ch.fx;
  }
  const long long ou = uidx<DIM>(g, a, b, ch.c0 + c);
  const double dt = stage ? *dtp : 0.0;
  double un[nv];
  // every load of the cell issued before any arithmetic (memory-level
  // parallelism; the operation order below is unchanged)
  double fr[DIM][nv][2], u0v[nv], ukv[nv];
#pragma unroll
  for (int v = 0; v < nv; ++v) {
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      fr[d][v][0] = F[(long long)(d * nv + v) * ch.nfb + fh[d]];
      fr[d][v][1] = F[(long long)(d * nv + v) * ch.nfb + f0];
    }
    ukv[v] = Uk[v * g.vstride + ou];
    u0v[v] = stage > 1 ? U0[v * g.vstride + ou] : ukv[v];
  }
#pragma unroll
  for (int v = 0; v < nv; ++v) {
    double acc = fr[0][v][0] - fr[0][v][1];
    acc = acc + (fr[1][v][0] - fr[1][v][1]);
    if (DIM == 3) acc = acc + (fr[DIM - 1][v][0] - fr[DIM - 1][v][1]);
    double L = -(acc / c_k.dx);
    if (GRAV) {  // gravity source from the cell average (P eq rtSource)
      if (v == 2) L = L + c_k.g2 * ukv[0];
      if (v == nv - 1) L = L + c_k.g2 * ukv[2];
    }
    if (stage == 0) {
      un[v] = L;
    } else if (stage > 10) {
      double uh = 0.0;
      un[v] = d_combine43(stage, U0[v * g.vstride + ou], ukv[v], L, dt, &uh);
      if (stage == 13 && valid) Uhat[v * g.vstride + ou] = uh;
    } else {
      un[v] = d_combine(stage, u0v[v], ukv[v], L, dt, c_k.c13, c_k.c23);
    }
    if (valid) Uout[v * g.vstride + ou] = un[v];
  }
  if (stage) {
    if (valid && !d_admissible<DIM>(c_k, un)) atomicOr(err, 2);
    if (stage == 3 && smax) block_max_atomic(smax, valid ? d_cell_speed<DIM>(c_k, un) : 0.0);
  }
}

template <int DIM>
__global__ void k_speed(const double* __restrict__ U, Geo g, unsigned long long* smax) {
  constexpr int nv = DIM + 2;
  const int nm = DIM == 3 ? g.nm : 1;
  const long long ncell = (long long)g.nx * nm * g.np_loc;
  const long long tid0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long tid = tid0 < ncell ? tid0 : ncell - 1;
  const int a = (int)(tid % g.nx);
  const long long r1 = tid / g.nx;
  const long long ou = uidx<DIM>(g, a, (int)(r1 % nm), (int)(r1 / nm));
  double u[nv];
#pragma unroll
  for (int v = 0; v < nv; ++v) u[v] = U[v * g.vstride + ou];
  block_max_atomic(smax, d_cell_speed<DIM>(c_k, u));
}

// dt = cfl*dx / smax on the device (select_dt), clipped so the
// last step lands exactly on t_end (advance_to); tt = {t, t_end}.
__global__ void k_dt(unsigned long long* smax, double* dt_cur, double* dt_seq, int* step,
                     int cap, int* err, double* tt, int* nprod) {
  const double s = __longlong_as_double((long long)*smax);
  double dt = (c_k.cfl * c_k.dx) / s;
  if (!(dt > 0.0) || !isfinite(dt)) atomicOr(err, 2);
  const double rem = tt[1] - tt[0];
  if (rem < dt) dt = rem > 0.0 ? rem : 0.0;
  tt[0] = tt[0] + dt;
  *dt_cur = dt;
  const int st = *step;
  if (st < cap) dt_seq[st] = dt;
  *step = st + 1;
  if (dt > 0.0) *nprod += 1;  // productive steps (advance_to: the clipped tail is dt = 0)
  *smax = 0ULL;
}

// slab-axis halo planes of a global end from the rank's own planes (whole
// padded planes, so the corner ghosts compose as T_slab(T_mid(T_x(U)))).
// which: bit0 = low side, bit1 = high side.
__global__ void k_halo_local(double* __restrict__ U, Geo g, int nv, int nglob, int p0, int which) {
  const long long per = (long long)g.H * g.pstride;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= 2 * per * nv) return;
  const int side = (int)(tid / (per * nv));
  if (!((which >> side) & 1)) return;
  const long long r = tid % (per * nv);
  const int v = (int)(r / per);
  const long long e = r % per;
  const int l = (int)(e / g.pstride);
  const long long o = e % g.pstride;
  const int p = side == 0 ? -g.H + l : g.np_loc + l;
  const int sa = c_k.dim - 1;
  const int src = bc_src(p0 + p, nglob, c_k.bcs[2 * sa + side]) - p0;
  int c[3], n[3];
  c[0] = (int)(o % g.nxp) - g.xo;
  n[0] = g.nx;
  c[1] = (int)(o / g.nxp) - g.Gm;  // 3-D mid row (2-D: overwritten below)
  n[1] = g.nm;
  c[sa] = p0 + p;
  n[sa] = nglob;
  const double u = U[v * g.vstride + (long long)(src + g.H) * g.pstride + o];
  U[v * g.vstride + (long long)(p + g.H) * g.pstride + o] = bc_value(u, sa, side, v, c);
}

// Ghost cells (fill_ghost) in one launch: every ghost cell of the
// padded local block — the x ghost columns and mid ghost rows of the planes
// [-hp, np + hp) and, with hp = H (one rank), the interior block of the
// slab-axis halo planes — gets the value of the cell its boundary kinds map
// to, the index maps and value transforms composed over the axes in order
// x, mid, slab (bc_src / bc_compose: periodic wrap, outflow clamp,
// reflecting mirror with the normal momentum negated, dirichlet / slit
// inflow states).  With
// several ranks (hp = 0) the halo planes are exchanged afterwards as whole
// padded planes.
__global__ void k_ghost(double* __restrict__ U, Geo g, int nv, int nsa, int p0, int hp) {
  const int P = g.np_loc + 2 * hp, rows = g.nm + 2 * g.Gm;
  const long long nA = 2LL * g.G * rows * P, nB = 2LL * g.Gm * g.nx * P,
                  nC = 2LL * hp * g.nm * g.nx, n = nA + nB + nC;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * nv) return;
  const int v = (int)(t / n);
  long long e = t % n;
  int x, j, p;
  if (e < nA) {  // x ghost columns, every row and plane
    const int gi = (int)(e % (2 * g.G));
    e /= 2 * g.G;
    x = gi < g.G ? gi - g.G : g.nx + gi - g.G;
    j = (int)(e % rows) - g.Gm;
    p = (int)(e / rows) - hp;
  } else if ((e -= nA) < nB) {  // mid ghost rows, interior columns
    x = (int)(e % g.nx);
    e /= g.nx;
    const int gj = (int)(e % (2 * g.Gm));
    j = gj < g.Gm ? gj - g.Gm : g.nm + gj - g.Gm;
    p = (int)(e / (2 * g.Gm)) - hp;
  } else {  // halo planes, interior block
    e -= nB;
    x = (int)(e % g.nx);
    e /= g.nx;
    j = (int)(e % g.nm);
    const int l = (int)(e / g.nm);
    p = l < hp ? l - hp : g.np_loc + l - hp;
  }
  // physical coordinates and extents (the slab axis is y in 2-D, z in 3-D)
  const int sa = c_k.dim - 1;
  int c[3], ext[3];
  c[0] = x;
  ext[0] = g.nx;
  if (sa == 2) {
    c[1] = j;
    ext[1] = g.nm;
  }
  c[sa] = p0 + p;
  ext[sa] = nsa;
  const int xs = bc_src(x, g.nx, c_k.bcs[x < 0 ? 0 : 1]);
  const int js = g.Gm ? bc_src(j, g.nm, c_k.bcs[j < 0 ? 2 : 3]) : j;
  const int ps = hp ? bc_src(p, nsa, c_k.bcs[2 * sa + (p < 0 ? 0 : 1)]) : p;
  const long long vb = v * g.vstride;
  const double u = U[vb + (long long)(ps + g.H) * g.pstride + moff(g, js) + xoff(g, xs)];
  U[vb + (long long)(p + g.H) * g.pstride + moff(g, j) + xoff(g, x)] = bc_compose(u, v, c, ext);
}

// AoS (host order) <-> SoA interior planes
template <int DIR>
__global__ void k_transpose(double* __restrict__ soa, double* __restrict__ aos, Geo g, int nv) {
  const long long n = (long long)g.nx * g.nm * g.np_loc;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n * nv) return;
  const long long c = tid / nv;
  const int v = (int)(tid % nv);
  const long long r1 = c / g.nx;
  const long long o = (long long)((int)(r1 / g.nm) + g.H) * g.pstride + moff(g, (int)(r1 % g.nm)) +
                      xoff(g, (int)(c % g.nx));
  if (DIR == 0)
    soa[v * g.vstride + o] = aos[tid];
  else
    aos[tid] = soa[v * g.vstride + o];
}

// states of interior cells [cell][s][v] from the extended-box St
template <int DIM>
__global__ void k_extract_states(const double* __restrict__ St, double* __restrict__ out, Geo g,
                                 Chunk ch, int NP) {
  constexpr int nv = DIM + 2;
  const int nm = DIM == 3 ? g.nm : 1;
  const long long ncell = (long long)g.nx * nm * ch.C;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= ncell * NP * nv) return;
  const long long cell = tid / (NP * nv);
  const int sv = (int)(tid % (NP * nv));
  const int a = (int)(cell % g.nx);
  const long long r1 = cell / g.nx;
  const int b = (int)(r1 % nm);
  const int c = (int)(r1 / nm);
  out[tid] = St[(long long)sv * ch.next + sidx<DIM>(ch, a, DIM == 3 ? b : 0, c)];
}

// GPU IC generator (same arithmetic as the host generator)
__global__ void k_ic_norm(const ICPlan* P, int f, Geo g, int p0, unsigned long long* out) {
  const int nm = P->dim == 3 ? g.nm : 1;
  const long long n = (long long)g.nx * nm * P->n[P->dim - 1];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n) return;
  const int i = (int)(tid % g.nx);
  const long long r = tid / g.nx;
  const int b = (int)(r % nm);
  const int pl = (int)(r / nm);
  const double m = P->dim == 3 ? cell_field_max(*P, P->f[f], i, b, pl)
                               : cell_field_max(*P, P->f[f], i, pl, 0);
  if (m > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__global__ void k_ic_fill(const ICPlan* P, double* U, Geo g, int p0) {
  const int nm = P->dim == 3 ? g.nm : 1;
  const long long n = (long long)g.nx * nm * g.np_loc;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n) return;
  const int i = (int)(tid % g.nx);
  const long long r = tid / g.nx;
  const int b = (int)(r % nm);
  const int pl = (int)(r / nm);
  double out[5];
  if (P->dim == 3)
    cell_average(*P, i, b, p0 + pl, out);
  else
    cell_average(*P, i, p0 + pl, 0, out);
  const long long o = (long long)(pl + g.H) * g.pstride + moff(g, b) + xoff(g, i);
  for (int v = 0; v < P->dim + 2; ++v) U[v * g.vstride + o] = out[v];
}

}  // namespace kfvm_b200

using namespace kfvm_b200;

// ------------------------------------------------------------------- NCCL
namespace {
typedef struct {
  char internal[128];
} nccl_uid;
typedef void* nccl_comm;
struct NcclApi {
  bool ok = false;
  int (*GetUniqueId)(nccl_uid*);
  int (*CommInitRank)(nccl_comm*, int, nccl_uid, int);
  int (*CommDestroy)(nccl_comm);
  int (*Send)(const void*, size_t, int, int, nccl_comm, cudaStream_t);
  int (*Recv)(void*, size_t, int, int, nccl_comm, cudaStream_t);
  int (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t);
  int (*AllGather)(const void*, void*, size_t, int, nccl_comm, cudaStream_t);
  int (*GroupStart)();
  int (*GroupEnd)();
};
NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  const char* env = getenv("KFVM_NCCL_LIB");
  void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.GetUniqueId = (int (*)(nccl_uid*))dlsym(h, "ncclGetUniqueId");
  api.CommInitRank = (int (*)(nccl_comm*, int, nccl_uid, int))dlsym(h, "ncclCommInitRank");
  api.CommDestroy = (int (*)(nccl_comm))dlsym(h, "ncclCommDestroy");
  api.Send = (int (*)(const void*, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclSend");
  api.Recv = (int (*)(void*, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclRecv");
  api.AllReduce = (int (*)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t))dlsym(
      h, "ncclAllReduce");
  api.AllGather = (int (*)(const void*, void*, size_t, int, nccl_comm, cudaStream_t))dlsym(
      h, "ncclAllGather");
  api.GroupStart = (int (*)())dlsym(h, "ncclGroupStart");
  api.GroupEnd = (int (*)())dlsym(h, "ncclGroupEnd");
  api.ok = api.GetUniqueId && api.CommInitRank && api.Send && api.Recv && api.AllReduce &&
           api.AllGather &&
           api.GroupStart && api.GroupEnd && api.CommDestroy;
  return api;
}
const int kNcclUint8 = 1;   // ncclUint8
const int kNcclUint64 = 5;  // ncclUint64
const int kNcclDouble = 8;  // ncclFloat64
const int kNcclMax = 2;     // ncclMax
}  // namespace

#include "kfvm_loopback.cuh"

// SSP(4,3) controller state (device)
struct Ctl {
  double t, t_final, dt_err, err_prev, err;
  int nacc, nrej, accept, done, abort;
};

struct kfvm_handle {
  kfvm_config cfg{};
  DevConsts kc{};
  DevTable tab{};
  std::vector<int> gather;
  int dim = 0, R = 0, nv = 0, NP = 0;
  int nsa = 0, p0 = 0, rank = 0, nranks = 1, device = 0;
  // the NCCL slab path is on: several ranks, or KFVM_FORCE_NCCL=1 on one rank
  // (a one-rank communicator with self send/recv: exercises the multi-GPU
  // code path on a single GPU)
  bool multi = false;
  Geo g{};
  double *U0 = nullptr, *Ua = nullptr, *Ub = nullptr;
  double* Pr = nullptr;  // k_prims output: p, c, 1/rho, u_d per cell (incl. halos)
  double *St = nullptr, *F = nullptr, *aos = nullptr;
  double* Lb = nullptr;  // 3-D R=2 tensor engine: limiter bounds [3][extended cell] (inside St)
  CUtensorMap* d_tmap = nullptr;  // 3-D R=2: TMA maps of U0, Ua, Ub (ring-plane boxes)
  CUtensorMap* d_tmapw = nullptr; // ... with the 16-warp engine's box (k_states_w: 2R+4 rows)
  int* d_gatw = nullptr;          // k_states_w's slot tables
  int wide = 1;                   // 3-D R=2: the 16-warp W-cache engine where its TMA boxes apply
  int kz_auto = 1;                // 3-D tensor engines: shorter z blocks on small grids (no kz option set)
  int num_sm = 148;
  int bounds_z = 1;               // 3-D R=2: k_bounds_z (plane-marching) instead of k_bounds
  int tma = 1;                    // option "tma": ring planes by TMA when the segments allow
  int ring_tiles = 1;             // option "ring_tiles": ring columns on the tensor engine
  size_t st_elems = 0, f_elems = 0, aos_elems = 0;
  int chunk = 0;
  int ring_split = 1;  // option "ring_split": ring columns by k_states_fast
  int *d_gather = nullptr;
  double *d_face = nullptr, *d_deriv = nullptr;
  double *d_dt_seq = nullptr, *d_dt_cur = nullptr;
  int dt_cap = 0;
  unsigned long long* d_smax = nullptr;
  double* d_tt = nullptr;  // {t, t_end} for advance_to
  int *d_step = nullptr, *d_err = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t s_halo = nullptr;     // halo exchange, overlapped with interior planes
  cudaEvent_t ev_fork = nullptr, ev_halo = nullptr;
  int overlap = 0;                   // split each stage into interior / border planes
  cudaGraphExec_t graph = nullptr;
  bool timing = false;
  bool fast = true;
  // 0 generic (k_states), 1 unrolled DFMA (k_states_fast), 2 tensor core (k_states_u),
  // 3 fused 2-D stage, 4 row-marching DFMA (2-D), 5 fused 3-D stage (k_fused3)
  int engine = 2;
  int kz = 16;     // planes marched by one k_states_u CTA
  bool visc = false;  // Navier-Stokes fluxes (k_visc after the face fluxes)
  bool grav = false;  // gravity source in k_update
  double *d_Bd = nullptr, *d_Bf = nullptr;
  int* d_gat4 = nullptr;
  int* d_gat4c = nullptr;   // 3-D R=2: the chunk tables for the ring-column tiles ([36 rows][5 cols])
  int* d_gat8 = nullptr;    // chunk tables of the fused 3-D engine's 8x4 tile
  double* d_edges = nullptr;  // tile-edge face states of the fused 3-D engine
  size_t edge_elems = 0;
  Edges eds{};
  cudaEvent_t ev[2];
  double t_states = 0, t_flux = 0, t_update = 0, t_other = 0;
  nccl_comm comm = nullptr;
  // in-process loopback transport (kfvm_loopback_id): the ranks' handles
  // live in one process on one device and exchange by device copies
  kfvm_loop::Group* loop = nullptr;
  unsigned long long loop_key = 0;
  long long loop_op = -1;
  std::vector<kfvm_loop::Pending> pend;
  long long launches = 0;
  long long graph_launches = 0;
  long long st_budget = 16LL << 30;
  int integrator = KFVM_SSPRK3;
  double* Uh = nullptr;               // SSP(4,3): embedded SSP(3,2) solution
  double* d_rows = nullptr;           // error-norm row partials [plane][row]
  double* d_planes = nullptr;         // plane partials, [rank][npmax] after the gather
  int npmax = 0;
  struct Ctl* d_ctl = nullptr;        // controller state on the device
  int* d_nps = nullptr;               // planes per rank
  cudaGraphExec_t graph43 = nullptr;
  int nacc43 = 0, nrej43 = 0;
  long long graph43_launches = 0;
  bool kx = false;                    // KXRCF two-pass reconstruction
  bool registered = false;            // holds a reference on the device constant image
  double* ext = nullptr;              // kfvm_gpu_states staging buffer
  size_t ext_elems = 0;
  unsigned char* d_flags = nullptr;   // KXRCF flags of the extended box
  std::string err;
};

namespace {

int fail(kfvm_handle* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  return code;
}

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      return fail(h, KFVM_ERR_DEVICE, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)

// Slab-exchange transport: NCCL (one process per GPU) or the in-process
// loopback group; point-to-point transfers are byte counts.
int tx_start(kfvm_handle* h) {
  if (h->loop) {
    h->pend.clear();
    return 0;
  }
  return nccl().GroupStart();
}
int tx_send(kfvm_handle* h, const void* p, size_t bytes, int peer, cudaStream_t st) {
  if (h->loop) {
    h->pend.push_back({true, const_cast<void*>(p), bytes, peer, st});
    return 0;
  }
  return nccl().Send(p, bytes, kNcclUint8, peer, h->comm, st);
}
int tx_recv(kfvm_handle* h, void* p, size_t bytes, int peer, cudaStream_t st) {
  if (h->loop) {
    h->pend.push_back({false, p, bytes, peer, st});
    return 0;
  }
  return nccl().Recv(p, bytes, kNcclUint8, peer, h->comm, st);
}
int tx_end(kfvm_handle* h) {
  if (h->loop) {
    const int rc = kfvm_loop::group_end(h->loop, h->rank, h->pend);
    h->pend.clear();
    return rc;
  }
  return nccl().GroupEnd();
}
int tx_allreduce_max_u64(kfvm_handle* h, unsigned long long* p, cudaStream_t st) {
  if (h->loop) {
    h->launches++;
    return kfvm_loop::allreduce_max_u64(h->loop, h->rank, h->loop_op, p, st);
  }
  return nccl().AllReduce(p, p, 1, kNcclUint64, kNcclMax, h->comm, st);
}
int tx_allgather_f64(kfvm_handle* h, const double* src, double* dst, size_t count,
                     cudaStream_t st) {
  if (h->loop) return kfvm_loop::allgather_f64(h->loop, h->rank, h->loop_op, src, dst, count, st);
  return nccl().AllGather(src, dst, count, kNcclDouble, h->comm, st);
}

// The constant banks (c_k, c_t, c_gather and the generated weight arrays of
// kfvm_gen.cuh) are per device and shared by every handle on it.  A handle
// may only be created when its constant image equals that of the live
// handles on the same device (otherwise KFVM_ERR_CONFIG: two different
// configurations would silently run with the last one's constants); the
// device copy of the table that c_t points to is owned by this registry and
// freed with the last handle of the device.
struct DeviceImage {
  int users = 0;
  DevConsts k{};
  DevTable t{};
  std::vector<int> gather;
  uint64_t hash = 0;
  double *d_face = nullptr, *d_deriv = nullptr;
};
std::mutex g_image_mu;
std::map<int, DeviceImage> g_images;
thread_local std::string g_create_err;  // kfvm_gpu_last_error(NULL) after a failed create

inline unsigned blocks(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }
// extended cells of the planes [e0, e1) a states launch covers
inline long long ext_range(const Chunk& ch) { return (long long)ch.ex * ch.em * (ch.e1 - ch.e0); }

Chunk make_chunk(const kfvm_handle* h, int c0, int C) {
  Chunk ch;
  ch.c0 = c0;
  ch.C = C;
  ch.ex = h->g.nx + 2;
  ch.em = h->dim == 3 ? h->g.nm + 2 : 1;
  ch.ep = C + 2;
  ch.e0 = 0;
  ch.e1 = ch.ep;
  ch.next = (long long)ch.ex * ch.em * ch.ep;
  ch.fx = h->g.nx + 1;
  ch.fm = h->dim == 3 ? h->g.nm + 1 : 1;
  ch.fp = C + 1;
  ch.nfb = (long long)ch.fx * ch.fm * ch.fp;
  return ch;
}

void tic(kfvm_handle* h) {
  if (h->timing) cudaEventRecord(h->ev[0], h->stream);
}
void toc(kfvm_handle* h, double* acc) {
  if (!h->timing) return;
  cudaEventRecord(h->ev[1], h->stream);
  cudaEventSynchronize(h->ev[1]);
  float ms = 0;
  cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]);
  *acc += ms;
}

// KFVM_DEBUG_SYNC=1: synchronise after each launch outside graph capture and
// report the first failing kernel (debugging aid; off by default)
void dbg_sync(kfvm_handle* h, const char* what) {
  static const bool on = getenv("KFVM_DEBUG_SYNC") != nullptr;
  if (!on) return;
  cudaStreamCaptureStatus cs;
  cudaStreamIsCapturing(h->stream, &cs);
  if (cs != cudaStreamCaptureStatusNone) return;
  const cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) fprintf(stderr, "[kfvm] %s: %s\n", what, cudaGetErrorString(e));
}

// Periodic x: the extended box's two ring columns are periodic images of
// the interior columns x = nx-1 and x = 0 (their stencil neighbourhoods,
// ghost cells included, hold the same values), so their face states are the
// images' face states, copied instead of recomputed (bit-identical).
__global__ void k_ring_copy(double* __restrict__ St, Chunk ch, int nkv) {
  const long long n = 2LL * ch.em * (ch.e1 - ch.e0);
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * nkv) return;
  const int k = (int)(t / n);
  const long long r = t % n;
  const int side = (int)(r & 1);
  const long long rb = r >> 1;  // (plane, row)
  const int b = (int)(rb % ch.em), c = ch.e0 + (int)(rb / ch.em);
  const long long row = ((long long)c * ch.em + b) * ch.ex;
  const long long dst = row + (side ? ch.ex - 1 : 0), src = row + (side ? 1 : ch.ex - 2);
  St[(long long)k * ch.next + dst] = St[(long long)k * ch.next + src];
}

template <int DIM, int R>
void launch_states(kfvm_handle* h, const double* U, const Chunk& ch) {
  tic(h);
  const unsigned char* kfl = h->kx ? h->d_flags : nullptr;
  if (kfl) {  // KXRCF: flagged cells only, unlimited states (engines 4, 2, 0)
    const int eng = DIM == 2 ? (h->engine == 0 ? 0 : 4) : (h->engine == 0 ? 0 : 2);
    if constexpr (DIM == 2) {
      if (eng == 4) {
        const int KZ = h->kz;
        const long long nb = (long long)((ch.ex + 31) / 32) * ((ch.e1 - ch.e0 + KZ - 1) / KZ);
        k_stage_row<R, false, true><<<(unsigned)nb, 128, 0, h->stream>>>(
            U, h->Pr, h->St, h->F, h->g, ch, KZ, h->d_err, kfl);
      }
    } else {
      if (eng == 2) {
        const int KZ = h->kz;
        const long long nb =
            (long long)((ch.ex + 31) / 32) * ch.em * ((ch.e1 - ch.e0 + KZ - 1) / KZ);
        k_states_u<DIM, R, false, true><<<(unsigned)nb, 128, UCfg<DIM, R>::bytes(), h->stream>>>(
            U, h->Pr, h->St, h->g, ch, KZ, h->d_err, h->d_Bd, h->d_Bf, h->d_gat4, kfl);
      }
    }
    if (eng == 0)
      k_states<DIM, R><<<blocks(ext_range(ch), 128), 128, 0, h->stream>>>(U, h->Pr, h->St, h->g,
                                                                          ch, h->d_err, kfl);
    h->launches++;
    if (eng != 4) {  // the 2-D row engine limits every cell itself
      k_limit_states<DIM, R><<<blocks(ext_range(ch), 128), 128, 0, h->stream>>>(U, h->Pr, h->St,
                                                                              h->g, ch, h->d_err);
      h->launches++;
    }
    toc(h, &h->t_states);
    return;
  }
  if constexpr (DIM == 2) {
    if (h->engine == 3) {
      // fused states + interior face fluxes, then the tile-edge faces
      const int KZ = h->kz;
      const long long nblk3 = (long long)((ch.ex + 31) / 32) * ((ch.ep + KZ - 1) / KZ);
      k_stage_row<R, true><<<(unsigned)nblk3, 128, 0, h->stream>>>(U, h->Pr, h->St, h->F, h->g,
                                                                   ch, KZ, h->d_err);
      dbg_sync(h, "k_stage_row");
      h->launches++;
      toc(h, &h->t_states);
      tic(h);
      const long long nxb = h->g.nx >= 31 ? (h->g.nx - 31) / 32 + 1 : 0;
      const long long nyb = ch.C >= KZ - 1 ? (ch.C - (KZ - 1)) / KZ + 1 : 0;
      const long long ne = nxb * ch.C + nyb * h->g.nx;
      if (ne > 0) {
        k_flux_edges<R><<<blocks(ne, 128), 128, 0, h->stream>>>(h->St, h->F, h->g, ch, KZ);
        dbg_sync(h, "k_flux_edges");
        h->launches++;
      }
      toc(h, &h->t_flux);
      return;
    }
  }
  // ring split: when the two ring columns of the extended box would cost a
  // mostly-empty last 32-cell segment (e.g. 258 = 8 x 32 + 2 at 256^3), the
  // segment engines cover the interior x range and the unrolled DFMA engine
  // computes the ring columns (same bits: every engine runs the pinned
  // contract)
  // (3-D only: in 2-D the ring columns are ~2k cells, a 65-CTA launch whose
  // latency (13 us) exceeds the saved segment (10 us), measured config 2)
  // periodic x (engine 2): the ring columns are copies of their periodic
  // images (k_ring_copy), so the segments always cover interior x only
  const bool ringcopy = DIM == 3 && h->engine == 2 && h->kc.per[0] != 0 && h->ring_split;
  const int xsp = (ringcopy || (DIM == 3 && Gen<DIM, R>::UNROLLED && h->ring_split &&
                                (ch.ex - 2 + 31) / 32 < (ch.ex + 31) / 32)) ? 1 : 0;
  auto ring = [&]() {
    if (!xsp) return;
    if (ringcopy) {
      const long long n = 2LL * ch.em * (ch.e1 - ch.e0) * h->NP * h->nv;
      k_ring_copy<<<blocks(n, 256), 256, 0, h->stream>>>(h->St, ch, h->NP * h->nv);
      h->launches++;
      return;
    }
    if constexpr (DIM == 3 && R == 2) {
      if (h->engine == 2 && h->d_gat4c && h->ring_tiles) {  // ring columns on the tensor engine
        // few tiles (2 columns x mid/32): short z blocks for enough CTAs
        const int KZ = h->ring_tiles > 1 ? h->ring_tiles : 4;
        const long long nb = 2LL * ((ch.em + 31) / 32) * ((ch.e1 - ch.e0 + KZ - 1) / KZ);
        k_states_u<3, 2, false, false, true><<<(unsigned)nb, 128, UCfg<3, 2>::bytes(true),
                                                 h->stream>>>(
            U, h->Pr, h->St, h->g, ch, KZ, h->d_err, h->d_Bd, h->d_Bf, h->d_gat4c, nullptr, 1,
            h->Lb, nullptr);
        h->launches++;
        return;
      }
    }
    const long long nr = 2LL * ch.em * (ch.e1 - ch.e0);
    if constexpr (Gen<DIM, R>::UNROLLED)
      k_states_fast<DIM, R, true><<<(unsigned)((nr + 31) / 32), 32 * (DIM + 2), 0, h->stream>>>(
          U, h->Pr, h->St, h->g, ch, h->d_err);
    h->launches++;
  };
  if constexpr (DIM == 2) {
    if (h->engine == 4) {
      const int KZ = h->kz;
      const long long nblk4 =
          (long long)((ch.ex - 2 * xsp + 31) / 32) * ((ch.e1 - ch.e0 + KZ - 1) / KZ);
      k_stage_row<R, false><<<(unsigned)nblk4, 128, 0, h->stream>>>(U, h->Pr, h->St, h->F, h->g,
                                                                    ch, KZ, h->d_err, nullptr, xsp);
      h->launches++;
      ring();
      toc(h, &h->t_states);
      return;
    }
  }
  if (h->engine == 2) {
    constexpr bool LB = DIM == 3 && R == 2;
    const int ui = U == h->U0 ? 0 : (U == h->Ua ? 1 : (U == h->Ub ? 2 : -1));
    bool wide = false;
    if constexpr (LB) wide = h->tma && h->wide && h->d_tmapw && h->d_gatw && ui >= 0;
    // planes one CTA marches: kz (32), fewer on small grids so that the launch
    // still has ~60 waves of CTAs (measured: 64^3 4.97 -> 3.1 ms/step, 128^3
    // 16.3 -> 15.4, 256^3 103.3 -> 102.2, R=3 128^3 79.2 -> 75.6; >= 8: the
    // ring fill per CTA); an explicit kz option is taken as given
    int KZ = h->kz;
    if (DIM == 3 && h->kz_auto) {
      const long long per = (long long)((ch.ex - 2 * xsp + 31) / 32) *
                            (wide ? (ch.em + kWideRows - 1) / kWideRows : ch.em);
      const long long slots = (long long)h->num_sm * (wide ? 1 : UCfg<DIM, R>::MINB);
      const long long k = (ch.e1 - ch.e0) * per / (60 * slots);
      KZ = (int)std::max<long long>(std::min<long long>(8, h->kz), std::min<long long>(k, h->kz));
    }
    const long long nblk2 =
        (long long)((ch.ex - 2 * xsp + 31) / 32) * ch.em * ((ch.e1 - ch.e0 + KZ - 1) / KZ);
    if (LB) {
      if (h->bounds_z) {  // warps march the planes (a third of the L2 reads)
        const long long nw = (long long)((ch.ex + 29) / 30) * ch.em *
                             ((ch.e1 - ch.e0 + kBoundsKB - 1) / kBoundsKB);
        k_bounds_z<<<(unsigned)((nw + 3) / 4), 128, 0, h->stream>>>(U, h->Pr, h->Lb, h->g, ch, h->d_err);
      } else {
        const long long nw = (long long)((ch.ex + 29) / 30) * ch.em * (ch.e1 - ch.e0);
        k_bounds<3><<<(unsigned)((nw + 3) / 4), 128, 0, h->stream>>>(U, h->Pr, h->Lb, h->g, ch,
                                                                    h->d_err);
      }
      h->launches++;
    }
    // ring planes by TMA: k_states_u needs segments that start on an even x
    // (ring split); k_states_w's wider rows take either parity
    const CUtensorMap* tm = nullptr;
    if (LB && xsp && h->tma && h->d_tmap && ui >= 0) tm = h->d_tmap + ui;
    if constexpr (LB) {
      if (wide) {  // the 16-warp W-cache engine
        const long long nbw = (long long)((ch.ex - 2 * xsp + 31) / 32) *
                              ((ch.em + kWideRows - 1) / kWideRows) * ((ch.e1 - ch.e0 + KZ - 1) / KZ);
        if (xsp)
          k_states_w<kWideRows, 0><<<(unsigned)nbw, 128 * kWideRows, WCfg<kWideRows>::bytes(), h->stream>>>(
              h->Pr, h->St, h->g, ch, KZ, h->d_Bd, h->d_Bf, h->d_gatw, xsp, h->Lb, h->d_tmapw + ui);
        else  // segments start at x = -1: the box one column earlier
          k_states_w<kWideRows, 1><<<(unsigned)nbw, 128 * kWideRows, WCfg<kWideRows>::bytes(), h->stream>>>(
              h->Pr, h->St, h->g, ch, KZ, h->d_Bd, h->d_Bf, h->d_gatw, xsp, h->Lb, h->d_tmapw + ui);
      }
    }
    if (!wide)
    k_states_u<DIM, R><<<(unsigned)nblk2, 128, UCfg<DIM, R>::bytes(LB, UCfg<DIM, R>::TGM), h->stream>>>(
        U, h->Pr, h->St, h->g, ch, KZ, h->d_err, h->d_Bd, h->d_Bf, h->d_gat4, nullptr, xsp, h->Lb, tm);
    ring();
    dbg_sync(h, "k_states_u");
    if (UCfg<DIM, R>::NG > 1) {  // (the ring copies above precede the limiter)
      h->launches++;
      k_limit_states<DIM, R><<<blocks(ext_range(ch), 128), 128, 0, h->stream>>>(U, h->Pr, h->St, h->g, ch,
                                                                          h->d_err);
      dbg_sync(h, "k_limit_states");
    }
  } else if constexpr (Gen<DIM, R>::UNROLLED) {
    if (h->engine == 1) {
      const long long nblk = (long long)((ch.ex + 31) / 32) * ch.em * (ch.e1 - ch.e0);
      k_states_fast<DIM, R><<<(unsigned)nblk, 32 * (DIM + 2), 0, h->stream>>>(U, h->Pr, h->St, h->g,
                                                                            ch, h->d_err);
    } else {
      k_states<DIM, R><<<blocks(ext_range(ch), 128), 128, 0, h->stream>>>(U, h->Pr, h->St, h->g,
                                                                          ch, h->d_err);
    }
  } else {
    k_states<DIM, R><<<blocks(ext_range(ch), 128), 128, 0, h->stream>>>(U, h->Pr, h->St, h->g,
                                                                        ch, h->d_err);
  }
  h->launches++;
  toc(h, &h->t_states);
}

template <int DIM, int R>
void launch_flux(kfvm_handle* h, const Chunk& ch) {
  tic(h);
  k_flux<DIM, R><<<dim3((unsigned)blocks(ch.nfb, 128), DIM), 128, 0, h->stream>>>(h->St, h->F,
                                                                                 h->g, ch);
  h->launches++;
  toc(h, &h->t_flux);
}

// the fused 3-D stage engine (k_fused3 + k_edges3): no face-state scratch
bool fused3(const kfvm_handle* h) { return h->dim == 3 && h->R == 2 && h->engine == 5 && !h->kx; }

// z-block layout of the stage's fused launches: disjoint plane ranges of the
// extended box, sorted by their first plane
void set_ranges(kfvm_handle* h, int n, const int* r0, const int* r1) {
  Edges& E = h->eds;
  E.nr = n;
  for (int i = 0; i < n; ++i) {
    E.r0[i] = r0[i];
    E.r1[i] = r1[i];
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (E.r0[j] < E.r0[i]) {
        std::swap(E.r0[i], E.r0[j]);
        std::swap(E.r1[i], E.r1[j]);
      }
  int nb = 0;
  for (int i = 0; i < n; ++i) nb += edge_nblocks(E, i);
  E.nzs = nb - 1;
}

void launch_fused3(kfvm_handle* h, const double* U, const Chunk& ch) {
  tic(h);
  int rr = -1;
  for (int i = 0; i < h->eds.nr; ++i)
    if (h->eds.r0[i] == ch.e0 && h->eds.r1[i] == ch.e1) rr = i;
  if (rr < 0) {  // a plane range outside the stage's layout: a programming error
    fprintf(stderr, "kfvm: fused 3-D launch over an unregistered plane range\n");
    abort();
  }
  const long long ntx = (ch.ex + kTX - 1) / kTX, nty = (ch.em + kTY - 1) / kTY;
  const long long nb = ntx * nty * edge_nblocks(h->eds, rr);
  k_fused3<2><<<(unsigned)nb, 128, FCfg<2>::bytes(), h->stream>>>(
      U, h->Pr, h->F, h->g, ch, h->eds, rr, h->d_err, h->d_Bd, h->d_Bf, h->d_gat8);
  dbg_sync(h, "k_fused3");
  h->launches++;
  toc(h, &h->t_states);
}

void launch_edges3(kfvm_handle* h, const Chunk& ch) {
  tic(h);
  const Edges& E = h->eds;
  const long long n = (long long)E.nxe * ch.em * ch.ep + (long long)E.nye * ch.ex * ch.ep +
                      (long long)E.nzs * ch.em * ch.ex;
  k_edges3<2><<<blocks(n, 128), 128, 0, h->stream>>>(h->F, ch, E);
  dbg_sync(h, "k_edges3");
  h->launches++;
  toc(h, &h->t_flux);
}

// states of the chunk's extended planes [ch.e0, ch.e1) (the fused 2-D
// engine also produces the face fluxes)
void states_only(kfvm_handle* h, const double* U, const Chunk& ch) {
  if (fused3(h)) {
    launch_fused3(h, U, ch);
    return;
  }
  if (h->dim == 2 && h->R == 2) launch_states<2, 2>(h, U, ch);
  if (h->dim == 2 && h->R == 3) launch_states<2, 3>(h, U, ch);
  if (h->dim == 3 && h->R == 2) launch_states<3, 2>(h, U, ch);
  if (h->dim == 3 && h->R == 3) launch_states<3, 3>(h, U, ch);
}

bool fused_engine(const kfvm_handle* h) { return h->dim == 2 && h->engine == 3 && !h->kx; }
void flux_only(kfvm_handle* h, const Chunk& ch) {
  if (fused3(h)) {
    launch_edges3(h, ch);
  } else if (!fused_engine(h)) {
    if (h->dim == 2 && h->R == 2) launch_flux<2, 2>(h, ch);
    if (h->dim == 2 && h->R == 3) launch_flux<2, 3>(h, ch);
    if (h->dim == 3 && h->R == 2) launch_flux<3, 2>(h, ch);
    if (h->dim == 3 && h->R == 3) launch_flux<3, 3>(h, ch);
  }
  if (h->visc) {  // F -= F^(v) on the same faces (needs the stage's k_prims)
    tic(h);
    if (h->dim == 2)
      k_visc<2><<<dim3((unsigned)blocks(ch.nfb, 128), 2), 128, 0, h->stream>>>(h->Pr, h->F, h->g, ch);
    else
      k_visc<3><<<dim3((unsigned)blocks(ch.nfb, 128), 3), 128, 0, h->stream>>>(h->Pr, h->F, h->g, ch);
    dbg_sync(h, "k_visc");
    h->launches++;
    toc(h, &h->t_flux);
  }
}

void states_and_flux(kfvm_handle* h, const double* U, const Chunk& ch) {
  states_only(h, U, ch);
  flux_only(h, ch);
}

void update(kfvm_handle* h, const Chunk& ch, const double* U0, const double* Uk, double* Uout,
            int stage) {
  const long long n = (long long)h->g.nx * (h->dim == 3 ? h->g.nm : 1) * ch.C;
  tic(h);
  unsigned long long* sm = stage == 3 ? h->d_smax : nullptr;
  double* uh = stage == 13 ? h->Uh : nullptr;
  if (h->dim == 2 && !h->grav)
    k_update<2><<<blocks(n, 256), 256, 0, h->stream>>>(h->F, U0, Uk, Uout, h->g, ch, stage,
                                                       h->d_dt_cur, sm, h->d_err, uh);
  else if (h->dim == 2)
    k_update<2, true><<<blocks(n, 256), 256, 0, h->stream>>>(h->F, U0, Uk, Uout, h->g, ch, stage,
                                                             h->d_dt_cur, sm, h->d_err, uh);
  else if (!h->grav)
    k_update<3><<<blocks(n, 256), 256, 0, h->stream>>>(h->F, U0, Uk, Uout, h->g, ch, stage,
                                                       h->d_dt_cur, sm, h->d_err, uh);
  else
    k_update<3, true><<<blocks(n, 256), 256, 0, h->stream>>>(h->F, U0, Uk, Uout, h->g, ch, stage,
                                                             h->d_dt_cur, sm, h->d_err, uh);
  h->launches++;
  toc(h, &h->t_update);
}

// ghost cells of the local block (one rank: the halo planes too)
void ghost(kfvm_handle* h, double* U) {
  const Geo& g = h->g;
  const int hp = !h->multi ? g.H : 0, P = g.np_loc + 2 * hp;
  const long long n = 2LL * g.G * (g.nm + 2 * g.Gm) * P + 2LL * g.Gm * g.nx * P +
                      2LL * hp * g.nm * g.nx;
  tic(h);
  k_ghost<<<blocks(n * h->nv, 256), 256, 0, h->stream>>>(U, g, h->nv, h->nsa, h->p0, hp);
  h->launches++;
  toc(h, &h->t_other);
}

// fill the slab-axis halo planes of U (local copy and/or NCCL exchange)
int halo(kfvm_handle* h, double* U, cudaStream_t st) {
  const long long per = (long long)h->g.H * h->g.pstride;
  tic(h);
  if (!h->multi) {
    (void)per;  // k_ghost filled the halo planes
  } else {
    const bool periodic = h->kc.per[h->dim - 1] != 0;
    const int lo = h->rank - 1, hi = h->rank + 1;
    const bool has_lo = periodic || lo >= 0, has_hi = periodic || hi < h->nranks;
    const int plo = (lo + h->nranks) % h->nranks, phi = hi % h->nranks;
    int which = (has_lo ? 0 : 1) | (has_hi ? 0 : 2);
    if (which) {
      k_halo_local<<<blocks(2 * per * h->nv, 256), 256, 0, st>>>(U, h->g, h->nv, h->nsa,
                                                                         h->p0, which);
      h->launches++;
    }
    // per peer pair the order is: upward transfer (my top interior -> the
    // upper rank's bottom halo), then downward; this keeps send/recv matching
    // correct when both neighbours are the same rank (2 ranks, periodic).
    const size_t bytes = (size_t)per * sizeof(double);
    tx_start(h);
    for (int v = 0; v < h->nv; ++v) {
      double* base = U + (long long)v * h->g.vstride;
      double* top_int = base + (long long)h->g.np_loc * h->g.pstride;
      double* top_halo = base + (long long)(h->g.np_loc + h->g.H) * h->g.pstride;
      double* bot_int = base + per;
      double* bot_halo = base;
      if (has_hi) tx_send(h, top_int, bytes, phi, st);
      if (has_lo) tx_recv(h, bot_halo, bytes, plo, st);
      if (has_lo) tx_send(h, bot_int, bytes, plo, st);
      if (has_hi) tx_recv(h, top_halo, bytes, phi, st);
    }
    if (tx_end(h) != 0) return fail(h, KFVM_ERR_DEVICE, "halo exchange failed");
  }
  toc(h, &h->t_other);
  return KFVM_OK;
}

int reduce_smax(kfvm_handle* h) {
  if (!h->multi) return KFVM_OK;
  // positive doubles order like their bit patterns: max on uint64 is exact
  if (tx_allreduce_max_u64(h, h->d_smax, h->stream) != 0)
    return fail(h, KFVM_ERR_DEVICE, "allreduce (max wavespeed) failed");
  return KFVM_OK;
}

// one stage: halo, then per chunk states -> flux -> update
// per-cell quantities of slab planes [p0, p1) (p relative to the first
// interior plane; halo planes are negative / >= np_loc)
void prims(kfvm_handle* h, const double* U, int p0, int p1) {
  if (p1 <= p0) return;
  const long long t0 = (long long)(p0 + h->g.H) * h->g.pstride;
  const long long n = (long long)(p1 - p0) * h->g.pstride;
  tic(h);
  if (h->dim == 2)
    k_prims<2><<<blocks(n, 256), 256, 0, h->stream>>>(U, h->Pr, t0, n, h->g.vstride);
  else
    k_prims<3><<<blocks(n, 256), 256, 0, h->stream>>>(U, h->Pr, t0, n, h->g.vstride);
  h->launches++;
  toc(h, &h->t_other);
}
void prims(kfvm_handle* h, const double* U) { prims(h, U, -h->g.H, h->g.np_loc + h->g.H); }

// states -> flux -> update over the local planes [q0, q1), in scratch-sized chunks
void run_planes(kfvm_handle* h, const double* Uin, double* Uout, int stage, int q0, int q1) {
  for (int c0 = q0; c0 < q1; c0 += h->chunk) {
    const Chunk ch = make_chunk(h, c0, std::min(h->chunk, q1 - c0));
    states_and_flux(h, Uin, ch);
    update(h, ch, h->U0, Uin, Uout, stage);
  }
}

// One stage.  With overlap on, the halo exchange runs on s_halo while every
// state whose stencil, limiter neighbourhood and per-cell quantities lie in
// the rank's own planes is computed: the chunks that do not reach a halo
// plane, or — when the slab is one chunk — its extended planes
// [R+1, np-R+1); then the halo planes' per-cell quantities and the rest.
// Each state is still computed exactly once with unchanged arithmetic, so the
// results are bit-identical to the serial schedule.
// KXRCF passes 1-2: unlimited states, flags of the slab's cells,
// the neighbouring ranks' edge-plane flags, the ghost cells' flags.
template <int DIM, int R>
int kx_flags(kfvm_handle* h, const double* U, const Chunk& ch) {
  tic(h);
  if (DIM == 3 && h->engine == 2) {  // pass 1 on the tensor cores
    const int KZ = h->kz;
    const long long nb = (long long)((ch.ex + 31) / 32) * ch.em * ((ch.e1 - ch.e0 + KZ - 1) / KZ);
    k_states_u<DIM, R, true><<<(unsigned)nb, 128, UCfg<DIM, R>::bytes(), h->stream>>>(
        U, h->Pr, h->St, h->g, ch, KZ, h->d_err, h->d_Bd, h->d_Bf, h->d_gat4, nullptr);
  } else if (DIM == 2 && h->engine != 0) {  // pass 1 from the row rings
    if constexpr (DIM == 2) {
      const int KZ = h->kz;
      const long long nb = (long long)((ch.ex + 31) / 32) * ((ch.e1 - ch.e0 + KZ - 1) / KZ);
      k_stage_row<R, false, false, true><<<(unsigned)nb, 128, 0, h->stream>>>(
          U, h->Pr, h->St, h->F, h->g, ch, KZ, h->d_err, nullptr);
    }
  } else {
    k_pass1<DIM, R><<<blocks(ext_range(ch), 128), 128, 0, h->stream>>>(U, h->St, h->g, ch,
                                                                       h->d_face);
  }
  // face jumps into the flux scratch (k_flux overwrites it later in the stage)
  k_kx_face<DIM, R><<<dim3(blocks(ch.nfb, 128), DIM), 128, 0, h->stream>>>(h->St, h->F, h->g, ch);
  k_kx_flag<DIM><<<blocks(ch.next, 256), 256, 0, h->stream>>>(U, h->Pr, h->F, h->d_flags, h->g,
                                                              ch, h->p0, h->nsa);
  h->launches += 3;
  if (h->multi) {
    const bool periodic = h->kc.per[h->dim - 1] != 0;
    const int lo = h->rank - 1, hi = h->rank + 1;
    const bool has_lo = periodic || lo >= 0, has_hi = periodic || hi < h->nranks;
    const int plo = (lo + h->nranks) % h->nranks, phi = hi % h->nranks;
    const long long pl = (long long)ch.ex * ch.em;
    unsigned char* f = h->d_flags;
    tx_start(h);
    if (has_hi) tx_send(h, f + (long long)ch.C * pl, pl, phi, h->stream);
    if (has_lo) tx_recv(h, f, pl, plo, h->stream);
    if (has_lo) tx_send(h, f + pl, pl, plo, h->stream);
    if (has_hi) tx_recv(h, f + (long long)(ch.C + 1) * pl, pl, phi, h->stream);
    if (tx_end(h) != 0) return fail(h, KFVM_ERR_DEVICE, "flag exchange failed");
  }
  k_kx_mirror<DIM><<<blocks(ch.next, 256), 256, 0, h->stream>>>(h->d_flags, h->g, ch, h->p0,
                                                                h->nsa, h->multi ? 1 : 0);
  h->launches++;
  toc(h, &h->t_other);
  return KFVM_OK;
}

int run_stage(kfvm_handle* h, const double* Uin, double* Uout, int stage) {
  const int np = h->g.np_loc, R = h->R;
  if (h->kx) {  // single chunk (checked at create)
    ghost(h, const_cast<double*>(Uin));
    int rc = halo(h, const_cast<double*>(Uin), h->stream);
    if (rc) return rc;
    prims(h, Uin);
    const Chunk ch = make_chunk(h, 0, np);
    if (h->dim == 2 && R == 2) rc = kx_flags<2, 2>(h, Uin, ch);
    if (h->dim == 2 && R == 3) rc = kx_flags<2, 3>(h, Uin, ch);
    if (h->dim == 3 && R == 2) rc = kx_flags<3, 2>(h, Uin, ch);
    if (h->dim == 3 && R == 3) rc = kx_flags<3, 3>(h, Uin, ch);
    if (rc) return rc;
    states_and_flux(h, Uin, ch);
    update(h, ch, h->U0, Uin, Uout, stage);
    return KFVM_OK;
  }
  const int nch = (np + h->chunk - 1) / h->chunk;
  auto needs_halo = [&](int c0, int C) { return c0 - 1 - R < 0 || c0 + C + R > np - 1; };
  if (!h->overlap || fused_engine(h) || np < 2 * R + 3) {
    ghost(h, const_cast<double*>(Uin));
    int rc = halo(h, const_cast<double*>(Uin), h->stream);
    if (rc) return rc;
    prims(h, Uin);
    if (fused3(h)) {
      const int r0 = 0, r1 = np + 2;
      set_ranges(h, 1, &r0, &r1);
    }
    run_planes(h, Uin, Uout, stage, 0, np);
    return KFVM_OK;
  }
  ghost(h, const_cast<double*>(Uin));
  CK(cudaEventRecord(h->ev_fork, h->stream));
  CK(cudaStreamWaitEvent(h->s_halo, h->ev_fork, 0));
  int rc = halo(h, const_cast<double*>(Uin), h->s_halo);
  if (rc) return rc;
  CK(cudaEventRecord(h->ev_halo, h->s_halo));
  prims(h, Uin, 0, np);
  if (nch == 1) {
    Chunk ch = make_chunk(h, 0, np);
    if (fused3(h)) {
      const int r0[3] = {R + 1, 0, np - R + 1}, r1[3] = {np - R + 1, R + 1, ch.ep};
      set_ranges(h, 3, r0, r1);
    }
    ch.e0 = R + 1;
    ch.e1 = np - R + 1;
    states_only(h, Uin, ch);
    CK(cudaStreamWaitEvent(h->stream, h->ev_halo, 0));
    prims(h, Uin, -h->g.H, 0);
    prims(h, Uin, np, np + h->g.H);
    ch.e0 = 0;
    ch.e1 = R + 1;
    states_only(h, Uin, ch);
    ch.e0 = np - R + 1;
    ch.e1 = ch.ep;
    states_only(h, Uin, ch);
    flux_only(h, ch);
    update(h, ch, h->U0, Uin, Uout, stage);
    return KFVM_OK;
  }
  for (int c0 = 0; c0 < np; c0 += h->chunk) {
    const int C = std::min(h->chunk, np - c0);
    if (needs_halo(c0, C)) continue;
    const Chunk ch = make_chunk(h, c0, C);
    states_and_flux(h, Uin, ch);
    update(h, ch, h->U0, Uin, Uout, stage);
  }
  CK(cudaStreamWaitEvent(h->stream, h->ev_halo, 0));
  prims(h, Uin, -h->g.H, 0);
  prims(h, Uin, np, np + h->g.H);
  for (int c0 = 0; c0 < np; c0 += h->chunk) {
    const int C = std::min(h->chunk, np - c0);
    if (!needs_halo(c0, C)) continue;
    const Chunk ch = make_chunk(h, c0, C);
    states_and_flux(h, Uin, ch);
    update(h, ch, h->U0, Uin, Uout, stage);
  }
  return KFVM_OK;
}

// ----------------------------------------------- SSP(4,3) + PI controller
// (oracle kfo_advance43): dt from the CFL limit and the
// controller, 4 stages, the pinned three-level error-norm sum, accept/reject.
__global__ void k_dt43(const unsigned long long* __restrict__ smax, Ctl* c, double* dt_cur) {
  if (c->done || c->abort || !(c->t < c->t_final)) {
    c->done = 1;
    *dt_cur = 0.0;
    return;
  }
  double dt = (c_k.cfl * c_k.dx) / __longlong_as_double((long long)*smax);
  if (!(dt > 0.0) || !isfinite(dt)) {
    c->abort = 1;
    *dt_cur = 0.0;
    return;
  }
  dt = fmin(dt, c->dt_err);
  if (dt < c_k.dt_min) {  // unstable setup
    c->abort = 1;
    *dt_cur = 0.0;
    return;
  }
  dt = fmin(dt, c_k.dt_max);
  const double rem = c->t_final - c->t;
  if (rem < dt) dt = rem;
  *dt_cur = dt;
}

// row partials: sequential over x, then variables, of q^2 (fma)
template <int D>
__global__ void k_err_rows(const double* __restrict__ Up, const double* __restrict__ Uh,
                           double* __restrict__ rows, Geo g) {
  constexpr int nv = D + 2;
  const int nrow = D == 3 ? g.nm : 1;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)nrow * g.np_loc) return;
  const int j = (int)(t % nrow), p = (int)(t / nrow);
  const long long base = (long long)(p + g.H) * g.pstride + moff(g, j) + xoff(g, 0);
  double r = 0.0;
  for (int x = 0; x < g.nx; ++x)
#pragma unroll
    for (int v = 0; v < nv; ++v) {
      const long long i = v * g.vstride + base + x;
      const double up = Up[i];
      const double q = (up - Uh[i]) / fma(c_k.rtol, fabs(up), c_k.atol);
      r = fma(q, q, r);
    }
  rows[t] = r;
}

__global__ void k_err_planes(const double* __restrict__ rows, double* __restrict__ planes,
                             int nrow, int np) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  double pl = 0.0;
  for (int j = 0; j < nrow; ++j) pl = pl + rows[(long long)p * nrow + j];
  planes[p] = pl;
}

__device__ double d_pi_factor(bool accept, double err, double err_prev) {
  if (accept) {
    const double e = fmax(err, 1e-10);
    const double f = c_k.safety * d_kf_pow(e, -0.7 / 3.0) * d_kf_pow(err_prev, 0.4 / 3.0);
    return fmin(5.0, fmax(0.2, f));
  }
  if (!(err == err)) return 0.2;
  return fmax(0.2, c_k.safety * d_kf_pow(err, -1.0 / 3.0));
}

// planes: [rank][npmax] (global plane order = rank order); nps: planes per rank
__global__ void k_ctl43(Ctl* c, const double* __restrict__ planes, const int* __restrict__ nps,
                        int nranks, int npmax, double ncomp, int* err, const double* dt_cur,
                        double* dt_seq, int cap) {
  if (c->done || c->abort) {
    c->accept = 0;
    *err = 0;
    return;
  }
  double sum = 0.0;
  for (int r = 0; r < nranks; ++r)
    for (int p = 0; p < nps[r]; ++p) sum = sum + planes[(long long)r * npmax + p];
  const bool ok = *err == 0;
  *err = 0;
  const double e = ok ? sqrt(sum / ncomp) : __longlong_as_double(0x7ff8000000000000LL);
  const bool accept = ok && e <= 1.0;
  const double dt = *dt_cur;
  c->dt_err = dt * d_pi_factor(accept, e, c->err_prev);
  c->err = e;
  if (accept) {
    c->err_prev = fmax(e, 1e-10);
    c->t = c->t + dt;
    if (c->nacc < cap) dt_seq[c->nacc] = dt;
    c->nacc += 1;
  } else {
    c->nrej += 1;
  }
  c->accept = accept ? 1 : 0;
}

__global__ void k_accept43(const Ctl* c, double* __restrict__ U0, const double* __restrict__ Up,
                           long long n) {
  if (!c->accept) return;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) U0[t] = Up[t];
}

int enqueue_dt(kfvm_handle* h) {
  int rc = reduce_smax(h);
  if (rc) return rc;
  tic(h);
  k_dt<<<1, 1, 0, h->stream>>>(h->d_smax, h->d_dt_cur, h->d_dt_seq, h->d_step, h->dt_cap, h->d_err,
                               h->d_tt, h->d_step + 1);
  h->launches++;
  toc(h, &h->t_other);
  return KFVM_OK;
}

int enqueue_step(kfvm_handle* h) {
  int rc = enqueue_dt(h);
  if (rc) return rc;
  if ((rc = run_stage(h, h->U0, h->Ua, 1))) return rc;
  if ((rc = run_stage(h, h->Ua, h->Ub, 2))) return rc;
  if ((rc = run_stage(h, h->Ub, h->U0, 3))) return rc;
  return KFVM_OK;
}

int enqueue_speed(kfvm_handle* h) {
  const long long n = (long long)h->g.nx * (h->dim == 3 ? h->g.nm : 1) * h->g.np_loc;
  CK(cudaMemsetAsync(h->d_smax, 0, sizeof(unsigned long long), h->stream));
  if (h->dim == 2)
    k_speed<2><<<blocks(n, 256), 256, 0, h->stream>>>(h->U0, h->g, h->d_smax);
  else
    k_speed<3><<<blocks(n, 256), 256, 0, h->stream>>>(h->U0, h->g, h->d_smax);
  h->launches++;
  return KFVM_OK;
}

// one SSP(4,3) attempt (graph-captured by kfvm_gpu_advance_to)
int enqueue_attempt43(kfvm_handle* h) {
  int rc = enqueue_speed(h);
  if (rc) return rc;
  if ((rc = reduce_smax(h))) return rc;
  k_dt43<<<1, 1, 0, h->stream>>>(h->d_smax, h->d_ctl, h->d_dt_cur);
  h->launches++;
  if ((rc = run_stage(h, h->U0, h->Ua, 11))) return rc;
  if ((rc = run_stage(h, h->Ua, h->Ub, 12))) return rc;
  if ((rc = run_stage(h, h->Ub, h->Ua, 13))) return rc;
  if ((rc = run_stage(h, h->Ua, h->Ub, 14))) return rc;
  const int nrow = h->dim == 3 ? h->g.nm : 1, np = h->g.np_loc;
  const long long nr = (long long)nrow * np;
  if (h->dim == 2)
    k_err_rows<2><<<blocks(nr, 128), 128, 0, h->stream>>>(h->Ub, h->Uh, h->d_rows, h->g);
  else
    k_err_rows<3><<<blocks(nr, 128), 128, 0, h->stream>>>(h->Ub, h->Uh, h->d_rows, h->g);
  double* loc = h->d_planes + (long long)h->nranks * h->npmax;  // this rank's partials
  k_err_planes<<<blocks(np, 128), 128, 0, h->stream>>>(h->d_rows, h->multi ? loc : h->d_planes,
                                                       nrow, np);
  h->launches += 2;
  if (h->multi) {
    if (tx_allgather_f64(h, loc, h->d_planes, (size_t)h->npmax, h->stream) != 0)
      return fail(h, KFVM_ERR_DEVICE, "allgather (error norm) failed");
  }
  const double ncomp = (double)h->g.nx * h->g.nm * h->nsa * h->nv;
  k_ctl43<<<1, 1, 0, h->stream>>>(h->d_ctl, h->d_planes, h->d_nps, h->nranks, h->npmax, ncomp,
                                  h->d_err, h->d_dt_cur, h->d_dt_seq, h->dt_cap);
  const long long n = h->g.vstride * h->nv;
  k_accept43<<<blocks(n, 256), 256, 0, h->stream>>>(h->d_ctl, h->U0, h->Ub, n);
  h->launches += 2;
  return KFVM_OK;
}

int check_err(kfvm_handle* h) {
  CK(cudaStreamSynchronize(h->stream));
  int e = 0;
  CK(cudaMemcpy(&e, h->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (e) {
    CK(cudaMemset(h->d_err, 0, sizeof(int)));
    return fail(h, KFVM_ERR_RUNTIME, "device reported an inadmissible state (NaN, rho<=0 or p<=0)");
  }
  return KFVM_OK;
}

void drop_graphs(kfvm_handle* h) {
  if (h->graph) cudaGraphExecDestroy(h->graph);
  if (h->graph43) cudaGraphExecDestroy(h->graph43);
  h->graph = nullptr;
  h->graph43 = nullptr;
}

int ensure_dt_cap(kfvm_handle* h, int n) {
  if (n <= h->dt_cap) return KFVM_OK;
  drop_graphs(h);
  if (h->d_dt_seq) cudaFree(h->d_dt_seq);
  h->d_dt_seq = nullptr;
  CK(cudaMalloc(&h->d_dt_seq, sizeof(double) * n));
  h->dt_cap = n;
  return KFVM_OK;
}

// interior cells x variables of the rank (the AoS host / staging layout)
long long interior_elems(const kfvm_handle* h) {
  return (long long)h->g.nx * h->g.nm * h->g.np_loc * h->nv;
}

int ensure_aos(kfvm_handle* h) {
  const size_t n = (size_t)interior_elems(h);
  if (h->aos_elems >= n) return KFVM_OK;
  if (h->aos) cudaFree(h->aos);
  CK(cudaMalloc(&h->aos, n * sizeof(double)));
  h->aos_elems = n;
  return KFVM_OK;
}

// Scratch of the current engine.  The fused 3-D engine keeps no face states:
// it needs the whole slab's face fluxes and the compact tile-edge buffers (one
// chunk).  The other engines get a chunked face-state + flux scratch within
// the budget: half the device memory still free after the state buffers (at
// least st_budget = 16 GB when that much is free), or `chunk_planes` planes
// when given (each chunk recomputes its two edge planes).
int configure_scratch(kfvm_handle* h, long long chunk_planes) {
  drop_graphs(h);
  for (double** p : {&h->St, &h->F, &h->d_edges})
    if (*p) {
      cudaFree(*p);
      *p = nullptr;
    }
  h->st_elems = h->f_elems = h->edge_elems = 0;
  const int np = h->g.np_loc;
  if (fused3(h)) {
    h->chunk = np;
    const Chunk ch = make_chunk(h, 0, np);
    Edges& E = h->eds;
    E.KZ = h->kz;
    E.nxe = (ch.ex + kTX - 1) / kTX - 1;
    E.nye = (ch.em + kTY - 1) / kTY - 1;
    const int nzcap = (ch.ep + E.KZ - 1) / E.KZ + 3;  // the overlapped split adds <= 2 starts
    E.sx = (long long)E.nxe * ch.em * ch.ep;
    E.sy = (long long)E.nye * ch.ex * ch.ep;
    E.sz = (long long)nzcap * ch.em * ch.ex;
    const long long rows = 2LL * h->R * h->R * h->nv;  // [side][m][v]
    h->edge_elems = (size_t)(rows * (E.sx + E.sy + E.sz));
    h->f_elems = (size_t)ch.nfb * h->dim * h->nv;
    CK(cudaMalloc(&h->F, h->f_elems * sizeof(double)));
    CK(cudaMalloc(&h->d_edges, h->edge_elems * sizeof(double)));
    E.x = h->d_edges;
    E.y = E.x + rows * E.sx;
    E.z = E.y + rows * E.sy;
    const int r0 = 0, r1 = ch.ep;
    set_ranges(h, 1, &r0, &r1);
    return KFVM_OK;
  }
  const int nlb = (h->dim == 3 && h->R == 2) ? 3 : 0;  // k_bounds output per extended cell
  const long long per_plane =
      ((long long)(h->g.nx + 2) * (h->dim == 3 ? h->g.nm + 2 : 1) * (h->NP * h->nv + nlb) +
       (long long)(h->g.nx + 1) * (h->dim == 3 ? h->g.nm + 1 : 1) * h->dim * h->nv) *
      (long long)sizeof(double);
  long long c = chunk_planes;
  if (c <= 0) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    long long budget = (long long)(0.5 * (double)fr);
    if (budget < h->st_budget) budget = std::min(h->st_budget, (long long)(0.8 * (double)fr));
    c = budget / per_plane - 2;
  }
  c = std::max(1LL, std::min(c, (long long)np));
  if (h->kx && c < np)  // the flags of a chunk's edge planes need the pass-1 states beyond them
    return fail(h, KFVM_ERR_CONFIG,
                "kxrcf: the slab's face states must fit one chunk (scratch budget: half the "
                "free device memory)");
  h->chunk = (int)c;
  const Chunk ch = make_chunk(h, 0, h->chunk);
  h->st_elems = (size_t)ch.next * h->NP * h->nv;
  h->f_elems = (size_t)ch.nfb * h->dim * h->nv;
  CK(cudaMalloc(&h->St, (h->st_elems + (size_t)ch.next * nlb) * sizeof(double)));
  CK(cudaMalloc(&h->F, h->f_elems * sizeof(double)));
  h->Lb = nlb ? h->St + h->st_elems : nullptr;
  return KFVM_OK;
}

// TMA tensor maps of the three state buffers for the tensor engine's ring
// planes: 4-D (x, mid row, slab plane, variable) over the ghost-padded
// storage, box = one region plane [var][2R+1 rows][32+2R columns].
int make_tmaps(kfvm_handle* h) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }();
  if (!encode) {  // no driver entry point: the ring loads by cp.async
    h->tma = 0;
    return KFVM_OK;
  }
  using M = UCfg<3, 2>;
  CUtensorMap maps[3];
  double* bufs[3] = {h->U0, h->Ua, h->Ub};
  const Geo& g = h->g;
  cuuint64_t dims[4] = {(cuuint64_t)g.nxp, (cuuint64_t)(g.nm + 2 * g.Gm),
                        (cuuint64_t)(g.np_loc + 2 * g.H), (cuuint64_t)h->nv};
  cuuint64_t strides[3] = {(cuuint64_t)g.nxp * 8, (cuuint64_t)g.pstride * 8,
                           (cuuint64_t)g.vstride * 8};
  cuuint32_t box[4] = {(cuuint32_t)M::RX, (cuuint32_t)M::RY, 1, (cuuint32_t)h->nv};
  cuuint32_t es[4] = {1, 1, 1, 1};
  for (int i = 0; i < 3; ++i) {
    CUresult r = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, bufs[i], dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(h, KFVM_ERR_DEVICE, "cuTensorMapEncodeTiled failed");
  }
  CK(cudaMalloc(&h->d_tmap, sizeof(maps)));
  CK(cudaMemcpy(h->d_tmap, maps, sizeof(maps), cudaMemcpyHostToDevice));
  // the 16-warp engine's boxes: 4 rows of cells per CTA (rows past the grid
  // are zero-filled by the TMA unit and never stored)
  box[0] = (cuuint32_t)WCfg<kWideRows>::RX;
  box[1] = (cuuint32_t)WCfg<kWideRows>::RY;
  for (int i = 0; i < 3; ++i) {
    CUresult r = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, bufs[i], dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(h, KFVM_ERR_DEVICE, "cuTensorMapEncodeTiled failed");
  }
  CK(cudaMalloc(&h->d_tmapw, sizeof(maps)));
  CK(cudaMemcpy(h->d_tmapw, maps, sizeof(maps), cudaMemcpyHostToDevice));
  return KFVM_OK;
}

// Upload the weights into the generated __constant__ arrays after checking
// that the table's geometry is the structure compiled into kfvm_gen.cuh
// (once per device: the registry's first handle).
template <int D, int R>
int upload_const(kfvm_handle* h, const kfvm_table* t) {
  using G = Gen<D, R>;
  if (t->n_full != G::N0 || t->total_cells != G::NTOT || t->n_points != G::NP ||
      t->n_alpha != G::NA || t->n_stencils != G::NS)
    return fail(h, KFVM_ERR_CONFIG, "table does not match the generated kernel structure");
  for (int i = 0; i < G::N0; ++i)
    for (int a = 0; a < 3; ++a)
      if (t->offsets[3 * i + a] != G::OFF[i][a])
        return fail(h, KFVM_ERR_CONFIG, "table stencil order differs from kfvm_gen.cuh");
  for (int i = 0; i < G::NTOT; ++i)
    if (t->gather[i] != G::GATHER[i])
      return fail(h, KFVM_ERR_CONFIG, "table substencils differ from kfvm_gen.cuh");
  if constexpr (G::UNROLLED) {
    // face weights transposed per stencil to [q][h][s] (generated weno() order)
    std::vector<double> ft((size_t)G::NTOT * G::NP);
    for (int q = 0; q < G::NS; ++q) {
      const int N = t->size[q], o = t->cell_offset[q];
      for (int hh = 0; hh < N; ++hh)
        for (int sp = 0; sp < G::NP; ++sp)
          ft[(size_t)(o + hh) * G::NP + sp] = t->face[(size_t)o * G::NP + (size_t)sp * N + hh];
    }
    CK(cudaMemcpyToSymbol(G::face_symbol(), ft.data(), sizeof(double) * G::NTOT * G::NP));
    CK(cudaMemcpyToSymbol(G::deriv_symbol(), t->deriv, sizeof(double) * G::NTOT * G::NA));
  }
  return KFVM_OK;
}

// Per-handle DMMA operands (B fragments, chunk tables) and kernel attributes.
template <int D, int R>
int upload_gen(kfvm_handle* h, const kfvm_table* t) {
  using G = Gen<D, R>;
  if (t->n_full != G::N0 || t->total_cells != G::NTOT || t->n_points != G::NP ||
      t->n_alpha != G::NA || t->n_stencils != G::NS)
    return fail(h, KFVM_ERR_CONFIG, "table does not match the generated kernel structure");
  // DMMA operands: per 4-entry chunk of each stencil (zero-padded at the
  // front), B fragments in lane order (k = lane%4, column = lane/4) and the
  // S0 position of every chunk slot
  using M = UCfg<D, R>;
  std::vector<double> bd((size_t)G::NCHUNK * M::ND * 32, 0.0), bf((size_t)G::NCHUNK * M::NPT * 32, 0.0);
  // per chunk slot {region offset in the plane, z offset}, then sQ (stencil | last<<8)
  std::vector<int> g4((size_t)G::NCHUNK * 9, 0);
  for (int q = 0, ck = 0; q < G::NS; ++q) {
    const int N = t->size[q], o = t->cell_offset[q];
    const int kcq = (N + 3) / 4, pad = 4 * kcq - N;
    for (int jj = 0; jj < kcq; ++jj, ++ck) {
      g4[(size_t)G::NCHUNK * 8 + ck] = q | (jj == kcq - 1 ? 256 : 0);
      for (int k = 0; k < 4; ++k) {
        const int hh = 4 * jj + k - pad;
        const int e = t->gather[o + (hh < 0 ? 0 : hh)];
        const int ox = G::OFF[e][0], oy = D == 3 ? G::OFF[e][1] : 0;
        const int oz = D == 3 ? G::OFF[e][2] : G::OFF[e][1];
        g4[(size_t)(ck * 4 + k) * 2] = (oy + (D == 3 ? R : 0)) * M::RX + ox + R;
        g4[(size_t)(ck * 4 + k) * 2 + 1] = oz;
      }
      for (int lane = 0; lane < 32; ++lane) {
        const int k = lane % 4, col = lane / 4, hh = 4 * jj + k - pad;
        for (int n = 0; n < M::ND; ++n) {
          const int al = 8 * n + col;
          bd[((size_t)ck * M::ND + n) * 32 + lane] =
              (hh >= 0 && al < G::NA) ? t->deriv[(size_t)o * G::NA + (size_t)al * N + hh] : 0.0;
        }
        for (int n = 0; n < M::NPT; ++n) {
          const int sp = 8 * n + col;
          bf[((size_t)ck * M::NPT + n) * 32 + lane] =
              (hh >= 0 && sp < G::NP) ? t->face[(size_t)o * G::NP + (size_t)sp * N + hh] : 0.0;
        }
      }
    }
  }
  if constexpr (M::PK) {
    // pass 2 packed: the NTOT stencil slots in stencil order, 4 per chunk,
    // zero B (pads) only in the last chunk; slot word = region offset |
    // (z offset + R) << 9 | stencil << 12
    const size_t b0 = bf.size();
    bf.resize(b0 + (size_t)M::NCH2 * M::NPT * 32, 0.0);
    const size_t g0 = g4.size();
    g4.resize(g0 + (size_t)M::NCH2 * 4, 0);
    int sl = 0;
    for (int q = 0; q < G::NS; ++q) {
      const int N = t->size[q], o = t->cell_offset[q];
      for (int hh = 0; hh < N; ++hh, ++sl) {
        const int ck = sl / 4, k = sl % 4;
        const int e = t->gather[o + hh];
        const int inpl = (G::OFF[e][1] + R) * M::RX + G::OFF[e][0] + R;
        g4[g0 + sl] = inpl | ((G::OFF[e][2] + R) << 9) | (q << 12);
        for (int col = 0; col < 8; ++col)
          for (int n = 0; n < M::NPT; ++n) {
            const int sp = 8 * n + col;
            bf[b0 + ((size_t)ck * M::NPT + n) * 32 + col * 4 + k] =
                sp < G::NP ? t->face[(size_t)o * G::NP + (size_t)sp * N + hh] : 0.0;
          }
      }
    }
    for (; sl < 4 * M::NCH2; ++sl) {  // trailing pads: any valid slot, zero weights
      g4[g0 + sl] = g4[g0 + sl - 1];
    }
  }
  if constexpr (D == 3) {
    // the fused 3-D engine's region geometry (8 x 4 tile): same chunks and slots
    std::vector<int> g8(g4);
    constexpr int RX8 = kTX + 2 * R;
    for (int q = 0, ck = 0; q < G::NS; ++q) {
      const int N = t->size[q], o = t->cell_offset[q];
      const int kcq = (N + 3) / 4, pad = 4 * kcq - N;
      for (int jj = 0; jj < kcq; ++jj, ++ck)
        for (int k = 0; k < 4; ++k) {
          const int hh = 4 * jj + k - pad;
          const int e = t->gather[o + (hh < 0 ? 0 : hh)];
          g8[(size_t)(ck * 4 + k) * 2] = (G::OFF[e][1] + R) * RX8 + G::OFF[e][0] + R;
        }
    }
    CK(cudaMalloc(&h->d_gat8, g8.size() * sizeof(int)));
    CK(cudaMemcpy(h->d_gat8, g8.data(), g8.size() * sizeof(int), cudaMemcpyHostToDevice));
    if constexpr (R == 2)
      CK(cudaFuncSetAttribute(k_fused3<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)FCfg<2>::bytes()));
  }
  if constexpr (D == 3 && R == 2) {
    // the same slots in the ring-column tile's layout [36 rows][5 columns]:
    // region offset (oy + R) * 5 + ox + R
    std::vector<int> gc(g4);
    constexpr int CX = 2 * R + 1;
    auto col_inpl = [&](int inpl_row) {  // row-tile offset (oy + R) * RX + ox + R -> column tile
      const int oyr = inpl_row / M::RX, oxr = inpl_row % M::RX;
      return oyr * CX + oxr;
    };
    for (int ck = 0; ck < G::NCHUNK; ++ck)
      for (int k = 0; k < 4; ++k) gc[(size_t)(ck * 4 + k) * 2] = col_inpl(g4[(size_t)(ck * 4 + k) * 2]);
    const size_t g0 = (size_t)G::NCHUNK * 9;
    for (size_t i = g0; i < gc.size(); ++i) {
      const int w = g4[i];
      gc[i] = col_inpl(w & 511) | (w & ~511);
    }
    CK(cudaMalloc(&h->d_gat4c, gc.size() * sizeof(int)));
    CK(cudaMemcpy(h->d_gat4c, gc.data(), gc.size() * sizeof(int), cudaMemcpyHostToDevice));
    // k_states_w's slot words: region offset | (oz + R) << 9 | stencil << 12 |
    // W-cache position of the S0 cell << 16 | last chunk of the stencil << 22;
    // the pass-1 chunks (front-padded per stencil), then the packed pass-2 chunks
    using WC = WCfg<kWideRows>;
    // stencil 0 must list every cell of S0 (the W cache is filled from it)
    {
      std::vector<char> seen(G::N0, 0);
      for (int hh = 0; hh < t->size[0]; ++hh) seen[t->gather[t->cell_offset[0] + hh]] = 1;
      for (int e = 0; e < G::N0; ++e)
        if (!seen[e]) return fail(h, KFVM_ERR_CONFIG, "stencil 0 does not cover S0");
    }
    // the chunks that READ the cache: pass 1 from stencil 1 on, all of pass 2
    std::vector<std::array<int, 4>> rd;
    for (int q = 1; q < G::NS; ++q) {
      const int N = t->size[q], o = t->cell_offset[q];
      const int kcq = (N + 3) / 4, pad = 4 * kcq - N;
      for (int jj = 0; jj < kcq; ++jj) {
        std::array<int, 4> c;
        for (int k = 0; k < 4; ++k) c[k] = t->gather[o + std::max(4 * jj + k - pad, 0)];
        rd.push_back(c);
      }
    }
    {
      std::vector<int> flat;
      for (int q = 0; q < G::NS; ++q)
        for (int hh = 0; hh < t->size[q]; ++hh) flat.push_back(t->gather[t->cell_offset[q] + hh]);
      while (flat.size() % 4) flat.push_back(flat.back());
      for (size_t i = 0; i < flat.size(); i += 4) rd.push_back({flat[i], flat[i + 1], flat[i + 2], flat[i + 3]});
    }
    // 4-colouring of S0 (bank window of a cell's cache row = colour): minimise
    // the half-warp wavefronts, sum over chunks of the largest number of
    // distinct cells of one colour; balanced colours (N0 positions suffice);
    // seeded multi-start pair-swap descent, deterministic
    std::vector<int> col(G::N0), bestc;
    auto cost = [&](const std::vector<int>& c) {
      int tot = 0;
      for (const auto& ck : rd) {
        int cnt[4] = {0, 0, 0, 0};
        for (int k = 0; k < 4; ++k) {
          bool dup = false;
          for (int k2 = 0; k2 < k; ++k2) dup |= ck[k2] == ck[k];
          if (!dup) cnt[c[ck[k]]]++;
        }
        tot += std::max(std::max(cnt[0], cnt[1]), std::max(cnt[2], cnt[3]));
      }
      return tot;
    };
    int bestv = 1 << 30;
    unsigned long long rng = 0x9e3779b97f4a7c15ull;
    for (int trial = 0; trial < 64; ++trial) {
      std::vector<int> perm(G::N0);
      for (int e = 0; e < G::N0; ++e) perm[e] = e;
      for (int e = G::N0 - 1; e > 0; --e) {
        rng = rng * 6364136223846793005ull + 1442695040888963407ull;
        std::swap(perm[e], perm[(int)((rng >> 33) % (unsigned)(e + 1))]);
      }
      for (int i = 0; i < G::N0; ++i) col[perm[i]] = i % 4;
      int cv = cost(col);
      for (bool imp = true; imp;) {
        imp = false;
        for (int a2 = 0; a2 < G::N0; ++a2)
          for (int b2 = a2 + 1; b2 < G::N0; ++b2) {
            if (col[a2] == col[b2]) continue;
            std::swap(col[a2], col[b2]);
            const int c2 = cost(col);
            if (c2 < cv) {
              cv = c2;
              imp = true;
            } else {
              std::swap(col[a2], col[b2]);
            }
          }
      }
      if (cv < bestv) {
        bestv = cv;
        bestc = col;
      }
    }
    // position of a cell: the next free one with position mod 4 = colour
    // (i % 4 colours: sizes 9, 8, 8, 8 -> the 9 of colour 0 end at position 32)
    std::vector<int> pos(G::N0);
    {
      int cnt[4] = {0, 0, 0, 0}, big = 0;
      for (int e = 0; e < G::N0; ++e) cnt[bestc[e]]++;
      for (int k = 1; k < 4; ++k)
        if (cnt[k] > cnt[big]) big = k;
      int nxt[4] = {0, 0, 0, 0};
      for (int e = 0; e < G::N0; ++e) {
        const int c = bestc[e] == big ? 0 : (bestc[e] == 0 ? big : bestc[e]);  // largest colour first
        pos[e] = c + 4 * nxt[c]++;
        if (pos[e] >= G::N0) return fail(h, KFVM_ERR_CONFIG, "W-cache colouring does not fit");
      }
    }
    std::vector<int> gw((size_t)WC::NT1 + WC::NT2, 0);
    for (int q = 0, ck = 0; q < G::NS; ++q) {
      const int N = t->size[q], o = t->cell_offset[q];
      const int kcq = (N + 3) / 4, pad = 4 * kcq - N;
      for (int jj = 0; jj < kcq; ++jj, ++ck)
        for (int k = 0; k < 4; ++k) {
          const int hh = 4 * jj + k - pad;
          const int e = t->gather[o + (hh < 0 ? 0 : hh)];
          const int inpl = (G::OFF[e][1] + R) * WC::RX + G::OFF[e][0] + R;
          gw[(size_t)ck * 4 + k] = inpl | ((G::OFF[e][2] + R) << 9) | (q << 12) | (pos[e] << 16) |
                                   (jj == kcq - 1 ? 1 << 22 : 0);
        }
    }
    {
      int sl = 0;
      for (int q = 0; q < G::NS; ++q) {
        const int N = t->size[q], o = t->cell_offset[q];
        for (int hh = 0; hh < N; ++hh, ++sl) {
          const int e = t->gather[o + hh];
          const int inpl = (G::OFF[e][1] + R) * WC::RX + G::OFF[e][0] + R;
          gw[(size_t)WC::NT1 + sl] = inpl | ((G::OFF[e][2] + R) << 9) | (q << 12) | (pos[e] << 16);
        }
      }
      for (; sl < WC::NT2; ++sl) gw[(size_t)WC::NT1 + sl] = gw[(size_t)WC::NT1 + sl - 1];
    }
    CK(cudaMalloc(&h->d_gatw, gw.size() * sizeof(int)));
    CK(cudaMemcpy(h->d_gatw, gw.data(), gw.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(k_states_w<kWideRows, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)WC::bytes()));
    CK(cudaFuncSetAttribute(k_states_w<kWideRows, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)WC::bytes()));
  }
  CK(cudaMalloc(&h->d_Bd, bd.size() * sizeof(double)));
  CK(cudaMalloc(&h->d_Bf, bf.size() * sizeof(double)));
  CK(cudaMalloc(&h->d_gat4, g4.size() * sizeof(int)));
  CK(cudaMemcpy(h->d_Bd, bd.data(), bd.size() * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->d_Bf, bf.data(), bf.size() * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->d_gat4, g4.data(), g4.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_states_u<D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)M::bytes(D == 3 && R == 2, M::TGM)));
  if constexpr (D == 3 && R == 2)
    CK(cudaFuncSetAttribute(k_states_u<D, R, false, false, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)M::bytes(true)));
  CK(cudaFuncSetAttribute(k_states_u<D, R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)M::bytes()));
  CK(cudaFuncSetAttribute(k_states_u<D, R, false, true>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)M::bytes()));
  return KFVM_OK;
}

}  // namespace

// ------------------------------------------------------------------ C-ABI
extern "C" int kfvm_nccl_unique_id(unsigned char id[128]) {
  NcclApi& N = nccl();
  if (!N.ok) return KFVM_ERR_DEVICE;
  nccl_uid u;
  if (N.GetUniqueId(&u) != 0) return KFVM_ERR_DEVICE;
  std::memcpy(id, u.internal, 128);
  return KFVM_OK;
}

extern "C" int kfvm_loopback_id(unsigned char id[128]) {
  kfvm_loop::make_id(id);
  return KFVM_OK;
}

// Boundary kinds per physical side (bc, or bc_side[] when bc_per_side) into
// the device constants; false for an invalid combination: unknown kind,
// unpaired periodic side, a mirror deeper than the axis (reflecting needs
// n >= R+1), an inadmissible dirichlet / inflow state, a non-positive slit.
static bool resolve_bcs(const kfvm_config* cfg, DevConsts* k) {
  const int dim = cfg->dim, H = cfg->radius + 1;
  const int n[3] = {cfg->nx, cfg->ny, dim == 3 ? cfg->nz : 1};
  const double gm1 = cfg->gamma - 1.0;
  for (int a = 0; a < 3; ++a) {
    for (int s = 0; s < 2; ++s) {
      const int side = 2 * a + s;
      int kind = cfg->bc_per_side ? cfg->bc_side[side] : cfg->bc;
      if (a >= dim) kind = KFVM_BC_PERIODIC;
      if (kind < KFVM_BC_PERIODIC || kind > KFVM_BC_SLIT) return false;
      if (!cfg->bc_per_side && kind > KFVM_BC_REFLECTING) return false;
      if (kind == KFVM_BC_REFLECTING && n[a] < H) return false;
      k->bcs[side] = kind;
      for (int v = 0; v < 5; ++v) k->bst[side][v] = 0.0;
      k->slc[side][0] = k->slc[side][1] = 0.0;
      k->slr2[side] = 0.0;
      if (kind == KFVM_BC_DIRICHLET || kind == KFVM_BC_SLIT) {
        const double* u = cfg->bc_state[side];
        for (int v = 0; v < dim + 2; ++v) {
          if (!std::isfinite(u[v])) return false;
          k->bst[side][v] = u[v];
        }
        double q = 0.0;
        for (int m = 0; m < dim; ++m) q += u[1 + m] * u[1 + m];
        if (!(u[0] > 0.0) || !(gm1 * (u[dim + 1] - 0.5 * q / u[0]) > 0.0)) return false;
      }
      if (kind == KFVM_BC_SLIT) {
        const double r = cfg->slit_radius[side];
        if (!(r > 0.0) || !std::isfinite(r)) return false;
        k->slc[side][0] = cfg->slit_center[side][0];
        k->slc[side][1] = cfg->slit_center[side][1];
        k->slr2[side] = r * r;
      }
    }
    const bool p0 = k->bcs[2 * a] == KFVM_BC_PERIODIC, p1 = k->bcs[2 * a + 1] == KFVM_BC_PERIODIC;
    if (p0 != p1) return false;  // periodic sides come in matching pairs
    k->per[a] = p0 ? 1 : 0;
  }
  return true;
}

extern "C" int kfvm_gpu_create(const kfvm_config* cfg, const kfvm_table* t, const kfvm_dist* dist,
                               kfvm_handle** out) {
  g_create_err.clear();
  if (!cfg || !t || !out) return KFVM_ERR_CONFIG;
  *out = nullptr;
  if ((cfg->dim != 2 && cfg->dim != 3) || (cfg->radius != 2 && cfg->radius != 3) ||
      t->dim != cfg->dim || t->radius != cfg->radius)
    return KFVM_ERR_CONFIG;
  if (cfg->nx < 1 || cfg->ny < 1 || (cfg->dim == 3 && cfg->nz < 1) || !(cfg->dx > 0) ||
      (cfg->riemann != KFVM_RIEMANN_HLLC && cfg->riemann != KFVM_RIEMANN_HLL))
    return KFVM_ERR_CONFIG;
  if (cfg->viscous && !(cfg->reynolds > 0 && cfg->prandtl > 0 && cfg->mach > 0))
    return KFVM_ERR_CONFIG;  // the viscous terms need Re, Pr, Ma
  if (!std::isfinite(cfg->inv_froude2)) return KFVM_ERR_CONFIG;
  {
    DevConsts probe{};
    if (!resolve_bcs(cfg, &probe)) return KFVM_ERR_CONFIG;
  }
  kfvm_handle* h = new kfvm_handle();
  h->cfg = *cfg;
  h->dim = cfg->dim;
  h->R = cfg->radius;
  h->nv = cfg->dim + 2;
  h->NP = t->n_points;
  // measured: row-marching DFMA for 2-D, tensor cores for 3-D.
  // The fused 3-D stage engine (5) is bit-identical but slower on B200: config
  // 3 132.3 vs 128.8 ms/step, config 4 1118.7 vs 1019.3 (profiles/r02) — the
  // in-kernel Riemann solves run at the reconstruction kernel's 12 warps/SM
  // instead of k_flux's full occupancy, and the face-state round trip they
  // save is not the bound (the stage is FP64-datapath bound)
  h->engine = cfg->dim == 2 ? 4 : 2;
  h->kz = cfg->dim == 2 ? 8 : 32;  // 3-D R=2: 32 measured 0.4 % faster than 16 (configs 3, 4)
  if (dist) {
    h->rank = dist->rank;
    h->nranks = dist->nranks;
    h->device = dist->device;
  }
  if (cudaSetDevice(h->device) != cudaSuccess) {
    delete h;
    return KFVM_ERR_DEVICE;
  }
  if (cudaDeviceGetAttribute(&h->num_sm, cudaDevAttrMultiProcessorCount, h->device) != cudaSuccess ||
      h->num_sm < 1)
    h->num_sm = 148;
  const int sa = cfg->dim - 1;
  h->nsa = sa == 2 ? cfg->nz : cfg->ny;
  if (h->nranks < 1 || h->nranks > h->nsa) {
    delete h;
    return KFVM_ERR_CONFIG;
  }
  int np;
  kfvm_slab_range(h->nsa, h->nranks, h->rank, &h->p0, &np);
  {
    const char* fe = std::getenv("KFVM_FORCE_NCCL");
    h->multi = h->nranks > 1 || (fe && fe[0] == '1');
  }
  h->g.nx = cfg->nx;
  h->g.nm = cfg->dim == 3 ? cfg->ny : 1;
  h->g.np_loc = np;
  h->g.H = cfg->radius + 1;
  if (np < h->g.H && h->nranks > 1) {
    delete h;
    return fail(nullptr, KFVM_ERR_CONFIG, "slab thinner than the halo");
  }
  h->g.G = h->g.H;
  h->g.Gm = cfg->dim == 3 ? h->g.H : 0;
  // rows start 128-byte aligned and cell 0 sits at a 128-byte boundary, so
  // the engines' 32-cell segments keep the alignment of an unpadded row
  h->g.xo = 16;
  h->g.nxp = (h->g.xo + h->g.nx + h->g.G + 15) / 16 * 16;
  h->g.pstride = (long long)h->g.nxp * (h->g.nm + 2 * h->g.Gm);
  h->g.vstride = h->g.pstride * (np + 2 * h->g.H);
  // constants (pinned on the host once)
  DevConsts& k = h->kc;
  k.dim = cfg->dim;
  k.nv = h->nv;
  k.R = cfg->radius;
  k.riemann = cfg->riemann;
  k.bc = cfg->bc;
  resolve_bcs(cfg, &k);
  k.n[0] = cfg->nx;
  k.n[1] = h->g.nm;
  k.n[2] = h->nsa;
  k.gamma = cfg->gamma;
  k.gm1 = cfg->gamma - 1.0;
  k.inv_gm1 = 1.0 / (cfg->gamma - 1.0);
  k.dx = cfg->dx;
  k.cfl = cfg->cfl;
  k.eps = cfg->eps;
  k.kappa = cfg->kappa;
  k.kf = cfg->flattener_kf;
  k.onepk = 1.0 + cfg->kappa;
  k.onemk = 1.0 - cfg->kappa;
  k.c13 = 1.0 / 3.0;
  k.c23 = 2.0 / 3.0;
  k.atol = cfg->atol;
  k.rtol = cfg->rtol;
  k.safety = cfg->safety;
  k.dt_min = cfg->dt_min;
  k.dt_max = cfg->dt_max > 0.0 ? cfg->dt_max : INFINITY;
  h->integrator = cfg->integrator;
  k.visc = cfg->viscous ? 1 : 0;
  k.inv_re = 1.0 / cfg->reynolds;  // the oracle computes the same doubles
  k.inv_prre = 1.0 / (cfg->prandtl * cfg->reynolds);
  k.gmm = cfg->gamma * (cfg->mach * cfg->mach);
  k.g2 = cfg->inv_froude2;
  h->visc = cfg->viscous != 0;
  h->grav = cfg->inv_froude2 != 0.0;
  k.kx = cfg->kxrcf ? 1 : 0;
  k.dm = std::pow(cfg->dx, cfg->kxrcf_m);  // the oracle computes the same std::pow
  h->kx = cfg->kxrcf != 0;
  DevTable& T = h->tab;
  T.n_full = t->n_full;
  T.n_points = t->n_points;
  T.n_alpha = t->n_alpha;
  T.n_stencils = t->n_stencils;
  T.rp = t->n_points / (2 * t->dim);
  for (int q = 0; q < t->n_stencils; ++q) {
    T.size[q] = t->size[q];
    T.cell_offset[q] = t->cell_offset[q];
    T.gamma_lin[q] = t->gamma_lin[q];
  }
  T.inv_g0 = 1.0 / t->gamma_lin[0];
  for (int hh = 0; hh < t->n_full; ++hh) {
    T.off_x[hh] = t->offsets[3 * hh];
    if (cfg->dim == 3) {
      T.off_m[hh] = t->offsets[3 * hh + 1];
      T.off_p[hh] = t->offsets[3 * hh + 2];
    } else {
      T.off_m[hh] = 0;
      T.off_p[hh] = t->offsets[3 * hh + 1];
    }
  }
  for (int s = 0; s < t->n_points; ++s) T.face_w[s] = t->face_weights[s];
  for (int a = 0; a < t->n_alpha; ++a) {
    const int ord = t->alpha[3 * a] + t->alpha[3 * a + 1] + t->alpha[3 * a + 2];
    double s = 1.0;
    for (int e = 0; e < 2 * ord; ++e) s *= cfg->dx;  // Delta^(2|alpha|)
    T.scale[a] = s;
  }
  int rc = KFVM_OK;
  auto bad = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && rc == KFVM_OK) {
      rc = KFVM_ERR_DEVICE;
      h->err = std::string(what) + ": " + cudaGetErrorString(e);
    }
  };
  const size_t nface = (size_t)t->total_cells * t->n_points;
  const size_t nder = (size_t)t->total_cells * t->n_alpha;
  T.gather = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_image_mu);
    DeviceImage& im = g_images[h->device];
    if (im.users > 0) {
      T.face = im.d_face;
      T.deriv = im.d_deriv;
      if (std::memcmp(&im.k, &k, sizeof(k)) != 0 || std::memcmp(&im.t, &T, sizeof(T)) != 0 ||
          im.hash != t->hash ||
          im.gather != std::vector<int>(t->gather, t->gather + t->total_cells)) {
        delete h;
        g_create_err = "another live handle on this device uses a different configuration or table "
                       "(the constant banks are per device)";
        return KFVM_ERR_CONFIG;
      }
      ++im.users;
      h->registered = true;
    } else {
      bad(cudaMalloc(&im.d_face, nface * sizeof(double)), "cudaMalloc face");
      bad(cudaMalloc(&im.d_deriv, nder * sizeof(double)), "cudaMalloc deriv");
      if (rc == KFVM_OK) {
        bad(cudaMemcpy(im.d_face, t->face, nface * sizeof(double), cudaMemcpyHostToDevice), "copy face");
        bad(cudaMemcpy(im.d_deriv, t->deriv, nder * sizeof(double), cudaMemcpyHostToDevice),
            "copy deriv");
      }
      T.face = im.d_face;
      T.deriv = im.d_deriv;
      bad(cudaMemcpyToSymbol(c_k, &k, sizeof(k)), "constants");
      bad(cudaMemcpyToSymbol(c_t, &T, sizeof(T)), "table");
      bad(cudaMemcpyToSymbol(c_gather, t->gather, sizeof(int) * t->total_cells), "gather");
      if (rc == KFVM_OK) {
        if (cfg->dim == 2 && cfg->radius == 2) rc = upload_const<2, 2>(h, t);
        if (cfg->dim == 2 && cfg->radius == 3) rc = upload_const<2, 3>(h, t);
        if (cfg->dim == 3 && cfg->radius == 2) rc = upload_const<3, 2>(h, t);
        if (cfg->dim == 3 && cfg->radius == 3) rc = upload_const<3, 3>(h, t);
      }
      if (rc == KFVM_OK) {
        im.users = 1;
        im.k = k;
        im.t = T;
        im.hash = t->hash;
        im.gather.assign(t->gather, t->gather + t->total_cells);
        h->registered = true;
      } else {
        if (im.d_face) cudaFree(im.d_face);
        if (im.d_deriv) cudaFree(im.d_deriv);
        im = DeviceImage();
      }
    }
  }
  h->d_face = const_cast<double*>(T.face);
  h->d_deriv = const_cast<double*>(T.deriv);
  if (rc == KFVM_OK) {
    if (cfg->dim == 2 && cfg->radius == 2) rc = upload_gen<2, 2>(h, t);
    if (cfg->dim == 2 && cfg->radius == 3) rc = upload_gen<2, 3>(h, t);
    if (cfg->dim == 3 && cfg->radius == 2) rc = upload_gen<3, 2>(h, t);
    if (cfg->dim == 3 && cfg->radius == 3) rc = upload_gen<3, 3>(h, t);
  }
  const size_t ufull = (size_t)h->g.vstride * h->nv;
  bad(cudaMalloc(&h->U0, ufull * sizeof(double)), "cudaMalloc U0");
  bad(cudaMalloc(&h->Ua, ufull * sizeof(double)), "cudaMalloc Ua");
  bad(cudaMalloc(&h->Ub, ufull * sizeof(double)), "cudaMalloc Ub");
  bad(cudaMalloc(&h->Pr, (size_t)h->g.vstride * (cfg->dim + 3) * sizeof(double)), "cudaMalloc prims");
  if (rc == KFVM_OK && cfg->dim == 3 && cfg->radius == 2) rc = make_tmaps(h);
  if (rc == KFVM_OK) {
    bad(cudaMemset(h->U0, 0, ufull * sizeof(double)), "memset");
    bad(cudaMemset(h->Ua, 0, ufull * sizeof(double)), "memset");
    bad(cudaMemset(h->Ub, 0, ufull * sizeof(double)), "memset");
  }
  if (rc == KFVM_OK) rc = configure_scratch(h, 0);
  if (h->kx && rc == KFVM_OK) {
    const Chunk ch = make_chunk(h, 0, h->chunk);
    bad(cudaMalloc(&h->d_flags, (size_t)ch.next), "cudaMalloc flags");
    if (rc == KFVM_OK) bad(cudaMemset(h->d_flags, 0, (size_t)ch.next), "memset flags");
  }
  if (h->integrator == KFVM_SSP43 && rc == KFVM_OK) {
    const int nrow = h->dim == 3 ? h->g.nm : 1;
    h->npmax = (h->nsa + h->nranks - 1) / h->nranks;
    bad(cudaMalloc(&h->Uh, (size_t)h->g.vstride * h->nv * sizeof(double)), "cudaMalloc uhat");
    bad(cudaMalloc(&h->d_rows, (size_t)nrow * h->g.np_loc * sizeof(double)), "cudaMalloc rows");
    bad(cudaMalloc(&h->d_planes, (size_t)(h->nranks + 1) * h->npmax * sizeof(double)),
        "cudaMalloc planes");
    bad(cudaMalloc(&h->d_ctl, sizeof(Ctl)), "cudaMalloc ctl");
    std::vector<int> nps(h->nranks);
    for (int r = 0; r < h->nranks; ++r) {
      int q0, nq;
      kfvm_slab_range(h->nsa, h->nranks, r, &q0, &nq);
      nps[r] = nq;
    }
    bad(cudaMalloc(&h->d_nps, sizeof(int) * h->nranks), "cudaMalloc nps");
    if (rc == KFVM_OK) {
      bad(cudaMemcpy(h->d_nps, nps.data(), sizeof(int) * h->nranks, cudaMemcpyHostToDevice), "nps");
      bad(cudaMemset(h->Uh, 0, (size_t)h->g.vstride * h->nv * sizeof(double)), "memset");
      bad(cudaMemset(h->d_planes, 0, (size_t)(h->nranks + 1) * h->npmax * sizeof(double)),
          "memset");
    }
  }
  bad(cudaMalloc(&h->d_dt_cur, sizeof(double)), "cudaMalloc dt");
  bad(cudaMalloc(&h->d_smax, sizeof(unsigned long long)), "cudaMalloc smax");
  bad(cudaMalloc(&h->d_tt, 2 * sizeof(double)), "cudaMalloc t");
  if (rc == KFVM_OK) {
    const double tt0[2] = {0.0, INFINITY};
    bad(cudaMemcpy(h->d_tt, tt0, sizeof(tt0), cudaMemcpyHostToDevice), "init t");
  }
  bad(cudaMalloc(&h->d_step, 2 * sizeof(int)), "cudaMalloc step");  // {step, productive steps}
  bad(cudaMalloc(&h->d_err, sizeof(int)), "cudaMalloc err");
  if (rc == KFVM_OK) {
    bad(cudaMemset(h->d_err, 0, sizeof(int)), "memset");
    bad(cudaMemset(h->d_step, 0, 2 * sizeof(int)), "memset");
    bad(cudaMemset(h->d_smax, 0, sizeof(unsigned long long)), "memset");
  }
  bad(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "stream");
  bad(cudaStreamCreateWithFlags(&h->s_halo, cudaStreamNonBlocking), "stream");
  bad(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming), "event");
  bad(cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming), "event");
  h->overlap = h->multi ? 1 : 0;
  bad(cudaEventCreate(&h->ev[0]), "event");
  bad(cudaEventCreate(&h->ev[1]), "event");
  if (rc == KFVM_OK) rc = ensure_dt_cap(h, 1024);
  if (rc == KFVM_OK && h->multi && dist && kfvm_loop::is_id(dist->nccl_id)) {
    h->loop_key = kfvm_loop::id_key(dist->nccl_id);
    h->loop = kfvm_loop::join(h->loop_key, h->nranks, h->device);
    if (!h->loop) {
      rc = KFVM_ERR_CONFIG;
      h->err = "loopback group: rank count or device differs from the group's";
    }
  } else if (rc == KFVM_OK && h->multi) {
    NcclApi& N = nccl();
    if (!N.ok) {
      rc = KFVM_ERR_DEVICE;
      h->err = "libnccl.so.2 not loadable";
    } else {
      nccl_uid u;
      if (dist && h->nranks > 1)
        std::memcpy(u.internal, dist->nccl_id, 128);
      else if (N.GetUniqueId(&u) != 0)  // KFVM_FORCE_NCCL: a one-rank communicator
        rc = KFVM_ERR_DEVICE;
      if (rc == KFVM_OK && N.CommInitRank(&h->comm, h->nranks, u, h->rank) != 0) {
        rc = KFVM_ERR_DEVICE;
        h->err = "ncclCommInitRank failed";
      }
    }
  }
  if (rc != KFVM_OK) {
    fprintf(stderr, "kfvm_gpu_create: %s\n", h->err.c_str());
    kfvm_gpu_destroy(h);
    return rc;
  }
  *out = h;
  return KFVM_OK;
}

extern "C" void kfvm_gpu_destroy(kfvm_handle* h) {
  if (!h) return;
  if (h->graph) cudaGraphExecDestroy(h->graph);
  if (h->graph43) cudaGraphExecDestroy(h->graph43);
  if (h->comm) nccl().CommDestroy(h->comm);
  if (h->loop) kfvm_loop::leave(h->loop_key, h->loop);
  cudaSetDevice(h->device);
  if (h->registered) {
    std::lock_guard<std::mutex> lk(g_image_mu);
    DeviceImage& im = g_images[h->device];
    if (--im.users == 0) {
      cudaFree(im.d_face);
      cudaFree(im.d_deriv);
      im = DeviceImage();
    }
  }
  for (void* p : {(void*)h->d_gat4c, (void*)h->d_gatw, (void*)h->d_tmapw, (void*)h->d_tmap, (void*)h->U0, (void*)h->Ua, (void*)h->Ub, (void*)h->Pr, (void*)h->St, (void*)h->F,
                  (void*)h->aos, (void*)h->d_dt_seq,
                  (void*)h->d_dt_cur, (void*)h->d_smax, (void*)h->d_step, (void*)h->d_err,
                  (void*)h->d_Bd, (void*)h->d_Bf, (void*)h->d_gat4, (void*)h->d_gat8, (void*)h->d_edges, (void*)h->d_tt,
                  (void*)h->d_flags, (void*)h->Uh, (void*)h->d_rows, (void*)h->d_planes,
                  (void*)h->d_ctl, (void*)h->d_nps, (void*)h->ext})
    if (p) cudaFree(p);
  if (h->stream) cudaStreamDestroy(h->stream);
  if (h->s_halo) cudaStreamDestroy(h->s_halo);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_halo) cudaEventDestroy(h->ev_halo);
  delete h;
}

extern "C" int kfvm_gpu_set_state_device(kfvm_handle* h, const double* U_dev) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  const long long n = interior_elems(h);
  k_transpose<0><<<blocks(n, 256), 256, 0, h->stream>>>(h->U0, const_cast<double*>(U_dev), h->g,
                                                         h->nv);
  h->launches++;
  // the captured step graph reads the fixed state buffers: it stays valid
  CK(cudaMemsetAsync(h->d_step, 0, 2 * sizeof(int), h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return KFVM_OK;
}

extern "C" int kfvm_gpu_get_state_device(kfvm_handle* h, double* U_dev) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  const long long n = interior_elems(h);
  k_transpose<1><<<blocks(n, 256), 256, 0, h->stream>>>(h->U0, U_dev, h->g, h->nv);
  h->launches++;
  CK(cudaStreamSynchronize(h->stream));
  return KFVM_OK;
}

extern "C" int kfvm_gpu_set_state(kfvm_handle* h, const double* U_host) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  int rc = ensure_aos(h);
  if (rc) return rc;
  const size_t n = (size_t)interior_elems(h);
  CK(cudaMemcpyAsync(h->aos, U_host, n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  return kfvm_gpu_set_state_device(h, h->aos);
}

extern "C" int kfvm_gpu_get_state(kfvm_handle* h, double* U_host) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  int rc = ensure_aos(h);
  if (rc) return rc;
  rc = kfvm_gpu_get_state_device(h, h->aos);
  if (rc) return rc;
  const size_t n = (size_t)interior_elems(h);
  CK(cudaMemcpyAsync(U_host, h->aos, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return KFVM_OK;
}

// Asynchronous variants on the handle's stream (no host synchronisation; the
// host buffer must stay untouched until kfvm_gpu_sync): upload + transpose,
// transpose + download.  With pinned buffers and one handle per field, the
// copies of one field overlap the steps of another on the copy engines.
extern "C" int kfvm_gpu_set_state_async(kfvm_handle* h, const double* U_host) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  int rc = ensure_aos(h);
  if (rc) return rc;
  const long long n = interior_elems(h);
  CK(cudaMemcpyAsync(h->aos, U_host, (size_t)n * sizeof(double), cudaMemcpyHostToDevice,
                     h->stream));
  k_transpose<0><<<blocks(n, 256), 256, 0, h->stream>>>(h->U0, h->aos, h->g, h->nv);
  h->launches++;
  CK(cudaMemsetAsync(h->d_step, 0, 2 * sizeof(int), h->stream));
  return KFVM_OK;
}

extern "C" int kfvm_gpu_get_state_async(kfvm_handle* h, double* U_host) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  int rc = ensure_aos(h);
  if (rc) return rc;
  const long long n = interior_elems(h);
  k_transpose<1><<<blocks(n, 256), 256, 0, h->stream>>>(h->U0, h->aos, h->g, h->nv);
  h->launches++;
  CK(cudaMemcpyAsync(U_host, h->aos, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  return KFVM_OK;
}

extern "C" int kfvm_gpu_rhs(kfvm_handle* h, double* dUdt_host) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  int rc = run_stage(h, h->U0, h->Ua, 0);
  if (rc) return rc;
  if ((rc = check_err(h))) return rc;
  if ((rc = ensure_aos(h))) return rc;
  const long long n = interior_elems(h);
  k_transpose<1><<<blocks(n, 256), 256, 0, h->stream>>>(h->Ua, h->aos, h->g, h->nv);
  h->launches++;
  CK(cudaMemcpyAsync(dUdt_host, h->aos, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return KFVM_OK;
}

extern "C" int kfvm_gpu_states(kfvm_handle* h, double* states_host) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  ghost(h, h->U0);
  int rc = halo(h, h->U0, h->stream);
  if (rc) return rc;
  prims(h, h->U0);
  const long long per_cell = (long long)h->NP * h->nv;
  const long long plane_cells = (long long)h->g.nx * h->g.nm;  // interior cells per plane
  if (h->kx) {  // the troubled-cell flags of this state first (one chunk, S:565 steps 1-2)
    const Chunk ch = make_chunk(h, 0, h->g.np_loc);
    if (h->dim == 2 && h->R == 2) rc = kx_flags<2, 2>(h, h->U0, ch);
    if (h->dim == 2 && h->R == 3) rc = kx_flags<2, 3>(h, h->U0, ch);
    if (h->dim == 3 && h->R == 2) rc = kx_flags<3, 2>(h, h->U0, ch);
    if (h->dim == 3 && h->R == 3) rc = kx_flags<3, 3>(h, h->U0, ch);
    if (rc) return rc;
  }
  // the fused 3-D engine keeps no face states: this call runs the tensor-core
  // states engine (same bits) over a temporary chunked scratch
  const int eng_saved = h->engine;
  const bool tmp_scratch = fused3(h);
  if (tmp_scratch) {
    h->engine = 2;
    if ((rc = configure_scratch(h, 0))) {
      h->engine = eng_saved;
      configure_scratch(h, 0);
      return rc;
    }
  }
  const size_t nbuf = (size_t)plane_cells * h->chunk * per_cell;
  if (h->ext_elems < nbuf) {
    if (h->ext) cudaFree(h->ext);
    h->ext = nullptr;
    h->ext_elems = 0;
    CK(cudaMalloc(&h->ext, nbuf * sizeof(double)));
    h->ext_elems = nbuf;
  }
  for (int c0 = 0; c0 < h->g.np_loc; c0 += h->chunk) {
    const Chunk ch = make_chunk(h, c0, std::min(h->chunk, h->g.np_loc - c0));
    states_and_flux(h, h->U0, ch);
    const long long n = plane_cells * ch.C * per_cell;
    if (h->dim == 2)
      k_extract_states<2><<<blocks(n, 256), 256, 0, h->stream>>>(h->St, h->ext, h->g, ch, h->NP);
    else
      k_extract_states<3><<<blocks(n, 256), 256, 0, h->stream>>>(h->St, h->ext, h->g, ch, h->NP);
    h->launches++;
    CK(cudaMemcpyAsync(states_host + plane_cells * c0 * per_cell, h->ext, n * sizeof(double),
                       cudaMemcpyDeviceToHost, h->stream));
  }
  CK(cudaStreamSynchronize(h->stream));
  rc = check_err(h);
  if (tmp_scratch) {
    h->engine = eng_saved;
    const int rc2 = configure_scratch(h, 0);
    if (!rc) rc = rc2;
  }
  return rc;
}

// KXRCF flags (1 = WENO) of the rank's cells for the current state, AoS order
// (the indicator pass of kfvm_gpu_states / the stage, S:565 steps 1-2).
__global__ void k_extract_flags(const unsigned char* __restrict__ fl, unsigned char* __restrict__ out,
                                Geo g, Chunk ch) {
  const long long t = (long long)blockIdx.x * 256 + threadIdx.x;
  const long long n = (long long)g.nx * g.nm * ch.C;
  if (t >= n) return;
  const int x = (int)(t % g.nx);
  const long long r = t / g.nx;
  const int j = (int)(r % g.nm), p = (int)(r / g.nm);
  const bool d3 = ch.em > 1;
  out[t] = fl[((long long)(p + 1) * ch.em + (d3 ? j + 1 : 0)) * ch.ex + (x + 1)];
}

extern "C" int kfvm_gpu_kxrcf_flags(kfvm_handle* h, unsigned char* flags_host) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  if (!h->kx) return fail(h, KFVM_ERR_CONFIG, "kxrcf is off in this handle's config");
  ghost(h, h->U0);
  int rc = halo(h, h->U0, h->stream);
  if (rc) return rc;
  prims(h, h->U0);
  const Chunk ch = make_chunk(h, 0, h->g.np_loc);
  if (h->dim == 2 && h->R == 2) rc = kx_flags<2, 2>(h, h->U0, ch);
  if (h->dim == 2 && h->R == 3) rc = kx_flags<2, 3>(h, h->U0, ch);
  if (h->dim == 3 && h->R == 2) rc = kx_flags<3, 2>(h, h->U0, ch);
  if (h->dim == 3 && h->R == 3) rc = kx_flags<3, 3>(h, h->U0, ch);
  if (rc) return rc;
  const long long n = (long long)h->g.nx * h->g.nm * ch.C;
  unsigned char* d = nullptr;
  CK(cudaMalloc(&d, (size_t)n));
  k_extract_flags<<<blocks(n, 256), 256, 0, h->stream>>>(h->d_flags, d, h->g, ch);
  h->launches++;
  CK(cudaMemcpyAsync(flags_host, d, (size_t)n, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  cudaFree(d);
  return KFVM_OK;
}

extern "C" int kfvm_gpu_select_dt(kfvm_handle* h, double* dt) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  int rc = enqueue_speed(h);
  if (rc) return rc;
  if ((rc = reduce_smax(h))) return rc;
  unsigned long long bits = 0;
  CK(cudaMemcpyAsync(&bits, h->d_smax, sizeof(bits), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  double s;
  std::memcpy(&s, &bits, sizeof(s));
  *dt = (h->cfg.cfl * h->cfg.dx) / s;
  return (*dt > 0 && std::isfinite(*dt)) ? KFVM_OK : fail(h, KFVM_ERR_RUNTIME, "bad dt");
}

extern "C" int kfvm_gpu_stage(kfvm_handle* h, int stage, double dt) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  if (stage < 1 || stage > 3) return fail(h, KFVM_ERR_CONFIG, "stage must be 1..3");
  CK(cudaMemcpyAsync(h->d_dt_cur, &dt, sizeof(double), cudaMemcpyHostToDevice, h->stream));
  double* in = stage == 1 ? h->U0 : (stage == 2 ? h->Ua : h->Ub);
  double* outp = stage == 1 ? h->Ua : (stage == 2 ? h->Ub : h->U0);
  int rc = run_stage(h, in, outp, stage);
  if (rc) return rc;
  return check_err(h);
}

// nsteps SSP-RK3 steps (graph-replayed on one rank); reset = start a new dt
// sequence (advance_to keeps counting across its batches)
int run_steps(kfvm_handle* h, int nsteps, bool reset) {
  if (reset) {
    int rc = ensure_dt_cap(h, nsteps);
    if (rc) return rc;
    CK(cudaMemsetAsync(h->d_step, 0, 2 * sizeof(int), h->stream));
  }
  int rc = enqueue_speed(h);
  if (rc) return rc;
  // loopback rendezvous is host-side (not capturable); NCCL multi-rank steps
  // are captured unless KFVM_NCCL_GRAPHS=0 (eager fallback for an NCCL build
  // that cannot capture p2p)
  static const bool nccl_graphs = [] {
    const char* e = std::getenv("KFVM_NCCL_GRAPHS");
    return !(e && e[0] == '0');
  }();
  if (h->timing || h->loop || (h->multi && !nccl_graphs)) {
    for (int s = 0; s < nsteps; ++s)
      if ((rc = enqueue_step(h))) return rc;
    return KFVM_OK;
  }
  if (!h->graph) {
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    const long long l0 = h->launches;
    rc = enqueue_step(h);
    cudaError_t e = cudaStreamEndCapture(h->stream, &graph);
    if (rc) return rc;
    if (e != cudaSuccess) return fail(h, KFVM_ERR_DEVICE, "graph capture failed");
    CK(cudaGraphInstantiate(&h->graph, graph, 0));
    cudaGraphDestroy(graph);
    h->graph_launches = h->launches - l0;  // kernels in one captured step
    h->launches = l0;
  }
  for (int s = 0; s < nsteps; ++s) CK(cudaGraphLaunch(h->graph, h->stream));
  h->launches += h->graph_launches * nsteps;
  return KFVM_OK;
}

extern "C" int kfvm_gpu_run_async(kfvm_handle* h, int nsteps) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  return run_steps(h, nsteps, true);
}

extern "C" int kfvm_gpu_sync(kfvm_handle* h) { return check_err(h); }

extern "C" int kfvm_gpu_dt_sequence(kfvm_handle* h, double* dt_seq, int nsteps) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  if (nsteps > h->dt_cap) return fail(h, KFVM_ERR_CONFIG, "nsteps exceeds dt capacity");
  CK(cudaMemcpyAsync(dt_seq, h->d_dt_seq, sizeof(double) * nsteps, cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return KFVM_OK;
}

extern "C" int kfvm_gpu_run(kfvm_handle* h, int nsteps, double* dt_seq) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  int rc = kfvm_gpu_run_async(h, nsteps);
  if (rc) return rc;
  if ((rc = kfvm_gpu_sync(h))) return rc;
  if (dt_seq) return kfvm_gpu_dt_sequence(h, dt_seq, nsteps);
  return KFVM_OK;
}

extern "C" int kfvm_gpu_step(kfvm_handle* h, double* dt_out) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  double dt;
  int rc = kfvm_gpu_run(h, 1, &dt);
  if (rc) return rc;
  if (dt_out) *dt_out = dt;
  return KFVM_OK;
}

// advance_to with fixed-CFL steps: runs until t = t_final (the last
// step is clipped) or max_steps; *t_reached is the simulation time reached.
// advance_to with SSP(4,3)+SSP(3,2) and the PI controller: graph-
// replayed attempts until t_final, an abort, or max_attempts.
int advance43(kfvm_handle* h, double t_final, int max_attempts, int* steps, double* t_reached) {
  if ((int)ensure_dt_cap(h, 4096)) return KFVM_ERR_DEVICE;
  Ctl c0{};
  c0.t = 0.0;
  c0.t_final = t_final;
  c0.dt_err = INFINITY;
  c0.err_prev = 1.0;
  CK(cudaMemcpyAsync(h->d_ctl, &c0, sizeof(c0), cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemsetAsync(h->d_err, 0, sizeof(int), h->stream));
  if (!h->graph43 && !h->loop) {
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    const long long l0 = h->launches;
    int rc = enqueue_attempt43(h);
    cudaError_t e = cudaStreamEndCapture(h->stream, &graph);
    if (rc) return rc;
    if (e != cudaSuccess) return fail(h, KFVM_ERR_DEVICE, "graph capture failed");
    CK(cudaGraphInstantiate(&h->graph43, graph, 0));
    cudaGraphDestroy(graph);
    h->graph43_launches = h->launches - l0;
    h->launches = l0;
  }
  Ctl c = c0;
  int attempts = 0;
  while (attempts < max_attempts) {
    const int n = std::min(8, max_attempts - attempts);
    for (int i = 0; i < n; ++i) {
      if (h->loop) {
        const int rc = enqueue_attempt43(h);
        if (rc) return rc;
      } else {
        CK(cudaGraphLaunch(h->graph43, h->stream));
        h->launches += h->graph43_launches;
      }
    }
    attempts += n;
    CK(cudaMemcpyAsync(&c, h->d_ctl, sizeof(c), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (c.abort) return fail(h, KFVM_ERR_RUNTIME, "dt below dt_min or not finite (S:611)");
    if (c.done || !(c.t < t_final)) break;
  }
  h->nacc43 = c.nacc;
  h->nrej43 = c.nrej;
  if (steps) *steps = c.nacc;
  if (t_reached) *t_reached = c.t;
  CK(cudaMemsetAsync(h->d_step, 0, 2 * sizeof(int), h->stream));
  return KFVM_OK;
}

extern "C" int kfvm_gpu_step_stats(kfvm_handle* h, int* accepted, int* rejected) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  if (accepted) *accepted = h->nacc43;
  if (rejected) *rejected = h->nrej43;
  return KFVM_OK;
}

extern "C" int kfvm_gpu_advance_to(kfvm_handle* h, double t_final, int max_steps, int* steps,
                                   double* t_reached) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  if (h->integrator == KFVM_SSP43) return advance43(h, t_final, max_steps, steps, t_reached);
  // batches of graph-replayed steps; the batch size follows the remaining
  // time / last dt, so at most one dt = 0 step runs past t_final; the dt
  // sequence and the productive-step count run over the whole call
  int rc = ensure_dt_cap(h, std::min(std::max(max_steps, 1), 1 << 16));
  if (rc) return rc;
  double tt[2] = {0.0, t_final};
  CK(cudaMemcpyAsync(h->d_tt, tt, sizeof(tt), cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemsetAsync(h->d_step, 0, 2 * sizeof(int), h->stream));
  int done = 0, batch = 1;
  while (done < max_steps) {
    const int n = std::min(batch, max_steps - done);
    if ((rc = run_steps(h, n, false))) return rc;
    if ((rc = kfvm_gpu_sync(h))) return rc;
    double dt = 0.0;
    CK(cudaMemcpy(tt, h->d_tt, sizeof(tt), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&dt, h->d_dt_cur, sizeof(dt), cudaMemcpyDeviceToHost));
    done += n;
    if (tt[0] >= t_final) break;
    const double est = dt > 0.0 ? std::ceil((t_final - tt[0]) / dt) : 32.0;
    batch = (int)std::max(1.0, std::min(32.0, est));
  }
  int cnt[2] = {0, 0};
  CK(cudaMemcpy(cnt, h->d_step, sizeof(cnt), cudaMemcpyDeviceToHost));
  if (steps) *steps = cnt[1];  // steps with dt > 0
  if (t_reached) *t_reached = tt[0];
  const double reset[2] = {tt[0], INFINITY};
  CK(cudaMemcpy(h->d_tt, reset, sizeof(reset), cudaMemcpyHostToDevice));
  return KFVM_OK;
}

// Per-phase cycle counters of the reconstruction kernels (built with
// -DKFVM_PHASE_TIMING; zeros otherwise).  reset != 0 clears them.
extern "C" int kfvm_phase_cycles(unsigned long long* out8, int reset) {
#ifdef KFVM_PHASE_TIMING
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out8, g_phase_cycles, 8 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
#else
  for (int i = 0; i < 8; ++i) out8[i] = 0;
  (void)reset;
#endif
  return KFVM_OK;
}

extern "C" void* kfvm_gpu_stream(kfvm_handle* h) { return (void*)h->stream; }
extern "C" long long kfvm_gpu_launch_count(kfvm_handle* h) { return h->launches; }

extern "C" int kfvm_gpu_set_option(kfvm_handle* h, const char* name, long long value) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  std::string n(name ? name : "");
  if (n == "fast_states" || n == "engine") {
    if (n == "engine") {
      if (value < 0 || value > 5 || ((value == 3 || value == 4) && h->dim != 2) ||
          (value == 5 && !(h->dim == 3 && h->R == 2)))
        return fail(h, KFVM_ERR_CONFIG,
                    "engine: 0 generic, 1 DFMA, 2 tensor core, 3 fused 2-D stage, "
                    "4 row-marching DFMA (2-D), 5 fused 3-D stage (3-D R=2)");
      h->engine = (int)value;
    } else {
      h->engine = value ? 2 : 0;
    }
    return configure_scratch(h, 0);
  }
  if (n == "ring_tiles") {
    drop_graphs(h);
    h->ring_tiles = value < 0 ? 0 : (int)value;  // 0 off, 1 on (KZ 4), > 1: its KZ
    return KFVM_OK;
  }
  if (n == "tma") {
    drop_graphs(h);
    h->tma = value ? 1 : 0;
    return KFVM_OK;
  }
  if (n == "bounds_z") {
    drop_graphs(h);
    h->bounds_z = value ? 1 : 0;
    return KFVM_OK;
  }
  if (n == "wide") {  // 3-D R=2: 1 = the 16-warp W-cache engine (k_states_w), 0 = k_states_u
    drop_graphs(h);
    h->wide = value ? 1 : 0;
    return KFVM_OK;
  }
  if (n == "ring_split") {
    drop_graphs(h);
    h->ring_split = value ? 1 : 0;
    return KFVM_OK;
  }
  if (n == "overlap") {
    h->overlap = value != 0;
    drop_graphs(h);
    return KFVM_OK;
  }
  if (n == "kz") {
    if (value < 1) return fail(h, KFVM_ERR_CONFIG, "kz must be >= 1");
    h->kz = (int)value;
    h->kz_auto = 0;
    drop_graphs(h);
    return fused3(h) ? configure_scratch(h, 0) : KFVM_OK;
  }
  if (n == "timing") {
    h->timing = value != 0;
    h->t_states = h->t_flux = h->t_update = h->t_other = 0;
    return KFVM_OK;
  }
  if (n == "chunk_planes" || n == "scratch_bytes") {
    // chunking applies to the face-state engines; the fused 3-D engine has no
    // face-state scratch and always runs the slab as one chunk
    long long c;
    if (n == "chunk_planes") {
      c = value;
    } else {
      const long long per_plane = (long long)(h->g.nx + 2) * (h->dim == 3 ? h->g.nm + 2 : 1) *
                                  h->NP * h->nv * (long long)sizeof(double);
      c = std::max(1LL, value / per_plane - 2);
    }
    if (h->kx && std::min(c, (long long)h->g.np_loc) < h->g.np_loc)
      return fail(h, KFVM_ERR_CONFIG, "kxrcf: the slab's face states must fit one chunk");
    return configure_scratch(h, c);
  }
  return fail(h, KFVM_ERR_CONFIG, "unknown option " + n);
}

extern "C" int kfvm_gpu_kernel_times(kfvm_handle* h, double* a, double* b, double* c, double* d) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  if (a) *a = h->t_states;
  if (b) *b = h->t_flux;
  if (c) *c = h->t_update;
  if (d) *d = h->t_other;
  return KFVM_OK;
}

extern "C" int kfvm_gpu_last_error(kfvm_handle* h, char* buf, size_t n) {
  if (!buf || n == 0) return KFVM_ERR_CONFIG;
  const std::string& e = h ? h->err : (g_create_err.empty() ? std::string("null handle") : g_create_err);
  std::snprintf(buf, n, "%s", e.c_str());
  return KFVM_OK;
}

// Seeded IC generated on the device directly into the handle's state (used
// by the bench at sizes where the host generator is slow); bit-identical to
// kfvm_ic_generate (same arithmetic, tables from the host).
extern "C" int kfvm_gpu_ic_generate(kfvm_handle* h, const kfvm_ic_params* ic) {
  if (!h) return KFVM_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  if (ic->kind != KFVM_IC_FOURIER && ic->kind != KFVM_IC_VORONOI &&
      ic->kind != KFVM_IC_FOURIER_SPHERE && ic->kind != KFVM_IC_UNIFORM)
    return fail(h, KFVM_ERR_CONFIG, "IC kind not available on the device");
  ICHostPlan hp;
  int rc = ic_plan_build(&h->cfg, ic, &hp);
  if (rc) return fail(h, rc, "bad IC parameters");
  ICPlan P = hp.plan;
  std::vector<void*> tmp;
  for (int a = 0; a < P.dim; ++a) {
    if (hp.fc[a].empty()) continue;
    double *dc, *ds;
    CK(cudaMalloc(&dc, hp.fc[a].size() * sizeof(double)));
    CK(cudaMalloc(&ds, hp.fs[a].size() * sizeof(double)));
    CK(cudaMemcpy(dc, hp.fc[a].data(), hp.fc[a].size() * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ds, hp.fs[a].data(), hp.fs[a].size() * sizeof(double), cudaMemcpyHostToDevice));
    P.fc[a] = dc;
    P.fs[a] = ds;
    tmp.push_back(dc);
    tmp.push_back(ds);
  }
  ICPlan* dP;
  CK(cudaMalloc(&dP, sizeof(ICPlan)));
  tmp.push_back(dP);
  CK(cudaMemcpy(dP, &P, sizeof(ICPlan), cudaMemcpyHostToDevice));
  // everything on the handle's stream, ordered after its queued work; the
  // state buffers are fixed, so the captured step graphs stay valid
  CK(cudaStreamSynchronize(h->stream));
  if (hp.needs_norm) {
    unsigned long long* dm;
    CK(cudaMalloc(&dm, sizeof(unsigned long long)));
    tmp.push_back(dm);
    const long long n = (long long)h->g.nx * h->g.nm * h->nsa;
    for (int f = 0; f < 1 + P.dim; ++f) {
      CK(cudaMemsetAsync(dm, 0, sizeof(unsigned long long), h->stream));
      k_ic_norm<<<blocks(n, 128), 128, 0, h->stream>>>(dP, f, h->g, h->p0, dm);
      unsigned long long bits;
      CK(cudaMemcpyAsync(&bits, dm, sizeof(bits), cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      std::memcpy(&P.f[f].norm, &bits, sizeof(double));
    }
    CK(cudaMemcpyAsync(dP, &P, sizeof(ICPlan), cudaMemcpyHostToDevice, h->stream));
  }
  const long long n = (long long)h->g.nx * h->g.nm * h->g.np_loc;
  k_ic_fill<<<blocks(n, 128), 128, 0, h->stream>>>(dP, h->U0, h->g, h->p0);
  CK(cudaMemsetAsync(h->d_step, 0, 2 * sizeof(int), h->stream));
  CK(cudaStreamSynchronize(h->stream));
  for (void* p : tmp) cudaFree(p);
  return KFVM_OK;
}

// ------------------------------------------------------- FP64 peak probes
// DFMA: 8 independent FMA chains per thread; DMMA: mma.sync m8n8k4 f64.
// Used once per pool to measure the roofline denominator.
namespace kfvm_b200 {
__global__ void k_dfma_peak(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma_peak(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
            : "+d"(c[i][0]), "+d"(c[i][1])
            : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
}  // namespace kfvm_b200

extern "C" int kfvm_fp64_peak(double* dfma_tflops, double* dmma_tflops, double* sm_clock_ghz) {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double* d;
  if (cudaMalloc(&d, 64) != cudaSuccess) return KFVM_ERR_DEVICE;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 512, iters = 4096;
  const int grid = nsm * 4;
  float ms = 0;
  k_dfma_peak<<<grid, threads>>>(d, 16, 0.999, 1e-3);
  cudaEventRecord(e0);
  k_dfma_peak<<<grid, threads>>>(d, iters, 0.999, 1e-3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dfma = 2.0 * 8 * 16 * (double)iters * threads * grid;
  if (dfma_tflops) *dfma_tflops = dfma / (ms * 1e-3) / 1e12;
  k_dmma_peak<<<grid, threads>>>(d, 16);
  cudaEventRecord(e0);
  k_dmma_peak<<<grid, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  // one m8n8k4 per warp = 8*8*4 FMA = 512 flops
  const double dmma = 512.0 * 4 * 16 * (double)iters * (threads / 32) * grid;
  if (dmma_tflops) *dmma_tflops = dmma / (ms * 1e-3) / 1e12;
  if (sm_clock_ghz) {
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
    *sm_clock_ghz = khz * 1e-6;
  }
  cudaFree(d);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? KFVM_OK : KFVM_ERR_DEVICE;
}
