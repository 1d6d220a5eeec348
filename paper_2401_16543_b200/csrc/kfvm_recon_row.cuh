// kfvm_recon_row.cuh — the fused 2-D stage kernel: reconstruct_states
// with the unrolled DFMA contractions of k_states_fast, fed from
// shared memory, followed in the same kernel by the per-GL-point Riemann
// solves and the face quadrature — face states stay
// on chip except on the tile edges.
// Included inside namespace kfvm_b200 by kfvm_gpu.cu (after kfvm_recon.cuh).
//
// CTA = nv warps over a 32-cell x-segment that marches along the slab axis
// (y) over KZ extended rows.  The 2R+1 rows of U the stencils touch and the
// 3 rows of k_prims quantities the limiter touches live in cp.async ring
// buffers (one new row of each per step, prefetched while the current row
// computes), so the per-cell gathers and the neighbourhood statistics are
// shared-memory reads at compile-time offsets instead of remapped global
// loads.  Warp wv reconstructs variable wv of the 32 cells (same generated
// weno() as k_states_fast, same operation order), the shared Phi^-1 +
// limiter epilogue (epilogue_core) leaves the face states in shared memory,
// and the 2R Riemann point tasks of the row (x-faces between the segment's
// cells, y-faces against the previous row's N states, kept on chip) are
// spread over the warps; the face fluxes go to F for k_update.  Faces on the
// tile edges (x between segments, y between row blocks) get their states
// stored in St and are finished by k_flux_edges.
#ifndef KFVM_RECON_ROW_CUH_
#define KFVM_RECON_ROW_CUH_

#include <cuda_pipeline.h>

// resident CTAs per SM (register cap 80 / 96): measured on config 2
#ifndef KFVM_ROW_MINB
#define KFVM_ROW_MINB(R) ((R) == 2 ? 6 : 5)
#endif

template <int R>
struct RowCfg {
  static constexpr int nv = 4;
  static constexpr int RX = 32 + 2 * R;  // ring row: cells x0-R .. x0+31+R
  static constexpr int PL = nv * RX;
  static constexpr int RING = 2 * R + 2;
  static constexpr int NX = 34;          // prims row: cells x0-1 .. x0+32
  static constexpr int NF = 5;           // p, c, 1/rho, u, v
  static constexpr int PPL = NF * NX;
  static constexpr int PRING = 4;
};

// FUSE = false: the same row-marching reconstruction writing every face
// state to St (k_flux follows), for comparison.
// KX (with FUSE = false): KXRCF mode — the WENO part runs only for rows
// holding a flagged cell; every cell is limited here, unflagged ones from
// their pass-1 states in St.  P1: KXRCF pass 1 — raw conservative values
// through Gen::pass1 (r_0 vectors), unlimited states to St.
template <int R, bool FUSE, bool KX = false, bool P1 = false>
__global__ void __launch_bounds__(128, KFVM_ROW_MINB(R))
    k_stage_row(const double* __restrict__ U, const double* __restrict__ Pr,
                double* __restrict__ St, double* __restrict__ F, Geo g, Chunk ch, int KZ,
                int* __restrict__ err, const unsigned char* __restrict__ kfl = nullptr,
                int xsp = 0) {
  constexpr int D = 2, nv = 4;
  using G = Gen<2, R>;
  using C = RowCfg<R>;
  using E = EpiSmem<2, G::NP>;
  constexpr int NP = G::NP, RP = NP / 4;
  static_assert(E::SW >= NP * nv * 32, "face states alias the sW buffer");
  __shared__ __align__(16) double sRing[C::RING * C::PL];
  __shared__ __align__(16) double sPr[C::PRING * C::PPL];
  __shared__ double sW[E::SW];  // reconstruction-variable values, then face states [s][v][cell]
  __shared__ double sS[E::SS];
  __shared__ double sTh[E::STH];
  __shared__ double sN[RP * nv * 32];       // previous row's N states [m][v][cell]
  __shared__ double sFp[2 * RP * nv * 32];  // point fluxes [task][v][cell]
  double* sSt = sW;

  const int lane = threadIdx.x & 31, wv = threadIdx.x >> 5;
  // xsp = 1 (FUSE = false): the segments cover the interior x range only (the
  // two ring columns are computed by k_states_fast<2, R, true>)
  const int nseg = (ch.ex - 2 * xsp + 31) >> 5;
  const int seg = blockIdx.x % nseg;
  const int zblk = blockIdx.x / nseg;
  const int cstart = ch.e0 + zblk * KZ, cend = min(ch.e1, cstart + KZ);
  const int x0 = xsp + seg * 32 - 1;  // x of the segment's first extended cell
  const int a = xsp + seg * 32 + lane;
  const bool active = a < ch.ex - xsp;
  const int xr = lane + R;   // the lane's cell in a ring row
  const int icn = lane + 1;  // the lane's cell in a prims row

  // per-thread source offsets (the same for every row)
  constexpr int NLU = (C::PL + 127) / 128, NLP = (C::PPL + 127) / 128;
  unsigned offU[NLU], offP[NLP];
#pragma unroll
  for (int k = 0; k < NLU; ++k) {
    const int i = threadIdx.x + 128 * k;
    const int rx = i % C::RX, v = i / C::RX;
    offU[k] = i < C::PL ? (unsigned)(v * g.vstride + xoff(g, x0 - R + rx)) : 0u;
  }
#pragma unroll
  for (int k = 0; k < NLP; ++k) {
    const int i = threadIdx.x + 128 * k;
    const int rx = i % C::NX, f = i / C::NX;
    offP[k] = i < C::PPL ? (unsigned)(f * g.vstride + xoff(g, x0 - 1 + rx)) : 0u;
  }
  auto load_row = [&](int p) {
    double* dst = sRing + ((p + 4 * C::RING) % C::RING) * C::PL;
    const double* src = U + (long long)(p + g.H) * g.pstride;
#pragma unroll
    for (int k = 0; k < NLU; ++k) {
      const int i = threadIdx.x + 128 * k;
      if (i < C::PL) __pipeline_memcpy_async(dst + i, src + offU[k], sizeof(double));
    }
  };
  auto load_prims = [&](int p) {
    double* dst = sPr + ((p + 4 * C::PRING) % C::PRING) * C::PPL;
    const double* src = Pr + (long long)(p + g.H) * g.pstride;
#pragma unroll
    for (int k = 0; k < NLP; ++k) {
      const int i = threadIdx.x + 128 * k;
      if (i < C::PPL) __pipeline_memcpy_async(dst + i, src + offP[k], sizeof(double));
    }
  };
  {
    const int p = ch.c0 - 1 + cstart;
    for (int oz = -R; oz <= R; ++oz) load_row(p + oz);
    for (int oz = -1; oz <= 1; ++oz) load_prims(p + oz);
    __pipeline_commit();
    __pipeline_wait_prior(0);
  }
  __syncthreads();

  for (int c = cstart; c < cend; ++c) {
    const int p = ch.c0 - 1 + c;
    if (c + 1 < cend) {
      load_row(p + R + 1);
      load_prims(p + 2);
    }
    __pipeline_commit();
    bool anyflag = true;
    if constexpr (KX) anyflag = __syncthreads_or(active && kfl[(long long)c * ch.ex + a]) != 0;
    const int slot0 = (p - R + 4 * C::RING) % C::RING;  // ring slot of row p - R
    auto row = [&](int ozr) -> const double* {        // ozr = oz + R
      const int sl = slot0 + ozr;
      return sRing + (sl >= C::RING ? sl - C::RING : sl) * C::PL;
    };
    const double* pr0 = sPr + ((p + 4 * C::PRING) % C::PRING) * C::PPL;
    const double* prm = sPr + ((p - 1 + 4 * C::PRING) % C::PRING) * C::PPL;
    const double* prp = sPr + ((p + 1 + 4 * C::PRING) % C::PRING) * C::PPL;

    const double* rc = row(R);
    if constexpr (P1) {
      double u[G::N0], w[NP];
#pragma unroll
      for (int h = 0; h < G::N0; ++h)
        u[h] = row(G::off(h, 1) + R)[wv * C::RX + xr + G::off(h, 0)];
      G::pass1(u, w);
      if (active) {
        const long long tid = (long long)c * ch.ex + a;
#pragma unroll
        for (int s2 = 0; s2 < NP; ++s2) St[(long long)(s2 * nv + wv) * ch.next + tid] = w[s2];
      }
      __pipeline_wait_prior(0);
      __syncthreads();
      continue;
    }
    // ---- transform of the cell average (identical to tile_transform)
    DTransform T;
    T.rt = rc[xr];
    T.inv_r = pr0[2 * C::NX + icn];
    T.ut[0] = pr0[3 * C::NX + icn];
    T.ut[1] = pr0[4 * C::NX + icn];
    T.ut[2] = T.mt[2] = 0.0;
    T.mt[0] = rc[C::RX + xr];
    T.mt[1] = rc[2 * C::RX + xr];
    {
      double ke = T.ut[0] * T.ut[0];
      ke = fma(T.ut[1], T.ut[1], ke);
      T.ke = 0.5 * ke;
    }
    // ---- stencil values W_wv = (Phi U)_wv (same operations as gather_var)
    if (anyflag) {
      double gv[G::N0];
      if (wv == 0) {
#pragma unroll
        for (int h = 0; h < G::N0; ++h) gv[h] = row(G::off(h, 1) + R)[xr + G::off(h, 0)];
      } else if (wv <= D) {
        const double ut = wv == 1 ? T.ut[0] : T.ut[1];
        const int vo = wv * C::RX;
#pragma unroll
        for (int h = 0; h < G::N0; ++h) {
          const double* X = row(G::off(h, 1) + R) + xr + G::off(h, 0);
          gv[h] = fma(-ut, X[0], X[vo]) * T.inv_r;
        }
      } else {
#pragma unroll
        for (int h = 0; h < G::N0; ++h) {
          const double* X = row(G::off(h, 1) + R) + xr + G::off(h, 0);
          double t = fma(T.ke, X[0], X[3 * C::RX]);
          t = fma(-T.ut[0], X[C::RX], t);
          t = fma(-T.ut[1], X[2 * C::RX], t);
          gv[h] = c_k.gm1 * t;
        }
      }
      double w[NP];
      G::weno(gv, w, c_t.scale, c_t.gamma_lin, c_k.eps, c_t.inv_g0);
#pragma unroll
      for (int s2 = 0; s2 < NP; ++s2) sW[lane * (NP * nv + 1) + s2 * nv + wv] = w[s2];
    }
    // ---- neighbourhood statistics (same as tile_stats): warp wv -> stat wv
    {
      const int stat = wv;
      double r;
      if (stat < 2) {
        r = rc[xr];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
#pragma unroll
          for (int aa = -1; aa <= 1; ++aa) {
            const double v = row(R - 1 + cc)[xr + aa];
            r = stat == 0 ? fmax(r, v) : fmin(r, v);
          }
      } else {
        const int fo = (stat - 2) * C::NX + icn;
        r = pr0[fo];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          const double* prz = cc == 0 ? prm : (cc == 1 ? pr0 : prp);
#pragma unroll
          for (int aa = -1; aa <= 1; ++aa) r = fmin(r, prz[fo + aa]);
        }
      }
      sS[stat * 32 + lane] = r;
      if (wv == 0) {
        double dl = 0.5 * (pr0[3 * C::NX + icn + 1] - pr0[3 * C::NX + icn - 1]);
        dl = fma(0.5, prp[4 * C::NX + icn] - prm[4 * C::NX + icn], dl);
        sS[4 * 32 + lane] = dl;
      }
    }
    __syncthreads();
    // ---- Phi^-1 + limiter; face states to shared memory (and to St on the
    // tile edges, for k_flux_edges)
    {
      double Ubar[nv];
#pragma unroll
      for (int v = 0; v < nv; ++v) Ubar[v] = rc[v * C::RX + xr];
      const long long tid = (long long)c * ch.ex + a;
      const bool first = c == cstart, last = c == cend - 1;
      auto store = [&](int s2, int v, double u) {
                             if (!FUSE) {
                               St[(long long)(s2 * nv + v) * ch.next + tid] = u;
                               return;
                             }
                             sSt[(s2 * nv + v) * 32 + lane] = u;
                             const bool edge = (lane == 0 && s2 < RP) ||
                                               (lane == 31 && s2 >= RP && s2 < 2 * RP) ||
                                               (first && s2 >= 2 * RP && s2 < 3 * RP) ||
                                               (last && s2 >= 3 * RP);
                             if (edge) St[(long long)(s2 * nv + v) * ch.next + tid] = u;
                           };
      const double* p1 = KX && !(active && kfl[tid]) ? St + tid : nullptr;
      epilogue_core<D, NP, decltype(store)>(err, sW, sS, sTh, T, Ubar, pr0[icn], lane, wv, active,
                                            store, p1, ch.next);
    }
    if (!FUSE) {
      __pipeline_wait_prior(0);
      __syncthreads();
      continue;
    }
    __syncthreads();
    // ---- Riemann point tasks: x-faces (lane | lane+1), y-faces (row below | this row)
    const bool has_y = c > cstart;
    const int ln = lane < 31 ? lane + 1 : 31;
    for (int task = wv; task < 2 * RP; task += nv) {
      double UL[nv], UR[nv], Fp[nv];
      if (task < RP) {  // x-face point m: E of this lane's cell | W of the next cell
        const int m = task;
#pragma unroll
        for (int v = 0; v < nv; ++v) {
          UL[v] = sSt[((RP + m) * nv + v) * 32 + lane];
          UR[v] = sSt[(m * nv + v) * 32 + ln];
        }
        d_riemann<2>(c_k, 0, UL, UR, Fp);
      } else {  // y-face point m: N of the row below | S of this row
        if (!has_y) continue;
        const int m = task - RP;
#pragma unroll
        for (int v = 0; v < nv; ++v) {
          UL[v] = sN[(m * nv + v) * 32 + lane];
          UR[v] = sSt[((2 * RP + m) * nv + v) * 32 + lane];
        }
        d_riemann<2>(c_k, 1, UL, UR, Fp);
      }
#pragma unroll
      for (int v = 0; v < nv; ++v) sFp[(task * nv + v) * 32 + lane] = Fp[v];
    }
    __syncthreads();
    // ---- face quadrature -> F (k_flux's order), keep the N states for the next row
    const int cy = c - 1;  // interior-row index of this row (x-faces) / y-face index
    if (wv == 0) {
      if (lane < 31 && a <= g.nx && c >= 1 && c <= ch.C) {
        double Fb[nv];
#pragma unroll
        for (int v = 0; v < nv; ++v) Fb[v] = 0.0;
        for (int m = 0; m < RP; ++m)
#pragma unroll
          for (int v = 0; v < nv; ++v)
            Fb[v] = fma(c_t.face_w[m], sFp[(m * nv + v) * 32 + lane], Fb[v]);
        const long long f = (long long)cy * ch.fx + a;
#pragma unroll
        for (int v = 0; v < nv; ++v) F[(long long)v * ch.nfb + f] = Fb[v];
      }
    } else if (wv == 1) {
      if (has_y && a >= 1 && a <= g.nx) {
        double Fb[nv];
#pragma unroll
        for (int v = 0; v < nv; ++v) Fb[v] = 0.0;
        for (int m = 0; m < RP; ++m)
#pragma unroll
          for (int v = 0; v < nv; ++v)
            Fb[v] = fma(c_t.face_w[2 * RP + m], sFp[((RP + m) * nv + v) * 32 + lane], Fb[v]);
        const long long f = (long long)cy * ch.fx + (a - 1);
#pragma unroll
        for (int v = 0; v < nv; ++v) F[(long long)(nv + v) * ch.nfb + f] = Fb[v];
      }
    } else {
      for (int i = threadIdx.x - 64; i < RP * nv * 32; i += 64)
        sN[i] = sSt[3 * RP * nv * 32 + i];
    }
    __pipeline_wait_prior(0);
    __syncthreads();
  }
}

#endif
