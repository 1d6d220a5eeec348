// kfvm_fused3.cuh — 3-D stage kernel: reconstruction (FP64 tensor cores) fused
// with the per-quadrature-point Riemann solves and the face quadrature
// (BASELINE north_star (2); SURVEY.md §7 hard part 4(b)).  Face states never
// reach HBM except on tile edges.  Included inside namespace kfvm_b200 by
// kfvm_gpu.cu, after kfvm_recon_u.cuh (whose DMMA passes it shares: same
// chunk tables, same B fragments, same pinned contract — DESIGN.md §4).
//
// Work decomposition.  A CTA = 4 warps owns an 8 (x) x 4 (y) tile of the
// extended box and marches KZ planes along z.  Warp w is tile row w; lane
// (r8, k4) = quad r8 is the cell in column r8, k4 its DMMA k-slot (the A
// fragment row is the lane's own cell, as in k_states_u).  After the passes
// and the limiter, lane k4 holds the states of points s = 8n + 2k4 + e
// (n = 0: W|E, 1: S|N, 2: B|T; k4 0,1 the minus faces, 2,3 the plus faces).
// Every cell solves its three minus faces, lane k4 the GL point m = k4 of each
// (3 HLLC/HLL solves per lane):
//   x (W face): right states from the lane's own quad, left states (E) from
//     quad r8 - 1 of the same warp, by shuffles;
//   y (S face): left states (N) of tile row w - 1 through shared memory;
//   z (B face): left states (T) of the previous plane, kept in shared memory
//     by the same lanes.
// The quad then forms the GL quadrature of each face (one fma chain per face
// and variable in point order, the oracle's order) and writes the face flux.
// Faces on a tile edge (column 0's W face, row 0's S face, the first plane of
// a z-block) have their two sides written to compact edge buffers and are
// solved by k_edges3, which runs the same Riemann + quadrature code.
#ifndef KFVM_FUSED3_CUH_
#define KFVM_FUSED3_CUH_

constexpr int kTX = 8, kTY = 4;  // tile: 8 x-cells x 4 rows, warp = row
// KFVM_ABL_* (timing ablations for tools/gpu/r2_abl.sh; results are wrong
// when any is set): NOPHI skips the stencil transforms in both passes,
// NORIEMANN the Riemann solves, NOLIMIT the limiter, NOBETA the smoothness
// indicators, NOTAIL the tail derivative chains.
#ifndef KFVM_F3_MINB  // resident CTAs per SM the register budget is sized for
#define KFVM_F3_MINB 3
#endif

template <int R>
struct FCfg {
  using G = Gen<3, R>;
  static constexpr int nv = 5;
  static constexpr int ND = (G::NA + 7) / 8;
  static constexpr int NDM = G::NA / 8;
  static constexpr int NT = G::NA - 8 * NDM;
  static constexpr int NPT = (G::NP + 7) / 8;
  static constexpr int RX = kTX + 2 * R, RY = kTY + 2 * R;
  static constexpr int RROW = RY * RX;   // one variable of a region plane
  static constexpr int PL = nv * RROW;   // one region plane
  static constexpr int RING = 2 * R + 2;
  static constexpr int NX = kTX + 2, NY = kTY + 2, NF = 6;  // prims neighbourhood
  static constexpr int PROW = NY * NX, PPL = NF * PROW, PRING = 4;
  static constexpr int SCW = G::NS * nv * 8;     // beta / c_q per warp
  static constexpr int RP = R * R;               // GL points per face
  static constexpr int XB = kTY * kTX * RP * nv;  // one face-state exchange buffer
  static constexpr size_t bytes() {
    return sizeof(double) * (RING * PL + PRING * PPL + 4 * SCW + 2 * XB) +
           sizeof(int) * (9 * G::NCHUNK);
  }
};

// Edge-face buffers (two sides, [side][m][v][face]) and the z-block layout
// of the stage's launches (disjoint plane ranges [r0, r1) of the extended
// box, sorted by r0, blocks of KZ planes from each r0).
struct Edges {
  double *x, *y, *z;
  long long sx, sy, sz;  // elements per (side, m, v) row
  int nxe, nye, nzs;     // x / y edge positions, z edge slots
  int KZ, nr;
  int r0[3], r1[3];
};

__host__ __device__ __forceinline__ int edge_nblocks(const Edges& E, int r) {
  return (E.r1[r] - E.r0[r] + E.KZ - 1) / E.KZ;
}
// slot of the z-edge at block start c > 0: block starts below c, minus plane 0
__device__ __forceinline__ int zslot(const Edges& E, int c) {
  int n = 0;
  for (int r = 0; r < E.nr; ++r) {
    if (c <= E.r0[r]) continue;
    const int k = (c - E.r0[r] + E.KZ - 1) / E.KZ;
    const int nb = edge_nblocks(E, r);
    n += k < nb ? k : nb;
  }
  return n - 1;
}
__device__ __forceinline__ int zslot_plane(const Edges& E, int s) {
  int i = s + 1;
  for (int r = 0; r < E.nr; ++r) {
    const int nb = edge_nblocks(E, r);
    if (i < nb) return E.r0[r] + i * E.KZ;
    i -= nb;
  }
  return -1;
}

template <int R, int DIR>
__device__ __forceinline__ void edge_store(double* buf, long long rowlen, int side, int m,
                                           long long idx, const double* u) {
#pragma unroll
  for (int v = 0; v < 5; ++v) buf[((long long)(side * R * R + m) * 5 + v) * rowlen + idx] = u[v];
}

template <int R>
__global__ void __launch_bounds__(128, KFVM_F3_MINB)
    k_fused3(const double* __restrict__ U, const double* __restrict__ Pr, double* __restrict__ F,
             Geo g, Chunk ch, Edges E, int rng, int* __restrict__ err,
             const double* __restrict__ Bd, const double* __restrict__ Bf,
             const int* __restrict__ gat8) {
  using G = Gen<3, R>;
  using C = FCfg<R>;
  constexpr int nv = 5, NP = G::NP, NS = G::NS, ND = C::ND, NPT = C::NPT, RP = C::RP;
  static_assert(NPT == 3 && NP == 24, "the fused engine holds the 24 points of 3-D R=2 in registers");
  extern __shared__ double smem[];
  double* sRing = smem;                          // [RING][nv][RY][RX]
  double* sPr = sRing + C::RING * C::PL;         // [PRING][NF][NY][NX]
  double* sC = sPr + C::PRING * C::PPL;          // [warp][q][v][8]
  double* sN = sC + 4 * C::SCW;                  // N states [row][col][m][v]
  double* sT = sN + C::XB;                       // T states of the previous plane
  int* sTab = reinterpret_cast<int*>(sT + C::XB);  // [chunk][4] {inplane, oz}
  int* sQ = sTab + 8 * G::NCHUNK;                  // stencil | last << 8

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k4 = lane & 3, r8 = lane >> 2;
  for (int i = threadIdx.x; i < 9 * G::NCHUNK; i += 128) sTab[i] = gat8[i];

  const int ntx = (ch.ex + kTX - 1) / kTX, nty = (ch.em + kTY - 1) / kTY;
  int bid = blockIdx.x;
  const int tx = bid % ntx;
  bid /= ntx;
  const int ty = bid % nty;
  const int zb = bid / nty;
  const int cstart = E.r0[rng] + zb * E.KZ, cend = min(E.r1[rng], cstart + E.KZ);
  const int a = tx * kTX + r8, b = ty * kTY + w;  // extended cell of this lane
  const bool active = a < ch.ex && b < ch.em;
  const int x0 = tx * kTX - 1, j0 = ty * kTY - 1;  // storage x / row of the tile's first cell
  const int xlo = -g.G, xhi = g.nx + g.G - 1, jlo = -g.Gm, jhi = g.nm + g.Gm - 1;

  auto load_plane = [&](int p) {  // region plane p -> ring slot (clamped: only inactive cells see it)
    double* dst = sRing + ((p + 4 * C::RING) % C::RING) * C::PL;
    const long long pbase = (long long)(p + g.H) * g.pstride;
    for (int i = threadIdx.x; i < C::PL; i += 128) {
      const int rx = i % C::RX, rr = i / C::RX;
      const int ry = rr % C::RY, v = rr / C::RY;
      const int xx = min(max(x0 - R + rx, xlo), xhi), jj = min(max(j0 - R + ry, jlo), jhi);
      __pipeline_memcpy_async(dst + i, U + v * g.vstride + pbase + xoff(g, xx) + moff(g, jj),
                              sizeof(double));
    }
  };
  auto load_prims = [&](int p) {
    double* dst = sPr + ((p + 4 * C::PRING) % C::PRING) * C::PPL;
    const long long pbase = (long long)(p + g.H) * g.pstride;
    for (int i = threadIdx.x; i < C::PPL; i += 128) {
      const int rx = i % C::NX, rr = i / C::NX;
      const int ry = rr % C::NY, f = rr / C::NY;
      const int xx = min(max(x0 - 1 + rx, xlo), xhi), jj = min(max(j0 - 1 + ry, jlo), jhi);
      __pipeline_memcpy_async(dst + i, Pr + f * g.vstride + pbase + xoff(g, xx) + moff(g, jj),
                              sizeof(double));
    }
  };
  {
    const int p = ch.c0 - 1 + cstart;
    for (int oz = -R; oz <= R; ++oz) load_plane(p + oz);
    for (int oz = -1; oz <= 1; ++oz) load_prims(p + oz);
    __pipeline_commit();
    __pipeline_wait_prior(0);
  }
  __syncthreads();

  double* sCw = sC + w * C::SCW;
  const int cb = w * C::RX + r8;                          // the cell's region base
  const int icr = (w + R) * C::RX + r8 + R;               // cell centre in a region plane
  const int icn = (w + 1) * C::NX + r8 + 1;               // cell centre in a prims plane
  const int qb = lane & ~3;
  PHASE_T0();
  for (int c = cstart; c < cend; ++c) {
    const int p = ch.c0 - 1 + c;
    if (c + 1 < cend) {
      load_plane(p + R + 1);
      load_prims(p + 2);
    }
    __pipeline_commit();
    const int slot0 = (p - R + 4 * C::RING) % C::RING;
    auto plane = [&](int ozr) -> const double* {
      const int sl = slot0 + ozr;
      return sRing + (sl >= C::RING ? sl - C::RING : sl) * C::PL;
    };
    const double* pr0 = sPr + ((p + 4 * C::PRING) % C::PRING) * C::PPL;
    const double* prm = sPr + ((p - 1 + 4 * C::PRING) % C::PRING) * C::PPL;
    const double* prp = sPr + ((p + 1 + 4 * C::PRING) % C::PRING) * C::PPL;
    DTransform T;
    T.rt = plane(R)[icr];
    T.inv_r = pr0[2 * C::PROW + icn];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      T.ut[d] = pr0[(3 + d) * C::PROW + icn];
      T.mt[d] = plane(R)[(1 + d) * C::RROW + icr];
    }
    {
      double ke = T.ut[0] * T.ut[0];
      ke = fma(T.ut[1], T.ut[1], ke);
      ke = fma(T.ut[2], T.ut[2], ke);
      T.ke = 0.5 * ke;
    }
    PHASE_MARK(0);
    // ---- pass 1: derivative columns -> beta (k_states_u order).  The stencil
    // structure is unrolled at compile time and two accumulator sets
    // alternate between stencils, so the smoothness indicator of stencil q
    // (its partial sums, tail chains and quad reductions) is formed while the
    // DMMAs of stencil q + 1 are in flight instead of stalling on them.
    {
      constexpr int NDM = C::NDM, NT = C::NT, NTA = NT > 0 ? NT : 1;
      double acc[2][nv][NDM][2];
      double tl[2][nv][NTA];
      double av[nv], bv[NDM], bt[NTA];
      {
        const int inpl = sTab[2 * k4], oz = sTab[2 * k4 + 1];
        const double* ap = plane(oz + R) + inpl + cb;
#pragma unroll
        for (int u = 0; u < nv; ++u) av[u] = ap[u * C::RROW];
#pragma unroll
        for (int n = 0; n < NDM; ++n) bv[n] = Bd[n * 32 + lane];
#pragma unroll
        for (int t = 0; t < NT; ++t) bt[t] = Bd[(ND - 1) * 32 + 4 * t + k4];
      }
      // beta of stencil q from accumulator set s (k_states_u's operation order)
      auto beta = [&](int q, int s) {
        double bq[nv];
#pragma unroll
        for (int v = 0; v < nv; ++v) bq[v] = 0.0;
#pragma unroll
        for (int n = 0; n < NDM; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int al = 8 * n + 2 * k4 + e;
            const double sc = al < G::NA ? c_t.scale[al] : 0.0;
#pragma unroll
            for (int v = 0; v < nv; ++v)
              if (al < G::NA) bq[v] = fma(sc, acc[s][v][n][e] * acc[s][v][n][e], bq[v]);
          }
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int al = 8 * NDM + t;
#pragma unroll
          for (int v = 0; v < nv; ++v) {
            double d = tl[s][v][t] + __shfl_xor_sync(0xffffffffu, tl[s][v][t], 1);
            d = d + __shfl_xor_sync(0xffffffffu, d, 2);
            if ((t >> 1) == k4) bq[v] = fma(c_t.scale[al], d * d, bq[v]);
          }
        }
#pragma unroll
        for (int v = 0; v < nv; ++v) {
          bq[v] = bq[v] + __shfl_xor_sync(0xffffffffu, bq[v], 1);
          bq[v] = bq[v] + __shfl_xor_sync(0xffffffffu, bq[v], 2);
        }
        if (k4 == 0) {
#pragma unroll
          for (int v = 0; v < nv; ++v) sCw[(q * nv + v) * 8 + r8] = bq[v];
        }
      };
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        const int s = q & 1;
#pragma unroll
        for (int u = 0; u < nv; ++u) {
#pragma unroll
          for (int n = 0; n < NDM; ++n) acc[s][u][n][0] = acc[s][u][n][1] = 0.0;
#pragma unroll
          for (int t = 0; t < NTA; ++t) tl[s][u][t] = 0.0;
        }
#pragma unroll
        for (int jj = 0; jj < G::kc(q); ++jj) {
          const int ck = G::cbase(q) + jj;
          const int cn = ck + 1 < G::NCHUNK ? ck + 1 : ck;
          const int inpl = sTab[2 * (cn * 4 + k4)], oz = sTab[2 * (cn * 4 + k4) + 1];
          const double* ap = plane(oz + R) + inpl + cb;
          double an[nv], bn[NDM], btn[NTA];
#pragma unroll
          for (int u = 0; u < nv; ++u) an[u] = ap[u * C::RROW];
#pragma unroll
          for (int n = 0; n < NDM; ++n) bn[n] = Bd[(cn * ND + n) * 32 + lane];
#pragma unroll
          for (int t = 0; t < NT; ++t) btn[t] = Bd[(cn * ND + ND - 1) * 32 + 4 * t + k4];
          double aw[nv];
#pragma unroll
          for (int v = 0; v < nv; ++v) {
#ifdef KFVM_ABL_NOPHI
            aw[v] = av[v];
#else
            aw[v] = phi_row<3>(T, av, v);
#endif
          }
#pragma unroll
          for (int n = 0; n < NDM; ++n)
#pragma unroll
            for (int v = 0; v < nv; ++v) dmma(acc[s][v][n][0], acc[s][v][n][1], aw[v], bv[n]);
#pragma unroll
          for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int v = 0; v < nv; ++v) tl[s][v][t] = fma(bt[t], aw[v], tl[s][v][t]);
#pragma unroll
          for (int u = 0; u < nv; ++u) av[u] = an[u];
#pragma unroll
          for (int n = 0; n < NDM; ++n) bv[n] = bn[n];
#pragma unroll
          for (int t = 0; t < NT; ++t) bt[t] = btn[t];
          if (q > 0 && jj == 0) beta(q - 1, s ^ 1);  // after the first chunk of stencil q
        }
      }
      beta(NS - 1, (NS - 1) & 1);
    }
    __syncwarp();
    PHASE_MARK(1);
    // ---- nonlinear weights (k_states_u order)
#pragma unroll
    for (int q = k4; q < NS; q += 4)
#pragma unroll
      for (int v = 0; v < nv; ++v) {
        const double bb = sCw[(q * nv + v) * 8 + r8];
        sCw[(q * nv + v) * 8 + r8] = c_t.gamma_lin[q] * (1.0 / fma(bb, bb, c_k.eps));
      }
    __syncwarp();
    for (int v = k4; v < nv; v += 4) {
      double wt[NS];
#pragma unroll
      for (int q = 0; q < NS; ++q) wt[q] = sCw[(q * nv + v) * 8 + r8];
      double sum = wt[0];
#pragma unroll
      for (int q = 1; q < NS; ++q) sum = sum + wt[q];
      const double inv_sum = 1.0 / sum;
      const double c0 = (wt[0] * inv_sum) * c_t.inv_g0;
      sCw[v * 8 + r8] = c0;
#pragma unroll
      for (int q = 1; q < NS; ++q) sCw[(q * nv + v) * 8 + r8] = fma(-c0, c_t.gamma_lin[q], wt[q] * inv_sum);
    }
    __syncwarp();
    PHASE_MARK(2);
    // ---- pass 2: every face point, one chain per (variable, point) through all stencils
    double V[nv][NPT][2];
    {
#pragma unroll
      for (int u = 0; u < nv; ++u)
#pragma unroll
        for (int n = 0; n < NPT; ++n) V[u][n][0] = V[u][n][1] = 0.0;
      int q = 0;
      double cq[nv];
#pragma unroll
      for (int v = 0; v < nv; ++v) cq[v] = sCw[v * 8 + r8];
      double av[nv], bv[NPT];
      {
        const int inpl = sTab[2 * k4], oz = sTab[2 * k4 + 1];
        const double* ap = plane(oz + R) + inpl + cb;
#pragma unroll
        for (int u = 0; u < nv; ++u) av[u] = ap[u * C::RROW];
#pragma unroll
        for (int n = 0; n < NPT; ++n) bv[n] = Bf[n * 32 + lane];
      }
#pragma unroll kUChunkUnroll
      for (int ck = 0; ck < G::NCHUNK; ++ck) {
        const int cn = ck + 1 < G::NCHUNK ? ck + 1 : ck;
        const int inpl = sTab[2 * (cn * 4 + k4)], oz = sTab[2 * (cn * 4 + k4) + 1];
        const double* ap = plane(oz + R) + inpl + cb;
        double an[nv], bn[NPT];
#pragma unroll
        for (int u = 0; u < nv; ++u) an[u] = ap[u * C::RROW];
#pragma unroll
        for (int n = 0; n < NPT; ++n) bn[n] = Bf[(cn * NPT + n) * 32 + lane];
        double aw[nv];
#pragma unroll
        for (int v = 0; v < nv; ++v) {
#ifdef KFVM_ABL_NOPHI
          aw[v] = cq[v] * av[v];
#else
          aw[v] = cq[v] * phi_row<3>(T, av, v);
#endif
        }
#pragma unroll
        for (int n = 0; n < NPT; ++n)
#pragma unroll
          for (int v = 0; v < nv; ++v) dmma(V[v][n][0], V[v][n][1], aw[v], bv[n]);
#pragma unroll
        for (int u = 0; u < nv; ++u) av[u] = an[u];
#pragma unroll
        for (int n = 0; n < NPT; ++n) bv[n] = bn[n];
        if ((sQ[ck] & 256) && q + 1 < NS) {
          ++q;
#pragma unroll
          for (int v = 0; v < nv; ++v) cq[v] = sCw[(q * nv + v) * 8 + r8];
        }
      }
    }
    PHASE_MARK(3);
    // ---- Phi^-1 and the positivity limiter (the k_states_u epilogue)
    double st[NPT][2][nv];
#pragma unroll
    for (int n = 0; n < NPT; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double Wp[nv];
#pragma unroll
        for (int v = 0; v < nv; ++v) Wp[v] = V[v][n][e];
        d_from_recon(3, T, c_k.inv_gm1, Wp, st[n][e]);
      }
    double Ubar[nv];
    {
      double rbmax = T.rt, rbmin = T.rt, pbmin = pr0[icn], cmin = pr0[C::PROW + icn];
      for (int mm = k4; mm < 27; mm += 4) {
        const int aa = mm % 3 - 1, bb = (mm / 3) % 3 - 1, cc = mm / 9 - 1;
        const double r = plane(R + cc)[bb * C::RX + icr + aa];
        const double* prz = cc < 0 ? prm : (cc > 0 ? prp : pr0);
        const int ip = bb * C::NX + icn + aa;
        rbmax = fmax(rbmax, r);
        rbmin = fmin(rbmin, r);
        pbmin = fmin(pbmin, prz[ip]);
        cmin = fmin(cmin, prz[C::PROW + ip]);
      }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        rbmax = fmax(rbmax, __shfl_xor_sync(0xffffffffu, rbmax, o));
        rbmin = fmin(rbmin, __shfl_xor_sync(0xffffffffu, rbmin, o));
        pbmin = fmin(pbmin, __shfl_xor_sync(0xffffffffu, pbmin, o));
        cmin = fmin(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
      }
      double delta = 0.5 * (pr0[3 * C::PROW + icn + 1] - pr0[3 * C::PROW + icn - 1]);
      delta = fma(0.5, pr0[4 * C::PROW + icn + C::NX] - pr0[4 * C::PROW + icn - C::NX], delta);
      delta = fma(0.5, prp[5 * C::PROW + icn] - prm[5 * C::PROW + icn], delta);
      const double kc = c_k.kf * cmin;
      double eta = -(delta + kc) / kc;
      eta = fmin(1.0, fmax(0.0, eta));
      const double fup = fma(c_k.kappa, 1.0 - eta, 1.0);
      const double flo = fma(-c_k.kappa, 1.0 - eta, 1.0);
      const double rmax = rbmax * fup, rmin = rbmin * flo, pmin = pbmin * flo;
      const double rt = T.rt, pt = pr0[icn];
      if (!(rt > 0.0) || !(pt > 0.0) || !(rmin > 0.0) || !(pmin > 0.0))
        if (active && k4 == 0) atomicOr(err, 2);
      Ubar[0] = rt;
#pragma unroll
      for (int d = 0; d < 3; ++d) Ubar[1 + d] = T.mt[d];
      Ubar[nv - 1] = plane(R)[(nv - 1) * C::RROW + icr];
#ifndef KFVM_ABL_NOLIMIT
      double th = 1.0;
#pragma unroll
      for (int n = 0; n < NPT; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double r = st[n][e][0];
          if (r < rmin)
            th = fmin(th, (rt - rmin) / (rt - r));
          else if (r > rmax)
            th = fmin(th, (rmax - rt) / (r - rt));
        }
      th = fmin(th, __shfl_xor_sync(0xffffffffu, th, 1));
      th = fmin(th, __shfl_xor_sync(0xffffffffu, th, 2));
      if (th < 1.0) {
#pragma unroll
        for (int n = 0; n < NPT; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int v = 0; v < nv; ++v) st[n][e][v] = fma(th, st[n][e][v] - Ubar[v], Ubar[v]);
      }
      double thp = 1.0;
#pragma unroll
      for (int n = 0; n < NPT; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (d_p_below(3, st[n][e], c_k.gm1, pmin)) {
            StateV<3> a_, b_;
#pragma unroll
            for (int v = 0; v < nv; ++v) {
              a_.v[v] = st[n][e][v];
              b_.v[v] = Ubar[v];
            }
            thp = fmin(thp, theta_p_bisect<3>(a_, b_, pmin));
          }
      thp = fmin(thp, __shfl_xor_sync(0xffffffffu, thp, 1));
      thp = fmin(thp, __shfl_xor_sync(0xffffffffu, thp, 2));
      if (thp < 1.0) {
#pragma unroll
        for (int n = 0; n < NPT; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int v = 0; v < nv; ++v) st[n][e][v] = fma(thp, st[n][e][v] - Ubar[v], Ubar[v]);
      }
#endif
    }
    PHASE_MARK(4);
    // ---- face-state exchange.  Lane k4 holds face points m = 2 (k4 & 1) + e
    // of the minus (k4 < 2) or plus (k4 >= 2) faces.
    const bool plus = k4 >= 2;
    const int mb = 2 * (k4 & 1);
    if (plus) {  // N states -> the next tile row (shared memory)
      double* nb = sN + ((w * kTX + r8) * RP) * nv;
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int v = 0; v < nv; ++v) nb[(mb + e) * nv + v] = st[1][e][v];
    }
    if (active) {  // tile-edge faces: both sides to the edge buffers
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = mb + e;
        if (plus) {
          if (r8 == kTX - 1 && a + 1 < ch.ex)
            edge_store<R, 0>(E.x, E.sx, 0, m, ((long long)c * ch.em + b) * E.nxe + tx, st[0][e]);
          if (w == kTY - 1 && b + 1 < ch.em)
            edge_store<R, 1>(E.y, E.sy, 0, m, ((long long)c * E.nye + ty) * ch.ex + a, st[1][e]);
          if (c == cend - 1 && c + 1 < ch.ep)
            edge_store<R, 2>(E.z, E.sz, 0, m, ((long long)zslot(E, cend) * ch.em + b) * ch.ex + a,
                             st[2][e]);
        } else {
          if (r8 == 0 && tx >= 1)
            edge_store<R, 0>(E.x, E.sx, 1, m, ((long long)c * ch.em + b) * E.nxe + tx - 1, st[0][e]);
          if (w == 0 && ty >= 1)
            edge_store<R, 1>(E.y, E.sy, 1, m, ((long long)c * E.nye + ty - 1) * ch.ex + a, st[1][e]);
          if (c == cstart && c > 0)
            edge_store<R, 2>(E.z, E.sz, 1, m, ((long long)zslot(E, cstart) * ch.em + b) * ch.ex + a,
                             st[2][e]);
        }
      }
    }
    __syncthreads();  // N states of every tile row visible
    PHASE_MARK(5);
    // ---- Riemann solves: lane k4 takes point m = k4 of the cell's W, S, B faces
    const bool inx = a >= 1 && a <= ch.ex - 2, iny = b >= 1 && b <= ch.em - 2,
               inz = c >= 1 && c <= ch.ep - 2;
    const bool vx = active && r8 >= 1 && a >= 1 && iny && inz;
    const bool vy = active && w >= 1 && b >= 1 && inx && inz;
    const bool vz = active && c > cstart && c >= 1 && inx && iny;
    double FL[3][nv];
    {
      const int srcR = qb + (k4 >> 1), srcL = ((qb - 4) & 31) + 2 + (k4 >> 1);
      const bool odd = k4 & 1;
      double UR[3][nv], UL[nv];
#pragma unroll
      for (int n = 0; n < 3; ++n)
#pragma unroll
        for (int v = 0; v < nv; ++v) {
          const double x0v = __shfl_sync(0xffffffffu, st[n][0][v], srcR);
          const double x1v = __shfl_sync(0xffffffffu, st[n][1][v], srcR);
          UR[n][v] = odd ? x1v : x0v;
        }
#pragma unroll
      for (int v = 0; v < nv; ++v) {
        const double x0v = __shfl_sync(0xffffffffu, st[0][0][v], srcL);
        const double x1v = __shfl_sync(0xffffffffu, st[0][1][v], srcL);
        UL[v] = odd ? x1v : x0v;
      }
      // all three solves as straight-line code (interleaved for ILP); the
      // left states of an invalid face are whatever the buffers hold and the
      // result is discarded
      double ULy[nv], ULz[nv];
      const double* nb = sN + (((w > 0 ? w - 1 : 0) * kTX + r8) * RP + k4) * nv;
      const double* tb = sT + ((w * kTX + r8) * RP + k4) * nv;
#pragma unroll
      for (int v = 0; v < nv; ++v) {
        ULy[v] = nb[v];
        ULz[v] = tb[v];
      }
#ifdef KFVM_ABL_NORIEMANN
#pragma unroll
      for (int v = 0; v < nv; ++v) {
        FL[0][v] = UL[v] + UR[0][v];
        FL[1][v] = ULy[v] + UR[1][v];
        FL[2][v] = ULz[v] + UR[2][v];
      }
#else
      d_riemann_sel<3, 0>(c_k, UL, UR[0], FL[0]);
      d_riemann_sel<3, 1>(c_k, ULy, UR[1], FL[1]);
      d_riemann_sel<3, 2>(c_k, ULz, UR[2], FL[2]);
#endif
#pragma unroll
      for (int v = 0; v < nv; ++v) {
        FL[0][v] = vx ? FL[0][v] : 0.0;
        FL[1][v] = vy ? FL[1][v] : 0.0;
        FL[2][v] = vz ? FL[2][v] : 0.0;
      }
    }
    // ---- face quadrature: lane d of the quad forms face d's flux in point order
    {
      const int d = k4 < 3 ? k4 : 2;
      double Fq[nv];
#pragma unroll
      for (int v = 0; v < nv; ++v) Fq[v] = 0.0;
#pragma unroll
      for (int m = 0; m < RP; ++m) {
        const double wm = c_t.face_w[2 * d * RP + m];
#pragma unroll
        for (int v = 0; v < nv; ++v) {
          const double f0 = __shfl_sync(0xffffffffu, FL[0][v], qb + m);
          const double f1 = __shfl_sync(0xffffffffu, FL[1][v], qb + m);
          const double f2 = __shfl_sync(0xffffffffu, FL[2][v], qb + m);
          Fq[v] = fma(wm, d == 0 ? f0 : (d == 1 ? f1 : f2), Fq[v]);
        }
      }
      const bool vd = d == 0 ? vx : (d == 1 ? vy : vz);
      if (k4 < 3 && vd) {
        const long long f = ((long long)(c - 1) * ch.fm + (b - 1)) * ch.fx + (a - 1);
#pragma unroll
        for (int v = 0; v < nv; ++v) F[(long long)(d * nv + v) * ch.nfb + f] = Fq[v];
      }
    }
    __syncwarp();
    if (plus) {  // T states for the next plane's B faces (same lanes' quads)
      double* tb = sT + ((w * kTX + r8) * RP) * nv;
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int v = 0; v < nv; ++v) tb[(mb + e) * nv + v] = st[2][e][v];
    }
    PHASE_MARK(6);
    __pipeline_wait_prior(0);
    __syncthreads();
    PHASE_MARK(7);
  }
}

// Faces on the tile edges of k_fused3: both sides from the edge buffers, the
// same Riemann solve and quadrature order as the fused kernel.
template <int R>
__global__ void __launch_bounds__(128) k_edges3(double* __restrict__ F, Chunk ch, Edges E) {
  constexpr int nv = 5, RP = R * R;
  const long long nx_ = (long long)E.nxe * ch.em * ch.ep, ny_ = (long long)E.nye * ch.ex * ch.ep,
                  nz_ = (long long)E.nzs * ch.em * ch.ex;
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int d, a, b, c;
  const double* buf;
  long long rowlen, idx;
  if (t < nx_) {
    const int ix = (int)(t % E.nxe);
    const long long r = t / E.nxe;
    b = (int)(r % ch.em);
    c = (int)(r / ch.em);
    a = kTX * (ix + 1);
    d = 0;
    buf = E.x;
    rowlen = E.sx;
    idx = t;
    if (!(a <= ch.ex - 1 && b >= 1 && b <= ch.em - 2 && c >= 1 && c <= ch.ep - 2)) return;
  } else if ((t -= nx_) < ny_) {
    a = (int)(t % ch.ex);
    const long long r = t / ch.ex;
    const int iy = (int)(r % E.nye);
    c = (int)(r / E.nye);
    b = kTY * (iy + 1);
    d = 1;
    buf = E.y;
    rowlen = E.sy;
    idx = t;
    if (!(b <= ch.em - 1 && a >= 1 && a <= ch.ex - 2 && c >= 1 && c <= ch.ep - 2)) return;
  } else if ((t -= ny_) < nz_) {
    a = (int)(t % ch.ex);
    const long long r = t / ch.ex;
    b = (int)(r % ch.em);
    const int s = (int)(r / ch.em);
    c = zslot_plane(E, s);
    d = 2;
    buf = E.z;
    rowlen = E.sz;
    idx = t;
    if (!(c >= 1 && c <= ch.ep - 1 && a >= 1 && a <= ch.ex - 2 && b >= 1 && b <= ch.em - 2)) return;
  } else {
    return;
  }
  double Fb[nv];
#pragma unroll
  for (int v = 0; v < nv; ++v) Fb[v] = 0.0;
  for (int m = 0; m < RP; ++m) {
    double UL[nv], UR[nv], Fp[nv];
#pragma unroll
    for (int v = 0; v < nv; ++v) {
      UL[v] = buf[((long long)(0 * RP + m) * nv + v) * rowlen + idx];
      UR[v] = buf[((long long)(1 * RP + m) * nv + v) * rowlen + idx];
    }
    if (d == 0)
      d_riemann_dir<3, 0>(c_k, UL, UR, Fp);
    else if (d == 1)
      d_riemann_dir<3, 1>(c_k, UL, UR, Fp);
    else
      d_riemann_dir<3, 2>(c_k, UL, UR, Fp);
    const double wm = c_t.face_w[2 * d * RP + m];
#pragma unroll
    for (int v = 0; v < nv; ++v) Fb[v] = fma(wm, Fp[v], Fb[v]);
  }
  const long long f = ((long long)(c - 1) * ch.fm + (b - 1)) * ch.fx + (a - 1);
#pragma unroll
  for (int v = 0; v < nv; ++v) F[(long long)(d * nv + v) * ch.nfb + f] = Fb[v];
}

#endif
