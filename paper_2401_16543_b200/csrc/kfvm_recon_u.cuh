// kfvm_recon_u.cuh — reconstruct_states on the FP64 tensor cores,
// plane-marching CTAs with a cp.async ring buffer.
// Included inside namespace kfvm_b200 by kfvm_gpu.cu.
//
// Contract (oracle weno_field): the stencil values are the
// linearized primitives W = Phi U of the central cell; every derivative /
// face-point vector of every (sub)stencil is contracted with them in
// stencil-order fma chains, here as zero-padded 4-entry DMMA chunks
// (mma.sync.m8n8k4.f64 == the sequential fma chain, measured).  In the A
// fragment, lane (r8, k4) holds row r8 = its own cell, so each lane applies
// its own cell's Phi to the raw U it loads.
//
// Work decomposition.  CTA = 4 warps = a 32-cell x-segment of one row; it
// marches along the slab axis over KZ extended planes.  Warp w owns cells
// seg_cell(w, 0..7) of the segment and ALL variables: the DMMA A operand (8 cells x 4
// stencil entries) is transformed on the fly from the staged U region, B (4
// entries x 8 columns) is the weight table in fragment order.  The accumulator layout
// puts all nv variables of one (cell, column) in one thread, so Phi, the
// WENO-AO combination, Phi^-1 and the positivity limiter run in registers;
// the 4 lanes of a quad share a cell and reduce with shuffles.
#ifndef KFVM_RECON_U_CUH_
#define KFVM_RECON_U_CUH_

#include <cuda_pipeline.h>

#ifndef KFVM_U_UNR  // chunk-loop unroll factor
#define KFVM_U_UNR 4
#endif
constexpr int kUChunkUnroll = KFVM_U_UNR;
// Cell of the 32-cell segment owned by quad r8 of warp w: 8 contiguous cells
// per warp.  A chunk's four slots sit at arbitrary (x, row, plane) offsets of
// the region, and row and plane strides are multiples of 4 words, so with the
// cells of a warp 4 apart (w + 4 r8) two slots with equal x offsets mod 4 put
// 16 distinct words on 8 banks: measured 4.0-4.6 wavefronts per A-operand
// load against 2.1-2.4 with contiguous cells (bank model of the chunk tables
// = the ncu count), and the stores of a warp's 8 cells fill two sectors.
#ifdef KFVM_CELL_STRIDE4
__device__ __forceinline__ int seg_cell(int w, int r8) { return w + 4 * r8; }
#else
__device__ __forceinline__ int seg_cell(int w, int r8) { return 8 * w + r8; }
#endif
#ifndef KFVM_U_MINB
#define KFVM_U_MINB 2
#endif
// 3-D R=2: 4 CTAs/SM (128 registers, 32 B of spills) now that the limiter
// bounds come from k_bounds and the shared memory is 54.9 KB per CTA —
// measured 121.7 vs 125.3 ms/step (config 3) and 961.9 vs 994.4 (config 4)
// against 3 CTAs at 166 registers (profiles/r02/README.md)
#ifndef KFVM_U_MINB32
#define KFVM_U_MINB32 4
#endif
#ifndef KFVM_U_EXTRA_SMEM  // occupancy experiments: padding per CTA (bytes)
#define KFVM_U_EXTRA_SMEM 0
#endif
#ifndef KFVM_U_BSMEM_MAX
#define KFVM_U_BSMEM_MAX (48 * 1024)
#endif

template <int D, int R>
struct UCfg {
  using G = Gen<D, R>;
  static constexpr int nv = D + 2;
  static constexpr int ND = (G::NA + 7) / 8;             // derivative tiles in Bd
  // 3-D: the tail derivative columns (a partial last tile, oracle weno_field)
  // run as per-lane DFMA slot chains; NDM full tiles go through DMMA
  static constexpr int NDM = D == 3 ? G::NA / 8 : ND;
  static constexpr int NT = D == 3 ? G::NA - 8 * NDM : 0;
  static constexpr int NPT = (G::NP + 7) / 8;
  // region x extent (row stride): 32 + 2R columns are needed; 3-D R=3 keeps
  // rows 42 words apart (bank model of its chunk tables, tools/bank_model.py:
  // 2.4 wavefronts per A-operand load against 3.1 at 38)
  static constexpr int RXN = 32 + 2 * R;
  static constexpr int RX = (D == 3 && R == 3) ? 42 : RXN;
  static constexpr int RY = D == 3 ? 2 * R + 1 : 1;     // region mid extent
  static constexpr int RROW = RY * RX;                  // one variable of a plane
  static constexpr int PL = nv * RROW;                  // one region plane
  static constexpr int RING = 2 * R + 2;                // planes in the ring
  static constexpr int NX = 34, NY = D == 3 ? 3 : 1;    // prims neighbourhood
  static constexpr int NF = 3 + D;                      // p, c, 1/rho, u_d
  static constexpr int PROW = NY * NX;
  static constexpr int PPL = NF * PROW;
  static constexpr int PRING = 4;
  static constexpr int SCW = G::NS * nv * 8;            // beta / c_q per warp
  // 3-D R=2: B fragments from L1 so that 3 CTAs fit per SM (measured 6.6 %
  // faster than 2 CTAs with B in shared memory, profiles/r01/README.md)
  static constexpr bool BSMEM =
      !(D == 3 && R == 2) && G::NCHUNK * (ND + NPT) * 32 * 8 <= KFVM_U_BSMEM_MAX;
  static constexpr int MINB = D == 3 ? (R == 2 ? KFVM_U_MINB32 : KFVM_U_MINB) : 4;
  static constexpr int SB = BSMEM ? G::NCHUNK * (ND + NPT) * 32 : 0;  // B fragments
  // 3-D: pass 2 over chunks packed across stencil boundaries
  static constexpr bool PK = D == 3 && R == 2;  // R=3 (point groups) measured slower packed
  static constexpr int NCH2 = PK ? (G::NTOT + 3) / 4 : 0;
  static constexpr int PG = NPT <= 3 ? NPT : 4;         // point tiles per pass-2 group
  static constexpr int NG = (NPT + PG - 1) / PG;         // groups (>1: limiter separate)
  // LB: the instance whose limiter bounds come from k_bounds (3-D R=2 main
  // engine): no per-cell-quantity ring in shared memory
  // TG: the instances that take the transform's per-cell quantities from Pr in
  // global memory (no per-cell-quantity ring): LB, and the main 3-D instance
  // of the configurations limited by k_limit_states (NG > 1: 3-D R=3, whose
  // ring + per-cell-quantity ring allowed ONE 4-warp CTA per SM; without it two)
  static constexpr bool TGM = D == 3 && NG > 1;
  static constexpr size_t bytes(bool lb = false, bool tg = false) {
    return sizeof(double) * (RING * (lb ? (PL + 15) / 16 * 16 : PL) + (lb || tg ? 0 : PRING * PPL) + 4 * SCW + SB) +
           (lb ? sizeof(unsigned long long) * (RING + 3) : 0) +
           sizeof(int) * (4 * G::NCHUNK * 2 + G::NCHUNK + 4 * NCH2) + KFVM_U_EXTRA_SMEM;
  }
};

template <int D>
__device__ __forceinline__ double phi_row(const DTransform& T, const double* X, int v) {
  // W_v = (Phi X)_v, constant part dropped (same formula as d_to_recon)
#ifdef KFVM_ABL_NOPHI  // timing ablation (wrong results)
  return X[v];
#endif
  if (v == 0) return X[0];
  if (v <= D) return fma(-T.ut[v - 1], X[0], X[v]) * T.inv_r;
  double t = fma(T.ke, X[0], X[D + 1]);
  t = fma(-T.ut[0], X[1], t);
  t = fma(-T.ut[1], X[2], t);
  if (D == 3) t = fma(-T.ut[2], X[3], t);
  return c_k.gm1 * t;
}

// P1: KXRCF pass 1 on the tensor cores — only the chunks of stencil
// 0, raw conservative U as the A operand, the r_0 face vectors as B, the
// unlimited states stored as they come out of the accumulators.
template <int D, int R, bool P1 = false, bool KXM = false, bool COL = false>
__global__ void __launch_bounds__(128, (P1 || KXM) ? (D == 3 && R == 2 ? 3 : UCfg<D, R>::MINB) : UCfg<D, R>::MINB)
    k_states_u(const double* __restrict__ U, const double* __restrict__ Pr,
               double* __restrict__ St, Geo g, Chunk ch, int KZ, int* __restrict__ err,
               const double* __restrict__ Bd, const double* __restrict__ Bf,
               const int* __restrict__ gat4, const unsigned char* __restrict__ kfl = nullptr,
               int xsp = 0, const double* __restrict__ Lb = nullptr,
               const CUtensorMap* __restrict__ tmap = nullptr) {
  using G = Gen<D, R>;
  using C = UCfg<D, R>;
  // LB: per-cell limiter bounds {rho_max, rho_min, p_min} from k_bounds and
  // the transform's per-cell quantities from Pr in global memory (no ring)
  constexpr bool LB = D == 3 && R == 2 && !P1 && !KXM && C::NG == 1;
  constexpr bool col = COL && LB;  // ring-column tile instance
  constexpr bool TG = LB || (C::TGM && !P1 && !KXM);  // transform quantities from global Pr
  constexpr int nv = C::nv, NP = G::NP, NS = G::NS, ND = C::ND, NPT = C::NPT;
  // LB with a tensor map (tmap): the U planes arrive by TMA — one elected
  // thread, one 4-D box [var][row][x] per plane, an mbarrier per ring slot.
  // FP64 boxes must start on an even x, which holds for the ring-split
  // segments (x0 - R = 32 seg - 2); otherwise the host passes no map and the
  // planes load by cp.async.
  constexpr int RXk = C::RX;
  constexpr int RROWk = C::RY * RXk, PLk = C::nv * RROWk;
  // ring slot stride: TMA destinations are 128-byte aligned
  constexpr int SLk = LB ? (PLk + 15) / 16 * 16 : PLk;
  extern __shared__ __align__(128) double smem[];
  double* sRing = smem;                          // [RING][nv][RY][RX]
  double* sPr = sRing + C::RING * SLk;         // [PRING][NF][NY][NX]
  double* sC = sPr + (TG ? 0 : C::PRING * C::PPL);  // [warp][q][v][8]
  double* sBd = sC + 4 * C::SCW;                 // B fragments [chunk][n][lane]
  double* sBf = sBd + G::NCHUNK * ND * 32;
  int* sTab = reinterpret_cast<int*>(sBd + C::SB);  // [chunk][4] {inplane, oz}
  int* sQ = sTab + 8 * G::NCHUNK;                        // stencil | last << 8
  unsigned long long* sBar = reinterpret_cast<unsigned long long*>(
      sTab + ((9 * G::NCHUNK + 4 * C::NCH2 + 1) & ~1));   // LB: mbarrier per ring slot
  // TMA path: no CTA barrier per plane.  A warp arrives on sDone[it & 1] after
  // pass 2 of its it-th plane (its last read of the oldest ring plane); the
  // issuing thread waits for the four arrivals of plane it - 1 before the TMA
  // that overwrites that slot.  A warp can enter plane it only after every
  // warp arrived for it - 2 (the plane it waits for was issued behind that
  // wait), so two alternating barriers never mix phases.
  unsigned long long* sDone = sBar + C::RING;

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k4 = lane & 3, r8 = lane >> 2;
  // chunk tables (host-built): region offset and z offset of every chunk slot
  for (int i = threadIdx.x; i < 9 * G::NCHUNK + 4 * C::NCH2; i += 128) sTab[i] = gat4[i];
  if constexpr (C::BSMEM) {
    for (int i = threadIdx.x; i < G::NCHUNK * ND * 32; i += 128) sBd[i] = __ldg(Bd + i);
    for (int i = threadIdx.x; i < G::NCHUNK * NPT * 32; i += 128) sBf[i] = __ldg(Bf + i);
  }
  const double* Bdp = C::BSMEM ? sBd : Bd;
  const double* Bfp = C::BSMEM ? sBf : Bf;

  // xsp = 1: the segments cover the interior x range only (the two ring
  // columns of the extended box are computed by column tiles (col = 1, the
  // LB instance), copied from their periodic images, or by k_states_fast)
  // col = 1 (LB): a CTA takes 32 cells of one ring column (x = -1 or nx)
  // along the mid axis — the row tile transposed: the region plane is
  // [var][36 rows][5 columns] (the same size), the host passes the chunk
  // tables built for that layout, and the planes load by cp.async.
  int bid = blockIdx.x;
  int seg = 0, zblk, b, j0, a, cidx = seg_cell(w, r8);
  if (LB && col) {
    const int nys = (ch.em + 31) >> 5;
    const int side = bid & 1;
    bid >>= 1;
    seg = bid % nys;  // y segment
    zblk = bid / nys;
    a = side ? ch.ex - 1 : 0;
    b = seg * 32 + cidx;
    j0 = seg * 32 - 1;  // mid index of the tile's first cell
  } else {
    const int nseg = (ch.ex - 2 * xsp + 31) >> 5;
    seg = bid % nseg;
    bid /= nseg;
    b = bid % ch.em;  // extended mid index
    zblk = bid / ch.em;
    j0 = D == 3 ? b - 1 : 0;
    a = xsp + seg * 32 + cidx;  // extended x index of this lane's cell
  }
  const int cstart = ch.e0 + zblk * KZ, cend = min(ch.e1, cstart + KZ);
  const int j = (LB && col) ? b - 1 : j0;  // this lane's cell's mid index
  // region origin: x of column 0 (+R) and mid index of row 0 (+R)
  const int x0 = (LB && col) ? a - 1 : xsp + seg * 32 - 1;
  // warp w owns the cells seg_cell(w, 0..7) of the segment
  const bool active = (LB && col) ? b < ch.em : a < ch.ex - xsp;
  const int sx = 0;
  const bool use_tma = LB && tmap != nullptr && !col;
  const int xr = cidx + R + sx;       // the cell's x in the region (row tiles)
  const int cb = (LB && col) ? cidx * (2 * R + 1) : cidx + sx;  // the cell's offset in a region plane
  if constexpr (KXM) {  // KXRCF: a tile without a flagged cell has nothing to do
    bool any = false;
    for (int i = threadIdx.x; i < 32 * (cend - cstart); i += 128) {
      const int ai = xsp + seg * 32 + (i & 31), ci = cstart + (i >> 5);
      any |= ai < ch.ex - xsp && kfl[((long long)ci * ch.em + b) * ch.ex + ai];
    }
    if (!__syncthreads_or(any)) return;
  }

  // x indices (remapped) of the region columns this thread copies
  auto load_plane = [&](int p) {  // region plane p -> ring slot
    double* dst = sRing + ((p + 4 * C::RING) % C::RING) * SLk;
    const long long pbase = (long long)(p + g.H) * g.pstride;
    if (LB && col) {  // [var][36 rows][5 columns]
      constexpr int CX = 2 * R + 1, CY = 32 + 2 * R;
      for (int i = threadIdx.x; i < C::nv * CX * CY; i += 128) {
        const int rx = i % CX, rr = i / CX;
        const int ry = rr % CY, v = rr / CY;
        const long long off =
            v * g.vstride + pbase + xoff(g, x0 - R + rx) + moff(g, min(j0 - R + ry, g.nm + g.Gm - 1));
        __pipeline_memcpy_async(dst + i, U + off, sizeof(double));
      }
      return;
    }
    for (int i = threadIdx.x; i < PLk; i += 128) {
      const int rx = i % RXk, rr = i / RXk;
      const int ry = rr % C::RY, v = rr / C::RY;
      // (padding columns of a wider row stride repeat the last needed one)
      const int xx = xoff(g, x0 - R + (RXk > C::RXN ? min(rx, C::RXN - 1) : rx));
      const long long off = v * g.vstride + pbase + xx +
                            (D == 3 ? moff(g, j - R + ry) : 0);
      __pipeline_memcpy_async(dst + i, U + off, sizeof(double));
    }
  };
  auto load_prims = [&](int p) {  // prims plane p -> prims ring slot
    double* dst = sPr + ((p + 4 * C::PRING) % C::PRING) * C::PPL;
    const long long pbase = (long long)(p + g.H) * g.pstride;
    for (int i = threadIdx.x; i < C::PPL; i += 128) {
      const int rx = i % C::NX, rr = i / C::NX;
      const int ry = rr % C::NY, f = rr / C::NY;
      const int xx = xoff(g, x0 - 1 + rx);
      const long long off = f * g.vstride + pbase + xx +
                            (D == 3 ? moff(g, j - 1 + ry) : 0);
      __pipeline_memcpy_async(dst + i, Pr + off, sizeof(double));
    }
  };
  // LB: TMA of region plane q into its ring slot (thread 0); plane q's slot
  // completes its ((q - base) / RING)-th phase when the bytes have landed
  const int base = ch.c0 - 1 + cstart - R;
  auto tma_plane = [&](int q) {
    const int sl = (q + 4 * C::RING) % C::RING;
    mbar_expect_tx(&sBar[sl], (unsigned)(PLk * sizeof(double)));
    tma_load_4d(sRing + sl * SLk, tmap, &sBar[sl], g.xo + x0 - R - sx, j - R + g.Gm, q + g.H, 0);
  };
  auto wait_plane = [&](int q) {
    mbar_wait(&sBar[(q + 4 * C::RING) % C::RING], (unsigned)(((q - base) / C::RING) & 1));
  };
  {
    const int p = ch.c0 - 1 + cstart;
    if (use_tma) {
      if (threadIdx.x == 0) {
        for (int sl = 0; sl < C::RING; ++sl) mbar_init(&sBar[sl], 1);
        mbar_init(&sDone[0], 4);
        mbar_init(&sDone[1], 4);
        mbar_init_fence();
      }
      __syncthreads();
      if (threadIdx.x == 0)
        for (int oz = -R; oz <= R; ++oz) tma_plane(p + oz);
      for (int oz = -R; oz <= R; ++oz) wait_plane(p + oz);
    } else {
      for (int oz = -R; oz <= R; ++oz) load_plane(p + oz);
      if (!P1 && !TG)  // pass 1 needs neither the transform nor the limiter statistics
        for (int oz = -1; oz <= 1; ++oz) load_prims(p + oz);
      __pipeline_commit();
      __pipeline_wait_prior(0);
    }
  }
  __syncthreads();

  double* sCw = sC + w * C::SCW;
  // LB: the transform's per-cell quantities (1/rho, u_d) of the warp's 8
  // cells for plane q, staged in the warp's weight area sCw[f][cell] (free
  // from the end of pass 2 until the next plane's transform is read)
  auto load_t = [&](int q) {
    const int f = lane >> 3, cc = seg_cell(w, lane & 7);
    const int ac = (LB && col) ? a : min(xsp + seg * 32 + cc, ch.ex - 1);
    const int jc = (LB && col) ? min(seg * 32 + cc, ch.em - 1) - 1 : j;
    __pipeline_memcpy_async(sCw + f * 8 + (lane & 7),
                            Pr + (2 + f) * g.vstride + uidx<D>(g, ac - 1, jc, q), sizeof(double));
  };
  if constexpr (TG) {
    load_t(ch.c0 - 1 + cstart);
    __pipeline_commit();
    __pipeline_wait_prior(0);
    __syncwarp();
  }
  PHASE_T0();
  for (int c = cstart; c < cend; ++c) {
    const int p = ch.c0 - 1 + c;
    const int it = c - cstart;
    if (use_tma) {
#ifdef KFVM_U_CTASYNC
      if (threadIdx.x == 0 && c + 1 < cend) tma_plane(p + R + 1);
#endif
      if (c > cstart) wait_plane(p + R);  // issued in the previous iteration
    } else {
      if (c + 1 < cend) {
        load_plane(p + R + 1);
        if (!P1 && !TG) load_prims(p + 2);
      }
      __pipeline_commit();
    }
    // KXRCF: the WENO passes run only for planes of this segment holding a
    // flagged cell; the limiter epilogue runs for every cell (unflagged cells
    // limit their pass-1 states from St)
    bool anyflag = true;
    if constexpr (KXM) {  // KXRCF: planes without a flagged cell are skipped
      anyflag = __syncthreads_or(active && kfl[((long long)c * ch.em + b) * ch.ex + a]) != 0;
      if (!anyflag) {
        __pipeline_wait_prior(0);
        __syncthreads();
        continue;
      }
    }
    // ring slot of plane p + oz (oz in [-R, R]) without a local pointer array
    const int slot0 = (p - R + 4 * C::RING) % C::RING;  // slot of plane p - R
    auto plane = [&](int ozr) -> const double* {       // ozr = oz + R
      const int sl = slot0 + ozr;
      return sRing + (sl >= C::RING ? sl - C::RING : sl) * SLk;
    };
    const double* pr0 = sPr + ((p + 4 * C::PRING) % C::PRING) * C::PPL;
    const double* prm = sPr + ((p - 1 + 4 * C::PRING) % C::PRING) * C::PPL;
    const double* prp = sPr + ((p + 1 + 4 * C::PRING) % C::PRING) * C::PPL;
    const int icn = (D == 3 ? C::NX : 0) + xr - R + 1;  // cell centre in a prims plane
    // cell centre in a region plane
    const int icr = (LB && col) ? (cidx + R) * (2 * R + 1) + R : (D == 3 ? R * RXk : 0) + xr;
    // ---- transform of the cell average (identical to d_make_transform)
    DTransform T;
    // rho~ and m~ enter only Phi^-1 (after pass 2): with one point group they
    // are read from the ring there, out of the passes' register budget
    constexpr bool LATE_RM = C::NG == 1 && !KXM && !P1;
    auto load_rm = [&]() {
      T.rt = plane(R)[icr];
      T.mt[2] = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) T.mt[d] = plane(R)[(1 + d) * RROWk + icr];
    };
    if (!LATE_RM) load_rm();
    // LB: the cell's per-cell quantities straight from Pr (the quad's lanes
    // load the same words)
    T.inv_r = TG ? sCw[r8] : pr0[2 * C::PROW + icn];
    T.ut[2] = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) T.ut[d] = TG ? sCw[(1 + d) * 8 + r8] : pr0[(3 + d) * C::PROW + icn];
    if (TG) __syncwarp();  // every lane has its transform before pass 1 reuses sCw
    {
      double ke = T.ut[0] * T.ut[0];
      ke = fma(T.ut[1], T.ut[1], ke);
      if (D == 3) ke = fma(T.ut[2], T.ut[2], ke);
      T.ke = 0.5 * ke;
    }
    constexpr int PG = C::PG, NG = C::NG;
    double V[nv][PG][2];
    if (anyflag) {
    PHASE_MARK(0);
    // ---- pass 1: derivative columns -> beta_{q,v}
    if constexpr (!P1) {
      constexpr int NDM = C::NDM, NT = C::NT, NTA = NT > 0 ? NT : 1;
      double acc[nv][NDM][2];
      double tl[nv][NTA];  // tail derivative slot chains (slot k4 of the quad)
#pragma unroll
      for (int u = 0; u < nv; ++u) {
#pragma unroll
        for (int n = 0; n < NDM; ++n) acc[u][n][0] = acc[u][n][1] = 0.0;
#pragma unroll
        for (int t = 0; t < NTA; ++t) tl[u][t] = 0.0;
      }
      int q = 0;
      // software pipeline: fragments of chunk ck+1 load while chunk ck issues;
      // a tail weight of column 8 NDM + t at slot k4 is the B fragment word
      // of lane 4t + k4 in the last tile
      double av[nv], bv[NDM], bt[NTA];
      {
        const int inpl = sTab[2 * k4], oz = sTab[2 * k4 + 1];
        const double* ap = plane(oz + R) + inpl + cb;
#pragma unroll
        for (int u = 0; u < nv; ++u) av[u] = ap[u * RROWk];
#pragma unroll
        for (int n = 0; n < NDM; ++n) bv[n] = Bdp[n * 32 + lane];
#pragma unroll
        for (int t = 0; t < NT; ++t) bt[t] = Bdp[(ND - 1) * 32 + 4 * t + k4];
      }
#pragma unroll kUChunkUnroll
      for (int ck = 0; ck < G::NCHUNK; ++ck) {
        const int cn = ck + 1 < G::NCHUNK ? ck + 1 : ck;
        const int inpl = sTab[2 * (cn * 4 + k4)], oz = sTab[2 * (cn * 4 + k4) + 1];
        const double* ap = plane(oz + R) + inpl + cb;
        double an[nv], bn[NDM], btn[NTA];
#pragma unroll
        for (int u = 0; u < nv; ++u) an[u] = ap[u * RROWk];
#pragma unroll
        for (int n = 0; n < NDM; ++n) bn[n] = Bdp[(cn * ND + n) * 32 + lane];
#pragma unroll
        for (int t = 0; t < NT; ++t) btn[t] = Bdp[(cn * ND + ND - 1) * 32 + 4 * t + k4];
        double aw[nv];  // W = Phi U at the slot, with this lane's cell's Phi
#pragma unroll
        for (int v = 0; v < nv; ++v) aw[v] = phi_row<D>(T, av, v);
#pragma unroll
        for (int n = 0; n < NDM; ++n)
#pragma unroll
          for (int v = 0; v < nv; ++v) dmma(acc[v][n][0], acc[v][n][1], aw[v], bv[n]);
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int v = 0; v < nv; ++v) {
#ifndef KFVM_ABL_NOTAIL  // timing ablation (wrong results): no tail derivative chains
            tl[v][t] = fma(bt[t], aw[v], tl[v][t]);
#endif
          }
#pragma unroll
        for (int u = 0; u < nv; ++u) av[u] = an[u];
#pragma unroll
        for (int n = 0; n < NDM; ++n) bv[n] = bn[n];
#pragma unroll
        for (int t = 0; t < NT; ++t) bt[t] = btn[t];
#ifdef KFVM_ABL_NOBETA  // timing ablation (wrong results): no smoothness indicators
        if (sQ[ck] & 256) {
          if (k4 == 0) {
#pragma unroll
            for (int v = 0; v < nv; ++v) sCw[(q * nv + v) * 8 + r8] = acc[v][0][0];
          }
#pragma unroll
          for (int u = 0; u < nv; ++u)
#pragma unroll
            for (int n = 0; n < NDM; ++n) acc[u][n][0] = acc[u][n][1] = 0.0;
          ++q;
        }
        if (false) {
#else
        if (sQ[ck] & 256) {
#endif
          // acc[v][n][e]: variable v of cell r8, alpha = 8n + 2k4 + e; each
          // lane chains its own alphas (partial k4, (n, e) order) and the quad
          // combines (p0 + p1) + (p2 + p3) (oracle weno_field order; the xor
          // tree gives every lane that value since + is commutative)
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
                if (al < G::NA) bq[v] = fma(sc, acc[v][n][e] * acc[v][n][e], bq[v]);
            }
          // tail alphas 8 NDM + t: the quad combines the slot chains as
          // (s0 + s1) + (s2 + s3); partial (t >> 1) takes them in t order
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const int al = 8 * NDM + t;
#pragma unroll
            for (int v = 0; v < nv; ++v) {
              double d = tl[v][t] + __shfl_xor_sync(0xffffffffu, tl[v][t], 1);
              d = d + __shfl_xor_sync(0xffffffffu, d, 2);
              if ((t >> 1) == k4) bq[v] = fma(c_t.scale[al], d * d, bq[v]);
              tl[v][t] = 0.0;
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
#pragma unroll
          for (int u = 0; u < nv; ++u)
#pragma unroll
            for (int n = 0; n < NDM; ++n) acc[u][n][0] = acc[u][n][1] = 0.0;
          ++q;
        }
      }
    }
    __syncwarp();
    PHASE_MARK(1);
    // ---- nonlinear weights, in two balanced steps: lane k4 forms
    // omega~ = gamma_q / (beta^2 + eps) for the stencils q = k4 (+4) of every
    // variable of its cell (the divisions, 10 per lane), then lane k4 sums
    // and normalises variable v = k4 (+4) — the same operations as one
    // sequential pass per variable
    if (!P1) {
#ifdef KFVM_OMEGA_SEQ  // the plain divisions, one after the other (A/B timing)
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
        for (int q = 1; q < NS; ++q)
          sCw[(q * nv + v) * 8 + r8] = fma(-c0, c_t.gamma_lin[q], wt[q] * inv_sum);
      }
#else
      // the lane's reciprocals as ONE interleaved batch (rcp_batch: the same
      // bits as 1.0 / x; consecutive plain divisions run as serial chains)
      constexpr int NQ = (NS + 3) / 4, NVL = (nv + 3) / 4;
      {
        double xs[NQ * nv], ys[NQ * nv];
#pragma unroll
        for (int i = 0; i < NQ; ++i)
#pragma unroll
          for (int v = 0; v < nv; ++v) {
            const int q = k4 + 4 * i;
            const double bb = q < NS ? sCw[(q * nv + v) * 8 + r8] : 1.0;
            xs[i * nv + v] = fma(bb, bb, c_k.eps);
          }
        rcp_batch<NQ * nv>(xs, ys);
#pragma unroll
        for (int i = 0; i < NQ; ++i) {
          const int q = k4 + 4 * i;
          if (q < NS) {
            const double gq = c_t.gamma_lin[q];
#pragma unroll
            for (int v = 0; v < nv; ++v) sCw[(q * nv + v) * 8 + r8] = gq * ys[i * nv + v];
          }
        }
      }
      __syncwarp();
      {
        double wt[NVL][NS], sum[NVL], inv_sum[NVL];
#pragma unroll
        for (int i = 0; i < NVL; ++i) {
          const int v = k4 + 4 * i;
#pragma unroll
          for (int q = 0; q < NS; ++q) wt[i][q] = v < nv ? sCw[(q * nv + v) * 8 + r8] : 1.0;
          sum[i] = wt[i][0];
#pragma unroll
          for (int q = 1; q < NS; ++q) sum[i] = sum[i] + wt[i][q];
        }
        rcp_batch<NVL>(sum, inv_sum);
#pragma unroll
        for (int i = 0; i < NVL; ++i) {
          const int v = k4 + 4 * i;
          if (v < nv) {
            const double c0 = (wt[i][0] * inv_sum[i]) * c_t.inv_g0;
            sCw[v * 8 + r8] = c0;
#pragma unroll
            for (int q = 1; q < NS; ++q)
              sCw[(q * nv + v) * 8 + r8] = fma(-c0, c_t.gamma_lin[q], wt[i][q] * inv_sum[i]);
          }
        }
      }
#endif
    }
    __syncwarp();
    PHASE_MARK(2);
#ifndef KFVM_U_CTASYNC
    // the next plane's TMA, issued here (half a plane before it is needed)
    // so that the wait for the other warps' arrivals rarely blocks
    if (use_tma && threadIdx.x == 0 && c + 1 < cend) {
      if (it > 0) mbar_wait(&sDone[(it - 1) & 1], (unsigned)(((it - 1) >> 1) & 1));
      tma_plane(p + R + 1);
    }
#endif
    // ---- pass 2: face-point columns.  The A operand of a chunk of stencil q
    // is the transformed value scaled by the lane's cell's c_q, so ONE
    // accumulator chain per (variable, point) runs through all stencils and
    // ends as the WENO-AO value (oracle weno_field order).  Point tiles in
    // groups of PG (registers); with more than one group the limited states
    // are produced by k_limit_states from the unlimited ones stored here.
#pragma unroll
    for (int grp = 0; grp < NG; ++grp) {
      const int t0 = grp * PG;
#pragma unroll
      for (int u = 0; u < nv; ++u)
#pragma unroll
        for (int n = 0; n < PG; ++n) V[u][n][0] = V[u][n][1] = 0.0;
      int q = 0;
      double cq[nv];
#pragma unroll
      for (int v = 0; v < nv; ++v) cq[v] = P1 ? 1.0 : sCw[v * 8 + r8];
      // 3-D: the chunks of pass 2 are packed across stencil boundaries (C::PK:
      // no per-stencil zero padding; a pad is an exact no-op of the chain, so
      // the bits are unchanged) and each slot carries its own stencil, whose
      // c_q the lane reloads when it changes
      constexpr bool PK = C::PK && !P1;
      constexpr int NCK = P1 ? G::kc(0) : (PK ? C::NCH2 : G::NCHUNK);  // pass 1: stencil 0 only
      const int* sT2 = sTab + 9 * G::NCHUNK;
      const double* Bf2 = Bf + G::NCHUNK * NPT * 32;
      auto slot = [&](int ck, int& inpl, int& ozr, int& qs) {
        if constexpr (PK) {
          const int pk = sT2[ck * 4 + k4];
          inpl = pk & 511;
          ozr = (pk >> 9) & 7;
          qs = pk >> 12;
        } else {
          inpl = sTab[2 * (ck * 4 + k4)];
          ozr = sTab[2 * (ck * 4 + k4) + 1] + R;
          qs = 0;
        }
      };
      auto bfrag = [&](int ck, int n) -> double {
        if constexpr (PK) return ldB2(Bf2 + (ck * NPT + n) * 32 + lane);
        return Bfp[(ck * NPT + n) * 32 + lane];
      };
      int qa = 0, qcur = 0;
      // software pipeline: fragments of chunk ck+1 load while chunk ck issues
      double av[nv], bv[PG];
      {
        int inpl, ozr;
        slot(0, inpl, ozr, qa);
        const double* ap = plane(ozr) + inpl + cb;
#pragma unroll
        for (int u = 0; u < nv; ++u) av[u] = ap[u * RROWk];
#pragma unroll
        for (int n = 0; n < PG; ++n) bv[n] = t0 + n < NPT ? bfrag(0, t0 + n) : 0.0;
      }
#pragma unroll kUChunkUnroll
      for (int ck = 0; ck < NCK; ++ck) {
        const int cn = ck + 1 < NCK ? ck + 1 : ck;
        int inpl, ozr, qn;
        slot(cn, inpl, ozr, qn);
        const double* ap = plane(ozr) + inpl + cb;
        double an[nv], bn[PG];
#pragma unroll
        for (int u = 0; u < nv; ++u) an[u] = ap[u * RROWk];
#pragma unroll
        for (int n = 0; n < PG; ++n) bn[n] = t0 + n < NPT ? bfrag(cn, t0 + n) : 0.0;
        if (PK && qa != qcur) {  // this slot starts a new stencil
          qcur = qa;
#pragma unroll
          for (int v = 0; v < nv; ++v) cq[v] = sCw[(qcur * nv + v) * 8 + r8];
        }
        double aw[nv];  // c_q (Phi U)_v at the slot, with this lane's cell's Phi
#pragma unroll
        for (int v = 0; v < nv; ++v) aw[v] = P1 ? av[v] : cq[v] * phi_row<D>(T, av, v);
#pragma unroll
        for (int n = 0; n < PG; ++n)
          if (t0 + n < NPT)
#pragma unroll
            for (int v = 0; v < nv; ++v) dmma(V[v][n][0], V[v][n][1], aw[v], bv[n]);
#pragma unroll
        for (int u = 0; u < nv; ++u) av[u] = an[u];
#pragma unroll
        for (int n = 0; n < PG; ++n) bv[n] = bn[n];
        qa = qn;
        if (!P1 && !PK && (sQ[ck] & 256) && q + 1 < NS) {
          ++q;
#pragma unroll
          for (int v = 0; v < nv; ++v) cq[v] = sCw[(q * nv + v) * 8 + r8];
        }
      }
      if (P1 && active) {  // pass-1 states are conservative already
        const long long tid = ((long long)c * ch.em + b) * ch.ex + a;
#pragma unroll
        for (int n = 0; n < PG; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int sp = 8 * (t0 + n) + 2 * k4 + e;
            if (t0 + n < NPT && sp < NP)
#pragma unroll
              for (int v = 0; v < nv; ++v) St[(long long)(sp * nv + v) * ch.next + tid] = V[v][n][e];
          }
      } else if (NG > 1 || KXM) {
        // unlimited states of this group (Phi^-1); k_limit_states limits them
        const long long tid = ((long long)c * ch.em + b) * ch.ex + a;
        if (active && (!KXM || kfl[tid])) {
#pragma unroll
          for (int n = 0; n < PG; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int sp = 8 * (t0 + n) + 2 * k4 + e;
              if (t0 + n < NPT && sp < NP) {
                double Wp[nv], u5[nv];
#pragma unroll
                for (int v = 0; v < nv; ++v) Wp[v] = V[v][n][e];
                d_from_recon(D, T, c_k.inv_gm1, Wp, u5);
#pragma unroll
                for (int v = 0; v < nv; ++v) St[(long long)(sp * nv + v) * ch.next + tid] = u5[v];
              }
            }
        }
      }
    }
    }
    PHASE_MARK(3);
    if constexpr (TG) {  // the next plane's transform quantities, hidden by the epilogue
      __syncwarp();
#ifndef KFVM_U_CTASYNC
      if (use_tma && lane == 0) mbar_arrive(&sDone[it & 1]);  // done with the oldest plane
#endif
      if (c + 1 < cend) load_t(p + 1);
      __pipeline_commit();
    }
    if constexpr (NG == 1 && !P1 && !KXM) {
    {
    if (LATE_RM) load_rm();
    // ---- Phi^-1: conservative states at this lane's points s = 8n + 2k4 + e
    double st[NPT][2][nv];
#pragma unroll
    for (int n = 0; n < NPT; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double Wp[nv];
#pragma unroll
        for (int v = 0; v < nv; ++v) Wp[v] = V[v][n][e];
        d_from_recon(D, T, c_k.inv_gm1, Wp, st[n][e]);
      }
    // ---- positivity limiter: neighbourhood statistics, the 4
    // lanes of the quad split the 3^d neighbours and reduce (max/min exact)
    double rmax, rmin, pmin;
    if constexpr (LB) {
      const long long tidb = ((long long)c * ch.em + b) * ch.ex + a;
      rmax = __ldg(Lb + tidb);
      rmin = __ldg(Lb + ch.next + tidb);
      pmin = __ldg(Lb + 2 * ch.next + tidb);
    } else {
      double rbmax = T.rt, rbmin = T.rt, pbmin = pr0[icn], cmin = pr0[C::PROW + icn];
      {
        constexpr int NN = D == 3 ? 27 : 9;
        for (int m = k4; m < NN; m += 4) {
          const int aa = m % 3 - 1;
          const int bb = D == 3 ? (m / 3) % 3 - 1 : 0;
          const int cc = D == 3 ? m / 9 - 1 : m / 3 - 1;
          const double r = plane(R + cc)[(D == 3 ? bb * RXk : 0) + icr + aa];
          const double* prz = cc < 0 ? prm : (cc > 0 ? prp : pr0);
          const int ip = (D == 3 ? bb * C::NX : 0) + icn + aa;
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
      }
      double delta = 0.5 * (pr0[3 * C::PROW + icn + 1] - pr0[3 * C::PROW + icn - 1]);
      if (D == 3) {
        delta = fma(0.5, pr0[4 * C::PROW + icn + C::NX] - pr0[4 * C::PROW + icn - C::NX], delta);
        delta = fma(0.5, prp[5 * C::PROW + icn] - prm[5 * C::PROW + icn], delta);
      } else {
        delta = fma(0.5, prp[4 * C::PROW + icn] - prm[4 * C::PROW + icn], delta);
      }
      const double kc = c_k.kf * cmin;
      double eta = -(delta + kc) / kc;
      eta = fmin(1.0, fmax(0.0, eta));
      const double fup = fma(c_k.kappa, 1.0 - eta, 1.0);
      const double flo = fma(-c_k.kappa, 1.0 - eta, 1.0);
      rmax = rbmax * fup;
      rmin = rbmin * flo;
      pmin = pbmin * flo;
      const double rt = T.rt, pt = pr0[icn];
      if (!(rt > 0.0) || !(pt > 0.0) || !(rmin > 0.0) || !(pmin > 0.0))
        if (active && k4 == 0) atomicOr(err, 2);
    }
    const double rt = T.rt;
    double Ubar[nv];
    Ubar[0] = rt;
#pragma unroll
    for (int d = 0; d < D; ++d) Ubar[1 + d] = T.mt[d];
    Ubar[nv - 1] = plane(R)[(nv - 1) * RROWk + icr];
    double th = 1.0;
#pragma unroll
    for (int n = 0; n < NPT; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (8 * n + 2 * k4 + e < NP) {
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
        if (8 * n + 2 * k4 + e < NP && d_p_below(D, st[n][e], c_k.gm1, pmin)) {
          StateV<D> a_, b_;
#pragma unroll
          for (int v = 0; v < nv; ++v) {
            a_.v[v] = st[n][e][v];
            b_.v[v] = Ubar[v];
          }
          thp = fmin(thp, theta_p_bisect<D>(a_, b_, pmin));
        }
    thp = fmin(thp, __shfl_xor_sync(0xffffffffu, thp, 1));
    thp = fmin(thp, __shfl_xor_sync(0xffffffffu, thp, 2));
    if (thp < 1.0) {  // (a branch: the scaling is rare, its FP64 operations are not)
#pragma unroll
      for (int n = 0; n < NPT; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int v = 0; v < nv; ++v) st[n][e][v] = fma(thp, st[n][e][v] - Ubar[v], Ubar[v]);
    }
    if (active) {
      const long long tid = ((long long)c * ch.em + b) * ch.ex + a;
#pragma unroll
      for (int n = 0; n < NPT; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int sp = 8 * n + 2 * k4 + e;
          if (sp < NP) {
#pragma unroll
            for (int v = 0; v < nv; ++v) St[(long long)(sp * nv + v) * ch.next + tid] = st[n][e][v];
          }
        }
    }
    }
    }
    PHASE_MARK(4);
    __pipeline_wait_prior(0);
#ifndef KFVM_U_CTASYNC
    if (use_tma)
      __syncwarp();  // load_t's words are the warp's own
    else
#endif
    __syncthreads();
    PHASE_MARK(5);
  }
}

// ------------------------------------------------------- k_limit_states
// Positivity limiter over the stored face states of one
// extended cell, for the configurations whose points do not fit the
// registers of k_states_u (3-D R=3).  Same arithmetic as the fused epilogue.
template <int D, int R>
__global__ void __launch_bounds__(128) k_limit_states(const double* __restrict__ U,
                                                      const double* __restrict__ Pr,
                                                      double* __restrict__ St, Geo g, Chunk ch,
                                                      int* __restrict__ err) {
  constexpr int nv = D + 2, NP = Gen<D, R>::NP;
  const long long tid = (long long)ch.e0 * ch.ex * ch.em + (long long)blockIdx.x * 128 + threadIdx.x;
  if (tid >= (long long)ch.e1 * ch.ex * ch.em) return;
  const int a = (int)(tid % ch.ex);
  const long long r1 = tid / ch.ex;
  const int b = (int)(r1 % ch.em), c = (int)(r1 / ch.em);
  const int x = a - 1, j = D == 3 ? b - 1 : 0, p = ch.c0 - 1 + c;
  const long long ic = uidx<D>(g, x, j, p);
  double Ubar[nv];
#pragma unroll
  for (int v = 0; v < nv; ++v) Ubar[v] = __ldg(U + v * g.vstride + ic);
  double rbmax = Ubar[0], rbmin = Ubar[0], pbmin = __ldg(Pr + ic), cmin = __ldg(Pr + g.vstride + ic);
  for (int cc = -1; cc <= 1; ++cc)
    for (int bb = (D == 3 ? -1 : 0); bb <= (D == 3 ? 1 : 0); ++bb)
      for (int aa = -1; aa <= 1; ++aa) {
        const long long o = uidx<D>(g, x + aa, j + bb, p + cc);
        const double r = __ldg(U + o);
        rbmax = fmax(rbmax, r);
        rbmin = fmin(rbmin, r);
        pbmin = fmin(pbmin, __ldg(Pr + o));
        cmin = fmin(cmin, __ldg(Pr + g.vstride + o));
      }
  double delta = 0.5 * (__ldg(Pr + 3 * g.vstride + uidx<D>(g, x + 1, j, p)) -
                        __ldg(Pr + 3 * g.vstride + uidx<D>(g, x - 1, j, p)));
  if (D == 3) {
    delta = fma(0.5, __ldg(Pr + 4 * g.vstride + uidx<D>(g, x, j + 1, p)) -
                         __ldg(Pr + 4 * g.vstride + uidx<D>(g, x, j - 1, p)), delta);
    delta = fma(0.5, __ldg(Pr + 5 * g.vstride + uidx<D>(g, x, j, p + 1)) -
                         __ldg(Pr + 5 * g.vstride + uidx<D>(g, x, j, p - 1)), delta);
  } else {
    delta = fma(0.5, __ldg(Pr + 4 * g.vstride + uidx<D>(g, x, j, p + 1)) -
                         __ldg(Pr + 4 * g.vstride + uidx<D>(g, x, j, p - 1)), delta);
  }
  const double kc = c_k.kf * cmin;
  double eta = -(delta + kc) / kc;
  eta = fmin(1.0, fmax(0.0, eta));
  const double fup = fma(c_k.kappa, 1.0 - eta, 1.0);
  const double flo = fma(-c_k.kappa, 1.0 - eta, 1.0);
  const double rmax = rbmax * fup, rmin = rbmin * flo, pmin = pbmin * flo;
  const double rt = Ubar[0], pt = __ldg(Pr + ic);
  if (!(rt > 0.0) || !(pt > 0.0) || !(rmin > 0.0) || !(pmin > 0.0)) atomicOr(err, 2);
  double th = 1.0;
  for (int sp = 0; sp < NP; ++sp) {
    const double r = St[(long long)(sp * nv) * ch.next + tid];
    if (r < rmin)
      th = fmin(th, (rt - rmin) / (rt - r));
    else if (r > rmax)
      th = fmin(th, (rmax - rt) / (r - rt));
  }
  double thp = 1.0;
  for (int sp = 0; sp < NP; ++sp) {
    StateV<D> a_, b_;
#pragma unroll
    for (int v = 0; v < nv; ++v) {
      const double u = St[(long long)(sp * nv + v) * ch.next + tid];
      a_.v[v] = th < 1.0 ? fma(th, u - Ubar[v], Ubar[v]) : u;
      b_.v[v] = Ubar[v];
    }
    if (d_p_below(D, a_.v, c_k.gm1, pmin)) thp = fmin(thp, theta_p_bisect<D>(a_, b_, pmin));
  }
  if (th < 1.0 || thp < 1.0)
    for (int sp = 0; sp < NP; ++sp)
#pragma unroll
      for (int v = 0; v < nv; ++v) {
        double* q = St + (long long)(sp * nv + v) * ch.next + tid;
        double u = *q;
        if (th < 1.0) u = fma(th, u - Ubar[v], Ubar[v]);
        if (thp < 1.0) u = fma(thp, u - Ubar[v], Ubar[v]);
        *q = u;
      }
}

// ------------------------------------------------------------- k_bounds
// Positivity-limiter bounds of every extended cell of the plane range
// [e0, e1) (the same operations as the in-kernel statistics of
// k_states_u and k_limit_states): rho_max, rho_min, p_min into
// Lb[3][extended cell], and the admissibility check of the average.  The
// 3-D R=2 tensor engine reads them instead of keeping a ring of per-cell
// quantities in shared memory.  A warp takes 32 consecutive cells of one
// row: each lane reduces its own column's 3 x 3 (mid, slab) neighbourhood,
// the x neighbours' column results arrive by shuffles (min/max are exact,
// so the reduction order is free); 3-D only.
__device__ __forceinline__ void col_stats(const double* __restrict__ U,
                                          const double* __restrict__ Pr, const Geo& g, int x,
                                          int j, int p, double* st) {
  st[0] = -INFINITY;  // rho max
  st[1] = INFINITY;   // rho min
  st[2] = INFINITY;   // p min
  st[3] = INFINITY;   // c min
#pragma unroll
  for (int cc = -1; cc <= 1; ++cc)
#pragma unroll
    for (int bb = -1; bb <= 1; ++bb) {
      const long long o = uidx<3>(g, x, j + bb, p + cc);
      const double r = __ldg(U + o);
      st[0] = fmax(st[0], r);
      st[1] = fmin(st[1], r);
      st[2] = fmin(st[2], __ldg(Pr + o));
      st[3] = fmin(st[3], __ldg(Pr + g.vstride + o));
    }
}

template <int D>
__global__ void __launch_bounds__(128) k_bounds(const double* __restrict__ U,
                                                const double* __restrict__ Pr,
                                                double* __restrict__ Lb, Geo g, Chunk ch,
                                                int* __restrict__ err) {
  static_assert(D == 3, "k_bounds serves the 3-D tensor engine");
  // a warp covers 30 cells of a row: lane l reduces column a0 - 1 + l, lanes
  // 1..30 own the cells (no divergent edge work)
  const int lane = threadIdx.x & 31;
  const long long wid = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
  const int nseg = (ch.ex + 29) / 30;
  const int seg = (int)(wid % nseg);
  const long long r1 = wid / nseg;
  const int b = (int)(r1 % ch.em);
  const int c = ch.e0 + (int)(r1 / ch.em);
  if (c >= ch.e1) return;  // whole warp
  const int a = min(seg * 30 - 1 + lane, ch.ex);  // column of this lane (a = -1 .. ex)
  const int x = a - 1, j = b - 1, p = ch.c0 - 1 + c;
  double own[4], lft[4], rgt[4];
  col_stats(U, Pr, g, x, j, p, own);
  const double u0 = __ldg(Pr + 3 * g.vstride + uidx<3>(g, x, j, p));
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    lft[k] = __shfl_up_sync(0xffffffffu, own[k], 1);
    rgt[k] = __shfl_down_sync(0xffffffffu, own[k], 1);
  }
  const double ul = __shfl_up_sync(0xffffffffu, u0, 1), ur = __shfl_down_sync(0xffffffffu, u0, 1);
  if (lane == 0 || lane == 31 || a < 0 || a >= ch.ex) return;
  const long long ic = uidx<3>(g, x, j, p);
  const double rt = __ldg(U + ic), pt = __ldg(Pr + ic);
  const double rbmax = fmax(fmax(own[0], lft[0]), rgt[0]);
  const double rbmin = fmin(fmin(own[1], lft[1]), rgt[1]);
  const double pbmin = fmin(fmin(own[2], lft[2]), rgt[2]);
  const double cmin = fmin(fmin(own[3], lft[3]), rgt[3]);
  double delta = 0.5 * (ur - ul);
  delta = fma(0.5, __ldg(Pr + 4 * g.vstride + uidx<3>(g, x, j + 1, p)) -
                       __ldg(Pr + 4 * g.vstride + uidx<3>(g, x, j - 1, p)), delta);
  delta = fma(0.5, __ldg(Pr + 5 * g.vstride + uidx<3>(g, x, j, p + 1)) -
                       __ldg(Pr + 5 * g.vstride + uidx<3>(g, x, j, p - 1)), delta);
  const double kc = c_k.kf * cmin;
  double eta = -(delta + kc) / kc;
  eta = fmin(1.0, fmax(0.0, eta));
  const double fup = fma(c_k.kappa, 1.0 - eta, 1.0);
  const double flo = fma(-c_k.kappa, 1.0 - eta, 1.0);
  const double rmax = rbmax * fup, rmin = rbmin * flo, pmin = pbmin * flo;
  if (!(rt > 0.0) || !(pt > 0.0) || !(rmin > 0.0) || !(pmin > 0.0)) atomicOr(err, 2);
  const long long tid = ((long long)c * ch.em + b) * ch.ex + a;
  Lb[tid] = rmax;
  Lb[ch.next + tid] = rmin;
  Lb[2 * ch.next + tid] = pmin;
}

// k_bounds_z: the same bounds with each warp marching KB planes of its row
// segment along the slab axis: the (mid) row statistics of a plane are formed
// once and kept in registers for the three planes that use them (k_bounds
// re-reads every plane three times through L2: 9 instead of 27 neighbour
// loads per cell and field).  min / max are exact, so the grouping is free.
constexpr int kBoundsKB = 16;
__device__ __forceinline__ void row_stats(const double* __restrict__ U,
                                          const double* __restrict__ Pr, const Geo& g, int x,
                                          int j, int p, double* st, double& rc, double& pc) {
  st[0] = -INFINITY;
  st[1] = INFINITY;
  st[2] = INFINITY;
  st[3] = INFINITY;
#pragma unroll
  for (int bb = -1; bb <= 1; ++bb) {
    const long long o = uidx<3>(g, x, j + bb, p);
    const double r = __ldg(U + o), pp = __ldg(Pr + o);
    st[0] = fmax(st[0], r);
    st[1] = fmin(st[1], r);
    st[2] = fmin(st[2], pp);
    st[3] = fmin(st[3], __ldg(Pr + g.vstride + o));
    if (bb == 0) {
      rc = r;
      pc = pp;
    }
  }
}

__global__ void __launch_bounds__(128) k_bounds_z(const double* __restrict__ U,
                                                  const double* __restrict__ Pr,
                                                  double* __restrict__ Lb, Geo g, Chunk ch,
                                                  int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const long long wid = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
  const int nseg = (ch.ex + 29) / 30;
  const int seg = (int)(wid % nseg);
  const long long r1 = wid / nseg;
  const int b = (int)(r1 % ch.em);
  const int c0 = ch.e0 + (int)(r1 / ch.em) * kBoundsKB;
  if (c0 >= ch.e1) return;  // whole warp
  const int c1 = min(ch.e1, c0 + kBoundsKB);
  const int a = min(seg * 30 - 1 + lane, ch.ex);  // column of this lane (a = -1 .. ex)
  const int x = a - 1, j = b - 1;
  const bool owner = !(lane == 0 || lane == 31 || a < 0 || a >= ch.ex);
  // rolling rows of planes p - 1, p, p + 1: statistics, centre rho / p, w
  double s0[4], s1[4], s2[4], r0, r1c, r2, q0, q1, q2, w0, w1, w2;
  {
    const int p = ch.c0 - 1 + c0;
    row_stats(U, Pr, g, x, j, p - 1, s0, r0, q0);
    row_stats(U, Pr, g, x, j, p, s1, r1c, q1);
    w0 = __ldg(Pr + 5 * g.vstride + uidx<3>(g, x, j, p - 1));
    w1 = __ldg(Pr + 5 * g.vstride + uidx<3>(g, x, j, p));
  }
  for (int c = c0; c < c1; ++c) {
    const int p = ch.c0 - 1 + c;
    row_stats(U, Pr, g, x, j, p + 1, s2, r2, q2);
    w2 = __ldg(Pr + 5 * g.vstride + uidx<3>(g, x, j, p + 1));
    const double u0 = __ldg(Pr + 3 * g.vstride + uidx<3>(g, x, j, p));
    const double vp = __ldg(Pr + 4 * g.vstride + uidx<3>(g, x, j + 1, p));
    const double vm = __ldg(Pr + 4 * g.vstride + uidx<3>(g, x, j - 1, p));
    double own[4], lft[4], rgt[4];
    own[0] = fmax(fmax(s0[0], s1[0]), s2[0]);
#pragma unroll
    for (int k = 1; k < 4; ++k) own[k] = fmin(fmin(s0[k], s1[k]), s2[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      lft[k] = __shfl_up_sync(0xffffffffu, own[k], 1);
      rgt[k] = __shfl_down_sync(0xffffffffu, own[k], 1);
    }
    const double ul = __shfl_up_sync(0xffffffffu, u0, 1), ur = __shfl_down_sync(0xffffffffu, u0, 1);
    if (owner) {
      const double rt = r1c, pt = q1;
      const double rbmax = fmax(fmax(own[0], lft[0]), rgt[0]);
      const double rbmin = fmin(fmin(own[1], lft[1]), rgt[1]);
      const double pbmin = fmin(fmin(own[2], lft[2]), rgt[2]);
      const double cmin = fmin(fmin(own[3], lft[3]), rgt[3]);
      double delta = 0.5 * (ur - ul);
      delta = fma(0.5, vp - vm, delta);
      delta = fma(0.5, w2 - w0, delta);
      const double kc = c_k.kf * cmin;
      double eta = -(delta + kc) / kc;
      eta = fmin(1.0, fmax(0.0, eta));
      const double fup = fma(c_k.kappa, 1.0 - eta, 1.0);
      const double flo = fma(-c_k.kappa, 1.0 - eta, 1.0);
      const double rmax = rbmax * fup, rmin = rbmin * flo, pmin = pbmin * flo;
      if (!(rt > 0.0) || !(pt > 0.0) || !(rmin > 0.0) || !(pmin > 0.0)) atomicOr(err, 2);
      const long long tid = ((long long)c * ch.em + b) * ch.ex + a;
      Lb[tid] = rmax;
      Lb[ch.next + tid] = rmin;
      Lb[2 * ch.next + tid] = pmin;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      s0[k] = s1[k];
      s1[k] = s2[k];
    }
    r0 = r1c;
    r1c = r2;
    q0 = q1;
    q1 = q2;
    w0 = w1;
    w1 = w2;
  }
}

#endif
