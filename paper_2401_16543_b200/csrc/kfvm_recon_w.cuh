// kfvm_recon_w.cuh — the 3-D R=2 tensor engine as ONE 16-warp CTA per SM
// (k_states_w): reconstruct_states with the pinned contract of
// k_states_u (kfvm_recon_u.cuh), restructured around what
// bounds it on B200 — the scalar FP64 instructions that share the datapath
// with the DMMAs and the shared-memory wavefronts of the A-operand loads
// (profiles/r02/README.md).
//
//  * CTA = 16 warps = MR = 4 adjacent rows x 32 cells, marching along z.  The
//    four rows share one ring of region planes [var][2R+MR rows][42] (8 rows
//    for 4 instead of 5 for 1), each plane one TMA box.
//  * W cache.  The A operand of a chunk slot is W = Phi_i U_k of the lane's
//    cell i and stencil cell k.  A cell's stencil S0 has 33 cells but its 8
//    (sub)stencils list 106 slots, and both passes walk all of them: the
//    engine of kfvm_recon_u.cuh transforms 222 slots per cell and plane.
//    Here the transformed values of the variables 2..4 (9 of the 11 FP64
//    operations of a slot) are stored in shared memory while pass 1 walks
//    the chunks of stencil 0 (= S0, every stencil cell once) and every later
//    slot of either pass reads them back: the same values, so the same bits.
//    (The shared ring is what makes room: 16 warps x 3 variables x 33 cells
//    x 8 cells/warp x 8 B = 99 KB of cache next to 79 KB of ring.)
//  * Bank layout (tools/bank_model.py): rows 42 words apart, a warp's 8 cells
//    contiguous, the cache split by half-warp with the S0 cells 4-coloured by
//    the host so that the slots of a chunk fall in different bank windows.
//  * No CTA barrier per plane (mbarrier hand-off as in k_states_u's TMA path);
//    the rows run skewed in phase and the last row issues the TMAs.
// Included inside namespace kfvm_b200 by kfvm_gpu.cu (after kfvm_recon_u.cuh).
#ifndef KFVM_RECON_W_CUH_
#define KFVM_RECON_W_CUH_

template <int MR>
struct WCfg {
  using G = Gen<3, 2>;
  using C = UCfg<3, 2>;
  static constexpr int R = 2, nv = 5;
  static constexpr int NW = 4 * MR;                  // warps
  // region x extent: 36 columns are needed; rows 42 words apart (and the
  // warp's 8 cells contiguous) spread the four slots of a chunk — arbitrary
  // (x, row) offsets of the stencil — over the banks: 2.1 wavefronts per
  // A-operand load in the half-warp bank model of the chunk tables against
  // 3.4 at 36 (ncu: the model's numbers); the 6 extra columns ride in the box
  static constexpr int RX = 42;
  static constexpr int RY = 2 * R + MR;              // region rows
  static constexpr int RROW = RY * RX;               // one variable of a plane
  static constexpr int PL = nv * RROW;               // one region plane
  static constexpr int SL = (PL + 15) / 16 * 16;     // ring slot stride (TMA: 128-byte aligned)
  static constexpr int RING = 2 * R + 2;
  static constexpr int SCW = G::NS * nv * 8;         // beta / c_q per warp
  static constexpr int V0 = 2, NCV = nv - V0;        // cached variables V0 .. nv-1
  static constexpr int N0 = G::N0;                   // cells of S0
  // W cache per warp [v][half h of the 8 cells][position 0..N0-1][4 cells]: a
  // 64-bit load runs per half-warp (4 cells x 4 slots), which is conflict-free
  // when the four S0 cells sit in different 4-word bank windows — position mod
  // 4, a 4-colouring of S0 the host searches so that the cells of (nearly)
  // every chunk differ (upload_gen: 1.2 wavefronts per half against 2.1 with
  // rows of 8 cells)
  static constexpr int HP = N0 * 4;
  static constexpr int WCW = NCV * 2 * HP;
  static constexpr int K0 = G::kc(0);                // chunks of stencil 0
  static constexpr int NT1 = 4 * G::NCHUNK, NT2 = 4 * C::NCH2;  // table words
  static constexpr size_t bytes() {
    return sizeof(double) * (RING * SL + NW * SCW + NW * WCW) +
           sizeof(int) * ((NT1 + NT2 + 1) & ~1) + sizeof(unsigned long long) * (RING + 2);
  }
};

// table word of a chunk slot (host: upload_gen): region offset (oy+R)*RX+ox+R
// | (oz+R) << 9 | stencil << 12 | W-cache position of the S0 cell << 16 | last
// chunk of its stencil << 22
template <int MR, int SH = 0>
__global__ void __launch_bounds__(128 * MR, 1)
    k_states_w(const double* __restrict__ Pr, double* __restrict__ St, Geo g, Chunk ch, int KZ,
               const double* __restrict__ Bd, const double* __restrict__ Bf,
               const int* __restrict__ gatw, int xsp, const double* __restrict__ Lb,
               const CUtensorMap* __restrict__ tmap) {
  using G = Gen<3, 2>;
  using C = UCfg<3, 2>;
  using W = WCfg<MR>;
  constexpr int D = 3, R = 2, nv = 5, NP = G::NP, NS = G::NS, ND = C::ND, NPT = C::NPT;
  constexpr int RX = W::RX, RROW = W::RROW, SL = W::SL, V0 = W::V0, NCV = W::NCV;
  static_assert(C::NDM == 1 && C::NT == 1 && NPT == 3 && C::NG == 1, "3-D R=2 structure");
  extern __shared__ __align__(128) double smem[];
  double* sRing = smem;                                // [RING][nv][RY][RX]
  double* sC = sRing + W::RING * SL;                   // [warp][q][v][8]
  double* sWc = sC + W::NW * W::SCW;                   // [warp][v - V0][S0 cell][8]
  int* sT1 = reinterpret_cast<int*>(sWc + W::NW * W::WCW);  // pass-1 slots [chunk][4]
  int* sT2 = sT1 + W::NT1;                             // pass-2 slots (packed chunks) [chunk][4]
  unsigned long long* sBar =
      reinterpret_cast<unsigned long long*>(sT1 + ((W::NT1 + W::NT2 + 1) & ~1));
  unsigned long long* sDone = sBar + W::RING;

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k4 = lane & 3, r8 = lane >> 2;
  const int wr = w >> 2, wx = w & 3;  // the warp's row of the CTA, its cell phase
  for (int i = threadIdx.x; i < W::NT1 + W::NT2; i += 128 * MR) sT1[i] = gatw[i];

  int bid = blockIdx.x;
  const int nseg = (ch.ex - 2 * xsp + 31) >> 5;
  const int nrb = (ch.em + MR - 1) / MR;
  const int seg = bid % nseg;
  bid /= nseg;
  const int rb = bid % nrb, zblk = bid / nrb;
  const int cidx = seg_cell(wx, r8);         // the lane's cell of the segment (see k_states_u)
  const int a = xsp + seg * 32 + cidx;       // extended x index
  const int b = rb * MR + wr;                // extended mid index
  const bool active = a < ch.ex - xsp && b < ch.em;
  const int bc = min(b, ch.em - 1);          // rows past the box: loads stay in bounds
  const int j = bc - 1;
  const int cstart = ch.e0 + zblk * KZ, cend = min(ch.e1, cstart + KZ);
  const int x0 = xsp + seg * 32 - 1;
  // FP64 TMA boxes start on an even element: segments that start on an odd x
  // (xsp = 0: they include the ring columns) load one more column on the left
  // (the 42-word rows have the room) and shift the cell by one
  constexpr int sh = SH;  // = (x0 - R) & 1 = !xsp (host; a run-time shift cost 2 % in registers)
  const int xr = cidx + R + sh;
  const int cb = wr * RX + cidx + sh;        // the cell's offset in a region plane
  const int icr = (R + wr) * RX + xr;        // the cell itself

  const int base = ch.c0 - 1 + cstart - R;
  auto tma_plane = [&](int q) {
    const int sl = (q + 4 * W::RING) % W::RING;
    mbar_expect_tx(&sBar[sl], (unsigned)(W::PL * sizeof(double)));
    tma_load_4d(sRing + sl * SL, tmap, &sBar[sl], g.xo + x0 - R - sh, rb * MR - 1 - R + g.Gm, q + g.H, 0);
  };
  auto wait_plane = [&](int q) {
    mbar_wait(&sBar[(q + 4 * W::RING) % W::RING], (unsigned)(((q - base) / W::RING) & 1));
  };
  {
    const int p = ch.c0 - 1 + cstart;
    if (threadIdx.x == 0) {
      for (int sl = 0; sl < W::RING; ++sl) mbar_init(&sBar[sl], 1);
      mbar_init(&sDone[0], W::NW);
      mbar_init(&sDone[1], W::NW);
      mbar_init_fence();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int oz = -R; oz <= R; ++oz) tma_plane(p + oz);
    for (int oz = -R; oz <= R; ++oz) wait_plane(p + oz);
  }
  __syncthreads();

  double* sCw = sC + w * W::SCW;
  double* sWw = sWc + w * W::WCW + (r8 >> 2) * W::HP + (r8 & 3);  // + (v - V0) * 2 HP + 4 position
  // the transform's per-cell quantities (1/rho, u_d) of the warp's 8 cells for
  // plane q, staged in the warp's weight area (see k_states_u)
  auto load_t = [&](int q) {
    const int f = lane >> 3, cc = seg_cell(wx, lane & 7);
    const int ac = min(xsp + seg * 32 + cc, ch.ex - 1);
    __pipeline_memcpy_async(sCw + f * 8 + (lane & 7),
                            Pr + (2 + f) * g.vstride + uidx<D>(g, ac - 1, j, q), sizeof(double));
  };
  load_t(ch.c0 - 1 + cstart);
  __pipeline_commit();
  __pipeline_wait_prior(0);
  __syncwarp();

  const double* Bf2 = Bf + G::NCHUNK * NPT * 32;
  // Phase skew.  The CTA's 16 warps would otherwise run their planes in lock
  // step (all in the weights phase, all in pass 2, ...), and the four warps
  // that share an SM sub-partition are the four ROWS of one cell phase: row
  // wr starts wr / MR of a plane period late, so the latency-bound phases of
  // one row overlap the DMMA phases of the others.  The LAST row issues the
  // TMAs (at the top of its plane, when every other warp has long arrived),
  // which also keeps any warp from running a full plane ahead of it.
#ifndef KFVM_W_SKEW_NS
#define KFVM_W_SKEW_NS 3000
#endif
  if (wr > 0) __nanosleep(wr * KFVM_W_SKEW_NS);
  const bool issuer = threadIdx.x == 128 * (MR - 1);
  for (int c = cstart; c < cend; ++c) {
    const int p = ch.c0 - 1 + c, it = c - cstart;
    if (c > cstart) wait_plane(p + R);  // issued in the previous iteration
    // the next plane's TMA, behind every warp's arrival for the previous
    // plane: its slot is theirs until then
    if (issuer && c + 1 < cend) {
      if (it > 0) mbar_wait(&sDone[(it - 1) & 1], (unsigned)(((it - 1) >> 1) & 1));
      tma_plane(p + R + 1);
    }
    const int slot0 = (p - R + 4 * W::RING) % W::RING;  // slot of plane p - R
    auto plane = [&](int ozr) -> const double* {         // ozr = oz + R
      const int sl = slot0 + ozr;
      return sRing + (sl >= W::RING ? sl - W::RING : sl) * SL;
    };
    DTransform T;
    T.inv_r = sCw[r8];
#pragma unroll
    for (int d = 0; d < D; ++d) T.ut[d] = sCw[(1 + d) * 8 + r8];
    __syncwarp();  // every lane has its transform before pass 1 reuses sCw
    {
      double ke = T.ut[0] * T.ut[0];
      ke = fma(T.ut[1], T.ut[1], ke);
      ke = fma(T.ut[2], T.ut[2], ke);
      T.ke = 0.5 * ke;
    }
    // ---- pass 1: derivative columns -> beta_{q,v} (k_states_u's operations)
    {
      double acc[nv][2], tl[nv];
#pragma unroll
      for (int u = 0; u < nv; ++u) acc[u][0] = acc[u][1] = tl[u] = 0.0;
      int q = 0;
      // (-DKFVM_W_BETA_PAIRS, bitwise, not the default)
      // beta of a stencil = ((p0 + sc8 d^2) + p1) + (p2 + p3), with lane k4's
      // partial chain p_k4 over its two derivative columns and the tail
      // derivative d = (s0 + s1) + (s2 + s3) of the quad's slot chains (oracle
      // weno_field order).  The quad reduces TWO stencils at a time: the even
      // lanes take the earlier one, the odd lanes the later one — in the xor-1
      // exchanges every lane sends the partner's stencil's value and keeps its
      // own, so each butterfly step is one add per variable for both stencils
      // (the same sums: + commutes) instead of one per stencil.
#ifndef KFVM_W_BETA_PAIRS  // default: one stencil at a time (the pair reduction below measured 828.7 vs 822.4 ms/step on config 4: fewer FP64 operations and shuffles, more selects and registers)
      auto beta = [&]() {
        double bq[nv];
#pragma unroll
        for (int v = 0; v < nv; ++v) bq[v] = 0.0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double sc = c_t.scale[2 * k4 + e];
#pragma unroll
          for (int v = 0; v < nv; ++v) bq[v] = fma(sc, acc[v][e] * acc[v][e], bq[v]);
        }
#pragma unroll
        for (int v = 0; v < nv; ++v) {
          double d = tl[v] + __shfl_xor_sync(0xffffffffu, tl[v], 1);
          d = d + __shfl_xor_sync(0xffffffffu, d, 2);
          if (k4 == 0) bq[v] = fma(c_t.scale[8], d * d, bq[v]);
          tl[v] = 0.0;
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
        for (int u = 0; u < nv; ++u) acc[u][0] = acc[u][1] = 0.0;
        ++q;
      };
#else
      static_assert(NS % 2 == 0, "stencils reduce in pairs");
      double pE[nv], tE[nv];  // the even stencil's partials and tail slot sums
      auto beta = [&]() {
        double bq[nv];
#pragma unroll
        for (int v = 0; v < nv; ++v) bq[v] = 0.0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double sc = c_t.scale[2 * k4 + e];
#pragma unroll
          for (int v = 0; v < nv; ++v) bq[v] = fma(sc, acc[v][e] * acc[v][e], bq[v]);
        }
        if (!(q & 1)) {
#pragma unroll
          for (int v = 0; v < nv; ++v) {
            pE[v] = bq[v];
            tE[v] = tl[v];
          }
        } else {
          const bool odd = k4 & 1;
          const double sc8 = c_t.scale[8];
#pragma unroll
          for (int v = 0; v < nv; ++v) {
            // tail: own stencil's slot sum + the partner's slot sum of it
            const double tm = odd ? tl[v] : tE[v], ts = odd ? tE[v] : tl[v];
            const double u2 = tm + __shfl_xor_sync(0xffffffffu, ts, 1);
            const double d = u2 + __shfl_xor_sync(0xffffffffu, u2, 2);
            // partials: lanes 0, 1 end with (p0, p1), lanes 2, 3 with (p2, p3)
            const double pm = odd ? bq[v] : pE[v], ps = odd ? pE[v] : bq[v];
            const double pr = __shfl_xor_sync(0xffffffffu, ps, 1);
            double pa = odd ? pr : pm;
            const double pb = odd ? pm : pr;
            if (k4 < 2) pa = fma(sc8, d * d, pa);
            const double s2 = pa + pb;
            const double bt2 = s2 + __shfl_xor_sync(0xffffffffu, s2, 2);
            if (k4 < 2) sCw[((q - 1 + (int)odd) * nv + v) * 8 + r8] = bt2;
          }
        }
#pragma unroll
        for (int u = 0; u < nv; ++u) acc[u][0] = acc[u][1] = tl[u] = 0.0;
        ++q;
      };
#endif
      // -- stencil 0 (= S0): raw values, transformed here and cached
      {
        double av[nv], bv, bt;
        int wd = sT1[k4];
        {
          const double* ap = plane((wd >> 9) & 7) + (wd & 511) + cb;
#pragma unroll
          for (int u = 0; u < nv; ++u) av[u] = ap[u * RROW];
          bv = Bd[lane];
          bt = Bd[(ND - 1) * 32 + k4];
        }
#pragma unroll
        for (int ck = 0; ck < W::K0; ++ck) {
          const int cn = ck + 1 < W::K0 ? ck + 1 : ck;
          const int wn = sT1[cn * 4 + k4];
          const double* ap = plane((wn >> 9) & 7) + (wn & 511) + cb;
          double an[nv];
#pragma unroll
          for (int u = 0; u < nv; ++u) an[u] = ap[u * RROW];
          const double bn = Bd[(cn * ND) * 32 + lane];
          const double btn = Bd[(cn * ND + ND - 1) * 32 + k4];
          double aw[nv];
#pragma unroll
          for (int v = 0; v < nv; ++v) aw[v] = phi_row<D>(T, av, v);
          double* wc = sWw + ((wd >> 16) & 63) * 4;
#pragma unroll
          for (int v = V0; v < nv; ++v) wc[(v - V0) * 2 * W::HP] = aw[v];
#pragma unroll
          for (int v = 0; v < nv; ++v) dmma(acc[v][0], acc[v][1], aw[v], bv);
#pragma unroll
          for (int v = 0; v < nv; ++v) tl[v] = fma(bt, aw[v], tl[v]);
#pragma unroll
          for (int u = 0; u < nv; ++u) av[u] = an[u];
          bv = bn;
          bt = btn;
          wd = wn;
        }
        beta();
      }
      __syncwarp();  // the quad's lanes cached different cells of S0
      // -- stencils 1..: rho and m_x raw, the cached W_2.. of the slot's S0 cell
      {
        double a0, a1, aw2[NCV], bv, bt;
        int wd = sT1[W::K0 * 4 + k4];
        {
          const double* ap = plane((wd >> 9) & 7) + (wd & 511) + cb;
          a0 = ap[0];
          a1 = ap[RROW];
          const double* wc = sWw + ((wd >> 16) & 63) * 4;
#pragma unroll
          for (int v = 0; v < NCV; ++v) aw2[v] = wc[v * 2 * W::HP];
          bv = Bd[(W::K0 * ND) * 32 + lane];
          bt = Bd[(W::K0 * ND + ND - 1) * 32 + k4];
        }
#pragma unroll kUChunkUnroll
        for (int ck = W::K0; ck < G::NCHUNK; ++ck) {
          const int cn = ck + 1 < G::NCHUNK ? ck + 1 : ck;
          const int wn = sT1[cn * 4 + k4];
          const double* ap = plane((wn >> 9) & 7) + (wn & 511) + cb;
          const double n0 = ap[0], n1 = ap[RROW];
          const double* wc = sWw + ((wn >> 16) & 63) * 4;
          double an2[NCV];
#pragma unroll
          for (int v = 0; v < NCV; ++v) an2[v] = wc[v * 2 * W::HP];
          const double bn = Bd[(cn * ND) * 32 + lane];
          const double btn = Bd[(cn * ND + ND - 1) * 32 + k4];
          double aw[nv];
          aw[0] = a0;
          aw[1] = fma(-T.ut[0], a0, a1) * T.inv_r;
#pragma unroll
          for (int v = 0; v < NCV; ++v) aw[V0 + v] = aw2[v];
#pragma unroll
          for (int v = 0; v < nv; ++v) dmma(acc[v][0], acc[v][1], aw[v], bv);
#pragma unroll
          for (int v = 0; v < nv; ++v) tl[v] = fma(bt, aw[v], tl[v]);
          a0 = n0;
          a1 = n1;
#pragma unroll
          for (int v = 0; v < NCV; ++v) aw2[v] = an2[v];
          bv = bn;
          bt = btn;
          if (wd & (1 << 22)) beta();
          wd = wn;
        }
      }
    }
    __syncwarp();
    // ---- nonlinear weights (k_states_u's operations; reciprocals as a batch)
    {
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
    }
    __syncwarp();
    // ---- pass 2: face-point columns over the packed chunks, A = c_q W
    double V[nv][NPT][2];
    {
#pragma unroll
      for (int u = 0; u < nv; ++u)
#pragma unroll
        for (int n = 0; n < NPT; ++n) V[u][n][0] = V[u][n][1] = 0.0;
      double cq[nv];
#pragma unroll
      for (int v = 0; v < nv; ++v) cq[v] = sCw[v * 8 + r8];
      int qcur = 0;
      double a0, a1, aw2[NCV], bv[NPT];
      int wd = sT2[k4];
      {
        const double* ap = plane((wd >> 9) & 7) + (wd & 511) + cb;
        a0 = ap[0];
        a1 = ap[RROW];
        const double* wc = sWw + ((wd >> 16) & 63) * 4;
#pragma unroll
        for (int v = 0; v < NCV; ++v) aw2[v] = wc[v * 2 * W::HP];
#pragma unroll
        for (int n = 0; n < NPT; ++n) bv[n] = ldB2(Bf2 + n * 32 + lane);
      }
#pragma unroll kUChunkUnroll
      for (int ck = 0; ck < C::NCH2; ++ck) {
        const int cn = ck + 1 < C::NCH2 ? ck + 1 : ck;
        const int wn = sT2[cn * 4 + k4];
        const double* ap = plane((wn >> 9) & 7) + (wn & 511) + cb;
        const double n0 = ap[0], n1 = ap[RROW];
        const double* wc = sWw + ((wn >> 16) & 63) * 4;
        double an2[NCV], bn[NPT];
#pragma unroll
        for (int v = 0; v < NCV; ++v) an2[v] = wc[v * 2 * W::HP];
#pragma unroll
        for (int n = 0; n < NPT; ++n) bn[n] = ldB2(Bf2 + (cn * NPT + n) * 32 + lane);
        const int qa = (wd >> 12) & 7;
        if (qa != qcur) {  // this slot starts a new stencil
          qcur = qa;
#pragma unroll
          for (int v = 0; v < nv; ++v) cq[v] = sCw[(qcur * nv + v) * 8 + r8];
        }
        double aw[nv];
        aw[0] = cq[0] * a0;
        aw[1] = cq[1] * (fma(-T.ut[0], a0, a1) * T.inv_r);
#pragma unroll
        for (int v = 0; v < NCV; ++v) aw[V0 + v] = cq[V0 + v] * aw2[v];
#pragma unroll
        for (int n = 0; n < NPT; ++n)
#pragma unroll
          for (int v = 0; v < nv; ++v) dmma(V[v][n][0], V[v][n][1], aw[v], bv[n]);
        a0 = n0;
        a1 = n1;
#pragma unroll
        for (int v = 0; v < NCV; ++v) aw2[v] = an2[v];
#pragma unroll
        for (int n = 0; n < NPT; ++n) bv[n] = bn[n];
        wd = wn;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sDone[it & 1]);  // done with the oldest ring plane
    if (c + 1 < cend) load_t(p + 1);  // hidden by the epilogue
    __pipeline_commit();
    // ---- Phi^-1, positivity limiter, store (k_states_u's LB epilogue)
    {
      T.rt = plane(R)[icr];
#pragma unroll
      for (int d = 0; d < D; ++d) T.mt[d] = plane(R)[(1 + d) * RROW + icr];
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
      const long long tidb = ((long long)c * ch.em + bc) * ch.ex + min(a, ch.ex - 1);
      const double rmax = __ldg(Lb + tidb);
      const double rmin = __ldg(Lb + ch.next + tidb);
      const double pmin = __ldg(Lb + 2 * ch.next + tidb);
      const double rt = T.rt;
      double Ubar[nv];
      Ubar[0] = rt;
#pragma unroll
      for (int d = 0; d < D; ++d) Ubar[1 + d] = T.mt[d];
      Ubar[nv - 1] = plane(R)[(nv - 1) * RROW + icr];
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
          if (d_p_below(D, st[n][e], c_k.gm1, pmin)) {
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
      if (thp < 1.0) {  // (a branch: the scaling is rare, its 60 FP64 operations are not)
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
#pragma unroll
            for (int v = 0; v < nv; ++v) St[(long long)(sp * nv + v) * ch.next + tid] = st[n][e][v];
          }
      }
    }
    __pipeline_wait_prior(0);
    __syncwarp();  // load_t's words are the warp's own
  }
}

#endif
