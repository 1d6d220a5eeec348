// kfvm_kxrcf.cuh — the KXRCF two-pass reconstruction (
// P:343-357, §5.3 steps 1-3): unlimited full-stencil states in conservative
// variables for every extended cell (pass 1), the troubled-cell flags from
// the entropy jumps across the faces (pass 2), then the WENO engines run in
// flagged cells only (their tiles are skipped otherwise) and k_limit_states
// applies the positivity limiter to every cell.  Same operations as the
// oracle's pass1_cell / global_flags / flag_of.
// Included inside namespace kfvm_b200 by kfvm_gpu.cu.
#ifndef KFVM_KXRCF_CUH_
#define KFVM_KXRCF_CUH_

// Pass 1: St[s][v][cell] = r_0(s) . U_v over S_0, stencil-order fma chains.
template <int D, int R>
__global__ void __launch_bounds__(128) k_pass1(const double* __restrict__ U,
                                               double* __restrict__ St, Geo g, Chunk ch,
                                               const double* __restrict__ face) {
  using G = Gen<D, R>;
  constexpr int nv = D + 2, NP = npoints(D, R), N0 = full_size(D, R);
  const long long tid = (long long)ch.e0 * ch.ex * ch.em + (long long)blockIdx.x * 128 + threadIdx.x;
  if (tid >= (long long)ch.e1 * ch.ex * ch.em) return;
  const int a = (int)(tid % ch.ex);
  const long long r1 = tid / ch.ex;
  const int b = (int)(r1 % ch.em), c = (int)(r1 / ch.em);
  if constexpr (G::UNROLLED) {
    // remapped offsets once, weights as __constant__ operands (kfvm_gen.cuh)
    Tile t;
    t.x = a - 1;
    t.j = D == 3 ? b - 1 : 0;
    t.p = ch.c0 - 1 + c;
    int xs[2 * R + 1];
    long long ms[2 * R + 1], ps[2 * R + 1];
    tile_offsets<D, R>(g, t, xs, ms, ps);
#pragma unroll 1
    for (int v = 0; v < nv; ++v) {
      double u[N0], w[NP];
#pragma unroll
      for (int h = 0; h < N0; ++h) {
        const int ox = G::off(h, 0), om = D == 3 ? G::off(h, 1) : 0;
        const int op = D == 3 ? G::off(h, 2) : G::off(h, 1);
        u[h] = __ldg(U + v * g.vstride + ps[op + R] + ms[om + R] + xs[ox + R]);
      }
      G::pass1(u, w);
#pragma unroll
      for (int s = 0; s < NP; ++s) St[(long long)(s * nv + v) * ch.next + tid] = w[s];
    }
  } else {
    constexpr int HB = 32;  // stencil values held per block
    const int x = a - 1, j = D == 3 ? b - 1 : 0, p = ch.c0 - 1 + c;
    for (int v = 0; v < nv; ++v) {
      for (int s0 = 0; s0 < NP; s0 += 8) {
        double acc[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) acc[s] = 0.0;
        for (int h0 = 0; h0 < N0; h0 += HB) {
          double u[HB];
#pragma unroll
          for (int hh = 0; hh < HB; ++hh) {
            const int h = h0 + hh;
            u[hh] = h < N0 ? __ldg(U + v * g.vstride +
                                   uidx<D>(g, x + c_t.off_x[h], j + c_t.off_m[h], p + c_t.off_p[h]))
                           : 0.0;
          }
#pragma unroll
          for (int s = 0; s < 8; ++s)
#pragma unroll
            for (int hh = 0; hh < HB; ++hh)
              if (h0 + hh < N0 && s0 + s < NP)
                acc[s] = fma(__ldg(face + (s0 + s) * N0 + h0 + hh), u[hh], acc[s]);
        }
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s0 + s < NP) St[(long long)((s0 + s) * nv + v) * ch.next + tid] = acc[s];
      }
    }
  }
}

// Entropy jump of every face the fluxes need (direction d = blockIdx.y):
// J = max over the face's GL points of |q(right) - q(left)|, NaN if any
// point gives NaN.  Each pass-1 state belongs to exactly one face, so every
// entropy is evaluated once.  J goes to scratch[d * nfb + face].
template <int D, int R>
__global__ void __launch_bounds__(128) k_kx_face(const double* __restrict__ St,
                                                 double* __restrict__ J, Geo g, Chunk ch) {
  constexpr int nv = D + 2, NP = npoints(D, R), RP = NP / (2 * D);
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= ch.nfb) return;
  const int d = blockIdx.y;
  const int a = (int)(tid % ch.fx);
  const long long r1 = tid / ch.fx;
  const int b = (int)(r1 % ch.fm), c = (int)(r1 / ch.fm);
  const int nm = D == 3 ? g.nm : 1;
  const bool slab = d == D - 1, mid = D == 3 && d == 1;
  const bool valid = (d == 0 ? true : a < g.nx) && (mid ? true : (D == 3 ? b < nm : true)) &&
                     (slab ? true : c < ch.C);
  if (!valid) return;
  const int lx = a - (d == 0), lj = (D == 3 ? b : 0) - (mid ? 1 : 0), lp = c - (slab ? 1 : 0);
  const long long iL = sidx<D>(ch, lx, lj, lp), iR = sidx<D>(ch, a, D == 3 ? b : 0, c);
  double jm = 0.0;
  bool nan = false;
#pragma unroll
  for (int m = 0; m < RP; ++m) {
    const int sL = (2 * d + 1) * RP + m, sR = (2 * d) * RP + m;
    double uL[nv], uR[nv];
#pragma unroll
    for (int v = 0; v < nv; ++v) {
      uL[v] = St[(long long)(sL * nv + v) * ch.next + iL];
      uR[v] = St[(long long)(sR * nv + v) * ch.next + iR];
    }
    const double jq = fabs(d_entropy<D>(c_k, uR) - d_entropy<D>(c_k, uL));
    if (!(jq == jq)) nan = true;
    jm = fmax(jm, jq);
  }
  J[(long long)d * ch.nfb + tid] = nan ? __longlong_as_double(0x7ff8000000000000LL) : jm;
}

// Pass 2: flags of the slab's own cells (extended planes 1..C of the single
// chunk) from the jumps of their faces.  Physical-boundary faces of outflow
// domains are exempt; a NaN jump or cell entropy flags the cell.
// p0g / nsa: the slab's first global plane and the global slab-axis extent.
template <int D>
__global__ void __launch_bounds__(256) k_kx_flag(const double* __restrict__ U,
                                                 const double* __restrict__ Pr,
                                                 const double* __restrict__ J,
                                                 unsigned char* __restrict__ fl, Geo g, Chunk ch,
                                                 int p0g, int nsa) {
  const long long tid = (long long)blockIdx.x * 256 + threadIdx.x;
  if (tid >= ch.next) return;
  const int a = (int)(tid % ch.ex);
  const long long r1 = tid / ch.ex;
  const int b = (int)(r1 % ch.em), c = (int)(r1 / ch.em);
  const int x = a - 1, j = D == 3 ? b - 1 : 0, p = ch.c0 - 1 + c;
  if (x < 0 || x >= g.nx || (D == 3 && (j < 0 || j >= g.nm)) || c < 1 || c > ch.C) return;
  const long long ic = uidx<D>(g, x, j, p);
  const double rho = __ldg(U + ic);
  const double Q = rho > 0.0 ? __ldg(Pr + ic) / d_kf_pow(rho, c_k.gamma)
                             : __longlong_as_double(0x7ff8000000000000LL);
  bool nan = !(Q == Q);
  double jmax = 0.0;
  const int pg = p0g + p, pc = c - 1;  // chunk-relative interior plane
#pragma unroll
  for (int d = 0; d < D; ++d) {
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int coord = d == 0 ? x : (d == D - 1 ? pg : j);
      const int n = d == 0 ? g.nx : (d == D - 1 ? nsa : g.nm);
      // physical-boundary faces of non-periodic axes are exempt
      if (!c_k.per[d] && ((side == 0 && coord == 0) || (side == 1 && coord == n - 1))) continue;
      const int fa = x + (d == 0 ? side : 0);
      const int fb = j + ((D == 3 && d == 1) ? side : 0);
      const int fc = pc + (d == D - 1 ? side : 0);
      const double jf = J[(long long)d * ch.nfb + ((long long)fc * ch.fm + fb) * ch.fx + fa];
      if (!(jf == jf)) nan = true;
      jmax = fmax(jmax, jf);
    }
  }
  fl[tid] = (nan || jmax / Q >= c_k.dm) ? 1 : 0;
}

// Flags of the extended box's ghost cells: the flag of the cell they
// replicate (periodic image; the nearest interior cell for every other kind
// — with one ghost layer the reflecting mirror image is that cell, and the
// dirichlet / slit ghosts take the flag of the cell they border).  Slab-axis neighbours owned by
// another rank were received into extended planes 0 and C+1 (x, mid interior
// positions) before this runs.
template <int D>
__global__ void __launch_bounds__(256) k_kx_mirror(unsigned char* __restrict__ fl, Geo g,
                                                   Chunk ch, int p0g, int nsa, int exchanged) {
  const long long tid = (long long)blockIdx.x * 256 + threadIdx.x;
  if (tid >= ch.next) return;
  const int a = (int)(tid % ch.ex);
  const long long r1 = tid / ch.ex;
  const int b = (int)(r1 % ch.em), c = (int)(r1 / ch.em);
  const int x = a - 1, j = D == 3 ? b - 1 : 0;
  const bool xin = x >= 0 && x < g.nx, jin = D == 2 || (j >= 0 && j < g.nm);
  const bool pin = c >= 1 && c <= ch.C;
  if (xin && jin && pin) return;
  // one ghost layer: the reflecting mirror image is the clamp
  const int xt = remap(x, g.nx, c_k.per[0]), jt = D == 3 ? remap(j, g.nm, c_k.per[1]) : 0;
  int ct = c;
  if (!pin) {
    const int pg = p0g + ch.c0 - 1 + c;  // global plane of this extended plane
    const bool outside = pg < 0 || pg >= nsa;
    if (!exchanged || (outside && !c_k.per[D - 1])) {
      // replicated plane is local: periodic wrap (one rank) or outflow clamp
      const int pt = remap(pg, nsa, c_k.per[D - 1]) - p0g;  // local plane index
      ct = pt - (ch.c0 - 1);
    } else if (xin && jin) {
      return;  // received from the neighbouring rank
    }
  }
  fl[tid] = fl[((long long)ct * ch.em + (D == 3 ? jt + 1 : 0)) * ch.ex + (xt + 1)];
}

#endif
