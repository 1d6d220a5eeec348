// FP64 datapath utilisation when every warp interleaves D DMMAs with S
// independent scalar DFMAs per iteration (the chunk loops of the 3-D
// reconstruction engines: pass 1 ~ D=5, S=16; pass 2 ~ D=15, S=16).
// Utilisation = (256 D + 32 S) FMAs per warp-iteration / (64 FMA/clk/SM x
// elapsed SM cycles).  Prints one line per (warps/SM, D, S).
#include <cstdio>
#include <cuda_runtime.h>

template <int D, int S>
__global__ void kern(double* out, int iters, double x) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[D > 0 ? D : 1][2];
#pragma unroll
  for (int i = 0; i < (D > 0 ? D : 1); ++i) c[i][0] = c[i][1] = 0.0;
  double s[S > 0 ? S : 1];
#pragma unroll
  for (int i = 0; i < (S > 0 ? S : 1); ++i) s[i] = x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
      // spread the scalar work between the DMMAs
#pragma unroll
      for (int j = i * S / (D > 0 ? D : 1); j < (i + 1) * S / (D > 0 ? D : 1); ++j)
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(s[j]) : "d"(b), "d"(a));
    }
    if (D == 0) {
#pragma unroll
      for (int j = 0; j < S; ++j) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(s[j]) : "d"(b), "d"(a));
    }
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < (D > 0 ? D : 1); ++i) r += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < (S > 0 ? S : 1); ++i) r += s[i];
  if (r == 1.2345) out[0] = r;
}

template <int D, int S>
void run(int warps_per_sm, double clk_ghz) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 64);
  const int threads = 32 * (warps_per_sm < 16 ? warps_per_sm : 16);
  const int ctas = warps_per_sm * 32 / threads;
  const int grid = nsm * ctas, iters = 2000;
  kern<D, S><<<grid, threads>>>(d, 10, 0.5);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<D, S><<<grid, threads>>>(d, iters, 0.5);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fma = (256.0 * D + 32.0 * S) * iters * (threads / 32) * (double)grid;
  const double cap = 64.0 * nsm * clk_ghz * 1e9 * ms * 1e-3;
  printf("warps/SM=%2d D=%2d S=%2d  %.3f ms  datapath %.1f %%\n", warps_per_sm, D, S, ms,
         100.0 * fma / cap);
  cudaFree(d);
}

int main() {
  int khz;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double ghz = khz * 1e-6;
  for (int w : {8, 12, 16}) {
    run<8, 0>(w, ghz);
    run<0, 32>(w, ghz);
    run<5, 16>(w, ghz);
    run<15, 16>(w, ghz);
    run<15, 48>(w, ghz);
    run<5, 40>(w, ghz);
  }
  return 0;
}
