// Do FP64 tensor-core MMAs (DMMA) and DFMAs share execution resources?
// Each warp issues a DMMA stream and/or a DFMA stream (same per-warp counts
// in every mode); if the mixed run takes ~max(dmma, dfma) the pipes are
// independent, if ~sum they are shared.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_dfma_mix.cu -o mix
#include <cstdio>
#include <cuda_runtime.h>

template <bool DO_MMA, bool DO_FMA>
__global__ void k_mix(double* out, int iters, double fa, double fb) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
  double x[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (DO_MMA) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(c[i][0]), "+d"(c[i][1])
              : "d"(a), "d"(b));
      }
      if (DO_FMA) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = fma(x[i], fa, fb);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

template <bool M, bool F>
float run(int grid, int threads, int iters, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_mix<M, F><<<grid, threads>>>(d, 8, 0.999, 1e-3);
  cudaEventRecord(e0);
  k_mix<M, F><<<grid, threads>>>(d, iters, 0.999, 1e-3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  const int iters = 4096;
  for (int tpb : {128, 256, 512}) {
    const int grid = nsm * (1024 / tpb);
    const float mm = run<true, false>(grid, tpb, iters, d);
    const float ff = run<false, true>(grid, tpb, iters, d);
    const float mf = run<true, true>(grid, tpb, iters, d);
    const double warps = (double)grid * tpb / 32;
    const double mma_fl = 512.0 * 16 * iters * warps;        // 4 r x 4 chains per iter
    const double fma_fl = 2.0 * 128 * iters * warps * 32;    // 4 r x 4 k x 8 per thread
    printf("tpb %d: dmma %.3f ms (%.1f TF)  dfma %.3f ms (%.1f TF)  both %.3f ms (%.1f TF total)  sum %.3f max %.3f\n",
           tpb, mm, mma_fl / mm / 1e9, ff, fma_fl / ff / 1e9, mf, (mma_fl + fma_fl) / mf / 1e9,
           mm + ff, mm > ff ? mm : ff);
  }
  return 0;
}
