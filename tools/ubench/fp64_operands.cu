// Microbenchmark: FP64 DFMA throughput when the weight operand comes from
// (a) registers, (b) __constant__ via uniform loads, (c) shared memory
// broadcast, at different reuse ratios R = DFMAs per loaded weight.
// Each thread keeps NACC independent accumulators (ILP).
#include <cstdio>
#include <cuda_runtime.h>

__constant__ __align__(16) double cw[4096];

template <int MODE, int REUSE, int NACC>
__global__ void kern(double* out, int iters, const double* __restrict__ gw) {
  __shared__ __align__(16) double sw[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sw[i] = gw[i];
  __syncthreads();
  double acc[NACC];
  double g[REUSE];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = i * 1e-3;
#pragma unroll
  for (int r = 0; r < REUSE; ++r) g[r] = threadIdx.x * 1e-4 + r;
  int base = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < NACC / REUSE; k += 2) {
      double2 w;
      if (MODE == 0) { w.x = 0.999; w.y = 1.001; }
      else if (MODE == 1) w = *reinterpret_cast<const double2*>(cw + ((base + 2 * k) & 4095));
      else w = *reinterpret_cast<const double2*>(sw + ((base + 2 * k) & 4095));
#pragma unroll
      for (int r = 0; r < REUSE; ++r) {
        acc[(k * REUSE + r) % NACC] = fma(w.x, g[r], acc[(k * REUSE + r) % NACC]);
        acc[((k + 1) * REUSE + r) % NACC] = fma(w.y, g[r], acc[((k + 1) * REUSE + r) % NACC]);
      }
    }
    base += 2 * (NACC / REUSE);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 1.2345) out[0] = s;
}

template <int MODE, int REUSE, int NACC>
void run(const char* name, int threads, int ctas_per_sm, double* d, const double* gw) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * ctas_per_sm, iters = 2000;
  kern<MODE, REUSE, NACC><<<grid, threads>>>(d, 10, gw);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<MODE, REUSE, NACC><<<grid, threads>>>(d, iters, gw);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * NACC * (double)iters * threads * grid;
  printf("%-28s thr=%4d ctas/sm=%d  %.2f TFLOP/s\n", name, threads, ctas_per_sm, flops / (ms * 1e-3) / 1e12);
}

int main() {
  double *d, *gw;
  cudaMalloc(&d, 64);
  cudaMalloc(&gw, 4096 * 8);
  cudaMemset(gw, 0, 4096 * 8);
  double h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = 1.0 + i * 1e-6;
  cudaMemcpyToSymbol(cw, h, sizeof(h));
  cudaMemcpy(gw, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int w : {1, 2, 3, 4}) {
    printf("--- warps/SMSP ~ %d (160-thread CTAs x %d)\n", w, w * 4 * 32 / 160 > 0 ? w * 4 * 32 / 160 : 1);
  }
  for (int cps : {1, 2, 3, 4}) {
    printf("=== %d x 160-thread CTAs per SM\n", cps);
    run<0, 1, 24>("reg  reuse1 acc24", 160, cps, d, gw);
    run<1, 1, 24>("const reuse1 acc24", 160, cps, d, gw);
    run<1, 2, 24>("const reuse2 acc24", 160, cps, d, gw);
    run<1, 4, 24>("const reuse4 acc24", 160, cps, d, gw);
    run<2, 1, 24>("smem reuse1 acc24", 160, cps, d, gw);
    run<2, 2, 24>("smem reuse2 acc24", 160, cps, d, gw);
    run<2, 4, 24>("smem reuse4 acc24", 160, cps, d, gw);
    run<1, 1, 8>("const reuse1 acc8", 160, cps, d, gw);
  }
  return 0;
}
