// DMMA (mma.sync m8n8k4 f64) throughput vs warps per SM and independent
// accumulator tiles per warp (ILP).  Prints TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void kern(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}

template <int NACC>
void run(int warps_per_sm) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 64);
  const int threads = 32 * (warps_per_sm < 32 ? warps_per_sm : 32);
  const int ctas = warps_per_sm * 32 / threads;
  const int grid = nsm * ctas, iters = 4000;
  kern<NACC><<<grid, threads>>>(d, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<NACC><<<grid, threads>>>(d, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 512.0 * NACC * (double)iters * (threads / 32) * grid;
  printf("warps/SM=%2d acc/warp=%2d  %.2f TFLOP/s\n", warps_per_sm, NACC, flops / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run<1>(w);
    run<2>(w);
    run<4>(w);
    run<8>(w);
    run<12>(w);
  }
  return 0;
}
