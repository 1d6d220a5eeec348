// Dependent-issue latency (cycles) of the FP64 operations on the stage
// kernels' critical paths: DFMA, DMUL, DADD, DMMA (accumulator chain),
// SHFL of a double, correctly rounded division and square root.  One warp,
// one dependency chain each; clock64 around 256 unrolled links.
#include <cstdio>
#include <cuda_runtime.h>

#define N 256

__global__ void lat(double* out, long long* cyc, double x0, double y) {
  double x = x0 + threadIdx.x * 1e-9;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-3);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = x * y;
  t1 = clock64();
  cyc[1] = t1 - t0;
  // DADD chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = x + y;
  t1 = clock64();
  cyc[2] = t1 - t0;
  // DMMA accumulator chain
  double c0 = x, c1 = y;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(y), "d"(x0));
  t1 = clock64();
  cyc[3] = t1 - t0;
  x += c0 + c1;
  // SHFL chain (double)
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64();
  cyc[4] = t1 - t0;
  // division chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = y / x;
  t1 = clock64();
  cyc[5] = t1 - t0;
  // sqrt chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = sqrt(x) + 0.25;
  t1 = clock64();
  cyc[6] = t1 - t0;
  // LDS chain (pointer chase through shared memory)
  __shared__ double sh[64];
  sh[threadIdx.x] = 0.0;
  __syncwarp();
  int idx = 0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) idx = (int)sh[idx + (threadIdx.x & 0)];
  t1 = clock64();
  cyc[7] = t1 - t0;
  out[threadIdx.x] = x + idx;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 32 * sizeof(double));
  cudaMalloc(&c, 8 * sizeof(long long));
  lat<<<1, 32>>>(d, c, 1.0, 0.999999);
  lat<<<1, 32>>>(d, c, 1.0, 0.999999);
  long long h[8];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[8] = {"DFMA", "DMUL", "DADD", "DMMA", "SHFL.f64", "div", "sqrt(+add)", "LDS.f64"};
  for (int i = 0; i < 8; ++i) printf("%-12s %.1f cycles\n", names[i], (double)h[i] / N);
  return 0;
}
