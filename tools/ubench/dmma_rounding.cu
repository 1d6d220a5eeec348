// Does mma.sync.m8n8k4.f64 round like the sequential fma chain
// d = fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c)))) ?  Compare bitwise on
// random data with several orders.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, const double* C, double* D, double* R, int n) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n) return;
  const double* a = A + w * 32; const double* b = B + w * 32; const double* c = C + w * 64;
  double ar = a[(lane >> 2) * 4 + (lane & 3)];
  double br = b[(lane & 3) * 8 + (lane >> 2)];
  double c0 = c[(lane >> 2) * 8 + (lane & 3) * 2], c1 = c[(lane >> 2) * 8 + (lane & 3) * 2 + 1];
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(ar), "d"(br));
  D[w * 64 + (lane >> 2) * 8 + (lane & 3) * 2] = c0;
  D[w * 64 + (lane >> 2) * 8 + (lane & 3) * 2 + 1] = c1;
  // reference orders (thread computes 2 outputs)
  for (int e = 0; e < 2; ++e) {
    const int i = lane >> 2, j = (lane & 3) * 2 + e;
    double s = c[i * 8 + j];
    for (int kk = 0; kk < 4; ++kk) s = fma(a[i * 4 + kk], b[kk * 8 + j], s);  // order 0..3
    R[(w * 64 + i * 8 + j) * 3 + 0] = s;
    s = c[i * 8 + j];
    for (int kk = 3; kk >= 0; --kk) s = fma(a[i * 4 + kk], b[kk * 8 + j], s);  // order 3..0
    R[(w * 64 + i * 8 + j) * 3 + 1] = s;
    // exact-ish: products summed with c then single rounding (emulated by two-sum chain in fma)
    double p = 0.0;
    for (int kk = 0; kk < 4; ++kk) p = fma(a[i * 4 + kk], b[kk * 8 + j], p);
    R[(w * 64 + i * 8 + j) * 3 + 2] = p + c[i * 8 + j];
  }
}

static uint64_t st = 88172645463325252ULL;
static double rnd() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return ((st >> 11) * 0x1.0p-53) * 2 - 1; }

int main() {
  const int n = 4096;
  double *A, *B, *C, *D, *R;
  cudaMallocManaged(&A, n * 32 * 8); cudaMallocManaged(&B, n * 32 * 8);
  cudaMallocManaged(&C, n * 64 * 8); cudaMallocManaged(&D, n * 64 * 8); cudaMallocManaged(&R, n * 64 * 3 * 8);
  for (int t = 0; t < 3; ++t) {
    for (int i = 0; i < n * 32; ++i) { A[i] = rnd() * (t == 2 ? ldexp(1.0, (int)(rnd() * 40)) : 1.0); B[i] = rnd(); }
    for (int i = 0; i < n * 64; ++i) C[i] = (t == 1 ? 0.0 : rnd() * 3);
    k<<<n / 4, 128>>>(A, B, C, D, R, n);
    cudaDeviceSynchronize();
    long m[3] = {0, 0, 0};
    for (int i = 0; i < n * 64; ++i)
      for (int o = 0; o < 3; ++o) m[o] += (D[i] == R[i * 3 + o]);
    printf("trial %d: match seq 0..3: %ld/%d  seq 3..0: %ld  (sum p)+c: %ld\n", t, m[0], n * 64, m[1], m[2]);
  }
  return 0;
}
