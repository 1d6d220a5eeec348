// 1-D bulk copy (cp.async.bulk, no tensor map) + mbarrier, to isolate TMA issues.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__global__ void k_bulk(const double* src, double* out, int mode) {
  __shared__ __align__(128) double buf[256];
  __shared__ __align__(8) unsigned long long mbar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(2048) : "memory");
    if (mode == 0)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(buf)), "l"(src), "r"(2048), "r"(smem_u32(&mbar)) : "memory");
    else
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(buf)), "l"(src), "r"(2048), "r"(smem_u32(&mbar)) : "memory");
  }
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
               ::"r"(smem_u32(&mbar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  double *d, *o;
  cudaMalloc(&d, 2048);
  cudaMalloc(&o, 2048);
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = i;
  cudaMemcpy(d, h, 2048, cudaMemcpyHostToDevice);
  k_bulk<<<1, 128>>>(d, o, mode);
  printf("bulk mode %d: %s\n", mode, cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(h, o, 2048, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 256; ++i) bad += h[i] != i;
  printf("mismatches %d\n", bad);
  int dev; cudaGetDevice(&dev); cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev);
  printf("cc %d.%d %s\n", pr.major, pr.minor, pr.name);
  return 0;
}
