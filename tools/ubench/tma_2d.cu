// Plain 2-D FP32 TMA tile load (the canonical example) to check TMA support.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out) {
  __shared__ __align__(1024) float buf[32 * 32];
  __shared__ __align__(8) unsigned long long mbar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(4096) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(smem_u32(buf)), "l"(&tm), "r"(smem_u32(&mbar)), "r"(32), "r"(64) : "memory");
  }
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(smem_u32(&mbar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = buf[i];
}
int main() {
  float* d; float* o;
  cudaMalloc(&d, 256 * 256 * 4); cudaMalloc(&o, 4096);
  float* h = (float*)malloc(256 * 256 * 4);
  for (int i = 0; i < 65536; ++i) h[i] = i;
  cudaMemcpy(d, h, 65536 * 4, cudaMemcpyHostToDevice);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {256, 256}, str[1] = {256 * 4};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  k<<<1, 128>>>(tm, o);
  printf("encode %d, 2-D fp32 TMA: %s\n", (int)r, cudaGetErrorString(cudaDeviceSynchronize()));
  float hb[1024]; cudaMemcpy(hb, o, 4096, cudaMemcpyDeviceToHost);
  int bad = 0; for (int y = 0; y < 32; ++y) for (int x = 0; x < 32; ++x) bad += hb[y * 32 + x] != h[(64 + y) * 256 + 32 + x];
  printf("mismatches %d\n", bad);
  return 0;
}
