// Minimal check of the 2-D row staging through TMA (cp.async.bulk.tensor 3-D
// box of a (x, plane, var) array + one mbarrier phase), as used by
// k_stage_row.  nvcc -gencode arch=compute_100a,code=sm_100a tma_row.cu -o tma_row
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cuda/barrier>
#include <cstdio>
#include <cstdlib>
#include <vector>

using block_barrier = cuda::barrier<cuda::thread_scope_block>;
namespace cde = cuda::device::experimental;

// reference pattern (CUDA programming guide): libcu++ barrier + TMA
__global__ void k_tma_cuda(const __grid_constant__ CUtensorMap tm, double* out, int x0, int p0, int nbytes) {
  __shared__ __align__(128) double buf[4 * 36];
#pragma nv_diag_suppress static_var_with_dynamic_init
  __shared__ block_barrier bar;
  if (threadIdx.x == 0) {
    init(&bar, blockDim.x);
    cde::fence_proxy_async_shared_cta();
  }
  __syncthreads();
  block_barrier::arrival_token token;
  if (threadIdx.x == 0) {
    cde::cp_async_bulk_tensor_3d_global_to_shared(buf, &tm, x0, p0, 0, bar);
    token = cuda::device::barrier_arrive_tx(bar, 1, nbytes);
  } else {
    token = bar.arrive();
  }
  bar.wait(std::move(token));
  for (int i = threadIdx.x; i < 4 * 36; i += blockDim.x) out[i] = buf[i];
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__global__ void k_tma_g(const CUtensorMap* tmg, double* out, int x0, int p0, int nbytes) {
  __shared__ __align__(128) double buf[4 * 36];
  __shared__ __align__(8) unsigned long long mbar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)),
                 "r"(nbytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(buf)),
        "l"(tmg), "r"(smem_u32(&mbar)), "r"(x0), "r"(p0), "r"(0)
        : "memory");
  }
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(&mbar)),
      "r"(0)
      : "memory");
  for (int i = threadIdx.x; i < 4 * 36; i += blockDim.x) out[i] = buf[i];
}

__global__ void k_tma(const __grid_constant__ CUtensorMap tm, double* out, int x0, int p0, int mode) {
  __shared__ __align__(128) double buf[4 * 36];
  __shared__ __align__(8) unsigned long long mbar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    if (mode & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)),
                 "r"(4 * 36 * 8)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(buf)),
        "l"(&tm), "r"(smem_u32(&mbar)), "r"(x0), "r"(p0), "r"(0)
        : "memory");
  }
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(&mbar)),
      "r"(0)
      : "memory");
  for (int i = threadIdx.x; i < 4 * 36; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  const int nx = 96, np = 20, nv = 4;
  std::vector<double> h((size_t)nx * np * nv);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 4 * 36 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (argc > 3 && atoi(argv[3]) == 1)
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  else
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  printf("fn %p\n", fn);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)np, (cuuint64_t)nv};
  const cuuint64_t strides[2] = {(cuuint64_t)nx * 8, (cuuint64_t)nx * np * 8};
  const int variant = argc > 2 ? atoi(argv[2]) : 0;
  const cuuint32_t bx = variant == 1 ? 32 : 36;
  const cuuint32_t box[3] = {bx, 1, 4}, es[3] = {1, 1, 1};
  const CUtensorMapDataType dt = variant == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  CUresult r = enc(&tm, dt, 3, d, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d (query %d)\n", (int)r, (int)q);
  {
    const unsigned long long* w = (const unsigned long long*)&tm;
    for (int i = 0; i < 16; ++i) printf("%016llx%s", w[i], i % 4 == 3 ? "\n" : " ");
  }
  CUtensorMap* tmg;
  cudaMalloc(&tmg, sizeof(CUtensorMap));
  cudaMemcpy(tmg, &tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 4; ++mode) {
    if (only >= 0 && mode != only) continue;
    if (mode == 3)
      k_tma_g<<<1, 128>>>(tmg, o, 29, 5, (int)(bx * 4 * 8));
    else if (mode == 2)
      k_tma_cuda<<<1, 128>>>(tm, o, argc > 4 ? atoi(argv[4]) : 29, 5, (int)(bx * 4 * 8));
    else
      k_tma<<<1, 128>>>(tm, o, 29, 5, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) continue;
    std::vector<double> hb(4 * 36);
    cudaMemcpy(hb.data(), o, hb.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int v = 0; v < 4; ++v)
      for (int x = 0; x < 36; ++x)
        if (hb[v * 36 + x] != h[((size_t)v * np + 5) * nx + 29 + x]) ++bad;
    printf("mode %d mismatches %d\n", mode, bad);
  }
  return 0;
}
