// Minimal TMA repro: 4-D planar map (dims {W, H, 1, 16}, box {16, 1, 1, 16}, SWIZZLE_64B).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, int nload, float* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(nload * 1024) : "memory");
    for (int q = 0; q < nload; ++q)
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(su(sm + q * 1024)), "l"((uint64_t)&tm), "r"(q * 3), "r"(q), "r"(0), "r"(0), "r"(su(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W1;\n\t}" ::"r"(su(&bar)) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nload * 256; i += blockDim.x) out[i] = ((float*)sm)[i];
}
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  EncFn enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int W = 256, H = 256;
  float* d; cudaMalloc(&d, (size_t)W * H * 16 * 4);
  float* o; cudaMalloc(&o, 24 * 1024);
  for (int variant = 0; variant < 6; ++variant) {
    if (only >= 0 && variant != only) continue;
    CUtensorMap tm;
    cuuint64_t dims[4] = {W, H, 1, 16};
    cuuint64_t str[3] = {W * 4, (cuuint64_t)W * H * 4, (cuuint64_t)W * H * 4};
    cuuint32_t box[4] = {16, 1, 1, 16}, es[4] = {1, 1, 1, 1};
    CUtensorMapSwizzle sw = variant == 0 ? CU_TENSOR_MAP_SWIZZLE_64B : (variant == 1 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_64B);
    if (variant == 2) { dims[2] = 16; dims[3] = 1; box[2] = 16; box[3] = 1; str[1] = (cuuint64_t)W * H * 4; str[2] = (cuuint64_t)W * H * 16 * 4; }
    if (variant == 3) { str[2] = (cuuint64_t)W * H * 4 * 2; }          // distinct strides (dims[3]=16 over 2x range: just a layout test)
    if (variant == 4) { box[0] = 32; sw = CU_TENSOR_MAP_SWIZZLE_128B; }
    if (variant == 5) { sw = CU_TENSOR_MAP_SWIZZLE_NONE; box[3] = 8; }
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<<<1, 128, 64 * 1024>>>(tm, variant == 4 ? 12 : 24, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: encode %d, run %s\n", variant, (int)r, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
