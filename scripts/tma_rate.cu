// TMA load throughput: CTAs repeatedly load B-byte contiguous boxes (B = 1/4/16 KB) from a
// 64 MB buffer into a 4-deep ring, 24 boxes per stage; reports ns per op and GB/s.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(su(b)), "r"(ph) : "memory");
}
__global__ void k(const __grid_constant__ CUtensorMap tm, int rows_per_box, int stages_total, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[4];
  const int box_bytes = rows_per_box * 64;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[i])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  const int nbox = box_bytes >= 24 * 1024 ? 1 : 24 * 1024 / box_bytes;  // ~24 KB per stage
  for (int s = 0; s < stages_total + 4; ++s) {
    const int slot = s & 3;
    if (s >= 4) wait(&full[slot], ((s >> 2) - 1) & 1);
    if (s < stages_total) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[slot])), "r"(nbox * box_bytes) : "memory");
      for (int q = 0; q < nbox; ++q) {
        const int row = ((blockIdx.x * 977 + s * 131 + q * 37) % 4000) * 64;  // pseudo-random 64-row-aligned
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su(sm + slot * 24 * 1024 + q * box_bytes)), "l"((uint64_t)&tm), "r"(0), "r"(row), "r"(su(&full[slot])) : "memory");
      }
    }
  }
  cyc[blockIdx.x] = clock64() - t0;
}
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  EncFn enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const size_t rows = 1 << 20;  // 64 MB of 64-B rows
  float* d; cudaMalloc(&d, rows * 64);
  long long* c; cudaMalloc(&c, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int rpb : {16, 64, 128}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {16, rows}, str[1] = {64};
    cuuint32_t box[2] = {16, (cuuint32_t)rpb}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int grid : {1, 148}) {
      const int stages = 400;
      k<<<grid, 32, 100 * 1024>>>(tm, rpb, stages, c);
      k<<<grid, 32, 100 * 1024>>>(tm, rpb, stages, c);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, c, grid * 8, cudaMemcpyDeviceToHost);
      long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      const double nops = (double)stages * (24 * 1024 / (rpb * 64));  // rpb <= 128: 24 KB per stage exactly
      const double us = mx / 1965.0;
      printf("box %5d B grid %3d: %.1f cycles/op, %.1f GB/s total (%s)\n", rpb * 64, grid, mx / nops,
             grid * stages * 24 * 1024.0 / (us * 1e3), cudaGetErrorString(e));
    }
  }
  return 0;
}
