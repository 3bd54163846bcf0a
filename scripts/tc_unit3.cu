// tcgen05 unit test 3: K-major SWIZZLE_128B operands (32 fp32 K per row) from a planar array;
// derived from unit test 2: K-major SWIZZLE_64B operands loaded by TMA from a
// row-major [rows x 16 floats] array (64-B rows), with descriptor start
// addresses shifted by b rows (b = 0..4) to realise the Hankel overlap:
//   D_b[m, n] = sum_k A[b + m, k] * B[n, k],  m < 128, n < 16, k < 16.
// Variants: base_offset field 0 or (start >> 7) & 7.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_unit2 tc_unit2.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define ROWS 128
#define KK 32
#define NN 32

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw64(uint32_t addr, int base_mode) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;  // SBO = 8 rows x 128 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(base_mode == 0 ? 2 : 1) << 61;  // 2: SWIZZLE_128B (1: 128B with 32B atom, for comparison)
  return d;
}

__global__ void k(const __grid_constant__ CUtensorMap ta, const float* gB, int b, int base_mode, float* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = sm;              // ROWS x 64 B (swizzled by TMA)
  uint8_t* sb = sm + 16384;      // NN rows x 128 B, SW128 by hand
  __shared__ __align__(8) uint64_t bar, mbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // B by hand: row n at n*128, 16-B chunk u stored at u ^ (n & 7)
  for (int e = threadIdx.x; e < NN * KK; e += blockDim.x) {
    const int n = e / KK, kk = e % KK;
    const int u = (kk / 4) ^ (n & 7);
    *(float*)(sb + n * 128 + u * 16 + (kk % 4) * 4) = gB[n * KK + kk];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(ROWS * 128) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(sa)), "l"((uint64_t)&ta), "r"(0), "r"(0), "r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W1;\n\t}"
                 ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int ks = 0; ks < 4; ++ks) {
      const uint64_t ad = desc_sw64(smem_u32(sa) + ks * 32, base_mode);
      const uint64_t bd = desc_sw64(smem_u32(sb) + ks * 32, base_mode);
      const uint32_t acc = ks > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                   ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)) : "memory");
  }
  __syncwarp();
  asm volatile("{\n\t.reg .pred p;\n\tW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n\t}"
               ::"r"(smem_u32(&mbar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int half = 0; half < NN / 16; ++half) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tmem + ((uint32_t)(32 * warp) << 16) + half * 16));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int q = 0; q < 16; ++q) out[(32 * warp + lane) * NN + half * 16 + q] = __uint_as_float(r[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  EncFn enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  float *hA = (float*)malloc(ROWS * KK * 4), *hB = (float*)malloc(NN * KK * 4), *hO = (float*)malloc(128 * NN * 4);
  srand(3);
  for (int i = 0; i < ROWS * KK; ++i) hA[i] = (float)((rand() % 17) - 8) / 8.0f;
  for (int i = 0; i < NN * KK; ++i) hB[i] = (float)((rand() % 13) - 6) / 4.0f;
  float *dA, *dB, *dO;
  cudaMalloc(&dA, ROWS * KK * 4); cudaMalloc(&dB, NN * KK * 4); cudaMalloc(&dO, 128 * NN * 4);
  cudaMemcpy(dA, hA, ROWS * KK * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, NN * KK * 4, cudaMemcpyHostToDevice);
  CUtensorMap ta;
  cuuint64_t dims[2] = {KK, ROWS}, str[1] = {KK * 4};
  cuuint32_t box[2] = {KK, ROWS}, es[2] = {1, 1};
  CUresult rr = enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)rr);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  for (int base_mode = 0; base_mode < 1; ++base_mode)
    for (int b = 0; b < 1; ++b) {
      cudaMemset(dO, 0, 128 * NN * 4);
      k<<<1, 128, 32 * 1024>>>(ta, dB, b, base_mode, dO);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(hO, dO, 128 * NN * 4, cudaMemcpyDeviceToHost);
      double err = 0, mx = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < NN; ++n) {
          double s = 0;
          for (int kk = 0; kk < KK; ++kk) s += (double)hA[m * KK + kk] * hB[n * KK + kk];
          err = fmax(err, fabs(s - hO[m * NN + n]));
          mx = fmax(mx, fabs(s));
        }
      printf("base_mode=%d b=%d: err %g (max %g) %s\n", base_mode, b, err, mx, cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
