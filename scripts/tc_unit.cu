// Standalone tcgen05 unit test: D = A^T B, A (K x M) and B (K x N) row-major in
// global memory (MN contiguous).  Modes:
//   0: TMA-loaded MN-major SWIZZLE_64B tiles (16-float boxes)
//   1: manual fill of K-major no-swizzle (INTERLEAVE) core matrices
//   2: manual fill of MN-major SW64 tiles (no TMA) with the XOR pattern
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_unit tc_unit.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define M 128
#define N 64
#define K 16

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Variant {
  int mode;
  int a_major, b_major;  // idesc bits
  int layout;            // descriptor layout type
  int lbo, sbo;          // bytes
  int version;
};

__device__ __forceinline__ uint64_t mkdesc(uint32_t addr, const Variant& v) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((v.lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((v.sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)v.version << 46;
  d |= (uint64_t)v.layout << 61;
  return d;
}

__global__ void tc_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, Variant v,
                          const float* gA, const float* gB, float* out, unsigned long long* dbg) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = sm;
  uint8_t* sb = sm + 64 * 1024;
  __shared__ __align__(8) uint64_t bar, mbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const int nks = K / 8;
  if (v.mode == 1) {
    for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
      const int m = e % M, k = e / M;
      const int off = (k / 8) * M * 32 + (m / 8) * v.sbo + ((k % 8) / 4) * v.lbo + (m % 8) * 16 + (k % 4) * 4;
      *(float*)(sa + off) = gA[k * M + m];
    }
    for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
      const int n = e % N, k = e / N;
      const int off = (k / 8) * N * 32 + (n / 8) * v.sbo + ((k % 8) / 4) * v.lbo + (n % 8) * 16 + (k % 4) * 4;
      *(float*)(sb + off) = gB[k * N + n];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  } else if (v.mode == 2) {
    for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
      const int m = e % M, k = e / M;
      const int c = m / 16, u = (m % 16) / 4, w = m % 4;
      const int addr = c * 1024 + k * 64;
      const int sw = (u ^ ((addr >> 7) & 3));
      *(float*)(sa + addr + sw * 16 + w * 4) = gA[k * M + m];
    }
    for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
      const int n = e % N, k = e / N;
      const int c = n / 16, u = (n % 16) / 4, w = n % 4;
      const int addr = c * 1024 + k * 64;
      const int sw = (u ^ ((addr >> 7) & 3));
      *(float*)(sb + addr + sw * 16 + w * 4) = gB[k * N + n];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  } else if (v.mode == 3) {
    // MN-major INTERLEAVE: (mn, k) at (mn/4)*SBO + (k/8)*LBO + (k%8)*16 + (mn%4)*4
    for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
      const int m = e % M, k = e / M;
      *(float*)(sa + (m / 4) * v.sbo + (k / 8) * v.lbo + (k % 8) * 16 + (m % 4) * 4) = gA[k * M + m];
    }
    for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
      const int n = e % N, k = e / N;
      *(float*)(sb + (n / 4) * v.sbo + (k / 8) * v.lbo + (k % 8) * 16 + (n % 4) * 4) = gB[k * N + n];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  } else if (v.mode == 4 || v.mode == 5) {
    // MN-major swizzled, span W bytes (128 or 32): chunk c of W/4 elements at c*LBO; row k at (k%8)*W + (k/8)*SBO;
    // 16-B unit u stored at u ^ ((addr >> 7) & (W/16 - 1))
    const int W = v.mode == 4 ? 128 : 32;
    const int E = W / 4;
    for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
      const int m = e % M, k = e / M;
      const int c = m / E, u = (m % E) / 4, w = m % 4;
      const int addr = c * v.lbo + (k / 8) * v.sbo + (k % 8) * W;
      const int sw = u ^ ((addr >> 7) & (W / 16 - 1));
      *(float*)(sa + addr + sw * 16 + w * 4) = gA[k * M + m];
    }
    for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
      const int n = e % N, k = e / N;
      const int c = n / E, u = (n % E) / 4, w = n % 4;
      const int addr = c * v.lbo + (k / 8) * v.sbo + (k % 8) * W;
      const int sw = u ^ ((addr >> 7) & (W / 16 - 1));
      *(float*)(sb + addr + sw * 16 + w * 4) = gB[k * N + n];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  } else if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(12 * 1024)
                 : "memory");
    for (int c = 0; c < 8; ++c)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(sa + c * 1024)),
          "l"((uint64_t)&ta), "r"(c * 16), "r"(0), "r"(smem_u32(&bar))
          : "memory");
    for (int c = 0; c < 4; ++c)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(sb + c * 1024)),
          "l"((uint64_t)&tb), "r"(c * 16), "r"(0), "r"(smem_u32(&bar))
          : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W1;\n\t}" ::"r"(
            smem_u32(&bar))
        : "memory");
    for (int q = 0; q < 8; ++q) dbg[q] = ((unsigned long long*)sa)[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)v.a_major << 15) |
                           ((uint32_t)v.b_major << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int ks = 0; ks < nks; ++ks) {
      uint32_t koff_a = v.mode == 1 ? ks * M * 32 : ks * 512;
      uint32_t koff_b = v.mode == 1 ? ks * N * 32 : ks * 512;
      if (v.mode == 3 || v.mode == 4 || v.mode == 5) { koff_a = ks * (v.mode == 3 ? v.lbo : v.sbo); koff_b = koff_a; }
      const uint64_t ad = mkdesc(smem_u32(sa) + koff_a, v), bd = mkdesc(smem_u32(sb) + koff_b, v);
      dbg[8 + ks] = ad;
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(
              tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar))
                 : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n\t.reg .pred p;\n\tW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n\t}" ::"r"(
          smem_u32(&mbar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int col = 0; col < N; col += 16) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(tmem + ((uint32_t)(32 * warp) << 16) + col));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int q = 0; q < 16; ++q) out[(32 * warp + lane) * N + col + q] = __uint_as_float(r[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  EncFn enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  float *hA = (float*)malloc(K * M * 4), *hB = (float*)malloc(K * N * 4);
  srand(1);
  for (int i = 0; i < K * M; ++i) hA[i] = (float)((rand() % 17) - 8) / 8.0f;
  for (int i = 0; i < K * N; ++i) hB[i] = (float)((rand() % 13) - 6) / 4.0f;
  float *dA, *dB, *dO;
  unsigned long long* dbg;
  cudaMalloc(&dA, K * M * 4);
  cudaMalloc(&dB, K * N * 4);
  cudaMalloc(&dO, M * N * 4);
  cudaMalloc(&dbg, 256);
  cudaMemcpy(dA, hA, K * M * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, K * N * 4, cudaMemcpyHostToDevice);
  CUtensorMap ta, tb;
  cuuint64_t da[2] = {M, K}, sa[1] = {M * 4}, db[2] = {N, K}, sbs[1] = {N * 4};
  cuuint32_t box[2] = {16, 16}, es[2] = {1, 1};
  CUresult r1 = enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, da, sa, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, db, sbs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d  A[0..3]=%g %g %g %g\n", (int)r1, (int)r2, hA[0], hA[1], hA[2], hA[3]);
  float* ref = (float*)malloc(M * N * 4);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)hA[k * M + m] * hB[k * N + n];
      ref[m * N + n] = (float)s;
    }
  Variant vs[] = {
      {1, 0, 0, 0, 128, 256, 1},
      {3, 1, 1, 0, 4096, 128, 1},   // MN interleave: LBO = K-group stride (32 groups*128B), SBO = 128
      {3, 1, 1, 0, 128, 4096, 1},
      {4, 1, 1, 2, 1024, 2048, 1},  // SW128 MN: chunk (32 el) stride LBO=1024? (8 rows*128B), SBO = K group stride
      {4, 1, 1, 2, 2048, 1024, 1},
      {5, 1, 1, 6, 256, 4096, 1},   // SW32 MN: chunk (8 el) at 256 B, K groups at 4096
      {5, 1, 1, 6, 4096, 256, 1},
  };
  cudaFuncSetAttribute(tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024 + 1024);
  float* hO = (float*)malloc(M * N * 4);
  for (auto v : vs) {
    cudaMemset(dO, 0, M * N * 4);
    cudaMemset(dbg, 0, 256);
    tc_kernel<<<1, 128, 128 * 1024 + 1024>>>(ta, tb, v, dA, dB, dO, dbg);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hO, dO, M * N * 4, cudaMemcpyDeviceToHost);
    unsigned long long hd[16];
    cudaMemcpy(hd, dbg, 128, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int i = 0; i < M * N; ++i) {
      err = fmax(err, fabs(hO[i] - ref[i]));
      mx = fmax(mx, fabs(ref[i]));
    }
    float* f = (float*)hd;
    printf("mode=%d amaj=%d layout=%d lbo=%d sbo=%d: err %g (max %g) %s o=%g %g %g ref=%g %g %g | smem %g %g %g %g | desc %llx\n",
           v.mode, v.a_major, v.layout, v.lbo, v.sbo, err, mx, cudaGetErrorString(e), hO[0], hO[1], hO[N], ref[0],
           ref[1], ref[N], f[0], f[1], f[2], f[3], hd[8]);
    if (e != cudaSuccess) break;
  }
  return 0;
}
