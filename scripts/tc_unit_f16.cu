// tcgen05 unit test: kind::f16 (fp16 inputs, fp32 accumulate) with K-major
// SWIZZLE_32B operands (rows of 16 halfs = 32 B, 8-row atoms of 256 B),
// written by hand in shared memory; checks D = A B^T (M = 128, K = 16) for
// N in {32, 80, 160, 256}, then times back-to-back MMA chains of kind::f16
// (K = 16) against kind::tf32 (K = 8, SW64 rows of 16 floats) at equal N.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_unit_f16 tc_unit_f16.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, int sbo, int layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// sw32 K-major half layout: row r, half k (0..15) -> byte r*32 + ((k>>3) ^ ((r>>2)&1))*16 + (k&7)*2
__device__ __forceinline__ int off32(int r, int k) { return r * 32 + (((k >> 3) ^ ((r >> 2) & 1)) << 4) + (k & 7) * 2; }
// sw64 K-major float layout: row r, float k (0..15)
__device__ __forceinline__ int off64(int r, int k) { return r * 64 + (((k >> 2) ^ ((r >> 1) & 3)) << 4) + (k & 3) * 4; }

__global__ void k(const float* gA, const float* gB, int N, int mode, int reps, int nacc, float* out, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = sm;          // 128 rows
  uint8_t* sb = sm + 8192;   // N rows
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int e = threadIdx.x; e < 128 * 16; e += blockDim.x) {
    const int r = e / 16, kk = e % 16;
    if (mode == 0) *(__half*)(sa + off32(r, kk)) = __float2half_rn(gA[e]);
    else *(float*)(sa + off64(r, kk)) = gA[e];
  }
  for (int e = threadIdx.x; e < N * 16; e += blockDim.x) {
    const int r = e / 16, kk = e % 16;
    if (mode == 0) *(__half*)(sb + off32(r, kk)) = __float2half_rn(gB[e]);
    else *(float*)(sb + off64(r, kk)) = gB[e];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = mode == 0 ? ((1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24))
                                     : ((1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                                        ((uint32_t)(128 >> 4) << 24));
    const long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
      if (mode == 0) {
        const uint64_t ad = desc(smem_u32(sa), 256, 6), bd = desc(smem_u32(sb), 256, 6);
        const uint32_t acc = rep >= nacc;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem + (rep % nacc) * N), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      } else {
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t ad = desc(smem_u32(sa) + ks * 32, 512, 4), bd = desc(smem_u32(sb) + ks * 32, 512, 4);
          const uint32_t acc = rep >= nacc || ks > 0;
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(tmem + (rep % nacc) * N), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n\t}"
                 ::"r"(smem_u32(&mbar)) : "memory");
    *cyc = clock64() - t0;
  }
  __syncwarp();
  asm volatile("{\n\t.reg .pred p;\n\tW3:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W3;\n\t}"
               ::"r"(smem_u32(&mbar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tmem + ((uint32_t)(32 * warp) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int q = 0; q < 16; ++q) out[(32 * warp + lane) * N + c + q] = __uint_as_float(r[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int main() {
  const int NMAX = 256;
  float *hA = (float*)malloc(128 * 16 * 4), *hB = (float*)malloc(NMAX * 16 * 4), *hO = (float*)malloc(128 * NMAX * 4);
  srand(3);
  // values exactly representable in fp16 (and tf32)
  for (int i = 0; i < 128 * 16; ++i) hA[i] = (float)((rand() % 17) - 8) / 8.0f;
  for (int i = 0; i < NMAX * 16; ++i) hB[i] = (float)((rand() % 13) - 6) / 4.0f;
  float *dA, *dB, *dO;
  long long* dc;
  cudaMalloc(&dA, 128 * 16 * 4); cudaMalloc(&dB, NMAX * 16 * 4); cudaMalloc(&dO, 128 * NMAX * 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, hA, 128 * 16 * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, NMAX * 16 * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int Ns[4] = {32, 80, 160, 256};
  int bad = 0;
  for (int mode = 0; mode < 2; ++mode)
    for (int ni = 0; ni < 4; ++ni) {
      const int N = Ns[ni];
      for (int nacc : {1, 2, 3}) {
        if (nacc * N > 512) continue;
        const int reps = 2000 - 2000 % (nacc * 2);
        cudaMemset(dO, 0, 128 * NMAX * 4);
        k<<<1, 128, 64 * 1024>>>(dA, dB, N, mode, reps, nacc, dO, dc);
        cudaError_t e = cudaDeviceSynchronize();
        long long cyc = 0;
        cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(hO, dO, 128 * N * 4, cudaMemcpyDeviceToHost);
        double err = 0, mx = 0;
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int kk = 0; kk < 16; ++kk) s += (double)hA[m * 16 + kk] * hB[n * 16 + kk];
            s *= reps / nacc;
            err = fmax(err, fabs(s - hO[m * N + n]));
            mx = fmax(mx, fabs(s));
          }
        const int nmma = mode == 0 ? reps : 2 * reps;
        printf("%s N=%3d nacc=%d reps=%4d: rel err %.2e  cycles/MMA %.1f  (K=16 per %.1f cycles) %s\n",
               mode == 0 ? "f16 " : "tf32", N, nacc, reps, err / mx, (double)cyc / nmma, (double)cyc / reps,
               cudaGetErrorString(e));
        if (e != cudaSuccess || err / mx > 1e-6) bad = 1;
      }
    }
  return bad;
}
