// tcgen05 kind::f16 issue-rate probe (timing only, zeroed operands): cycles per
// MMA for back-to-back chains rotating over `nacc` accumulators, as a function
// of the operand swizzle (SW32 / SW64 / SW128 K-major rows: the K = 16 step
// is one row (SW32) or one of 2 / 4 sub-steps of a wider row), N, and
// cta_group (::1 with M = 128; ::2 with M = 256 over a CTA pair).
// Question it answers: is the convolution's ~142-cycle-per-MMA cost a
// per-instruction overhead (then fewer, wider MMAs / M = 256 pay) or the
// operand-read floor of narrow swizzles?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_rate2 tc_rate2.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

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

template <int CG>
__global__ void k(int N, int rowb, int reps, int nacc, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  uint8_t* sa = sm;              // 128 rows x rowb
  uint8_t* sb = sm + 128 * 128;  // N rows x rowb
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const int layout = rowb == 32 ? 6 : (rowb == 64 ? 4 : 2);
  const int ksub = rowb / 32;
  if (threadIdx.x == 0 && rank == 0) {
    const int M = 128 * CG;
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint64_t ad0 = desc(smem_u32(sa), 8 * rowb, layout), bd0 = desc(smem_u32(sb), 8 * rowb, layout);
    const long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
      const int ks = rep % ksub;
      const uint64_t ad = ad0 + (uint64_t)(2 * ks), bd = bd0 + (uint64_t)(2 * ks);
      const uint32_t acc = rep >= nacc;
      const uint32_t d = tmem + (uint32_t)((rep % nacc) * N);
      if (CG == 1)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    if (CG == 1)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   ::"r"(smem_u32(&mbar)), "h"((uint16_t)3) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n\t}"
                 ::"r"(smem_u32(&mbar)) : "memory");
    *cyc = clock64() - t0;
  }
  if (CG == 2 && rank == 1 && threadIdx.x == 0)
    asm volatile("{\n\t.reg .pred p;\n\tW3:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W3;\n\t}"
                 ::"r"(smem_u32(&mbar)) : "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int main() {
  long long* dc;
  cudaMalloc(&dc, 8);
  const int smem = 100 * 1024;
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int Ns[6] = {32, 80, 128, 160, 240, 256};
  for (int cg = 1; cg <= 2; ++cg)
    for (int rowb : {32, 64, 128})
      for (int ni = 0; ni < 6; ++ni)
        for (int nacc : {1, 2}) {
          const int N = Ns[ni];
          if (cg == 2 && (N % 16)) continue;
          if (nacc * N > 512) continue;
          const int reps = 4000;
          cudaError_t e;
          if (cg == 1) {
            k<1><<<1, 128, smem>>>(N, rowb, reps, nacc, dc);
          } else {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(2);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k<2>, N, rowb, reps, nacc, dc);
          }
          e = cudaDeviceSynchronize();
          long long cyc = 0;
          cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
          const double c = (double)cyc / reps;
          const double floor = 128.0 * N / 256.0;  // per-SM f16 floor (cycles per K = 16 MMA at M = 128 per SM)
          printf("cta_group::%d M=%3d rowB=%3d N=%3d nacc=%d: %.1f cyc/MMA  floor %.1f  eff %.2f %s\n", cg, 128 * cg,
                 rowb, N, nacc, c, floor, floor / c, cudaGetErrorString(e));
          if (e != cudaSuccess) return 1;
        }
  return 0;
}
