// mbarrier hand-off latency: two warps ping-pong through two mbarriers
// (count 1) with try_wait (default), try_wait + suspend-time hint, and a
// test_wait spin; plus the latency of a tcgen05.commit arrive with no MMA
// outstanding (the pipeline skeleton's empty-barrier hop).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
template <int MODE>
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  if (MODE == 0) {
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(sa(b)), "r"(ph) : "memory");
  } else if (MODE == 1) {
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 20;\n\t@!p bra W_%=;\n\t}" ::"r"(sa(b)), "r"(ph) : "memory");
  } else {
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(sa(b)), "r"(ph) : "memory");
  }
}
template <int MODE>
__global__ void pingpong(int iters, long long* out) {
  __shared__ __align__(8) uint64_t b[2];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&b[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&b[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (MODE == 3 && warp == 1)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(sa(&tslot)));
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t ph = i & 1;
    if (warp == 0) {
      if (lane == 0) arrive(&b[0]);
      if (MODE == 3) wait<0>(&b[1], ph); else wait<MODE>(&b[1], ph);
    } else if (warp == 1) {
      if (MODE == 3) {
        wait<0>(&b[0], ph);
        if (lane == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&b[1])) : "memory");
        __syncwarp();
      } else {
        wait<MODE>(&b[0], ph);
        if (lane == 0) arrive(&b[1]);
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *out = (t1 - t0) / iters;
  __syncthreads();
  if (MODE == 3 && warp == 1) {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tslot));
  }
}
int main() {
  long long* d; long long h;
  cudaMalloc(&d, 8);
  const char* names[] = {"try_wait", "try_wait hint 20ns", "test_wait spin", "tcgen05.commit hop"};
  for (int m = 0; m < 4; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) pingpong<0><<<1, 64>>>(2000, d);
      if (m == 1) pingpong<1><<<1, 64>>>(2000, d);
      if (m == 2) pingpong<2><<<1, 64>>>(2000, d);
      if (m == 3) pingpong<3><<<1, 64>>>(2000, d);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-22s round trip %lld cycles  (%s)\n", names[m], h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
