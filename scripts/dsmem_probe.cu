// DSMEM probe: cost of pulling a 4 KB vector from one CTA's shared memory
// into registers by many warps of an 8-CTA cluster, vs fewer pullers, vs
// local shared memory; and the cluster-barrier round trip.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

__device__ __forceinline__ double2 ld_dsmem(const double2* local_ptr, unsigned rank) {
  unsigned a = (unsigned)__cvta_generic_to_shared(local_ptr), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(ra) : "memory");
  return v;
}

// mode 0: all warps pull 8 x 16B/lane from CTA 0 (generic mapa pointer)
// mode 1: all warps pull via ld.shared::cluster
// mode 2: warp 0 of each CTA pulls (ld.shared::cluster)
// mode 3: only CTA 1 warp 0 pulls
// mode 4: all warps read local smem
// mode 5: 100 x (arrive.release + wait) round trips
// mode 6: 100 x (arrive.relaxed + wait)
// mode 7: all warps pull from CTA (warp's rank + 1) % 8 (spread sources)
__global__ void __cluster_dims__(8, 1, 1) k(int mode, long long* out) {
  __shared__ double2 buf[256];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = make_double2(rank + i * 1e-3, i);
  cl.sync();
  double acc = 0.0;
  long long t0 = clock64();
  bool pull = true;
  if (mode == 2) pull = wid == 0;
  if (mode == 3) pull = rank == 1 && wid == 0;
  if (mode <= 4 || mode == 7) {
    if (pull) {
      double2 w[8];
      if (mode == 0) {
        const double2* rb = cl.map_shared_rank(buf, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = rb[lane + 32 * u];
      } else if (mode == 4) {
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = buf[lane + 32 * u];
      } else {
        const unsigned src = mode == 7 ? (rank + 1) & 7 : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = ld_dsmem(&buf[lane + 32 * u], src);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += w[u].x + w[u].y;
    }
  } else {
    for (int i = 0; i < 100; ++i) {
      if (mode == 5) cl_arrive(); else cl_arrive_relaxed();
      cl_wait();
    }
  }
  long long t1 = clock64();
  if (lane == 0) out[rank * 32 + wid] = (t1 - t0) + (acc == 12345.0);
  cl.sync();
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 32 * sizeof(long long));
  const char* names[] = {"all warps pull (generic)", "all warps pull (ld.shared::cluster)", "warp0/CTA pulls",
                         "one warp pulls", "all warps local smem", "arrive.release+wait x100",
                         "arrive.relaxed+wait x100", "all warps pull, spread sources"};
  for (int warps : {4, 8, 16}) {
    for (int mode = 0; mode < 8; ++mode) {
      long long best[256];
      for (int rep = 0; rep < 3; ++rep) {
        k<<<8, warps * 32>>>(mode, d);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(best, d, 8 * 32 * sizeof(long long), cudaMemcpyDeviceToHost);
      long long mx = 0, mn = 1LL << 60;
      for (int r = 0; r < 8; ++r)
        for (int w = 0; w < warps; ++w) {
          mx = best[r * 32 + w] > mx ? best[r * 32 + w] : mx;
          mn = best[r * 32 + w] < mn ? best[r * 32 + w] : mn;
        }
      printf("warps/CTA %2d  %-38s max %7lld  min %7lld cycles%s\n", warps, names[mode], mx, mn,
             (mode == 5 || mode == 6) ? " (per 100)" : "");
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
