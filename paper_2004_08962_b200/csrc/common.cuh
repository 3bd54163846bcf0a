// Shared device helpers for the HICU B200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hicu_b200.h"

#define HICU_HD __host__ __device__ __forceinline__

// ---------------------------------------------------------------------------
// complex arithmetic on float2 / double2
// ---------------------------------------------------------------------------
HICU_HD float2 cf(float r, float i) { return make_float2(r, i); }
HICU_HD double2 cd(double r, double i) { return make_double2(r, i); }
HICU_HD float2 operator+(float2 a, float2 b) { return cf(a.x + b.x, a.y + b.y); }
HICU_HD float2 operator-(float2 a, float2 b) { return cf(a.x - b.x, a.y - b.y); }
HICU_HD double2 operator+(double2 a, double2 b) { return cd(a.x + b.x, a.y + b.y); }
HICU_HD double2 operator-(double2 a, double2 b) { return cd(a.x - b.x, a.y - b.y); }
HICU_HD double2 operator*(double s, double2 a) { return cd(s * a.x, s * a.y); }
HICU_HD float2 operator*(float s, float2 a) { return cf(s * a.x, s * a.y); }
HICU_HD double2 cmul(double2 a, double2 b) { return cd(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
HICU_HD double2 cmulc(double2 a, double2 b) {  // conj(a) * b
  return cd(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
HICU_HD double2 conjd(double2 a) { return cd(a.x, -a.y); }
HICU_HD double abs2d(double2 a) { return a.x * a.x + a.y * a.y; }
HICU_HD float abs2f(float2 a) { return a.x * a.x + a.y * a.y; }
// acc += a * b
HICU_HD void cfma(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}
// acc += conj(a) * b
HICU_HD void cfmac(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(-a.y, b.x, acc.y);
}
HICU_HD void zfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
HICU_HD void zfmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}

// ---------------------------------------------------------------------------
// geometry as seen by kernels (built on the host from hicu_geom)
// ---------------------------------------------------------------------------
struct DevGeom {
  int ndim;
  int n;
  int ncirc;               // number of circular axes
  int circ_axes[HICU_MAX_NDIM];
  int64_t dims[HICU_MAX_NDIM];
  int64_t stride[HICU_MAX_NDIM];   // k-space element strides (C order)
  int64_t roff[HICU_MAX_NDIM];
  int64_t rext[HICU_MAX_NDIM];
  int64_t rstride[HICU_MAX_NDIM];  // row-major strides of the region block
  int64_t s;                        // region size
  int64_t N;                        // k-space size
  const int32_t* pos;
  const int64_t* koff;
  // coil-structured fast path: last axis is the coil axis, the kernel spans
  // all Nc coils at every spatial tap (kappa = sp*Nc + c), the region has one
  // coil row (rext[last] == 1, roff[last] == 0, not circular).  nc = 0 when
  // the geometry does not have this structure (generic kernels are used).
  int nc;
  int nsp;  // spatial taps (n / nc)
  int64_t kext[HICU_MAX_NDIM];  // kernel bounding box (0 = unknown)
  uint32_t flags;               // hicu_geom flags (HICU_GEOM_*)
};

// Non-circular part of the flat address of row i, plus the region coordinates
// on circular axes (needed for the wrap).
__device__ __forceinline__ int64_t row_base(const DevGeom& g, int64_t i, int* cc) {
  int64_t base = 0;
  int ci = 0;
#pragma unroll
  for (int d = 0; d < HICU_MAX_NDIM; ++d) {
    if (d >= g.ndim) break;
    int64_t r = (i / g.rstride[d]) % g.rext[d];
    if (ci < g.ncirc && g.circ_axes[ci] == d) {
      cc[ci++] = (int)r;
    } else {
      base += (g.roff[d] + r) * g.stride[d];
    }
  }
  return base;
}

// wrap contribution for circular axes: sum_d ((r_d + pos_d) mod N_d) * stride_d
__device__ __forceinline__ int64_t circ_part(const DevGeom& g, const int* cc, const int32_t* pos_k) {
  int64_t a = 0;
  for (int c = 0; c < g.ncirc; ++c) {
    int d = g.circ_axes[c];
    int64_t v = cc[c] + pos_k[d];
    if (v >= g.dims[d]) v -= g.dims[d];
    a += v * g.stride[d];
  }
  return a;
}

// ---------------------------------------------------------------------------
// deterministic block reduction of NV doubles; result valid in thread 0
// ---------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void block_reduce_store(double (&v)[NV], double* out) {
  __shared__ double red[32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) red[warp][k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += red[w][k];
      out[k] = t;
    }
  }
}

// fixed-order warp sum of a strided partial array: parts[j*stride + off]
__device__ __forceinline__ double warp_sum_parts(const double* parts, int np, int stride, int off) {
  const int lane = threadIdx.x & 31;
  double t = 0.0;
  for (int j = lane; j < np; j += 32) t += parts[(size_t)j * stride + off];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// Programmatic dependent launch.  Every kernel of the library starts with
// hicu_pdl_entry(): it waits until the previous grid in the stream has
// completed (and its writes are visible) and then lets the next grid launch,
// so the next kernel's launch and CTA placement overlap this kernel's run.
// A no-op for kernels launched without the attribute.
__device__ __forceinline__ void hicu_pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

bool hicu_pdl_enabled();

// kernel<<<grid, block, smem, stream>>>(args...) with the programmatic
// stream serialization attribute (cudaLaunchKernelEx coerces the arguments to
// the kernel's parameter types); errors surface through hicu_check_launch.
template <typename... KArgs, typename... Args>
inline void hicu_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                        Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = hicu_pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  (void)cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

// hicu_launch for a kernel that runs as thread-block clusters of cluster_x CTAs.
template <typename... KArgs, typename... Args>
inline void hicu_launch_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = hicu_pdl_enabled() ? 1 : 0;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = cluster_x;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  (void)cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

// thread-block-cluster helpers (split arrive / wait)
__device__ __forceinline__ void hicu_cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void hicu_cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ unsigned hicu_cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

int hicu_set_error(int code, const char* msg);
int hicu_check_cuda(cudaError_t e, const char* where);
// count one kernel launch and check it
int hicu_check_launch(const char* where);
int hicu_make_devgeom(const hicu_geom* g, DevGeom* out);
int hicu_sm_count();
// raise a kernel's dynamic shared-memory limit to the device maximum (once)
void hicu_allow_max_smem(const void* func);
// Gram implementations (gram_lag.cu, gram_tc.cu, gram_simt.cu)
bool hicu_gram_lag_supported(const DevGeom& g);
size_t hicu_gram_lag_workspace(const DevGeom& g);
double hicu_gram_lag_flops(const DevGeom& g);
bool hicu_gram_lag_tc(const DevGeom& g);
int hicu_gram_lag(const DevGeom& g, const float2* x, double2* G, void* ws, size_t ws_bytes, cudaStream_t st);
