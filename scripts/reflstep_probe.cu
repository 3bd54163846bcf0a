// Cycles per "reflector step" (dot over l entries, warp reduction, axpy) in one warp,
// for several implementations.  l = 90 complex doubles, data in shared memory.
#include <cstdio>
#include <cuda_runtime.h>
struct z2 { double x, y; };
__device__ __forceinline__ double2 cm(double2 a, double2 b) { return make_double2(a.x*b.x - a.y*b.y, a.x*b.y + a.y*b.x); }
__device__ __forceinline__ void zfmac(double2& acc, double2 a, double2 b) {  // acc += conj(a) b
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(-a.y, b.x, acc.y);
}
template <int MODE>
__global__ void k(int l, int steps, const double2* __restrict__ gv, double2* out, long long* cyc) {
  __shared__ double2 v[60 * 40];
  __shared__ double2 x[128];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 60 * 40; i += blockDim.x) v[i] = gv[i];
  for (int i = threadIdx.x; i < l; i += blockDim.x) x[i] = make_double2(1.0 / (i + 1), 0.5);
  __syncthreads();
  double2 xr[3];
  for (int u = 0; u < 3; ++u) { const int i = lane + 32 * u; xr[u] = i < l ? x[i] : make_double2(0, 0); }
  long long t0 = clock64();
  if (MODE == 4) {
    for (int s = 0; s < steps; ++s) {
      const int kk = (s % 60);
      const double2* w = v + (size_t)(kk % 20) * 90;
      double2 wr[3];
#pragma unroll
      for (int u = 0; u < 3; ++u) { const int i = lane + 32 * u; wr[u] = (i > kk && i < l) ? w[i] : make_double2(0, 0); }
      double2 d0 = make_double2(0, 0), d1 = d0, d2 = d0;
      zfmac(d0, wr[0], xr[0]); zfmac(d1, wr[1], xr[1]); zfmac(d2, wr[2], xr[2]);
      double2 dot = make_double2(d0.x + d1.x + d2.x, d0.y + d1.y + d2.y);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double a = __shfl_xor_sync(0xffffffffu, dot.x, o), b = __shfl_xor_sync(0xffffffffu, dot.y, o);
        dot.x += a; dot.y += b;
      }
      const double2 f = cm(make_double2(0.3, 0.1), dot);
#pragma unroll
      for (int u = 0; u < 3; ++u) { xr[u].x -= wr[u].x*f.x - wr[u].y*f.y; xr[u].y -= wr[u].x*f.y + wr[u].y*f.x; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { *cyc = t1 - t0; out[0] = xr[0]; }
    return;
  }
  for (int s = 0; s < steps; ++s) {
    const int kk = (s % 60);
    const double2* w = v + (size_t)(kk % 20) * 90;
    double2 dot = make_double2(0, 0);
    if (MODE == 0) {  // 32-lane stride, 5-level xor reduction of two doubles
      for (int i = kk + 1 + lane; i < l; i += 32) zfmac(dot, w[i], x[i]);
      for (int o = 16; o > 0; o >>= 1) { dot.x += __shfl_xor_sync(0xffffffffu, dot.x, o); dot.y += __shfl_xor_sync(0xffffffffu, dot.y, o); }
    } else if (MODE == 1) {  // same but reduction interleaved manually
      for (int i = kk + 1 + lane; i < l; i += 32) zfmac(dot, w[i], x[i]);
      #pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double a = __shfl_xor_sync(0xffffffffu, dot.x, o), b = __shfl_xor_sync(0xffffffffu, dot.y, o);
        dot.x += a; dot.y += b;
      }
    } else if (MODE == 2) {  // no reduction at all (lower bound: loads + fma + axpy)
      for (int i = kk + 1 + lane; i < l; i += 32) zfmac(dot, w[i], x[i]);
    } else if (MODE == 4) {  // handled below (register-resident)
    } else if (MODE == 3) {  // reduction through shared memory by lane 0 (serial 32)
      for (int i = kk + 1 + lane; i < l; i += 32) zfmac(dot, w[i], x[i]);
      __shared__ double2 red[32];
      red[lane] = dot; __syncwarp();
      if (lane == 0) { double2 t = make_double2(0,0); for (int q = 0; q < 32; ++q) { t.x += red[q].x; t.y += red[q].y; } red[0] = t; }
      __syncwarp(); dot = red[0]; __syncwarp();
    }
    const double2 f = cm(make_double2(0.3, 0.1), dot);
    for (int i = kk + 1 + lane; i < l; i += 32) { const double2 wi = w[i]; x[i] = make_double2(x[i].x - (wi.x*f.x - wi.y*f.y), x[i].y - (wi.x*f.y + wi.y*f.x)); }
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { *cyc = t1 - t0; out[0] = x[5]; }
}
int main() {
  double2 *gv, *o; long long* c; long long h;
  cudaMalloc(&gv, sizeof(double2) * 128 * 96); cudaMemset(gv, 0, sizeof(double2) * 128 * 96);
  cudaMalloc(&o, 64); cudaMalloc(&c, 8);
  const char* names[] = {"xor-reduce 5 levels (2 doubles)", "xor-reduce interleaved", "no reduction", "smem serial reduce",
                         "register-resident x, loads up front"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<1, 32>>>(90, 600, gv, o, c);
      if (mode == 1) k<1><<<1, 32>>>(90, 600, gv, o, c);
      if (mode == 2) k<2><<<1, 32>>>(90, 600, gv, o, c);
      if (mode == 3) k<3><<<1, 32>>>(90, 600, gv, o, c);
      if (mode == 4) k<4><<<1, 32>>>(90, 600, gv, o, c);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-36s: %.1f cycles/step (%s)\n", names[mode], (double)h / 600, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
