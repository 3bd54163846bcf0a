// Rank-2 update throughput probe (hetrd6's D phase in isolation): W warps, each
// thread keeps a[3][8] complex in registers and applies
//   a -= v_i conj(w_j) + wp_i conj(v_j)
// for 8 columns x 3 row slots per iteration (192 DFMA per thread), with v/w
// read from shared memory (broadcast) or from registers.
#include <cstdio>
#include <cuda_runtime.h>
struct d2 { double x, y; };
template <bool SMEM>
__global__ void k(int iters, double* out, long long* cyc) {
  __shared__ d2 sv[96], sw[96];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int i = t; i < 96; i += blockDim.x) { sv[i] = {1e-3 * i, 2e-3}; sw[i] = {3e-3, 1e-3 * i}; }
  __syncthreads();
  d2 a[3][8];
#pragma unroll
  for (int u = 0; u < 3; ++u)
#pragma unroll
    for (int c = 0; c < 8; ++c) a[u][c] = {1.0 + u + c * 1e-3, 0.5 * c};
  d2 vr[3], wr[3];
#pragma unroll
  for (int u = 0; u < 3; ++u) { vr[u] = sv[lane + 32 * u]; wr[u] = sw[lane + 32 * u]; }
  d2 vreg[8], wreg[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { vreg[c] = sv[8 * w + c]; wreg[c] = sw[8 * w + c]; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const d2 vj = SMEM ? sv[(8 * w + c + it) % 96] : vreg[c];
      const d2 wj = SMEM ? sw[(8 * w + c + it) % 96] : wreg[c];
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        d2 x = a[u][c];
        x.x = fma(-vr[u].x, wj.x, fma(-vr[u].y, wj.y, x.x));
        x.x = fma(-wr[u].x, vj.x, fma(-wr[u].y, vj.y, x.x));
        x.y = fma(-vr[u].y, wj.x, fma(vr[u].x, wj.y, x.y));
        x.y = fma(-wr[u].y, vj.x, fma(wr[u].x, vj.y, x.y));
        a[u][c] = x;
      }
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int u = 0; u < 3; ++u)
#pragma unroll
    for (int c = 0; c < 8; ++c) s += a[u][c].x + a[u][c].y;
  out[t] = s;
  if (t == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; long long h;
  cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
  for (int smem = 0; smem < 2; ++smem)
    for (int warps : {1, 4, 8, 12}) {
      const int iters = 200;
      for (int rep = 0; rep < 2; ++rep) {
        if (smem) k<true><<<1, warps * 32>>>(iters, o, c); else k<false><<<1, warps * 32>>>(iters, o, c);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      const double per = (double)h / iters;
      printf("%s warps %2d: %.0f cycles per iteration (192 DFMA/thread) -> %.2f warp-DFMA/clk/SM\n",
             smem ? "v,w from smem" : "v,w in regs  ", warps, per, 192.0 * warps / per);
    }
  return 0;
}
