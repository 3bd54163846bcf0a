// Critical-path inflation probe: warp 0 times a dependent fp64 chain while the
// other warps of the CTA run background fp64 work (independent DFMA streams)
// until warp 0 is done.  Answers: how much slower is a latency-bound warp
// when it shares the SM's fp64 pipes with bulk-update warps?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int mode, int iters, double* out, long long* cyc) {
  __shared__ volatile int done;
  __shared__ double sm[1024];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) done = 0;
  sm[threadIdx.x] = 1.0 + threadIdx.x;
  __syncthreads();
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999, c = 1e-7;
  if (warp == 0) {
    long long t0 = clock64();
    double x = a;
    if (mode == 0 || mode == 2) {
      for (int i = 0; i < iters; ++i) x = fma(x, b, c);
    } else {
      for (int i = 0; i < iters; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      *cyc = t1 - t0;
      done = 1;
    }
    out[threadIdx.x] = x;
  } else {
    double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3;
    long long n = 0;
    while (!done) {
      if (mode == 2) {
#pragma unroll 4
        for (int i = 0; i < 16; ++i) { x0 += sm[(threadIdx.x + i) & 1023]; }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          x0 = fma(x0, b, c); x1 = fma(x1, b, c); x2 = fma(x2, b, c); x3 = fma(x3, b, c);
        }
      }
      ++n;
    }
    out[threadIdx.x] = x0 + x1 + x2 + x3 + n;
  }
}
int main() {
  double* o; long long* c; long long h;
  cudaMalloc(&o, 8192 * 8); cudaMalloc(&c, 8);
  const char* names[] = {"dfma chain vs bg dfma", "shfl+dadd chain vs bg dfma", "dfma chain vs bg lds+dadd"};
  for (int mode = 0; mode < 3; ++mode)
    for (int threads : {32, 64, 128, 256, 512, 1024}) {
      const int iters = 2048;
      k<<<1, threads>>>(mode, iters, o, c);
      k<<<1, threads>>>(mode, iters, o, c);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("%-30s warps %2d: %.2f cyc/op\n", names[mode], threads / 32, (double)h / iters);
    }
  return 0;
}
