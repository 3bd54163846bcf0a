// fp64 latency / throughput probe on one SM: dependent DFMA chain, independent
// DFMA streams, double division and sqrt, shared-memory load latency.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int mode, int iters, double* out, long long* cyc) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999, c = 1e-7;
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  __shared__ double sm[1024];
  sm[threadIdx.x] = a;
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0) {
    for (int i = 0; i < iters; ++i) x0 = fma(x0, b, c);
  } else if (mode == 1) {
    for (int i = 0; i < iters; ++i) {
      x0 = fma(x0, b, c); x1 = fma(x1, b, c); x2 = fma(x2, b, c); x3 = fma(x3, b, c);
      x4 = fma(x4, b, c); x5 = fma(x5, b, c); x6 = fma(x6, b, c); x7 = fma(x7, b, c);
    }
  } else if (mode == 2) {
    for (int i = 0; i < iters; ++i) x0 = 1.0 / (x0 + 1.0);
  } else if (mode == 3) {
    for (int i = 0; i < iters; ++i) x0 = sqrt(x0 + 1.0);
  } else if (mode == 4) {
    int idx = threadIdx.x;
    for (int i = 0; i < iters; ++i) { x0 += sm[idx]; idx = (idx + (int)x0) & 1023; }
  } else if (mode == 5) {
    for (int i = 0; i < iters; ++i) { x0 = __shfl_xor_sync(0xffffffffu, x0, 1) + 1.0; }
  } else if (mode == 6) {
    for (int i = 0; i < iters; ++i) __syncthreads();
  }
  long long t1 = clock64();
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; long long h;
  cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
  const char* names[] = {"dfma dependent chain (cyc/op)", "dfma 8 indep streams (cyc/iter of 8)", "ddiv chain (cyc/op)",
                         "dsqrt chain (cyc/op)", "lds dependent (cyc/op)", "shfl+dadd chain (cyc/op)", "syncthreads (cyc/op)"};
  for (int mode = 0; mode < 7; ++mode)
    for (int threads : {32, 128, 512, 1024}) {
      const int iters = 4096;
      k<<<1, threads>>>(mode, iters, o, c);
      k<<<1, threads>>>(mode, iters, o, c);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("%-40s threads %4d: %.2f\n", names[mode], threads, (double)h / iters);
    }
  return 0;
}
