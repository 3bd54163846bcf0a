// SVD coil compression: covariance over sampled locations and the apply
// pass.  HBM-bound; no reference function (SPEC.md:8 leaves it out of the
// reference package; the paper compresses before reconstruction,
// PAPER.md:170,179,184).
//   cov[a][b] = sum_{l: mask[l,0]==1} conj(x[l,a]) x[l,b]   (8*N_in bytes read)
//   y[l, j]   = sum_c x[l, c] basis[c, j]                   (8*N_in + 8*N_out)
#include "common.cuh"

namespace {

constexpr int kLocPerBlock = 64;

int cov_blocks(int64_t nloc) {
  int64_t b = (nloc + 1023) / 1024;
  int64_t cap = (int64_t)hicu_sm_count() * 4;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

// block b accumulates a contiguous slice of locations into parts[b][nc][nc]
__global__ void __launch_bounds__(1024) coil_cov_kernel(int64_t nloc, int nc, const float2* __restrict__ x, const uint8_t* __restrict__ mask,
                                int64_t per_block, double2* __restrict__ parts) {
  hicu_pdl_entry();
  __shared__ float2 xs[kLocPerBlock][33];
  __shared__ uint8_t ms[kLocPerBlock];
  const int64_t l0 = (int64_t)blockIdx.x * per_block;
  int64_t l1 = l0 + per_block;
  if (l1 > nloc) l1 = nloc;
  const int a = threadIdx.x / nc, b = threadIdx.x % nc;
  const bool active = threadIdx.x < nc * nc;
  double2 acc = cd(0.0, 0.0);
  for (int64_t lc = l0; lc < l1; lc += kLocPerBlock) {
    const int cnt = (int)((l1 - lc) < kLocPerBlock ? (l1 - lc) : kLocPerBlock);
    for (int e = threadIdx.x; e < cnt * nc; e += blockDim.x) {
      const int li = e / nc, c = e % nc;
      const int64_t idx = (lc + li) * nc + c;
      xs[li][c] = mask[idx] == 1 ? x[idx] : cf(0.f, 0.f);  // mask_apply fused (x may be raw k-space)
    }
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) ms[e] = mask[(lc + e) * nc];
    __syncthreads();
    if (active) {
      for (int li = 0; li < cnt; ++li) {
        if (ms[li] != 1) continue;
        const float2 xa = xs[li][a], xb = xs[li][b];
        acc.x += (double)xa.x * xb.x + (double)xa.y * xb.y;
        acc.y += (double)xa.x * xb.y - (double)xa.y * xb.x;
      }
    }
    __syncthreads();
  }
  if (active) parts[(size_t)blockIdx.x * nc * nc + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(1024) coil_cov_reduce(int nc, int nparts, const double2* __restrict__ parts, double2* __restrict__ cov) {
  hicu_pdl_entry();
  const int e = threadIdx.x;
  if (e >= nc * nc) return;
  double2 s = cd(0.0, 0.0);
  for (int k = 0; k < nparts; ++k) s = s + parts[(size_t)k * nc * nc + e];
  cov[e] = s;
}

__global__ void coil_apply_kernel(int64_t nloc, int nc, int nv, const float2* __restrict__ x,
                                  const uint8_t* __restrict__ mask, const double2* __restrict__ basis,
                                  float2* __restrict__ y, uint8_t* __restrict__ mask_out) {
  hicu_pdl_entry();
  __shared__ float2 sb[32 * 32];
  for (int e = threadIdx.x; e < nc * nv; e += blockDim.x) {
    const double2 v = basis[e];
    sb[e] = cf((float)v.x, (float)v.y);
  }
  __syncthreads();
  const int64_t total = nloc * nv;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = e / nv;
    const int j = (int)(e % nv);
    const float2* xl = x + l * nc;
    float2 acc = cf(0.f, 0.f);
    if (mask) {  // mask_apply fused (arrays.py:54-67): unobserved entries read as zero
      const uint8_t* ml = mask + l * nc;
      for (int c = 0; c < nc; ++c)
        if (ml[c] == 1) cfma(acc, xl[c], sb[c * nv + j]);
    } else {
      for (int c = 0; c < nc; ++c) cfma(acc, xl[c], sb[c * nv + j]);
    }
    y[e] = acc;
    if (mask_out) mask_out[e] = mask[l * nc];
  }
}

}  // namespace

extern "C" size_t hicu_coil_workspace(int64_t nloc, int nc) {
  return (size_t)cov_blocks(nloc) * nc * nc * sizeof(double2);
}

extern "C" int hicu_coil_cov(int64_t nloc, int nc, const void* x, const uint8_t* mask, void* cov, void* ws,
                             size_t ws_bytes, void* stream) {
  if (nloc < 1 || nc < 1 || nc > 32 || !x || !mask || !cov || !ws)
    return hicu_set_error(HICU_ERR_PARAMETER, "coil_cov: bad arguments");
  if (ws_bytes < hicu_coil_workspace(nloc, nc)) return hicu_set_error(HICU_ERR_WORKSPACE, "coil_cov: workspace");
  const int blocks = cov_blocks(nloc);
  const int64_t per = (nloc + blocks - 1) / blocks;
  cudaStream_t st = (cudaStream_t)stream;
  hicu_launch(coil_cov_kernel, blocks, 1024, 0, st, nloc, nc, (const float2*)x, mask, per, (double2*)ws);
  int s = hicu_check_launch("coil_cov_kernel");
  if (s) return s;
  hicu_launch(coil_cov_reduce, 1, 1024, 0, st, nc, blocks, (const double2*)ws, (double2*)cov);
  return hicu_check_launch("coil_cov_reduce");
}

extern "C" int hicu_coil_apply(int64_t nloc, int nc, int nv, const void* x, const uint8_t* mask, const void* basis,
                               void* y, uint8_t* mask_out, void* stream) {
  if (nloc < 1 || nc < 1 || nc > 32 || nv < 1 || nv > nc || !x || !basis || !y || (mask_out && !mask))
    return hicu_set_error(HICU_ERR_PARAMETER, "coil_apply: bad arguments");
  int64_t blocks = (nloc * nv + 255) / 256;
  int64_t cap = (int64_t)hicu_sm_count() * 8;
  if (blocks > cap) blocks = cap;
  hicu_launch(coil_apply_kernel, (int)blocks, 256, 0, (cudaStream_t)stream, nloc, nc, nv, (const float2*)x, mask,
                                                                   (const double2*)basis, (float2*)y, mask_out);
  return hicu_check_launch("coil_apply_kernel");
}
