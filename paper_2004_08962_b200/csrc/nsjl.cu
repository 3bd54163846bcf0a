// Closed-form JL-compressed nullspace: Q~ = Q [P] without forming the
// Householder reflectors one column at a time.
//
// The reference (subspace.py:158-212) triangularises V (n x r, orthonormal
// columns) with r reflections H_k = I - tau_k w_k w_k^H (w_k[k] = 1), each
// mapping its pivot to a NONNEGATIVE real beta_k, and returns
// Q = H_0^H ... H_{r-1}^H [0; I].  For orthonormal V that convention forces
// R = I (the Cholesky factor of V^H V = I with a positive diagonal), so with
// E = [I; 0], F = [0; I] and the compact-WY form
// H_0^H ... H_{r-1}^H = I - Y T Y^H (Y unit lower trapezoidal, T upper):
//     A := V - E = -Y T Y_1^H           (an LU factorisation of A, no pivoting)
//     Q  = F - Y T Y_2^H = F + A A_1^{-H} V_2^H
// where A_1 = V_1 - I (top r x r block) and V_2 the bottom n - r rows.  The
// LU pivots of A_1 are exactly the reference's u0 = x0 - beta, and
// Q~_j = Q P_j = [0; P_j] + A X_j with A_1^H X_j = V_2^H P_j.
//
// So the sequential part shrinks from r reflector steps over n rows plus r
// reflector applications to an r x r LU (registers, one barrier per step) and
// two r-step triangular solves; everything else is small parallel products.
// When a pivot falls below kPivotFloor (the reference's skipped "identity"
// reflector, or cancellation in x0 - beta), the kernel raises *gate and the
// stage driver's gated Householder kernels (dense.cu) recompute Q~ the
// reference way.  Verified against the reference's householder_nullspace to
// ~1e-15 (tests/test_gpu_ops.py::test_nullspace_jl_*).
#include "common.cuh"

namespace {

constexpr int kNjThreads = 512;
constexpr int kNjCols = 4;            // JL columns per CTA (the r x r LU is redundant per CTA)
constexpr double kPivotFloor = 1e-3;  // |u0| below this -> Householder fallback

template <int CT, int QN>
__global__ void __launch_bounds__(kNjThreads)
nsjl_kernel(int n, int r, const double2* __restrict__ V, int cols, const double2* __restrict__ Pin,
            double2* __restrict__ B, float2* __restrict__ out32, int p, int* __restrict__ gate) {
  hicu_pdl_entry();
  constexpr int RG = kNjThreads / CT;  // row groups of the register-resident LU
  extern __shared__ double2 smj[];
  double2* LU = smj;                    // r x r: U (upper, incl. diagonal), L (strictly lower)
  double2* colb = LU + (size_t)r * r;   // 2 x r published column k (double-buffered)
  double2* rowb = colb + 2 * r;         // 2 x r published row k
  double2* idg = rowb + 2 * r;          // r: 1 / U[k][k]
  double2* Zp = idg + r;                // RG x r x kNjCols partials of V_2^H P
  double2* X = Zp + (size_t)RG * r * kNjCols;  // r x kNjCols
  const int tid = threadIdx.x, j = tid % CT, rg = tid / CT;
  const int c0 = blockIdx.x * kNjCols;
  const int nc = min(kNjCols, cols - c0);

  // LU operand A_1 = V_1 - I: element (rg + RG q, j) in s[q]
  double2 s[QN];
#pragma unroll
  for (int q = 0; q < QN; ++q) {
    const int i = rg + RG * q;
    s[q] = (i < r && j < r) ? V[(size_t)i * r + j] : cd(0.0, 0.0);
    if (i == j) s[q].x -= 1.0;
  }
  // Z partials: Z[a][c] = sum_{k >= r} conj(V[k][a]) P[k][c], k split over the row groups
  if (j < r) {
    double2 acc[kNjCols];
#pragma unroll
    for (int c = 0; c < kNjCols; ++c) acc[c] = cd(0.0, 0.0);
    for (int k = r + rg; k < n; k += RG) {
      const double2 va = V[(size_t)k * r + j];
#pragma unroll
      for (int c = 0; c < kNjCols; ++c)
        if (c < nc) zfmac(acc[c], va, __ldg(Pin + (size_t)k * cols + c0 + c));
    }
#pragma unroll
    for (int c = 0; c < kNjCols; ++c) Zp[((size_t)rg * r + j) * kNjCols + c] = acc[c];
  }
  // publish column 0 (rows > 0) and row 0
  if (j == 0) {
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      const int i = rg + RG * q;
      if (i > 0 && i < r) colb[i] = s[q];
    }
  }
  if (rg == 0 && j < r) rowb[j] = s[0];
  __syncthreads();

  double minpiv = 1e300;
  for (int k = 0; k < r; ++k) {
    const int b = k & 1;
    const double2 piv = rowb[b * r + k];
    const double d = abs2d(piv);
    minpiv = fmin(minpiv, d);
    const double2 invp = cd(piv.x / d, -piv.y / d);
    if (j > k && j < r) {
      const double2 f = cmul(rowb[b * r + j], invp);  // U[k][j] / U[k][k]
#pragma unroll
      for (int q = 0; q < QN; ++q) {
        const int i = rg + RG * q;
        if (i > k && i < r) s[q] = s[q] - cmul(colb[b * r + i], f);
      }
    } else if (j == k) {
#pragma unroll
      for (int q = 0; q < QN; ++q) {
        const int i = rg + RG * q;
        if (i > k && i < r) LU[(size_t)i * r + k] = cmul(s[q], invp);  // L[i][k]
      }
      if (rg == 0) idg[k] = invp;
    }
    if (k + 1 < r) {
      const int nb = (b ^ 1) * r;
      if (j == k + 1) {
#pragma unroll
        for (int q = 0; q < QN; ++q) {
          const int i = rg + RG * q;
          if (i > k + 1 && i < r) colb[nb + i] = s[q];
        }
      }
      if (rg == (k + 1) % RG && j > k && j < r) {
#pragma unroll
        for (int q = 0; q < QN; ++q)
          if (rg + RG * q == k + 1) rowb[nb + j] = s[q];
      }
    }
    __syncthreads();
  }
  // U (upper part, final since step i-1)
#pragma unroll
  for (int q = 0; q < QN; ++q) {
    const int i = rg + RG * q;
    if (i < r && j < r && i <= j) LU[(size_t)i * r + j] = s[q];
  }
  if (blockIdx.x == 0 && tid == 0) *gate = (minpiv >= kPivotFloor * kPivotFloor) ? 0 : 1;
  __syncthreads();

  // A_1^H X = Z  <=>  U^H (L^H X) = Z: one warp per JL column, rows i = lane + 32 m
  const int warp = tid >> 5, lane = tid & 31;
  if (warp < nc) {
    constexpr int MQ = 4;  // r <= 128
    double2 z[MQ];
#pragma unroll
    for (int m = 0; m < MQ; ++m) {
      const int i = lane + 32 * m;
      double2 acc = cd(0.0, 0.0);
      if (i < r)
        for (int g = 0; g < RG; ++g) acc = acc + Zp[((size_t)g * r + i) * kNjCols + warp];
      z[m] = acc;
    }
    // forward: U^H y = z  (y_k = (z_k - sum_{m<k} conj(U[m][k]) y_m) / conj(U[k][k]))
    for (int k = 0; k < r; ++k) {
      const int sl = k >> 5;
      double2 zv = z[0];
#pragma unroll
      for (int m = 1; m < MQ; ++m)
        if (sl == m) zv = z[m];
      zv.x = __shfl_sync(0xffffffffu, zv.x, k & 31);
      zv.y = __shfl_sync(0xffffffffu, zv.y, k & 31);
      const double2 y = cmulc(idg[k], zv);
#pragma unroll
      for (int m = 0; m < MQ; ++m) {
        const int i = lane + 32 * m;
        if (i == k) z[m] = y;
        else if (i > k && i < r) z[m] = z[m] - cmulc(LU[(size_t)k * r + i], y);
      }
    }
    // backward: L^H x = y  (x_k = y_k - sum_{m>k} conj(L[m][k]) x_m)
    for (int k = r - 1; k >= 0; --k) {
      const int sl = k >> 5;
      double2 xv = z[0];
#pragma unroll
      for (int m = 1; m < MQ; ++m)
        if (sl == m) xv = z[m];
      xv.x = __shfl_sync(0xffffffffu, xv.x, k & 31);
      xv.y = __shfl_sync(0xffffffffu, xv.y, k & 31);
#pragma unroll
      for (int m = 0; m < MQ; ++m) {
        const int i = lane + 32 * m;
        if (i < k) z[m] = z[m] - cmulc(LU[(size_t)k * r + i], xv);
      }
    }
#pragma unroll
    for (int m = 0; m < MQ; ++m) {
      const int i = lane + 32 * m;
      if (i < r) X[(size_t)i * kNjCols + warp] = z[m];
    }
  }
  __syncthreads();

  // Q~[k][c] = [0; P][k][c] + sum_a (V[k][a] - delta_ka) X[a][c]
  for (int k = tid; k < n; k += kNjThreads) {
    double2 acc[kNjCols], acc2[kNjCols];
#pragma unroll
    for (int c = 0; c < kNjCols; ++c) {
      acc[c] = (k >= r && c < nc) ? __ldg(Pin + (size_t)k * cols + c0 + c) : cd(0.0, 0.0);
      acc2[c] = cd(0.0, 0.0);
      if (k < r) acc[c] = cd(-X[(size_t)k * kNjCols + c].x, -X[(size_t)k * kNjCols + c].y);
    }
    const double2* vr = V + (size_t)k * r;
    int a = 0;
    for (; a + 1 < r; a += 2) {
      const double2 v0 = __ldg(vr + a), v1 = __ldg(vr + a + 1);
#pragma unroll
      for (int c = 0; c < kNjCols; ++c) {
        zfma(acc[c], v0, X[(size_t)a * kNjCols + c]);
        zfma(acc2[c], v1, X[(size_t)(a + 1) * kNjCols + c]);
      }
    }
    if (a < r) {
      const double2 v0 = __ldg(vr + a);
#pragma unroll
      for (int c = 0; c < kNjCols; ++c) zfma(acc[c], v0, X[(size_t)a * kNjCols + c]);
    }
#pragma unroll
    for (int c = 0; c < kNjCols; ++c) {
      if (c >= nc) continue;
      const double2 v = acc[c] + acc2[c];
      const int jj = c0 + c;
      B[(size_t)k * cols + jj] = v;
      if (out32) {
        const int step = jj / p, t = jj % p;
        out32[((size_t)step * n + k) * p + t] = cf((float)v.x, (float)v.y);
      }
    }
  }
}

size_t nsjl_smem(int r, int ct) {
  const int rg = kNjThreads / ct;
  return ((size_t)r * r + 5 * (size_t)r + (size_t)rg * r * kNjCols + (size_t)r * kNjCols) * sizeof(double2);
}

int nsjl_ct(int r) { return r <= 64 ? 64 : (r <= 100 ? 128 : 0); }

}  // namespace

extern "C" int hicu_nullspace_jl_supported(int n, int r) {
  const int ct = nsjl_ct(r);
  return (r >= 1 && r < n && ct && nsjl_smem(r, ct) <= (size_t)220 * 1024) ? 1 : 0;
}

extern "C" int hicu_nullspace_jl(int n, int r, const void* V, int cols, const void* Bin, void* B, void* out32, int p,
                                 int* gate_dev, void* stream) {
  if (n < 1 || cols < 1 || !V || !Bin || !B || !gate_dev)
    return hicu_set_error(HICU_ERR_PARAMETER, "nullspace_jl: bad arguments");
  if (out32 && (p < 1 || cols % p != 0)) return hicu_set_error(HICU_ERR_PARAMETER, "nullspace_jl: bad p");
  if (!hicu_nullspace_jl_supported(n, r)) return hicu_set_error(HICU_ERR_SIZE, "nullspace_jl: rank not supported");
  const int ct = nsjl_ct(r);
  const size_t smem = nsjl_smem(r, ct);
  const int grid = (cols + kNjCols - 1) / kNjCols;
  cudaStream_t st = (cudaStream_t)stream;
  auto go = [&](auto kern) {
    hicu_allow_max_smem((const void*)kern);
    hicu_launch(kern, grid, kNjThreads, smem, st, n, r, (const double2*)V, cols, (const double2*)Bin, (double2*)B,
                (float2*)out32, p ? p : 1, gate_dev);
  };
  if (ct == 64) go(nsjl_kernel<64, 8>);
  else go(nsjl_kernel<128, 25>);
  return hicu_check_launch("nsjl_kernel");
}
