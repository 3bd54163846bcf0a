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
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace {

constexpr int kNjCols = 4;            // JL columns per CTA (the r x r LU is redundant per CTA)
constexpr double kPivotFloor = 1e-3;  // |u0| below this -> Householder fallback
__device__ unsigned long long g_nsjl_trace[8];  // phase clocks of CTA 0 (HICU_NSJL_TRACE)
#define NSJL_STAMP(i) \
  if (blockIdx.x == 0 && threadIdx.x == 0) g_nsjl_trace[i] = clock64();

// 1/d for 1e-30 < d < 1e30 to ~1 ulp: fp32 MUFU seed (no slow path) and two
// fp64 Newton steps.  Pivots outside that range raise the gate anyway.
__device__ __forceinline__ double nsjl_rcp(double d) {
  const float df = (float)fmin(fmax(d, 1e-30), 1e30);
  float x0;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(x0) : "f"(df));
  double x = (double)x0;
  x = fma(x, fma(-d, x, 1.0), x);
  x = fma(x, fma(-d, x, 1.0), x);
  return x;
}

__device__ __forceinline__ void nsjl_cp16(void* dst_smem, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst_smem)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void nsjl_cp_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ int nsjl_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];"
               : "=r"(v)
               : "r"((unsigned)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}
__device__ __forceinline__ void nsjl_st_release(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v)
               : "memory");
}

// 1 / z, published by the single thread that owns the pivot
__device__ __forceinline__ double2 nsjl_inv(double2 z) {
  const double t = nsjl_rcp(abs2d(z));
  return cd(z.x * t, -z.y * t);
}

// Z partials: Zp[g][a][c] = sum_{k >= r, k = r + g (mod RG)} conj(V[k][a]) P[k][c0 + c],
// thread (a = j, g = rg); P_2 already staged in shared memory (Ps, (n - r) x kNjCols),
// V loads issued in batches of 16 rows.
template <int RG>
__device__ __forceinline__ void nsjl_zpart(int n, int r, const double2* __restrict__ V, const double2* __restrict__ Ps,
                                           int j, int rg, double2* __restrict__ Zp) {
  if (j >= r) return;
  double2 acc[kNjCols];
#pragma unroll
  for (int c = 0; c < kNjCols; ++c) acc[c] = cd(0.0, 0.0);
  constexpr int kB = 16;
  for (int k0 = r + rg; k0 < n; k0 += kB * RG) {
    double2 va[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int k = k0 + u * RG;
      va[u] = k < n ? V[(size_t)k * r + j] : cd(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int k = k0 + u * RG;
      if (k < n) {
#pragma unroll
        for (int c = 0; c < kNjCols; ++c) zfmac(acc[c], va[u], Ps[(size_t)(k - r) * kNjCols + c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kNjCols; ++c) Zp[((size_t)rg * r + j) * kNjCols + c] = acc[c];
}

// Solves and Q~ (shared by the single-CTA-LU kernel and the global-LU path):
// LU / idg may live in shared or global memory (generic loads); V chunks are
// staged in `stage` (stage_elems double2, padded rows of r + 1).
template <int CT, int NT, int RG>
__device__ __forceinline__ void nsjl_finish(int n, int r, const double2* __restrict__ V, int cols, int c0, int nc,
                                            double2* __restrict__ B, float2* __restrict__ out32, int p,
                                            const double2* LU, const double2* idg, const double2* Zp, double2* X,
                                            const double2* Ps, double2* stage, int stage_elems) {
  const int tid = threadIdx.x;
  // A_1^H X = Z  <=>  U^H (L^H X) = Z: one warp per JL column, rows i = lane + 32 m;
  // the next row of U / L is loaded one step ahead
  const int warp = tid >> 5, lane = tid & 31;
  if (warp < nc) {
    constexpr int MQ = (CT + 31) / 32;  // r <= CT
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
    double2 un[MQ];
#pragma unroll
    for (int m = 0; m < MQ; ++m) {
      const int i = lane + 32 * m;
      un[m] = i < r ? LU[i] : cd(0.0, 0.0);
    }
    for (int k = 0; k < r; ++k) {
      double2 uc[MQ];
#pragma unroll
      for (int m = 0; m < MQ; ++m) {
        uc[m] = un[m];
        const int i = lane + 32 * m;
        un[m] = (k + 1 < r && i < r) ? LU[(size_t)(k + 1) * r + i] : cd(0.0, 0.0);
      }
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
        else if (i > k) z[m] = z[m] - cmulc(uc[m], y);
      }
    }
    // backward: L^H x = y  (x_k = y_k - sum_{m>k} conj(L[m][k]) x_m)
#pragma unroll
    for (int m = 0; m < MQ; ++m) {
      const int i = lane + 32 * m;
      un[m] = i < r - 1 ? LU[(size_t)(r - 1) * r + i] : cd(0.0, 0.0);
    }
    for (int k = r - 1; k >= 0; --k) {
      double2 lc[MQ];
#pragma unroll
      for (int m = 0; m < MQ; ++m) {
        lc[m] = un[m];
        const int i = lane + 32 * m;
        un[m] = (k >= 1 && i < k - 1) ? LU[(size_t)(k - 1) * r + i] : cd(0.0, 0.0);
      }
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
        if (i < k) z[m] = z[m] - cmulc(lc[m], xv);
      }
    }
#pragma unroll
    for (int m = 0; m < MQ; ++m) {
      const int i = lane + 32 * m;
      if (i < r) X[(size_t)i * kNjCols + warp] = z[m];
    }
  }
  __syncthreads();
  NSJL_STAMP(3)

  // Q~[k][c] = [0; P][k][c] + sum_a (V[k][a] - delta_ka) X[a][c]; V staged through
  // shared memory (LU and pivot areas) in chunks of CH rows with padded stride r + 1
  const int ld = r + 1;
  const int CH = stage_elems / ld;  // rows per staged V chunk (>= 1)
  for (int k0 = 0; k0 < n; k0 += CH) {
    const int rows = min(CH, n - k0);
    for (int e = tid; e < rows * r; e += NT) {
      const int kk = e / r, a = e - kk * r;
      nsjl_cp16(stage + (size_t)kk * ld + a, V + (size_t)(k0 + kk) * r + a);
    }
    nsjl_cp_wait_all();
    __syncthreads();
    // thread (row kk = tid % TR (+ TR, ...), column c = tid / TR): two rows per
    // pass as independent accumulation chains
    constexpr int TR = NT / kNjCols;
    const int c = tid / TR;
    for (int kk = tid % TR; kk < rows; kk += 2 * TR) {
      const bool two = kk + TR < rows;
      const int k = k0 + kk, k2 = k + TR;
      double2 acc = cd(0.0, 0.0), acc2 = cd(0.0, 0.0), bcc = cd(0.0, 0.0), bcc2 = cd(0.0, 0.0);
      if (c < nc) {
        acc = k >= r ? Ps[(size_t)(k - r) * kNjCols + c] : cd(-X[(size_t)k * kNjCols + c].x, -X[(size_t)k * kNjCols + c].y);
        if (two)
          bcc = k2 >= r ? Ps[(size_t)(k2 - r) * kNjCols + c]
                        : cd(-X[(size_t)k2 * kNjCols + c].x, -X[(size_t)k2 * kNjCols + c].y);
      }
      const double2* vr = stage + (size_t)kk * ld;
      const double2* vr2 = vr + (size_t)TR * ld;
      int a = 0;
      for (; a + 1 < r; a += 2) {
        const double2 x0 = X[(size_t)a * kNjCols + c], x1 = X[(size_t)(a + 1) * kNjCols + c];
        zfma(acc, vr[a], x0);
        zfma(acc2, vr[a + 1], x1);
        if (two) {
          zfma(bcc, vr2[a], x0);
          zfma(bcc2, vr2[a + 1], x1);
        }
      }
      if (a < r) {
        const double2 x0 = X[(size_t)a * kNjCols + c];
        zfma(acc, vr[a], x0);
        if (two) zfma(bcc, vr2[a], x0);
      }
      if (c < nc) {
        const int jj = c0 + c, step = jj / p, t = jj % p;
        const double2 v = acc + acc2;
        B[(size_t)k * cols + jj] = v;
        if (out32) out32[((size_t)step * n + k) * p + t] = cf((float)v.x, (float)v.y);
        if (two) {
          const double2 v2 = bcc + bcc2;
          B[(size_t)k2 * cols + jj] = v2;
          if (out32) out32[((size_t)step * n + k2) * p + t] = cf((float)v2.x, (float)v2.y);
        }
      }
    }
    __syncthreads();
  }
  NSJL_STAMP(4)
}

// CT threads per LU row group (>= r), NT threads, QN = ceil(r / (NT / CT)) rows per thread.
template <int CT, int QN, int NT, bool WARP_LU>
__global__ void __launch_bounds__(NT)
nsjl_kernel(int n, int r, const double2* __restrict__ V, int cols, const double2* __restrict__ Pin,
            double2* __restrict__ B, float2* __restrict__ out32, int p, int* __restrict__ gate) {
  hicu_pdl_entry();
  NSJL_STAMP(0)
  constexpr int RG = NT / CT;  // row groups of the register-resident LU (warp-uniform: CT % 32 == 0)
  extern __shared__ double2 smj[];
  double2* LU = smj;                           // RG*QN x r: U (upper, incl. diagonal), L (strictly lower)
  // generic LU: 2 x RG*QN published column k and 2 x CT row k (double-buffered);
  // warp LU: every step's column k kept (r x 64, no reuse, so no write-after-read hazard)
  constexpr int kColbPerR = WARP_LU ? 64 : 0;
  double2* colb = LU + (size_t)RG * QN * r;
  double2* rowb = colb + (WARP_LU ? (size_t)kColbPerR * r : 2 * RG * QN);
  double2* idg = rowb + (WARP_LU ? 0 : 2 * CT);  // r: 1 / U[k][k]
  double2* Zp = idg + r;                // RG x r x kNjCols partials of V_2^H P
  double2* X = Zp + (size_t)RG * r * kNjCols;  // r x kNjCols
  double* pd = (double*)(X + (size_t)r * kNjCols);  // r: |U[k][k]|^2
  int* ready = (int*)(pd + r);                       // r: column k published (warp LU)
  double2* Ps = (double2*)(((uintptr_t)(ready + r) + 15) & ~(uintptr_t)15);  // (n - r) x kNjCols: P_2
  const int tid = threadIdx.x, j = tid % CT, rg = tid / CT;
  const int c0 = blockIdx.x * kNjCols;
  const int nc = min(kNjCols, cols - c0);
  for (int e = tid; e < (n - r) * kNjCols; e += NT) {
    const int kk = e / kNjCols, c = e - kk * kNjCols;
    if (c < nc) nsjl_cp16(Ps + e, Pin + (size_t)(r + kk) * cols + c0 + c);
    else Ps[e] = cd(0.0, 0.0);
  }

  if constexpr (WARP_LU) {
    // Warp-column LU (r <= 64, 8 warps): warp w holds columns 8w..8w+7 of A_1
    // for rows lane and lane + 32 in registers.  Row k of the warp's columns
    // is a shuffle from lane k % 32; only column k crosses warps (shared
    // memory, one barrier per step), and warps whose columns are all <= k
    // skip the update entirely.
    static_assert(NT == 256, "warp LU is laid out for 8 warps x 8 columns");
    const int w = tid >> 5, ln = tid & 31;
    double2* colw = colb;  // r x 64
    double2 a0[8], a1[8];  // column w + 8c, rows ln and ln + 32
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int jj = w + 8 * c;
      a0[c] = (ln < r && jj < r) ? V[(size_t)ln * r + jj] : cd(0.0, 0.0);
      a1[c] = (ln + 32 < r && jj < r) ? V[(size_t)(ln + 32) * r + jj] : cd(0.0, 0.0);
      if (ln == jj) a0[c].x -= 1.0;
      if (ln + 32 == jj) a1[c].x -= 1.0;
    }
    nsjl_cp_wait_all();
    __syncthreads();
    nsjl_zpart<RG>(n, r, V, Ps, j, rg, Zp);
    for (int k = tid; k < r; k += NT) ready[k] = k == 0;
    if (w == 0) {
      colw[ln] = a0[0];
      colw[ln + 32] = a1[0];
      if (ln == 0) {
        idg[0] = nsjl_inv(a0[0]);
        pd[0] = abs2d(a0[0]);
      }
    }
    __syncthreads();
    NSJL_STAMP(1)
    for (int k = 0; k < r; ++k) {
      // wait for column k (published by warp k % 8 with release semantics)
      if (w != (k & 7))
        while (nsjl_ld_acquire(ready + k) == 0) {
        }
      const double2 invp = idg[k];
      const double2* ck = colw + (size_t)k * 64;
      const double2 l0 = ln > k ? cmul(ck[ln], invp) : cd(0.0, 0.0);
      const double2 l1 = ln + 32 > k ? cmul(ck[ln + 32], invp) : cd(0.0, 0.0);
      if (w == (k & 7)) {
        if (ln > k) LU[(size_t)ln * r + k] = l0;
        if (ln + 32 > k && ln + 32 < r) LU[(size_t)(ln + 32) * r + k] = l1;
      }
      const bool hi = k >= 32;
      const int kl = k & 31;
      if (k + 1 < r && w == ((k + 1) & 7)) {
        // this warp owns column k + 1: update and publish it (with 1 / pivot)
        // before its other columns; the other warps' trailing updates for
        // step k overlap this chain
        const int cc = (k + 1) >> 3;
        double2 v0 = a0[0], v1 = a1[0];
#pragma unroll
        for (int c = 1; c < 8; ++c)
          if (c == cc) {
            v0 = a0[c];
            v1 = a1[c];
          }
        double2 u = hi ? v1 : v0;
        u.x = __shfl_sync(0xffffffffu, u.x, kl);
        u.y = __shfl_sync(0xffffffffu, u.y, kl);
        v0 = v0 - cmul(l0, u);
        v1 = v1 - cmul(l1, u);
        double2* cn = colw + (size_t)(k + 1) * 64;
        cn[ln] = v0;
        cn[ln + 32] = v1;
        if (ln == ((k + 1) & 31)) {
          const double2 pv = k + 1 >= 32 ? v1 : v0;
          idg[k + 1] = nsjl_inv(pv);
          pd[k + 1] = abs2d(pv);
        }
        __syncwarp();
        if (ln == 0) nsjl_st_release(ready + k + 1, 1);
      }
      if (w + 56 > k) {  // warp-uniform; columns <= k get u = 0 (no branch per column:
                         // measured faster than skipping them, 61K vs 69K cycles per LU)
        double2 u[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          u[c] = hi ? a1[c] : a0[c];
          u[c].x = __shfl_sync(0xffffffffu, u[c].x, kl);
          u[c].y = __shfl_sync(0xffffffffu, u[c].y, kl);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double2 uc = w + 8 * c > k ? u[c] : cd(0.0, 0.0);
          a0[c] = a0[c] - cmul(l0, uc);
          a1[c] = a1[c] - cmul(l1, uc);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int jj = w + 8 * c;
      if (jj < r && ln <= jj) LU[(size_t)ln * r + jj] = a0[c];
      if (jj < r && ln + 32 <= jj) LU[(size_t)(ln + 32) * r + jj] = a1[c];
    }
  } else {
    // Generic LU (r <= 100): element (rg + RG q, j) of A_1 = V_1 - I in s[q]. = V_1 - I: element (rg + RG q, j) in s[q]
    double2 s[QN];
#pragma unroll
    for (int q = 0; q < QN; ++q) {
      const int i = rg + RG * q;
      s[q] = (i < r && j < r) ? V[(size_t)i * r + j] : cd(0.0, 0.0);
      if (i == j) s[q].x -= 1.0;
    }
    nsjl_cp_wait_all();
    __syncthreads();
    nsjl_zpart<RG>(n, r, V, Ps, j, rg, Zp);
    // Published column k (rows > k, zero elsewhere, RG*QN entries) and row k
    // (columns > k, zero elsewhere) make every thread's update unconditional:
    // s[q] -= colb[i] * (rowb[j] / U[k][k]) is a no-op outside the trailing block.
    // publish column 0, row 0 and 1 / pivot 0
    if (j == 0) {
#pragma unroll
      for (int q = 0; q < QN; ++q) {
        const int i = rg + RG * q;
        colb[i] = i > 0 ? s[q] : cd(0.0, 0.0);
      }
      if (rg == 0) {
        idg[0] = nsjl_inv(s[0]);
        pd[0] = abs2d(s[0]);
      }
    }
    if (rg == 0 && j < CT) rowb[j] = j > 0 ? s[0] : cd(0.0, 0.0);
    __syncthreads();
    NSJL_STAMP(1)

    // right-looking LU without pivoting, one barrier per step; the pivot's
    // owner publishes its inverse with the next row/column
    for (int k = 0; k < r; ++k) {
      const int b = k & 1;
      const double2 invp = idg[k];
      const double2* cb = colb + b * (RG * QN);
      const double2 f = cmul(rowb[b * CT + j], invp);  // U[k][j] / U[k][k], 0 unless j > k
      if (j == k) {
#pragma unroll
        for (int q = 0; q < QN; ++q) {
          const int i = rg + RG * q;
          if (i > k) LU[(size_t)i * r + k] = cmul(s[q], invp);  // L[i][k] (rows >= r land in spare rows)
        }
      }
#pragma unroll
      for (int q = 0; q < QN; ++q) s[q] = s[q] - cmul(cb[rg + RG * q], f);
      if (k + 1 < r) {
        double2* ncb = colb + (b ^ 1) * (RG * QN);
        if (j == k + 1) {
          double2 pv = s[0];
#pragma unroll
          for (int q = 0; q < QN; ++q) {
            const int i = rg + RG * q;
            ncb[i] = i > k + 1 ? s[q] : cd(0.0, 0.0);
            if (i == k + 1) pv = s[q];
          }
          if (rg == (k + 1) % RG) {
            idg[k + 1] = nsjl_inv(pv);
            pd[k + 1] = abs2d(pv);
          }
        }
        if (rg == (k + 1) % RG) {  // warp-uniform
          double2 v = s[0];
#pragma unroll
          for (int q = 1; q < QN; ++q)
            if (rg + RG * q == k + 1) v = s[q];
          rowb[(b ^ 1) * CT + j] = j > k + 1 ? v : cd(0.0, 0.0);
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
  }
  if (blockIdx.x == 0 && tid < 32) {
    double m = 1e300;
    for (int k = tid; k < r; k += 32) m = fmin(m, pd[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (tid == 0) *gate = (m >= kPivotFloor * kPivotFloor) ? 0 : 1;  // NaN -> fallback
  }
  __syncthreads();
  NSJL_STAMP(2)

  nsjl_finish<CT, NT, RG>(n, r, V, cols, c0, nc, B, out32, p, LU, idg, Zp, X, Ps, LU, (int)(idg - LU));
}

// ---------------------------------------------------------------------------
// Ranks whose r x r LU exceeds one SM (C4/C5: r = 150 / 120, n = 1000): the LU
// runs in one CTA over a global-memory (L2-resident) copy of A_1, right-looking
// with one block barrier per step; the Z / solve / Q~ phases then run in the
// usual per-JL-column CTAs reading U, L and 1/pivot from global memory.
// ---------------------------------------------------------------------------
constexpr int kLuThreads = 1024;

__global__ void __launch_bounds__(kLuThreads)
nsjl_lu_global_kernel(int r, const double2* __restrict__ V, double2* __restrict__ LUg, double2* __restrict__ Lg,
                      double2* __restrict__ idg, double* __restrict__ pd, int* __restrict__ gate) {
  hicu_pdl_entry();
  const int tid = threadIdx.x;
  for (int e = tid; e < r * r; e += kLuThreads) {
    const int i = e / r, j = e - i * r;
    double2 v = V[(size_t)i * r + j];
    if (i == j) v.x -= 1.0;
    LUg[e] = v;
  }
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    const double2 piv = __ldcg(LUg + (size_t)k * r + k);
    const double2 inv = nsjl_inv(piv);
    if (tid == 0) {
      idg[k] = inv;
      pd[k] = abs2d(piv);
    }
    // rows k+1.. x columns k.. : column k gives L[i][k] (kept aside: column k
    // is still being read this step), the rest take the rank-1 update
    const int m = r - k - 1;
    for (int e = tid; e < m * (m + 1); e += kLuThreads) {
      const int ii = e / (m + 1), jj = e - ii * (m + 1);
      const int i = k + 1 + ii;
      const double2 l = cmul(__ldcg(LUg + (size_t)i * r + k), inv);
      if (jj == 0) {
        Lg[(size_t)i * r + k] = l;
      } else {
        const int j = k + jj;
        double2* pij = LUg + (size_t)i * r + j;
        *pij = __ldcg(pij) - cmul(l, __ldcg(LUg + (size_t)k * r + j));
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < r * r; e += kLuThreads) {
    const int i = e / r, j = e - i * r;
    if (i > j) LUg[e] = Lg[e];
  }
  if (tid < 32) {
    double mn = 1e300;
    for (int k = tid; k < r; k += 32) mn = fmin(mn, pd[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (tid == 0) *gate = (mn >= kPivotFloor * kPivotFloor) ? 0 : 1;
  }
}

// The same LU on one 8-CTA thread-block cluster (the default for these
// ranks): row i of A_1 lives in the shared memory of CTA i % 8 (cyclic, so the
// shrinking trailing block stays balanced).  Step k: the owner of row k
// writes U[k][k..r) into every CTA's shared memory with DSMEM stores
// (double-buffered by step parity), one cluster barrier, then every CTA
// forms l = A[i][k] / U[k][k] for its rows i > k (stored to global at once:
// column k is never read again) and folds row k into them, a warp per row.
// Same arithmetic per element as nsjl_lu_global_kernel (l = a * (1 / pivot),
// a -= l * u), same outputs (LUg: U on and above the diagonal, L below;
// idg = 1 / pivot; pd = |pivot|^2; *gate).  The single CTA streaming the
// trailing block through L2 took 0.48 / 0.85 ms at r = 120 / 150.
constexpr int kLcCS = 8;
constexpr int kLcThreads = 512;
constexpr int kLcMaxR = 256;

__global__ void __cluster_dims__(kLcCS, 1, 1) __launch_bounds__(kLcThreads, 1)
nsjl_lu_cluster_kernel(int r, const double2* __restrict__ V, double2* __restrict__ LUg, double2* __restrict__ idg,
                       double* __restrict__ pd, int* __restrict__ gate) {
  hicu_pdl_entry();
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  extern __shared__ double2 lcA[];  // [nr][r]: rows cr, cr + 8, ...
  __shared__ double2 srow[2][kLcMaxR];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = kLcThreads / 32;
  const int nr = (r - cr + kLcCS - 1) / kLcCS;
  for (int q = tid; q < nr * r; q += kLcThreads) {
    const int rl = q / r, j = q - rl * r, i = cr + kLcCS * rl;
    double2 v = V[(size_t)i * r + j];
    if (i == j) v.x -= 1.0;
    lcA[q] = v;
  }
  bool bad = false;
  cluster.sync();
  for (int k = 0; k < r; ++k) {
    const int buf = k & 1;
    if (cr == k % kLcCS) {
      const double2* row = lcA + (size_t)(k / kLcCS) * r;
      const int m = r - k;
      for (int q = tid; q < kLcCS * m; q += kLcThreads) {
        const int c = q / m, j = k + (q - c * m);
        *cluster.map_shared_rank(&srow[buf][j], c) = row[j];
      }
    }
    cluster.sync();
    const double2 piv = srow[buf][k];
    const double p2 = abs2d(piv);
    const double2 inv = nsjl_inv(piv);
    bad |= !(p2 >= kPivotFloor * kPivotFloor);  // NaN -> fallback
    if (cr == k % kLcCS && tid == 0) {
      idg[k] = inv;
      pd[k] = p2;
    }
    // fold row k into this CTA's rows i > k
    const int first = k >= cr ? (k - cr) / kLcCS + 1 : 0;
    for (int rl = first + warp; rl < nr; rl += nw) {
      double2* Ai = lcA + (size_t)rl * r;
      const double2 l = cmul(Ai[k], inv);
      if (lane == 0) LUg[(size_t)(cr + kLcCS * rl) * r + k] = l;
      for (int j = k + 1 + lane; j < r; j += 32) Ai[j] = Ai[j] - cmul(l, srow[buf][j]);
    }
    __syncthreads();  // the next owner reads its updated row
  }
  // U: rows are final from their own step on
  for (int q = tid; q < nr * r; q += kLcThreads) {
    const int rl = q / r, j = q - rl * r, i = cr + kLcCS * rl;
    if (j >= i) LUg[(size_t)i * r + j] = lcA[q];
  }
  if (cr == 0 && tid == 0) *gate = bad ? 1 : 0;
  cluster.sync();
}

template <int CT, int NT>
__global__ void __launch_bounds__(NT)
nsjl_big_kernel(int n, int r, const double2* __restrict__ V, int cols, const double2* __restrict__ Pin,
                double2* __restrict__ B, float2* __restrict__ out32, int p, const double2* __restrict__ LUg,
                const double2* __restrict__ idg, int stage_elems) {
  hicu_pdl_entry();
  constexpr int RG = NT / CT;
  extern __shared__ double2 smj[];
  double2* Zp = smj;                              // RG x r x kNjCols
  double2* X = Zp + (size_t)RG * r * kNjCols;     // r x kNjCols
  double2* Ps = X + (size_t)r * kNjCols;          // (n - r) x kNjCols
  double2* stage = Ps + (size_t)(n - r) * kNjCols;
  const int tid = threadIdx.x, j = tid % CT, rg = tid / CT;
  const int c0 = blockIdx.x * kNjCols;
  const int nc = min(kNjCols, cols - c0);
  for (int e = tid; e < (n - r) * kNjCols; e += NT) {
    const int kk = e / kNjCols, c = e - kk * kNjCols;
    if (c < nc) nsjl_cp16(Ps + e, Pin + (size_t)(r + kk) * cols + c0 + c);
    else Ps[e] = cd(0.0, 0.0);
  }
  nsjl_cp_wait_all();
  __syncthreads();
  nsjl_zpart<RG>(n, r, V, Ps, j, rg, Zp);
  __syncthreads();
  nsjl_finish<CT, NT, RG>(n, r, V, cols, c0, nc, B, out32, p, LUg, idg, Zp, X, Ps, stage, stage_elems);
}

size_t nsjl_big_fixed(int n, int r, int ct, int nt) {
  return ((size_t)(nt / ct) * r * kNjCols + (size_t)r * kNjCols + (size_t)(n - r) * kNjCols) * sizeof(double2);
}

int nsjl_big_ct(int r) { return r <= 128 ? 128 : (r <= 160 ? 160 : 0); }
int nsjl_big_nt(int ct) { return ct == 128 ? 512 : 640; }
constexpr size_t kBigSmem = (size_t)200 * 1024;

size_t nsjl_big_ws(int r) { return ((size_t)2 * r * r + r) * sizeof(double2) + (size_t)r * sizeof(double) + 256; }

bool nsjl_big_ok(int n, int r) {
  const int ct = nsjl_big_ct(r);
  if (!ct || r < 1 || r >= n) return false;
  return nsjl_big_fixed(n, r, ct, nsjl_big_nt(ct)) + (size_t)(r + 1) * sizeof(double2) <= kBigSmem;
}

int nsjl_threads(int ct) { return ct == 64 ? 256 : 512; }

size_t nsjl_smem(int n, int r, int ct, bool warp_lu) {
  const int rg = nsjl_threads(ct) / ct, rows = ct == 64 ? rg * 16 : rg * 25;  // RG * QN of the instantiation
  const size_t pub = warp_lu ? (size_t)64 * r : 2 * (size_t)rows + 2 * (size_t)ct;
  return ((size_t)rows * r + pub + (size_t)r + (size_t)rg * r * kNjCols + (size_t)r * kNjCols) * sizeof(double2) +
         (size_t)r * (sizeof(double) + sizeof(int)) + 16 + (size_t)(n - r) * kNjCols * sizeof(double2);
}

int nsjl_ct(int r) { return r <= 64 ? 64 : (r <= 100 ? 128 : 0); }

}  // namespace

static bool nsjl_small_ok(int n, int r) {
  const int ct = nsjl_ct(r);
  return r >= 1 && r < n && ct && nsjl_smem(n, r, ct, ct == 64) <= (size_t)226 * 1024;
}

extern "C" int hicu_nullspace_jl_supported(int n, int r) { return (nsjl_small_ok(n, r) || nsjl_big_ok(n, r)) ? 1 : 0; }

// The cluster LU + per-column CTAs serve every rank above the warp-column LU
// (r > 64) that fits them: the single-CTA kernel's barrier-per-step LU,
// redundant in each of its CTAs, took 0.78 ms at C3's r = 100.
static bool nsjl_use_big(int n, int r) { return nsjl_big_ok(n, r) && (r > 64 || !nsjl_small_ok(n, r)); }

extern "C" size_t hicu_nullspace_jl_workspace(int n, int r) { return nsjl_use_big(n, r) ? nsjl_big_ws(r) : 0; }

extern "C" int hicu_nullspace_jl_ws(int n, int r, const void* V, int cols, const void* Bin, void* B, void* out32,
                                    int p, int* gate_dev, void* ws, size_t ws_bytes, void* stream) {
  if (n < 1 || cols < 1 || !V || !Bin || !B || !gate_dev)
    return hicu_set_error(HICU_ERR_PARAMETER, "nullspace_jl: bad arguments");
  if (out32 && (p < 1 || cols % p != 0)) return hicu_set_error(HICU_ERR_PARAMETER, "nullspace_jl: bad p");
  if (!hicu_nullspace_jl_supported(n, r)) return hicu_set_error(HICU_ERR_SIZE, "nullspace_jl: rank not supported");
  if (nsjl_use_big(n, r) && (!nsjl_small_ok(n, r) || (ws && ws_bytes >= nsjl_big_ws(r)))) {
    const size_t need = nsjl_big_ws(r);
    if (!ws || ws_bytes < need) return hicu_set_error(HICU_ERR_WORKSPACE, "nullspace_jl: workspace too small");
    uint8_t* w = (uint8_t*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    double2* LUg = (double2*)w;
    double2* Lg = LUg + (size_t)r * r;
    double2* idg = Lg + (size_t)r * r;
    double* pd = (double*)(idg + r);
    cudaStream_t st = (cudaStream_t)stream;
    // one 8-CTA cluster holds A_1 in distributed shared memory; the single-CTA
    // global-memory LU stays for ranks beyond it (and HICU_NSJL_LU_GLOBAL=1, tests)
    static const bool force_global = [] {
      const char* e = getenv("HICU_NSJL_LU_GLOBAL");
      return e && e[0] == '1';
    }();
    const size_t lsm = (size_t)((r + kLcCS - 1) / kLcCS) * r * sizeof(double2);
    int s;
    if (!force_global && r <= kLcMaxR && lsm <= (size_t)200 * 1024) {
      hicu_allow_max_smem((const void*)nsjl_lu_cluster_kernel);
      hicu_launch(nsjl_lu_cluster_kernel, kLcCS, kLcThreads, lsm, st, r, (const double2*)V, LUg, idg, pd, gate_dev);
      s = hicu_check_launch("nsjl_lu_cluster_kernel");
    } else {
      hicu_launch(nsjl_lu_global_kernel, 1, kLuThreads, 0, st, r, (const double2*)V, LUg, Lg, idg, pd, gate_dev);
      s = hicu_check_launch("nsjl_lu_global_kernel");
    }
    if (s) return s;
    const int ct = nsjl_big_ct(r), nt = nsjl_big_nt(ct);
    const size_t fixed = nsjl_big_fixed(n, r, ct, nt);
    const int stage_elems = (int)((kBigSmem - fixed) / sizeof(double2));
    const int grid = (cols + kNjCols - 1) / kNjCols;
    auto go = [&](auto kern) {
      hicu_allow_max_smem((const void*)kern);
      hicu_launch(kern, grid, nt, kBigSmem, st, n, r, (const double2*)V, cols, (const double2*)Bin, (double2*)B,
                  (float2*)out32, p ? p : 1, (const double2*)LUg, (const double2*)idg, stage_elems);
    };
    if (ct == 128) go(nsjl_big_kernel<128, 512>);
    else go(nsjl_big_kernel<160, 640>);
    return hicu_check_launch("nsjl_big_kernel");
  }
  return hicu_nullspace_jl(n, r, V, cols, Bin, B, out32, p, gate_dev, stream);
}

extern "C" int hicu_nullspace_jl(int n, int r, const void* V, int cols, const void* Bin, void* B, void* out32, int p,
                                 int* gate_dev, void* stream) {
  if (n < 1 || cols < 1 || !V || !Bin || !B || !gate_dev)
    return hicu_set_error(HICU_ERR_PARAMETER, "nullspace_jl: bad arguments");
  if (out32 && (p < 1 || cols % p != 0)) return hicu_set_error(HICU_ERR_PARAMETER, "nullspace_jl: bad p");
  if (!nsjl_small_ok(n, r))
    return hicu_set_error(HICU_ERR_SIZE, "nullspace_jl: rank needs the workspace entry (hicu_nullspace_jl_ws)");
  const int ct = nsjl_ct(r);
  const size_t smem = nsjl_smem(n, r, ct, ct == 64);
  const int grid = (cols + kNjCols - 1) / kNjCols;
  cudaStream_t st = (cudaStream_t)stream;
  auto go = [&](auto kern) {
    hicu_allow_max_smem((const void*)kern);
    hicu_launch(kern, grid, nsjl_threads(ct), smem, st, n, r, (const double2*)V, cols, (const double2*)Bin, (double2*)B,
                (float2*)out32, p ? p : 1, gate_dev);
  };
  if (ct == 64) go(nsjl_kernel<64, 16, 256, true>);
  else go(nsjl_kernel<128, 25, 512, false>);
  return hicu_check_launch("nsjl_kernel");
}
