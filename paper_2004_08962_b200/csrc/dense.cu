// Small dense complex128 algebra for the nullspace step.
//
// Reference: rsvd_right_vectors (subspace.py:67-155) is replaced by the
// Nystrom form of the same sketch (SURVEY §0 parity fact 1):
//   Y = G Omega, C = Omega^H Y, C_nu = R^H R (Cholesky, shifted only if C is
//   numerically indefinite), W = (Y + nu Omega) R^{-1}, M = W^H W = F L F^H
//   (cyclic parallel Jacobi), V = (W F)[:, top r] L^{-1/2}.
// W W^H = Y C^{-1} Y^H equals the reference's W_ref W_ref^H, so V spans the
// reference's subspace for the same Omega.
// householder_nullspace (subspace.py:158-212) and jl_compress (:215-229) are
// restated as a reflector build plus a column-parallel reflector apply.
//
// All kernels are fp64; single-CTA kernels keep their matrix in shared
// memory when it fits and fall back to a global workspace otherwise.
#include <cooperative_groups.h>

#include "common.cuh"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>

size_t hicu_heev_top_workspace(int l, int r);
int hicu_heev_top(int l, int r, const double2* A, double* lam, double2* F, void* ws, cudaStream_t st);

namespace {

constexpr int kSmemCap = 200 * 1024;

__device__ __forceinline__ double warp_sum_d_(double t) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// ---------------------------------------------------------------------------
// C = op(A) op(B), row-major, op in {N, C}
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 load_op(const double2* A, int lda, bool conjT, int i, int l) {
  // element (i, l) of op(A)
  return conjT ? conjd(A[(size_t)l * lda + i]) : A[(size_t)i * lda + l];
}

__global__ void zgemm_kernel(bool ca, bool cb, int m, int n, int k, const double2* __restrict__ A, int lda,
                             const double2* __restrict__ B, int ldb, double2* __restrict__ C, int ldc) {
  hicu_pdl_entry();
  __shared__ double2 As[16][17];
  __shared__ double2 Bs[16][17];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int row = blockIdx.y * 16 + ty, col = blockIdx.x * 16 + tx;
  double2 acc = cd(0.0, 0.0);
  for (int l0 = 0; l0 < k; l0 += 16) {
    As[ty][tx] = (row < m && l0 + tx < k) ? load_op(A, lda, ca, row, l0 + tx) : cd(0.0, 0.0);
    const int brow = l0 + ty;
    Bs[ty][tx] = (brow < k && col < n) ? load_op(B, ldb, cb, brow, col) : cd(0.0, 0.0);
    __syncthreads();
#pragma unroll
    for (int l = 0; l < 16; ++l) zfma(acc, As[ty][l], Bs[l][tx]);
    __syncthreads();
  }
  if (row < m && col < n) C[(size_t)row * ldc + col] = acc;
}

// Small-K variant: the whole K panel of a 16 x 16 output tile is staged in
// shared memory with one batch of loads and one barrier; each thread then
// runs its K loop with four independent accumulators (DFMA latency ~9
// cycles).  The nullspace GEMMs (K = n or ell <= 256) are latency-bound, and
// the tiled kernel above pays one L2 round trip per 16-wide K chunk.
constexpr int kZgK = 256;
__device__ __forceinline__ void zp_cp16(double2* dst_smem, const double2* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst_smem)),
               "l"(src)
               : "memory");
}
__global__ void __launch_bounds__(256)
zgemm_panel_kernel(bool ca, bool cb, int m, int n, int k, const double2* __restrict__ A, int lda,
                   const double2* __restrict__ B, int ldb, double2* __restrict__ C, int ldc) {
  hicu_pdl_entry();
  extern __shared__ double2 zp[];
  double2* As = zp;              // 16 x (k+1): row r of op(A), padded
  double2* Bs = zp + 16 * (k + 1);  // k x 17: op(B) rows, padded
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int row0 = blockIdx.y * 16, col0 = blockIdx.x * 16;
  // staged with cp.async (every element's copy in flight at once; a
  // load-then-store loop paid one L2 round trip per iteration, ~15 us per
  // call); conjugation is applied when the panels are read
  for (int e = threadIdx.x; e < 16 * k; e += 256) {
    const int r = ca ? e % 16 : e / k, l = ca ? e / 16 : e % k;  // coalesced along the contiguous index
    const int row = row0 + r;
    double2* dst = As + r * (k + 1) + l;
    if (row < m) zp_cp16(dst, ca ? A + (size_t)l * lda + row : A + (size_t)row * lda + l);
    else *dst = cd(0.0, 0.0);
  }
  for (int e = threadIdx.x; e < 16 * k; e += 256) {
    const int c = cb ? e / k : e % 16, l = cb ? e % k : e / 16;
    const int col = col0 + c;
    double2* dst = Bs + l * 17 + c;
    if (col < n) zp_cp16(dst, cb ? B + (size_t)col * ldb + l : B + (size_t)l * ldb + col);
    else *dst = cd(0.0, 0.0);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const double2* a = As + ty * (k + 1);
  double2 c0 = cd(0.0, 0.0), c1 = c0, c2 = c0, c3 = c0;
  int l = 0;
  if (!ca && !cb) {
    for (; l + 3 < k; l += 4) {
      zfma(c0, a[l], Bs[l * 17 + tx]);
      zfma(c1, a[l + 1], Bs[(l + 1) * 17 + tx]);
      zfma(c2, a[l + 2], Bs[(l + 2) * 17 + tx]);
      zfma(c3, a[l + 3], Bs[(l + 3) * 17 + tx]);
    }
    for (; l < k; ++l) zfma(c0, a[l], Bs[l * 17 + tx]);
  } else {
    const double sa = ca ? -1.0 : 1.0, sb = cb ? -1.0 : 1.0;  // conjugation as a sign on the imaginary part
    for (; l + 3 < k; l += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 x = a[l + u], y = Bs[(l + u) * 17 + tx];
        double2& cc = u == 0 ? c0 : (u == 1 ? c1 : (u == 2 ? c2 : c3));
        zfma(cc, cd(x.x, sa * x.y), cd(y.x, sb * y.y));
      }
    }
    for (; l < k; ++l) {
      const double2 x = a[l], y = Bs[l * 17 + tx];
      zfma(c0, cd(x.x, sa * x.y), cd(y.x, sb * y.y));
    }
  }
  const int row = row0 + ty, col = col0 + tx;
  if (row < m && col < n) C[(size_t)row * ldc + col] = (c0 + c1) + (c2 + c3);
}

// Long-K variant (K > kZgK: the Nystrom products over n = 490 / 1000 rows):
// 32 x 32 output tiles, 2 x 2 outputs per thread, K chunks of 32 staged
// K-major through a double-buffered cp.async ring (coalesced along the
// contiguous global index for either op), conjugation applied as a sign when
// the panels are read.  zgemm_kernel above pays two block barriers and an L2
// round trip per 16-wide chunk with one output per thread (120 - 145 us per
// call at C5 / C4).
constexpr int kZtT = 32, kZtK = 32, kZtLd = kZtT + 1;

__global__ void __launch_bounds__(256)
zgemm_tile_kernel(bool ca, bool cb, int m, int n, int k, const double2* __restrict__ A, int lda,
                  const double2* __restrict__ B, int ldb, double2* __restrict__ C, int ldc) {
  hicu_pdl_entry();
  extern __shared__ double2 zt[];
  double2* As = zt;                        // [2][kZtK][kZtLd]: op(A)(row0 + i, l0 + l) at [l][i]
  double2* Bs = zt + 2 * kZtK * kZtLd;     // [2][kZtK][kZtLd]: op(B)(l0 + l, col0 + j) at [l][j]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int row0 = blockIdx.y * kZtT, col0 = blockIdx.x * kZtT;
  auto stage = [&](int c, int buf) {
    const int l0 = c * kZtK;
    for (int e = tid; e < kZtT * kZtK; e += 256) {
      const int i = ca ? e % kZtT : e / kZtK, l = ca ? e / kZtT : e % kZtK;
      double2* dst = As + ((size_t)buf * kZtK + l) * kZtLd + i;
      const int row = row0 + i, ll = l0 + l;
      if (row < m && ll < k) zp_cp16(dst, ca ? A + (size_t)ll * lda + row : A + (size_t)row * lda + ll);
      else *dst = cd(0.0, 0.0);
    }
    for (int e = tid; e < kZtT * kZtK; e += 256) {
      const int j = cb ? e / kZtK : e % kZtT, l = cb ? e % kZtK : e / kZtT;
      double2* dst = Bs + ((size_t)buf * kZtK + l) * kZtLd + j;
      const int col = col0 + j, ll = l0 + l;
      if (col < n && ll < k) zp_cp16(dst, cb ? B + (size_t)col * ldb + ll : B + (size_t)ll * ldb + col);
      else *dst = cd(0.0, 0.0);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const double sa = ca ? -1.0 : 1.0, sb = cb ? -1.0 : 1.0;
  double2 c00 = cd(0.0, 0.0), c01 = c00, c10 = c00, c11 = c00;
  const int nch = (k + kZtK - 1) / kZtK;
  stage(0, 0);
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) {
      stage(c + 1, buf ^ 1);  // last read in chunk c - 1 (barrier at the end of that chunk)
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double2* a = As + (size_t)buf * kZtK * kZtLd;
    const double2* b = Bs + (size_t)buf * kZtK * kZtLd;
#pragma unroll 8
    for (int l = 0; l < kZtK; ++l) {
      double2 a0 = a[l * kZtLd + ty], a1 = a[l * kZtLd + ty + 16];
      double2 b0 = b[l * kZtLd + tx], b1 = b[l * kZtLd + tx + 16];
      a0.y *= sa, a1.y *= sa, b0.y *= sb, b1.y *= sb;
      zfma(c00, a0, b0);
      zfma(c01, a0, b1);
      zfma(c10, a1, b0);
      zfma(c11, a1, b1);
    }
    __syncthreads();
  }
  const int r0 = row0 + ty, r1 = r0 + 16, q0 = col0 + tx, q1 = q0 + 16;
  if (r0 < m && q0 < n) C[(size_t)r0 * ldc + q0] = c00;
  if (r0 < m && q1 < n) C[(size_t)r0 * ldc + q1] = c01;
  if (r1 < m && q0 < n) C[(size_t)r1 * ldc + q0] = c10;
  if (r1 < m && q1 < n) C[(size_t)r1 * ldc + q1] = c11;
}

int zgemm_launch(char opa, char opb, int m, int n, int k, const double2* A, int lda, const double2* B, int ldb,
                 double2* C, int ldc, cudaStream_t st) {
  if (k <= kZgK) {
    const size_t smem = ((size_t)16 * (k + 1) + (size_t)k * 17) * sizeof(double2);
    hicu_allow_max_smem((const void*)zgemm_panel_kernel);
    dim3 grid((n + 15) / 16, (m + 15) / 16);
    hicu_launch(zgemm_panel_kernel, grid, 256, smem, st, opa == 'C', opb == 'C', m, n, k, A, lda, B, ldb, C, ldc);
    return hicu_check_launch("zgemm_panel_kernel");
  }
  if (m * (size_t)n >= 4096) {
    const size_t smem = (size_t)4 * kZtK * kZtLd * sizeof(double2);
    hicu_allow_max_smem((const void*)zgemm_tile_kernel);
    dim3 grid((n + kZtT - 1) / kZtT, (m + kZtT - 1) / kZtT);
    hicu_launch(zgemm_tile_kernel, grid, 256, smem, st, opa == 'C', opb == 'C', m, n, k, A, lda, B, ldb, C, ldc);
    return hicu_check_launch("zgemm_tile_kernel");
  }
  dim3 grid((n + 15) / 16, (m + 15) / 16);
  hicu_launch(zgemm_kernel, grid, 256, 0, st, opa == 'C', opb == 'C', m, n, k, A, lda, B, ldb, C, ldc);
  return hicu_check_launch("zgemm_kernel");
}

// ---------------------------------------------------------------------------
// Cholesky C_nu = C + nu*O = R^H R (upper R, in place in C)
// nu starts at 0; on a non-positive pivot it escalates (stabilised Nystrom).
// ---------------------------------------------------------------------------
template <bool SMEM>
__global__ void __launch_bounds__(512)
chol_kernel(int ell, double2* __restrict__ Cg, const double2* __restrict__ Og, const double2* __restrict__ G,
            int n, double2* __restrict__ gws, double* __restrict__ nu_out, int* __restrict__ status) {
  hicu_pdl_entry();
  extern __shared__ double2 sA[];
  double2* A = SMEM ? sA : gws;
  __shared__ double s_scale;
  __shared__ int s_fail;
  __shared__ double s_nu;
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int i = 0; i < n; ++i) tr += G[(size_t)i * n + i].x;
    s_scale = tr > 0.0 ? tr / n : 1.0;
    s_nu = 0.0;
  }
  __syncthreads();
  for (int attempt = 0; attempt < 12; ++attempt) {
    const double nu = s_nu;
    for (int e = threadIdx.x; e < ell * ell; e += blockDim.x) {
      const double2 o = Og[e];
      A[e] = Cg[e] + nu * o;
    }
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    for (int kk = 0; kk < ell; ++kk) {
      const double d = A[(size_t)kk * ell + kk].x;
      if (!(d > 0.0) || !isfinite(d)) {
        if (threadIdx.x == 0) s_fail = 1;
        __syncthreads();
        break;
      }
      const double rs = sqrt(d), inv = 1.0 / rs;
      __syncthreads();
      for (int j = kk + threadIdx.x; j < ell; j += blockDim.x) {
        if (j == kk) A[(size_t)kk * ell + kk] = cd(rs, 0.0);
        else A[(size_t)kk * ell + j] = inv * A[(size_t)kk * ell + j];
      }
      __syncthreads();
      // trailing update of the upper triangle, one warp per row
      {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int i = kk + 1 + warp; i < ell; i += nw) {
          const double2 a = A[(size_t)kk * ell + i];
#pragma unroll 4
          for (int j = i + lane; j < ell; j += 32) {
            // A[i][j] -= conj(R[kk][i]) * R[kk][j]
            A[(size_t)i * ell + j] = A[(size_t)i * ell + j] - cmulc(a, A[(size_t)kk * ell + j]);
          }
        }
      }
      __syncthreads();
    }
    __syncthreads();
    if (!s_fail) break;
    if (threadIdx.x == 0) s_nu = (s_nu == 0.0) ? 1e-14 * s_scale : s_nu * 100.0;
    __syncthreads();
    if (attempt == 11 && threadIdx.x == 0) *status = HICU_ERR_DEGENERATE_INPUT;
  }
  // write back R (upper triangle, zero below)
  for (int e = threadIdx.x; e < ell * ell; e += blockDim.x) {
    const int i = e / ell, j = e % ell;
    Cg[e] = (j >= i) ? A[e] : cd(0.0, 0.0);
  }
  if (threadIdx.x == 0) *nu_out = s_nu;
}

// Cholesky on an 8-CTA cluster for ell > 96 when C does not fit one SM's
// shared memory (C3 / C4 / C5: ell = 150 / 225 / 180).  Row i of the upper
// triangle lives in CTA i % 8 (cyclic); per step the owner of row k takes
// the pivot's square root, scales its row and writes it into every CTA's
// shared memory (double-buffered by step parity); one cluster barrier; each
// CTA folds row k into its rows.  Same arithmetic per element as chol_kernel
// (A[i][j] -= conj(R[k][i]) R[k][j]); the shift escalation on a non-positive
// pivot is decided identically by every CTA (the failing pivot's owner
// broadcasts the flag with the row).
constexpr int kCcCS = 8;
constexpr int kCcThreads = 512;
constexpr int kCcMaxL = 256;

__global__ void __cluster_dims__(kCcCS, 1, 1) __launch_bounds__(kCcThreads, 1)
chol_cluster_kernel(int ell, double2* __restrict__ Cg, const double2* __restrict__ Og, const double2* __restrict__ G,
                    int n, double* __restrict__ nu_out, int* __restrict__ status) {
  hicu_pdl_entry();
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  extern __shared__ double2 ccA[];  // [nr][ell]
  __shared__ double2 srow[2][kCcMaxL];
  __shared__ int sfail[2];
  __shared__ double s_scale;
  __shared__ double wred[kCcThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = kCcThreads / 32;
  const int nr = (ell - cr + kCcCS - 1) / kCcCS;
  {  // shift scale: trace(G) / n, summed warp-parallel in a fixed order (every CTA the same value)
    double t = 0.0;
    for (int i = tid; i < n; i += kCcThreads) t += G[(size_t)i * n + i].x;
    t = warp_sum_d_(t);
    if (lane == 0) wred[warp] = t;
    __syncthreads();
    if (tid == 0) {
      double tr = 0.0;
      for (int w = 0; w < nw; ++w) tr += wred[w];
      s_scale = tr > 0.0 ? tr / n : 1.0;
    }
    __syncthreads();
  }
  double nu = 0.0;
  bool failed = false;
  for (int attempt = 0; attempt < 12; ++attempt) {
    for (int q = tid; q < nr * ell; q += kCcThreads) {
      const int r = q / ell, j = q - r * ell;
      const size_t gi = (size_t)(cr + kCcCS * r) * ell + j;
      ccA[q] = Cg[gi] + nu * Og[gi];
    }
    if (tid < 2) sfail[tid] = 0;
    cluster.sync();
    failed = false;
    for (int k = 0; k < ell; ++k) {
      const int buf = k & 1;
      if (cr == k % kCcCS) {
        double2* row = ccA + (size_t)(k / kCcCS) * ell;
        const double dg = row[k].x;
        const bool bad = !(dg > 0.0) || !isfinite(dg);
        if (bad) {
          if (tid < kCcCS) *cluster.map_shared_rank(&sfail[buf], tid) = 1;
        } else {
          const double rs = sqrt(dg), inv = 1.0 / rs;
          for (int q = tid; q < kCcCS * (ell - k); q += kCcThreads) {
            const int c = q / (ell - k), j = k + (q - c * (ell - k));
            const double2 v = j == k ? cd(rs, 0.0) : inv * row[j];
            *cluster.map_shared_rank(&srow[buf][j], c) = v;
          }
          __syncthreads();  // every thread has read the unscaled row
          for (int j = k + tid; j < ell; j += kCcThreads) row[j] = srow[buf][j];
        }
      }
      cluster.sync();
      if (sfail[buf]) {
        failed = true;
        break;
      }
      // fold row k into this CTA's rows i > k (upper triangle j >= i)
      for (int r = warp; r < nr; r += nw) {
        const int i = cr + kCcCS * r;
        if (i <= k) continue;
        const double2 a = srow[buf][i];
        double2* Ai = ccA + (size_t)r * ell;
        for (int j = i + lane; j < ell; j += 32) Ai[j] = Ai[j] - cmulc(a, srow[buf][j]);
      }
      __syncthreads();  // the next owner reads its updated row
    }
    if (!failed) break;
    nu = nu == 0.0 ? 1e-14 * s_scale : nu * 100.0;
    cluster.sync();  // every CTA has seen the failure before the flags are cleared
    if (attempt == 11 && cr == 0 && tid == 0) *status = HICU_ERR_DEGENERATE_INPUT;
  }
  for (int q = tid; q < nr * ell; q += kCcThreads) {
    const int r = q / ell, j = q - r * ell, i = cr + kCcCS * r;
    Cg[(size_t)i * ell + j] = j >= i ? ccA[q] : cd(0.0, 0.0);
  }
  if (cr == 0 && tid == 0) *nu_out = nu;
  cluster.sync();
}

// Register-resident variant (ell <= 96): row i of the upper triangle lives
// in warp i % 16 (slot i / 16), lane t holding columns t + 32u.  Step k: the
// owner warp finalises row k (sqrt + one reciprocal on every lane, no
// reduction) and publishes it in a double-buffered shared row guarded by
// mbarriers (full: owner -> all, empty: all 16 warps -> next writer), so
// there is no block barrier: the owner of row k+1 folds row k into row k+1
// first and publishes it while the other warps are still folding row k into
// their rows (one-step lookahead).  Same arithmetic per element as
// chol_kernel up to FMA contraction; the shift-scale trace is summed
// warp-parallel in a fixed order.
__device__ unsigned g_chol_trace[12];  // debug (HICU_CHOL_TRACE)

template <int PER, int RPW>
__device__ __forceinline__ void chol3_publish(int k, int ell, int lane, double2 (&a)[RPW][PER], double2* buf,
                                              int* fail_flag) {
  const int os = k >> 4, uk = k >> 5;
  double2 rk[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    rk[u] = a[0][u];
#pragma unroll
    for (int s = 1; s < RPW; ++s) rk[u] = (s == os) ? a[s][u] : rk[u];
  }
  double dk = rk[0].x;
#pragma unroll
  for (int u = 1; u < PER; ++u) dk = (u == uk) ? rk[u].x : dk;
  dk = __shfl_sync(0xffffffffu, dk, k & 31);
  const bool ok = (dk > 0.0) && isfinite(dk);
  const double rs = sqrt(dk), inv = 1.0 / rs;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int j = lane + 32 * u;
    const double2 val = (j == k) ? cd(rs, 0.0) : inv * rk[u];
    buf[j] = val;
#pragma unroll
    for (int s = 0; s < RPW; ++s)
      if (s == os) a[s][u] = val;
  }
  if (lane == 0) *fail_flag = ok ? 0 : 1;
}

template <int PER, int RPW>
__device__ __forceinline__ void chol3_fold(int k, int warp, int ell, int only, int skip, const double2* buf,
                                           const double2 (&rj)[PER], double2 (&a)[RPW][PER]) {
#pragma unroll
  for (int s = 0; s < RPW; ++s) {
    const int i = warp + 16 * s;
    if (i > k && i < ell && (only < 0 || s == only) && s != skip) {
      const double2 ai = buf[i];
#pragma unroll
      for (int u = 0; u < PER; ++u)
        if (32 * (u + 1) > k + 1) {
          a[s][u].x = fma(-ai.x, rj[u].x, fma(-ai.y, rj[u].y, a[s][u].x));
          a[s][u].y = fma(-ai.x, rj[u].y, fma(ai.y, rj[u].x, a[s][u].y));
        }
    }
  }
}

template <int PER, int RPW>
__global__ void __launch_bounds__(512)
chol2_kernel(int ell, double2* __restrict__ Cg, const double2* __restrict__ Og, const double2* __restrict__ G, int n,
             double* __restrict__ nu_out, int* __restrict__ status) {
  hicu_pdl_entry();
  __shared__ double2 rowk[2][PER * 32];
  __shared__ double red[16];
  __shared__ int s_fail[2];
  __shared__ __align__(8) uint64_t bars[12][4];  // per attempt: full[2], empty[2]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  {
    double tr = 0.0;
    for (int i = t; i < n; i += 512) tr += G[(size_t)i * n + i].x;
    for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
    if (lane == 0) red[warp] = tr;
  }
  if (t < 48) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(&bars[t >> 2][t & 3]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"((t & 3) < 2 ? 1 : 16));
  }
  __syncthreads();
  double scale = 0.0;
#pragma unroll
  for (int w = 0; w < 16; ++w) scale += red[w];
  scale = scale > 0.0 ? scale / n : 1.0;
  const unsigned c0 = (unsigned)clock();
  double nu = 0.0;
  double2 a[RPW][PER];
  bool failed = true;
  auto arrive = [](uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(b)) : "memory");
  };
  auto wait = [](uint64_t* b, uint32_t par) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
        "r"(par)
        : "memory");
  };
  for (int attempt = 0; attempt < 12; ++attempt) {
    uint64_t* full = bars[attempt];
    uint64_t* empty = bars[attempt] + 2;
#pragma unroll
    for (int s = 0; s < RPW; ++s) {
      const int i = warp + 16 * s;
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int j = lane + 32 * u;
        a[s][u] = (i < ell && j < ell) ? Cg[(size_t)i * ell + j] + nu * Og[(size_t)i * ell + j] : cd(0.0, 0.0);
      }
    }
    bool fail = false;
    const unsigned c1 = (unsigned)clock();
    if (warp == 0) {
      chol3_publish<PER, RPW>(0, ell, lane, a, rowk[0], &s_fail[0]);
      __syncwarp();
      if (lane == 0) arrive(&full[0]);
    }
    for (int k = 0; k < ell; ++k) {
      const int b = k & 1;
      wait(&full[b], (k >> 1) & 1);
      double2 rj[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) rj[u] = rowk[b][lane + 32 * u];
      if (s_fail[b]) {
        fail = true;
        break;
      }
      const int k1 = k + 1;
      if (k1 < ell && warp == (k1 & 15)) {
        const int s1 = k1 >> 4;
        const bool tr = (k == 30 || k == 31) && lane == 0;
        const int tb = (k - 30) * 5;
        if (tr) g_chol_trace[2 + tb] = (unsigned)clock();
        chol3_fold<PER, RPW>(k, warp, ell, s1, -1, rowk[b], rj, a);
        if (tr) g_chol_trace[3 + tb] = (unsigned)(clock() + (int)(a[0][0].x > 1e300));
        if (k1 >= 2) wait(&empty[k1 & 1], ((k1 >> 1) - 1) & 1);
        if (tr) g_chol_trace[4 + tb] = (unsigned)clock();
        chol3_publish<PER, RPW>(k1, ell, lane, a, rowk[k1 & 1], &s_fail[k1 & 1]);
        __syncwarp();
        if (lane == 0) arrive(&full[k1 & 1]);
        if (tr) g_chol_trace[5 + tb] = (unsigned)clock();
        chol3_fold<PER, RPW>(k, warp, ell, -1, s1, rowk[b], rj, a);
        if (tr) g_chol_trace[6 + tb] = (unsigned)(clock() + (int)(a[0][0].x > 1e300));
      } else {
        chol3_fold<PER, RPW>(k, warp, ell, -1, -1, rowk[b], rj, a);
      }
      __syncwarp();
      if (lane == 0) arrive(&empty[b]);
    }
    __syncthreads();
    if (t == 0) {
      g_chol_trace[0] = c1 - c0;
      g_chol_trace[1] = (unsigned)clock() - c1;
    }
    if (!fail) {
      failed = false;
      break;
    }
    nu = (nu == 0.0) ? 1e-14 * scale : nu * 100.0;
  }
  if (failed) {
    if (t == 0) *status = HICU_ERR_DEGENERATE_INPUT;
  }
#pragma unroll
  for (int s = 0; s < RPW; ++s) {
    const int i = warp + 16 * s;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int j = lane + 32 * u;
      if (i < ell && j < ell) Cg[(size_t)i * ell + j] = (j >= i) ? a[s][u] : cd(0.0, 0.0);
    }
  }
  if (t == 0) *nu_out = nu;
}

// W = (Y + nu*Omega) R^{-1}; one warp per row, R staged in smem when it fits.
__global__ void trsm_rows_kernel(int n, int ell, const double2* __restrict__ Y, const double2* __restrict__ Om,
                                 const double* __restrict__ nu_p, const double2* __restrict__ R, bool r_smem,
                                 double2* __restrict__ W) {
  hicu_pdl_entry();
  extern __shared__ double2 sm[];
  const int warps = blockDim.x >> 5;
  double2* sR = sm;
  double2* rowbuf = sm + (r_smem ? (size_t)ell * ell : 0);
  if (r_smem) {
    for (int e = threadIdx.x; e < ell * ell; e += blockDim.x) sR[e] = R[e];
    __syncthreads();
  }
  const double2* RR = r_smem ? sR : R;
  const double nu = *nu_p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* w = rowbuf + (size_t)warp * ell;
  for (int row = blockIdx.x * warps + warp; row < n; row += gridDim.x * warps) {
    for (int j = 0; j < ell; ++j) {
      double2 part = cd(0.0, 0.0);
      for (int k = lane; k < j; k += 32) zfma(part, w[k], RR[(size_t)k * ell + j]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        part.x += __shfl_xor_sync(0xffffffffu, part.x, o);
        part.y += __shfl_xor_sync(0xffffffffu, part.y, o);
      }
      if (lane == 0) {
        const double2 yv = Y[(size_t)row * ell + j] + nu * Om[(size_t)row * ell + j];
        const double2 num = yv - part;
        const double rjj = RR[(size_t)j * ell + j].x;
        w[j] = cd(num.x / rjj, num.y / rjj);
      }
      __syncwarp();
    }
    for (int j = lane; j < ell; j += 32) W[(size_t)row * ell + j] = w[j];
    __syncwarp();
  }
}

// Right-looking variant: one warp per row, lane t owns entries j = t, t+32,
// t+64, ... of the row.  For each j the owner finishes w_j (one multiply by the
// precomputed 1/R_jj), broadcasts it with one shuffle, and every lane folds
// w_j R[j][k] into its pending entries k > j: no reduction per column.
constexpr int kTrsmMaxPer = 8;  // ell <= 256
__device__ unsigned g_trsm_trace[4];  // debug (HICU_TRSM_TRACE): block 0 warp 0 cycles of the first row
// PER = ceil(ell / 32).  Every per-column step is branch-free: the row of R
// is loaded for all PER slots before the owner's shuffle (clamped index, so
// the loads never wait on w_j) and the fold is a select, so a step costs one
// shuffle + two dependent FMAs instead of PER serialised load latencies.
template <int PER>
__global__ void __launch_bounds__(128) trsm_rl_kernel(int n, int ell, const double2* __restrict__ Y,
                                                      const double2* __restrict__ Om, const double* __restrict__ nu_p,
                                                      const double2* __restrict__ R, double2* __restrict__ W) {
  hicu_pdl_entry();
  extern __shared__ double2 smr[];
  double2* sR = smr;                                       // ell x ell (upper)
  double* rinv = reinterpret_cast<double*>(sR + (size_t)ell * ell);  // 1 / R_jj
  for (int e = threadIdx.x; e < ell * ell; e += blockDim.x) sR[e] = R[e];
  for (int j = threadIdx.x; j < ell; j += blockDim.x) rinv[j] = 1.0 / R[(size_t)j * ell + j].x;
  __syncthreads();
  const unsigned c1 = (unsigned)clock();
  const double nu = *nu_p;
  const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int kc[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) kc[u] = min(lane + 32 * u, ell - 1);
  for (int row = blockIdx.x * warps + warp; row < n; row += gridDim.x * warps) {
    double2 acc[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int j = lane + 32 * u;
      acc[u] = (j < ell) ? Y[(size_t)row * ell + j] + nu * Om[(size_t)row * ell + j] : cd(0.0, 0.0);
    }
    for (int j = 0; j < ell; ++j) {
      const double2* Rj = sR + (size_t)j * ell;
      double2 rj[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) rj[u] = Rj[kc[u]];
      const double ri = rinv[j];
      const int uj = j >> 5;
      double2 wj = acc[0];
#pragma unroll
      for (int u = 1; u < PER; ++u) wj = (u == uj) ? acc[u] : wj;
      wj = ri * wj;
      wj.x = __shfl_sync(0xffffffffu, wj.x, j & 31);
      wj.y = __shfl_sync(0xffffffffu, wj.y, j & 31);
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int k = lane + 32 * u;
        const double2 t = acc[u] - cmul(wj, rj[u]);
        acc[u] = (k == j) ? wj : ((k > j) ? t : acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int j = lane + 32 * u;
      if (j < ell) W[(size_t)row * ell + j] = acc[u];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) g_trsm_trace[1] = (unsigned)clock() - c1;
  }
}

template <int PER>
void trsm_rl_launch(int n, int ell, const double2* Y, const double2* Om, const double* nu, const double2* R,
                    double2* W, size_t smem, cudaStream_t st) {
  if (PER * 32 < ell) {
    if constexpr (PER < kTrsmMaxPer) trsm_rl_launch<PER + 1>(n, ell, Y, Om, nu, R, W, smem, st);
    return;
  }
  const int warps = 4;
  hicu_allow_max_smem((const void*)trsm_rl_kernel<PER>);
  hicu_launch(trsm_rl_kernel<PER>, (n + warps - 1) / warps, warps * 32, smem, st, n, ell, Y, Om, nu, R, W);
}

// Streaming variant for ell > 112 (R no longer fits one SM's shared memory:
// C3 / C4 / C5, ell = 150 / 225 / 180): the same right-looking steps, with the
// rows of R staged kTrsJB at a time through a double-buffered cp.async ring
// shared by the CTA's warps (one row of Y per warp, every warp walks the
// blocks in lockstep).  trsm_rows_kernel read R column-wise from L2 with a
// warp reduction per column: 250 / 430 us at ell = 180 / 225.
constexpr int kTrsJB = 16;
constexpr int kTrsWarps = 8;

template <int PER>
__global__ void __launch_bounds__(kTrsWarps * 32)
trsm_rls_kernel(int n, int ell, const double2* __restrict__ Y, const double2* __restrict__ Om,
                const double* __restrict__ nu_p, const double2* __restrict__ R, double2* __restrict__ W) {
  hicu_pdl_entry();
  extern __shared__ double2 smr[];
  double2* sR = smr;                                                          // 2 x kTrsJB x ell
  double* rinv = reinterpret_cast<double*>(sR + (size_t)2 * kTrsJB * ell);   // 1 / R_jj
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nblk = (ell + kTrsJB - 1) / kTrsJB;
  auto stage = [&](int b) {
    const int j0 = b * kTrsJB, rows = min(kTrsJB, ell - j0);
    double2* dst = sR + (size_t)(b & 1) * kTrsJB * ell;
    const double2* src = R + (size_t)j0 * ell;
    for (int e = tid; e < rows * ell; e += kTrsWarps * 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst + e)),
                   "l"(src + e)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage(0);
  for (int j = tid; j < ell; j += kTrsWarps * 32) rinv[j] = 1.0 / R[(size_t)j * ell + j].x;
  const double nu = *nu_p;
  const int row = blockIdx.x * kTrsWarps + warp;
  const bool live = row < n;
  int kc[PER];
  double2 acc[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int j = lane + 32 * u;
    kc[u] = min(j, ell - 1);
    acc[u] = (live && j < ell) ? Y[(size_t)row * ell + j] + nu * Om[(size_t)row * ell + j] : cd(0.0, 0.0);
  }
  for (int b = 0; b < nblk; ++b) {
    if (b + 1 < nblk) {
      stage(b + 1);  // its buffer was last read in block b - 1 (barrier at the end of that block)
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double2* blk = sR + (size_t)(b & 1) * kTrsJB * ell;
    const int j0 = b * kTrsJB, rows = min(kTrsJB, ell - j0);
    for (int jj = 0; jj < rows; ++jj) {
      const int j = j0 + jj;
      const double2* Rj = blk + (size_t)jj * ell;
      double2 rj[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) rj[u] = Rj[kc[u]];
      const double ri = rinv[j];
      const int uj = j >> 5;
      double2 wj = acc[0];
#pragma unroll
      for (int u = 1; u < PER; ++u) wj = (u == uj) ? acc[u] : wj;
      wj = ri * wj;
      wj.x = __shfl_sync(0xffffffffu, wj.x, j & 31);
      wj.y = __shfl_sync(0xffffffffu, wj.y, j & 31);
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int k = lane + 32 * u;
        const double2 t = acc[u] - cmul(wj, rj[u]);
        acc[u] = (k == j) ? wj : ((k > j) ? t : acc[u]);
      }
    }
    __syncthreads();  // block b's buffer is free for block b + 2
  }
  if (live) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int j = lane + 32 * u;
      if (j < ell) W[(size_t)row * ell + j] = acc[u];
    }
  }
}

template <int PER>
void trsm_rls_launch(int n, int ell, const double2* Y, const double2* Om, const double* nu, const double2* R,
                     double2* W, cudaStream_t st) {
  if (PER * 32 < ell) {
    if constexpr (PER < kTrsmMaxPer) trsm_rls_launch<PER + 1>(n, ell, Y, Om, nu, R, W, st);
    return;
  }
  const size_t smem = (size_t)2 * kTrsJB * ell * sizeof(double2) + (size_t)ell * sizeof(double);
  hicu_allow_max_smem((const void*)trsm_rls_kernel<PER>);
  hicu_launch(trsm_rls_kernel<PER>, (n + kTrsWarps - 1) / kTrsWarps, kTrsWarps * 32, smem, st, n, ell, Y, Om, nu, R,
              W);
}

// ---------------------------------------------------------------------------
// Cyclic parallel two-sided Jacobi for a Hermitian PSD matrix (round-robin
// ordering).  Logs every rotation (p, q, c, s*e^{i phi}) so the same unitary
// can be applied to W afterwards; emits eigenvalues and their descending order.
// ---------------------------------------------------------------------------
struct RotEntry {
  int p, q;
  double c;
  double2 se;
};

__device__ __forceinline__ void rr_pair(int m, int round, int i, int& p, int& q) {
  if (i == 0) {
    p = m - 1;
    q = round;
  } else {
    p = (round + i) % (m - 1);
    q = (round - i + (m - 1)) % (m - 1);
  }
  if (p > q) { int t = p; p = q; q = t; }
}

__global__ void __launch_bounds__(1024)
jacobi_kernel(int ell, const double2* __restrict__ Mg, double2* __restrict__ gws, bool use_smem, int max_sweeps,
              double tol, RotEntry* __restrict__ log, int* __restrict__ nrounds_out, double* __restrict__ evals,
              int* __restrict__ order, int* __restrict__ status) {
  hicu_pdl_entry();
  extern __shared__ double2 sA[];
  double2* A = use_smem ? sA : gws;
  const int m = ell + (ell & 1);
  const int half = m / 2;
  __shared__ RotEntry rot[128];
  __shared__ int s_any;
  __shared__ double s_floor;
  for (int e = threadIdx.x; e < ell * ell; e += blockDim.x) A[e] = Mg[e];
  __syncthreads();
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int i = 0; i < ell; ++i) tr += fabs(A[(size_t)i * ell + i].x);
    s_floor = 1e-300 + 1e-15 * tr;  // below fp64 round-off of the largest eigenvalues
  }
  __syncthreads();
  int rounds = 0;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
    for (int rd = 0; rd < m - 1; ++rd) {
      if (threadIdx.x < half) {
        int p, q;
        rr_pair(m, rd, threadIdx.x, p, q);
        RotEntry r{p, q, 1.0, cd(0.0, 0.0)};
        if (q < ell) {
          const double a = A[(size_t)p * ell + p].x, d = A[(size_t)q * ell + q].x;
          const double2 b = A[(size_t)p * ell + q];
          const double bb = sqrt(abs2d(b));
          if (bb > s_floor && bb > tol * sqrt(fabs(a * d))) {
            const double th = (d - a) / (2.0 * bb);
            const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(1.0 + th * th));
            const double c = 1.0 / sqrt(1.0 + t * t);
            const double s = t * c;
            r.c = c;
            r.se = cd(s * b.x / bb, s * b.y / bb);
            s_any = 1;
          }
        }
        rot[threadIdx.x] = r;
        log[(size_t)rounds * half + threadIdx.x] = r;
      }
      __syncthreads();
      // rows: (A_p, A_q) <- (c A_p - se A_q, conj(se) A_p + c A_q)
      for (int e = threadIdx.x; e < half * ell; e += blockDim.x) {
        const RotEntry r = rot[e / ell];
        if (r.q >= ell || (r.se.x == 0.0 && r.se.y == 0.0)) continue;
        const int j = e % ell;
        const double2 ap = A[(size_t)r.p * ell + j], aq = A[(size_t)r.q * ell + j];
        A[(size_t)r.p * ell + j] = r.c * ap - cmul(r.se, aq);
        A[(size_t)r.q * ell + j] = cmulc(r.se, ap) + r.c * aq;
      }
      __syncthreads();
      // cols: (A_:p, A_:q) <- (c A_:p - conj(se) A_:q, se A_:p + c A_:q)
      for (int e = threadIdx.x; e < half * ell; e += blockDim.x) {
        const RotEntry r = rot[e / ell];
        if (r.q >= ell || (r.se.x == 0.0 && r.se.y == 0.0)) continue;
        const int j = e % ell;
        const double2 ap = A[(size_t)j * ell + r.p], aq = A[(size_t)j * ell + r.q];
        A[(size_t)j * ell + r.p] = r.c * ap - cmulc(r.se, aq);
        A[(size_t)j * ell + r.q] = cmul(r.se, ap) + r.c * aq;
      }
      __syncthreads();
      ++rounds;
    }
    if (!s_any) break;
  }
  if (threadIdx.x == 0) *nrounds_out = rounds;
  for (int i = threadIdx.x; i < ell; i += blockDim.x) evals[i] = A[(size_t)i * ell + i].x;
  __syncthreads();
  // descending order by rank counting (ties broken by index: stable)
  for (int i = threadIdx.x; i < ell; i += blockDim.x) {
    const double v = evals[i];
    int rank = 0;
    for (int j = 0; j < ell; ++j) {
      const double w = evals[j];
      rank += (w > v) || (w == v && j < i);
    }
    order[rank] = i;
  }
}

// Apply the logged rotations to the rows of W (n x ell), one warp per row,
// then V[row, t] = W'[row, order[t]] / sqrt(evals[order[t]]) for t < r.
__global__ void rot_apply_kernel(int n, int ell, int r, const double2* __restrict__ W, const RotEntry* __restrict__ log,
                                 const int* __restrict__ nrounds_p, const double* __restrict__ evals,
                                 const int* __restrict__ order, double2* __restrict__ V, int* __restrict__ status,
                                 bool scale) {
  hicu_pdl_entry();
  extern __shared__ double2 sw[];
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = ell + (ell & 1), half = m / 2;
  const int nrounds = *nrounds_p;
  double2* w = sw + (size_t)warp * ell;
  for (int row = blockIdx.x * warps + warp; row < n; row += gridDim.x * warps) {
    for (int j = lane; j < ell; j += 32) w[j] = W[(size_t)row * ell + j];
    __syncwarp();
    for (int rd = 0; rd < nrounds; ++rd) {
      const RotEntry* lr = log + (size_t)rd * half;
      for (int i = lane; i < half; i += 32) {
        const RotEntry e = lr[i];
        if (e.q >= ell || (e.se.x == 0.0 && e.se.y == 0.0)) continue;
        const double2 xp = w[e.p], xq = w[e.q];
        w[e.p] = e.c * xp - cmulc(e.se, xq);
        w[e.q] = cmul(e.se, xp) + e.c * xq;
      }
      __syncwarp();
    }
    for (int t = lane; t < r; t += 32) {
      const int src = order[t];
      const double lam = evals[src];
      double2 v = cd(0.0, 0.0);
      if (!scale) {
        v = w[src];
      } else if (lam > 0.0) {
        const double inv = 1.0 / sqrt(lam);
        v = inv * w[src];
      } else if (status) {
        *status = HICU_ERR_DEGENERATE_INPUT;
      }
      V[(size_t)row * r + t] = v;
    }
    __syncwarp();
  }
}

// Canonical phase of each column of V (n x r): rotate so the largest-|.|
// entry (first on ties) is real positive.  The reference's V carries LAPACK
// zgesdd's phases, which are an implementation detail; fixing a documented
// convention makes the Householder basis (subspace.py:158-212), and with it
// the free-running trajectory, reproducible by the oracle.
__global__ void canon_phase_kernel(int n, int r, double2* __restrict__ V, const double* __restrict__ lam,
                                   int* __restrict__ status) {
  hicu_pdl_entry();
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = blockIdx.x * warps + warp; t < r; t += gridDim.x * warps) {
    if (lam) {
      // V = W F Lambda^{-1/2}: unit columns (left singular vectors of W)
      const double lv = lam[t];
      const double sc = lv > 0.0 ? 1.0 / sqrt(lv) : 0.0;
      if (!(lv > 0.0) && lane == 0 && status) *status = HICU_ERR_DEGENERATE_INPUT;
      for (int k = lane; k < n; k += 32) V[(size_t)k * r + t] = sc * V[(size_t)k * r + t];
      __syncwarp();
    }
    double best = -1.0;
    int bk = 0;
    for (int k = lane; k < n; k += 32) {
      const double a = abs2d(V[(size_t)k * r + t]);
      if (a > best) { best = a; bk = k; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
      if (ob > best || (ob == best && ok < bk)) { best = ob; bk = ok; }
    }
    const double2 e = V[(size_t)bk * r + t];
    const double mag = sqrt(abs2d(e));
    if (!(mag > 0.0)) continue;
    const double2 ph = cd(e.x / mag, -e.y / mag);  // conj(e)/|e|
    __syncwarp();
    for (int k = lane; k < n; k += 32) V[(size_t)k * r + t] = cmul(V[(size_t)k * r + t], ph);
  }
}

// ---------------------------------------------------------------------------
// Householder triangularisation of V (subspace.py:158-201).  refl is r x n
// (row j = w_j, zero before entry j), tau r, flags r.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024)
householder_kernel(int n, int r, const double2* __restrict__ Vg, double tol, double2* __restrict__ gws,
                   bool use_smem, double2* __restrict__ refl, double2* __restrict__ tau, int* __restrict__ flags,
                   int* __restrict__ status,
    const int* __restrict__ gate) {
  hicu_pdl_entry();
  if (gate && *gate == 0) return;  // closed-form path succeeded (nsjl.cu)
  extern __shared__ double2 sV[];
  double2* sw = sV;                                   // current reflector w (n)
  double2* v = use_smem ? sV + n : gws;  // column-major: element (k, j) at v[j*n + k] (conflict-free)
  __shared__ double red[32];
  __shared__ double2 s_u0inv, s_tau;
  __shared__ int s_active;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = threadIdx.x; e < n * r; e += blockDim.x) v[(size_t)(e % r) * n + e / r] = Vg[e];
  for (int e = threadIdx.x; e < n * r; e += blockDim.x) refl[e] = cd(0.0, 0.0);
  __syncthreads();
  for (int col = 0; col < r; ++col) {
    double t = 0.0;
    for (int k = col + 1 + threadIdx.x; k < n; k += blockDim.x) t += abs2d(v[(size_t)col * n + k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[warp] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tail = 0.0;
      for (int w = 0; w < nw; ++w) tail += red[w];
      const double2 x0 = v[(size_t)col * n + col];
      const double beta = sqrt(tail + x0.x * x0.x + x0.y * x0.y);
      int active = 1;
      if (beta < tol) {
        *status = HICU_ERR_DEGENERATE_INPUT;
        active = 0;
      } else if (tail == 0.0 && x0.y == 0.0 && x0.x >= 0.0) {
        active = 0;
      }
      double2 u0 = cd(0.0, 0.0), tv = cd(0.0, 0.0);
      if (active) {
        if (x0.x > 0.0) {
          // (-tail + 2i beta x0.im) / (conj(x0) + beta)
          const double2 nume = cd(-tail, 2.0 * beta * x0.y);
          const double2 deno = cd(x0.x + beta, -x0.y);
          const double dd = abs2d(deno);
          u0 = cd((nume.x * deno.x + nume.y * deno.y) / dd, (nume.y * deno.x - nume.x * deno.y) / dd);
        } else {
          u0 = cd(x0.x - beta, x0.y);
        }
        tv = cd((beta - x0.x) / beta, x0.y / beta);  // (beta - conj(x0)) / beta
      }
      const double uu = abs2d(u0);
      s_u0inv = active ? cd(u0.x / uu, -u0.y / uu) : cd(0.0, 0.0);
      s_tau = tv;
      s_active = active;
      flags[col] = active;
      tau[col] = tv;
    }
    __syncthreads();
    if (s_active) {
      const double2 ui = s_u0inv;
      // w = xvec / u0, w[0] = 1
      for (int k = col + threadIdx.x; k < n; k += blockDim.x) {
        const double2 wv = (k == col) ? cd(1.0, 0.0) : cmul(v[(size_t)col * n + k], ui);
        refl[(size_t)col * n + k] = wv;
        sw[k] = wv;
      }
      __syncthreads();
      // rest -= (tau w)(w^H rest), one warp per remaining column
      const double2 tv = s_tau;
      const double2* wrow = sw;
      // two columns per warp pass so the two shuffle-reduction chains overlap
      for (int j0 = col + 1 + warp; j0 < r; j0 += 2 * nw) {
        const int j1 = j0 + nw;
        const bool two = j1 < r;
        double2 d0 = cd(0.0, 0.0), d1 = cd(0.0, 0.0);
        for (int k = col + lane; k < n; k += 32) {
          const double2 wk = wrow[k];
          zfmac(d0, wk, v[(size_t)j0 * n + k]);
          if (two) zfmac(d1, wk, v[(size_t)j1 * n + k]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          d0.x += __shfl_xor_sync(0xffffffffu, d0.x, o);
          d0.y += __shfl_xor_sync(0xffffffffu, d0.y, o);
          d1.x += __shfl_xor_sync(0xffffffffu, d1.x, o);
          d1.y += __shfl_xor_sync(0xffffffffu, d1.y, o);
        }
        const double2 f0 = cmul(tv, d0), f1 = cmul(tv, d1);
        for (int k = col + lane; k < n; k += 32) {
          const double2 wk = wrow[k];
          v[(size_t)j0 * n + k] = v[(size_t)j0 * n + k] - cmul(wk, f0);
          if (two) v[(size_t)j1 * n + k] = v[(size_t)j1 * n + k] - cmul(wk, f1);
        }
      }
    }
    __syncthreads();
  }
}

// Latency-oriented Householder triangularisation (same reflectors as
// householder_kernel): one block barrier per column.  Warp 0 owns column
// col+1: it applies reflector col to it, then immediately builds reflector
// col+1 (norm by shuffles, w into the other half of a double-buffered smem
// vector, refl row to global).  Warps 1.. apply reflector col to the other
// remaining columns, two per pass so their reduction chains overlap.
__device__ __forceinline__ void hh2_reflector(int n, int c, const double2* vc, double tol, int lane,
                                              double2* __restrict__ refl, double2* __restrict__ tau,
                                              int* __restrict__ flags, int* __restrict__ status, double2* s_tau,
                                              int* s_act, double2* w_next) {
  double t = 0.0;
  for (int k = c + 1 + lane; k < n; k += 32) t += abs2d(vc[k]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  double2 ui = cd(0.0, 0.0);
  int active = 0;
  if (lane == 0) {
    const double tail = t;
    const double2 x0 = vc[c];
    const double beta = sqrt(tail + x0.x * x0.x + x0.y * x0.y);
    active = 1;
    if (beta < tol) {
      *status = HICU_ERR_DEGENERATE_INPUT;
      active = 0;
    } else if (tail == 0.0 && x0.y == 0.0 && x0.x >= 0.0) {
      active = 0;
    }
    double2 u0 = cd(0.0, 0.0), tv = cd(0.0, 0.0);
    if (active) {
      if (x0.x > 0.0) {
        const double2 nume = cd(-tail, 2.0 * beta * x0.y);
        const double2 deno = cd(x0.x + beta, -x0.y);
        const double dd = abs2d(deno);
        u0 = cd((nume.x * deno.x + nume.y * deno.y) / dd, (nume.y * deno.x - nume.x * deno.y) / dd);
      } else {
        u0 = cd(x0.x - beta, x0.y);
      }
      tv = cd((beta - x0.x) / beta, x0.y / beta);
      const double uu = abs2d(u0);
      ui = cd(u0.x / uu, -u0.y / uu);
    }
    *s_tau = tv;
    *s_act = active;
    flags[c] = active;
    tau[c] = tv;
  }
  active = __shfl_sync(0xffffffffu, active, 0);
  ui.x = __shfl_sync(0xffffffffu, ui.x, 0);
  ui.y = __shfl_sync(0xffffffffu, ui.y, 0);
  if (!active) return;
  for (int k = c + lane; k < n; k += 32) {
    const double2 wv = (k == c) ? cd(1.0, 0.0) : cmul(vc[k], ui);
    refl[(size_t)c * n + k] = wv;
    w_next[k] = wv;
  }
}

__global__ void __launch_bounds__(1024)
householder2_kernel(int n, int r, const double2* __restrict__ Vg, double tol, double2* __restrict__ refl,
                    double2* __restrict__ tau, int* __restrict__ flags, int* __restrict__ status,
    const int* __restrict__ gate) {
  hicu_pdl_entry();
  if (gate && *gate == 0) return;  // closed-form path succeeded (nsjl.cu)
  extern __shared__ double2 sh2[];
  double2* sw = sh2;           // 2 x n (double-buffered reflector w)
  double2* v = sh2 + 2 * n;    // column-major: element (k, j) at v[j*n + k]
  __shared__ double2 s_tau[2];
  __shared__ int s_act[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = threadIdx.x; e < n * r; e += blockDim.x) v[(size_t)(e % r) * n + e / r] = Vg[e];
  for (int e = threadIdx.x; e < n * r; e += blockDim.x) refl[e] = cd(0.0, 0.0);
  __syncthreads();
  if (warp == 0) hh2_reflector(n, 0, v, tol, lane, refl, tau, flags, status, &s_tau[0], &s_act[0], sw);
  __syncthreads();
  for (int col = 0; col < r; ++col) {
    const int par = col & 1;
    const double2 tv = s_tau[par];
    const double2* w = sw + (size_t)par * n;
    if (s_act[par]) {
      if (warp == 0) {
        const int j = col + 1;
        if (j < r) {
          double2 d0 = cd(0.0, 0.0);
          for (int k = col + lane; k < n; k += 32) zfmac(d0, w[k], v[(size_t)j * n + k]);
          d0 = cd(warp_sum_d_(d0.x), warp_sum_d_(d0.y));
          const double2 f0 = cmul(tv, d0);
          for (int k = col + lane; k < n; k += 32) v[(size_t)j * n + k] = v[(size_t)j * n + k] - cmul(w[k], f0);
        }
      } else {
        for (int j0 = col + 2 + (warp - 1); j0 < r; j0 += 2 * (nw - 1)) {
          const int j1 = j0 + (nw - 1);
          const bool two = j1 < r;
          double2 d0 = cd(0.0, 0.0), d1 = cd(0.0, 0.0);
          for (int k = col + lane; k < n; k += 32) {
            const double2 wk = w[k];
            zfmac(d0, wk, v[(size_t)j0 * n + k]);
            if (two) zfmac(d1, wk, v[(size_t)j1 * n + k]);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            d0.x += __shfl_xor_sync(0xffffffffu, d0.x, o);
            d0.y += __shfl_xor_sync(0xffffffffu, d0.y, o);
            d1.x += __shfl_xor_sync(0xffffffffu, d1.x, o);
            d1.y += __shfl_xor_sync(0xffffffffu, d1.y, o);
          }
          const double2 f0 = cmul(tv, d0), f1 = cmul(tv, d1);
          for (int k = col + lane; k < n; k += 32) {
            const double2 wk = w[k];
            v[(size_t)j0 * n + k] = v[(size_t)j0 * n + k] - cmul(wk, f0);
            if (two) v[(size_t)j1 * n + k] = v[(size_t)j1 * n + k] - cmul(wk, f1);
          }
        }
      }
    }
    if (warp == 0 && col + 1 < r) {
      __syncwarp();
      hh2_reflector(n, col + 1, v + (size_t)(col + 1) * n, tol, lane, refl, tau, flags, status, &s_tau[par ^ 1],
                    &s_act[par ^ 1], sw + (size_t)(par ^ 1) * n);
    }
    __syncthreads();
  }
}

// Register-staged variant of householder2 (n <= 32 PER): every per-step
// column access is one predicated batch of PER loads per lane (lane owns rows
// lane + 32u), the dot, the reduction (x and y interleaved in one shuffle
// tree) and the axpy run on registers, so a column is read once and written
// once per step; warp 0 builds reflector col+1 from the registers that hold
// the freshly updated column instead of re-reading it.  Same arithmetic as
// hh2_reflector.
template <int PER>
__device__ __forceinline__ void hh2r_build(int n, int c, double tol, int lane, const double2 (&x)[PER],
                                           double2* __restrict__ refl, double2* __restrict__ tau, int* __restrict__ flags,
                                           int* __restrict__ status, double2* s_tau, int* s_act, double2* w_next) {
  double t0 = 0.0, t1 = 0.0;
  double2 x0 = cd(0.0, 0.0);
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int k = lane + 32 * u;
    const double a = (k > c && k < n) ? abs2d(x[u]) : 0.0;
    if (u & 1) t1 += a;
    else t0 += a;
    x0 = (k == c) ? x[u] : x0;
  }
  double t = t0 + t1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  x0.x = __shfl_sync(0xffffffffu, x0.x, c & 31);
  x0.y = __shfl_sync(0xffffffffu, x0.y, c & 31);
  double2 ui = cd(0.0, 0.0);
  int active = 0;
  if (lane == 0) {
    const double tail = t;
    const double beta = sqrt(tail + x0.x * x0.x + x0.y * x0.y);
    active = 1;
    if (beta < tol) {
      *status = HICU_ERR_DEGENERATE_INPUT;
      active = 0;
    } else if (tail == 0.0 && x0.y == 0.0 && x0.x >= 0.0) {
      active = 0;
    }
    double2 u0 = cd(0.0, 0.0), tv = cd(0.0, 0.0);
    if (active) {
      if (x0.x > 0.0) {
        const double2 nume = cd(-tail, 2.0 * beta * x0.y);
        const double2 deno = cd(x0.x + beta, -x0.y);
        const double dd = abs2d(deno);
        u0 = cd((nume.x * deno.x + nume.y * deno.y) / dd, (nume.y * deno.x - nume.x * deno.y) / dd);
      } else {
        u0 = cd(x0.x - beta, x0.y);
      }
      tv = cd((beta - x0.x) / beta, x0.y / beta);
      const double uu = abs2d(u0);
      ui = cd(u0.x / uu, -u0.y / uu);
    }
    *s_tau = tv;
    *s_act = active;
    flags[c] = active;
    tau[c] = tv;
  }
  active = __shfl_sync(0xffffffffu, active, 0);
  ui.x = __shfl_sync(0xffffffffu, ui.x, 0);
  ui.y = __shfl_sync(0xffffffffu, ui.y, 0);
  if (!active) return;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int k = lane + 32 * u;
    if (k < c || k >= n) continue;
    const double2 wv = (k == c) ? cd(1.0, 0.0) : cmul(x[u], ui);
    refl[(size_t)c * n + k] = wv;
    w_next[k] = wv;
  }
}

template <int PER>
__global__ void __launch_bounds__(512)
householder2r_kernel(int n, int r, const double2* __restrict__ Vg, double tol, double2* __restrict__ refl,
                     double2* __restrict__ tau, int* __restrict__ flags, int* __restrict__ status,
    const int* __restrict__ gate) {
  hicu_pdl_entry();
  if (gate && *gate == 0) return;  // closed-form path succeeded (nsjl.cu)
  extern __shared__ double2 sh2[];
  double2* sw = sh2;           // 2 x n (double-buffered reflector w)
  double2* v = sh2 + 2 * n;    // column-major: element (k, j) at v[j*n + k]
  __shared__ double2 s_tau[2];
  __shared__ int s_act[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = threadIdx.x; e < n * r; e += blockDim.x) v[(size_t)(e % r) * n + e / r] = Vg[e];
  for (int e = threadIdx.x; e < n * r; e += blockDim.x) refl[e] = cd(0.0, 0.0);
  for (int e = threadIdx.x; e < 2 * n; e += blockDim.x) sw[e] = cd(0.0, 0.0);
  __syncthreads();
  if (warp == 0) {
    double2 x[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int k = lane + 32 * u;
      x[u] = k < n ? v[k] : cd(0.0, 0.0);
    }
    hh2r_build<PER>(n, 0, tol, lane, x, refl, tau, flags, status, &s_tau[0], &s_act[0], sw);
  }
  __syncthreads();
  for (int col = 0; col < r; ++col) {
    const int par = col & 1;
    const double2 tv = s_tau[par];
    const double2* w = sw + (size_t)par * n;
    const int act = s_act[par];
    // w_col is zero above row col (entries of the buffer below col were cleared)
    double2 wr[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int k = lane + 32 * u;
      wr[u] = (k >= col && k < n) ? w[k] : cd(0.0, 0.0);
    }
    if (warp == 0) {
      const int j = col + 1;
      if (j < r) {
        double2 x[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int k = lane + 32 * u;
          x[u] = k < n ? v[(size_t)j * n + k] : cd(0.0, 0.0);
        }
        if (act) {
          double2 d0 = cd(0.0, 0.0), d1 = cd(0.0, 0.0);
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            if (u & 1) zfmac(d1, wr[u], x[u]);
            else zfmac(d0, wr[u], x[u]);
          }
          double2 d = d0 + d1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            d.x += __shfl_xor_sync(0xffffffffu, d.x, o);
            d.y += __shfl_xor_sync(0xffffffffu, d.y, o);
          }
          const double2 f0 = cmul(tv, d);
#pragma unroll
          for (int u = 0; u < PER; ++u) x[u] = x[u] - cmul(wr[u], f0);
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int k = lane + 32 * u;
            if (k < n) v[(size_t)j * n + k] = x[u];
          }
        }
        // the entries of the other buffer below row j must read as zero
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int k = lane + 32 * u;
          if (k < j && k < n) sw[(size_t)(par ^ 1) * n + k] = cd(0.0, 0.0);
        }
        __syncwarp();
        hh2r_build<PER>(n, j, tol, lane, x, refl, tau, flags, status, &s_tau[par ^ 1], &s_act[par ^ 1],
                        sw + (size_t)(par ^ 1) * n);
      }
    } else if (act) {
      for (int j0 = col + 2 + (warp - 1); j0 < r; j0 += 2 * (nw - 1)) {
        const int j1 = j0 + (nw - 1);
        const bool two = j1 < r;
        double2 a[PER], b[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int k = lane + 32 * u;
          a[u] = k < n ? v[(size_t)j0 * n + k] : cd(0.0, 0.0);
          b[u] = (two && k < n) ? v[(size_t)j1 * n + k] : cd(0.0, 0.0);
        }
        double2 d0 = cd(0.0, 0.0), d1 = cd(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          zfmac(d0, wr[u], a[u]);
          zfmac(d1, wr[u], b[u]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          d0.x += __shfl_xor_sync(0xffffffffu, d0.x, o);
          d0.y += __shfl_xor_sync(0xffffffffu, d0.y, o);
          d1.x += __shfl_xor_sync(0xffffffffu, d1.x, o);
          d1.y += __shfl_xor_sync(0xffffffffu, d1.y, o);
        }
        const double2 f0 = cmul(tv, d0), f1 = cmul(tv, d1);
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int k = lane + 32 * u;
          if (k >= n) continue;
          v[(size_t)j0 * n + k] = a[u] - cmul(wr[u], f0);
          if (two) v[(size_t)j1 * n + k] = b[u] - cmul(wr[u], f1);
        }
      }
    }
    __syncthreads();
  }
}

// B <- H_0^H ... applied for col = r-1 .. 0: block -= conj(tau) w (w^H block).
// One warp per column of B (held in shared memory); the reflectors stream
// through shared memory in chunks so each is read from L2 once per CTA.
constexpr int kReflChunk = 8;
__global__ void apply_reflectors_kernel(int n, int r, const double2* __restrict__ refl, const double2* __restrict__ tau,
                                        const int* __restrict__ flags, int cols, const double2* __restrict__ Bin,
                                        double2* __restrict__ B, float2* __restrict__ out32, int p,
    const int* __restrict__ gate) {
  hicu_pdl_entry();
  if (gate && *gate == 0) return;  // closed-form path succeeded (nsjl.cu)
  extern __shared__ double2 sb[];
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* b = sb + (size_t)warp * n;
  double2* ws = sb + (size_t)warps * n;  // kReflChunk reflectors
  __shared__ double2 ts[kReflChunk];
  __shared__ int fs[kReflChunk];
  const int j = blockIdx.x * warps + warp;
  const bool active = j < cols;
  if (active)
    for (int k = lane; k < n; k += 32) b[k] = Bin[(size_t)k * cols + j];
  for (int c1 = r - 1; c1 >= 0; c1 -= kReflChunk) {
    const int c0 = max(0, c1 - kReflChunk + 1);
    __syncthreads();
    for (int q = threadIdx.x; q < (c1 - c0 + 1) * n; q += blockDim.x)
      ws[q] = refl[(size_t)(c0 + q / n) * n + q % n];
    for (int q = threadIdx.x; q <= c1 - c0; q += blockDim.x) {
      ts[q] = tau[c0 + q];
      fs[q] = flags[c0 + q];
    }
    __syncthreads();
    if (!active) continue;
    for (int col = c1; col >= c0; --col) {
      if (!fs[col - c0]) continue;
      const double2* w = ws + (size_t)(col - c0) * n;
      double2 dot = cd(0.0, 0.0);
      for (int k = col + lane; k < n; k += 32) zfmac(dot, w[k], b[k]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        dot.x += __shfl_xor_sync(0xffffffffu, dot.x, o);
        dot.y += __shfl_xor_sync(0xffffffffu, dot.y, o);
      }
      const double2 f = cmulc(ts[col - c0], dot);  // conj(tau) * dot
      for (int k = col + lane; k < n; k += 32) b[k] = b[k] - cmul(w[k], f);
      __syncwarp();
    }
  }
  if (!active) return;
  for (int k = lane; k < n; k += 32) {
    const double2 v = b[k];
    B[(size_t)k * cols + j] = v;
    if (out32) {
      const int step = j / p, t = j % p;
      out32[((size_t)step * n + k) * p + t] = cf((float)v.x, (float)v.y);
    }
  }
}

// Resident variant: n <= 32 * kArPer rows held in registers (res2 below).
constexpr int kArWarps = 4;
constexpr int kArPer = 8;  // n <= 256 for the resident apply

// Streaming variant (n <= 32 kArPer): each warp carries two columns of B in
// registers and reads the reflectors straight from L2 one step ahead (no
// 192 KB shared-memory staging per CTA); the two columns' dot products are
// reduced together, interleaving the x and y parts (one 5-level shuffle tree
// for four doubles instead of four sequential trees).
constexpr int kAr2Warps = 4;
__global__ void __launch_bounds__(kAr2Warps * 32)
apply_reflectors_res2_kernel(int n, int r, const double2* __restrict__ refl, const double2* __restrict__ tau,
                             const int* __restrict__ flags, int cols, const double2* __restrict__ Bin,
                             double2* __restrict__ B, float2* __restrict__ out32, int p,
    const int* __restrict__ gate) {
  hicu_pdl_entry();
  if (gate && *gate == 0) return;  // closed-form path succeeded (nsjl.cu)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = 2 * (blockIdx.x * kAr2Warps + warp);
  if (j0 >= cols) return;
  const bool two = j0 + 1 < cols;
  double2 b0[kArPer], b1[kArPer];
#pragma unroll
  for (int u = 0; u < kArPer; ++u) {
    const int k = lane + 32 * u;
    b0[u] = k < n ? Bin[(size_t)k * cols + j0] : cd(0.0, 0.0);
    b1[u] = (k < n && two) ? Bin[(size_t)k * cols + j0 + 1] : cd(0.0, 0.0);
  }
  double2 wn[kArPer];
  auto load_w = [&](int col) {
#pragma unroll
    for (int u = 0; u < kArPer; ++u) {
      const int k = lane + 32 * u;
      wn[u] = (col >= 0 && k < n) ? __ldg(refl + (size_t)col * n + k) : cd(0.0, 0.0);  // zero above col
    }
  };
  load_w(r - 1);
  for (int col = r - 1; col >= 0; --col) {
    double2 wr[kArPer];
#pragma unroll
    for (int u = 0; u < kArPer; ++u) wr[u] = wn[u];
    load_w(col - 1);  // next reflector in flight while this one is applied
    const int act = __ldg(flags + col);
    if (!act) continue;
    double2 d0 = cd(0.0, 0.0), d1 = cd(0.0, 0.0), e0 = cd(0.0, 0.0), e1 = cd(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < kArPer; u += 2) {
      zfmac(d0, wr[u], b0[u]);
      zfmac(e0, wr[u], b1[u]);
      if (u + 1 < kArPer) {
        zfmac(d1, wr[u + 1], b0[u + 1]);
        zfmac(e1, wr[u + 1], b1[u + 1]);
      }
    }
    double2 d = d0 + d1, e = e0 + e1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      d.x += __shfl_xor_sync(0xffffffffu, d.x, o);
      d.y += __shfl_xor_sync(0xffffffffu, d.y, o);
      e.x += __shfl_xor_sync(0xffffffffu, e.x, o);
      e.y += __shfl_xor_sync(0xffffffffu, e.y, o);
    }
    const double2 tc = __ldg(tau + col);
    const double2 f = cmulc(tc, d), g = cmulc(tc, e);  // conj(tau) * dot
#pragma unroll
    for (int u = 0; u < kArPer; ++u) {
      b0[u] = b0[u] - cmul(wr[u], f);
      b1[u] = b1[u] - cmul(wr[u], g);
    }
  }
#pragma unroll
  for (int u = 0; u < kArPer; ++u) {
    const int k = lane + 32 * u;
    if (k >= n) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = j0 + h;
      if (h == 1 && !two) continue;
      const double2 v = h ? b1[u] : b0[u];
      B[(size_t)k * cols + j] = v;
      if (out32) {
        const int step = j / p, t = j % p;
        out32[((size_t)step * n + k) * p + t] = cf((float)v.x, (float)v.y);
      }
    }
  }
}

struct NysWs {
  double2 *Y, *O, *C, *W, *M, *scratch, *F;
  void* heev;
  double* evals;
  double* nu;
  int* order;
  int* nrounds;
  RotEntry* log;
  size_t bytes;
};

constexpr int kMaxSweeps = 30;

NysWs nystrom_layout(int n, int ell, char* base) {
  NysWs w;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? base + off : nullptr;
    off += (bytes + 255) & ~(size_t)255;
    return p;
  };
  const int m = ell + (ell & 1);
  w.Y = (double2*)take((size_t)n * ell * sizeof(double2));
  w.O = (double2*)take((size_t)ell * ell * sizeof(double2));
  w.C = (double2*)take((size_t)ell * ell * sizeof(double2));
  w.W = (double2*)take((size_t)n * ell * sizeof(double2));
  w.M = (double2*)take((size_t)ell * ell * sizeof(double2));
  w.scratch = (double2*)take((size_t)ell * ell * sizeof(double2));
  w.evals = (double*)take((size_t)ell * sizeof(double));
  w.nu = (double*)take(sizeof(double));
  w.order = (int*)take((size_t)ell * sizeof(int));
  w.nrounds = (int*)take(sizeof(int));
  w.log = (RotEntry*)take((size_t)kMaxSweeps * (m - 1) * (m / 2) * sizeof(RotEntry));
  w.F = (double2*)take((size_t)ell * ell * sizeof(double2));
  w.heev = (void*)take(hicu_heev_top_workspace(ell, ell));
  w.bytes = off;
  return w;
}

}  // namespace

extern "C" int hicu_zgemm(char opa, char opb, int m, int n, int k, const void* A, int lda, const void* B, int ldb,
                          void* C, int ldc, void* stream) {
  if (!A || !B || !C || m < 1 || n < 1 || k < 1) return hicu_set_error(HICU_ERR_PARAMETER, "zgemm: bad arguments");
  if ((opa != 'N' && opa != 'C') || (opb != 'N' && opb != 'C'))
    return hicu_set_error(HICU_ERR_PARAMETER, "zgemm: op must be N or C");
  return zgemm_launch(opa, opb, m, n, k, (const double2*)A, lda, (const double2*)B, ldb, (double2*)C, ldc,
                      (cudaStream_t)stream);
}

extern "C" size_t hicu_nystrom_workspace(int n, int ell) { return nystrom_layout(n, ell, nullptr).bytes; }

extern "C" int hicu_nystrom(int n, int ell, int r, const void* G, const void* omega, void* V, void* ws,
                            size_t ws_bytes, int* status_dev, void* stream) {
  if (!(1 <= r && r < n)) return hicu_set_error(HICU_ERR_PARAMETER, "nystrom: rank must satisfy 1 <= r < n");
  if (ell < r || ell > 256) return hicu_set_error(HICU_ERR_PARAMETER, "nystrom: sketch width out of range");
  if (!G || !omega || !V || !ws || !status_dev) return hicu_set_error(HICU_ERR_PARAMETER, "nystrom: null pointer");
  NysWs w = nystrom_layout(n, ell, (char*)ws);
  if (ws_bytes < w.bytes) return hicu_set_error(HICU_ERR_WORKSPACE, "nystrom: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  auto Gp = (const double2*)G;
  auto Om = (const double2*)omega;
  int s;
  if ((s = zgemm_launch('N', 'N', n, ell, n, Gp, n, Om, ell, w.Y, ell, st))) return s;
  if ((s = zgemm_launch('C', 'N', ell, ell, n, Om, ell, w.Y, ell, w.C, ell, st))) return s;
  if ((s = zgemm_launch('C', 'N', ell, ell, n, Om, ell, Om, ell, w.O, ell, st))) return s;
  {
    const size_t bytes = (size_t)ell * ell * sizeof(double2);
    const bool sm = bytes <= kSmemCap;
    if (ell <= 96) {
      auto args = [&](auto kern) {
        hicu_launch(kern, 1, 512, 0, st, ell, w.C, (const double2*)w.O, Gp, n, w.nu, status_dev);
      };
      if (ell <= 16) args(chol2_kernel<1, 1>);
      else if (ell <= 32) args(chol2_kernel<1, 2>);
      else if (ell <= 48) args(chol2_kernel<2, 3>);
      else if (ell <= 64) args(chol2_kernel<2, 4>);
      else if (ell <= 80) args(chol2_kernel<3, 5>);
      else args(chol2_kernel<3, 6>);
    } else if (sm) {
      hicu_allow_max_smem((const void*)chol_kernel<true>);
      hicu_launch(chol_kernel<true>, 1, 512, bytes, st, ell, w.C, w.O, Gp, n, w.scratch, w.nu, status_dev);
    } else if (ell <= kCcMaxL) {
      const size_t csm = (size_t)((ell + kCcCS - 1) / kCcCS) * ell * sizeof(double2);
      hicu_allow_max_smem((const void*)chol_cluster_kernel);
      hicu_launch(chol_cluster_kernel, kCcCS, kCcThreads, csm, st, ell, w.C, (const double2*)w.O, Gp, n, w.nu,
                  status_dev);
    } else {
      hicu_launch(chol_kernel<false>, 1, 512, 0, st, ell, w.C, w.O, Gp, n, w.scratch, w.nu, status_dev);
    }
    if ((s = hicu_check_launch("chol_kernel"))) return s;
  }
  {
    const size_t rbytes = (size_t)ell * ell * sizeof(double2);
    if (rbytes + (size_t)ell * sizeof(double) <= kSmemCap) {
      trsm_rl_launch<1>(n, ell, w.Y, Om, w.nu, w.C, w.W, rbytes + (size_t)ell * sizeof(double), st);
      if ((s = hicu_check_launch("trsm_rl_kernel"))) return s;
    } else if (ell <= 32 * kTrsmMaxPer) {
      trsm_rls_launch<4>(n, ell, w.Y, Om, w.nu, w.C, w.W, st);
      if ((s = hicu_check_launch("trsm_rls_kernel"))) return s;
    } else {
    const int warps = 8;
    const size_t rowb = (size_t)warps * ell * sizeof(double2);
    const bool sm = rbytes + rowb <= kSmemCap;
    const size_t smem = (sm ? rbytes : 0) + rowb;
    hicu_allow_max_smem((const void*)trsm_rows_kernel);
    const int blocks = (n + warps - 1) / warps;
    hicu_launch(trsm_rows_kernel, blocks, warps * 32, smem, st, n, ell, w.Y, Om, w.nu, w.C, sm, w.W);
    if ((s = hicu_check_launch("trsm_rows_kernel"))) return s;
    }
  }
  if ((s = zgemm_launch('C', 'N', ell, ell, n, w.W, ell, w.W, ell, w.M, ell, st))) return s;
  // top-r eigenpairs of M = W^H W (tridiagonal + bisection + inverse iteration)
  if ((s = hicu_heev_top(ell, r, w.M, w.evals, w.F, w.heev, st))) return s;
  // V = W F Lambda^{-1/2}
  if ((s = zgemm_launch('N', 'N', n, r, ell, w.W, ell, w.F, r, (double2*)V, r, st))) return s;
  hicu_launch(canon_phase_kernel, (r + 7) / 8, 256, 0, st, n, r, (double2*)V, w.evals, status_dev);
  if ((s = hicu_check_launch("canon_phase_kernel"))) return s;
  return HICU_OK;
}

int hicu_householder_gated(int n, int r, const void* V, double tol, void* refl, void* tau, int* flags,
                           int* status_dev, const int* gate, void* stream) {
  if (r < 0 || r > n || !refl || !tau || !flags || !status_dev)
    return hicu_set_error(HICU_ERR_DEGENERATE_INPUT, "householder: bad arguments");
  if (r == 0) return HICU_OK;
  if (!V) return hicu_set_error(HICU_ERR_PARAMETER, "householder: null V");
  const size_t bytes = (size_t)n * r * sizeof(double2);
  const bool sm = bytes + (size_t)n * sizeof(double2) <= kSmemCap;
  void* gws = nullptr;
  if (!sm) {
    // large V: work in place in the caller's refl buffer is not possible (different layout);
    // require the caller to size refl at 2*n*r and use its upper half as scratch.
    gws = (double2*)refl + (size_t)n * r;
  }
  if (bytes + (size_t)2 * n * sizeof(double2) <= kSmemCap && n <= 256) {
    const size_t sm2 = bytes + (size_t)2 * n * sizeof(double2);
    auto go = [&](auto kern) {
      hicu_allow_max_smem((const void*)kern);
      hicu_launch(kern, 1, 512, sm2, (cudaStream_t)stream, n, r, (const double2*)V, tol, (double2*)refl, (double2*)tau,
                  flags, status_dev, gate);
    };
    if (n <= 128) go(householder2r_kernel<4>);
    else if (n <= 192) go(householder2r_kernel<6>);
    else go(householder2r_kernel<8>);
    return hicu_check_launch("householder2r_kernel");
  }
  if (bytes + (size_t)2 * n * sizeof(double2) <= kSmemCap) {
    hicu_allow_max_smem((const void*)householder2_kernel);
    // 512 threads: 32 us faster than 1024 (less MIO contention on warp 0)
    hicu_launch(householder2_kernel, 1, 512, bytes + (size_t)2 * n * sizeof(double2), (cudaStream_t)stream, 
        n, r, (const double2*)V, tol, (double2*)refl, (double2*)tau, flags, status_dev, gate);
    return hicu_check_launch("householder2_kernel");
  }
  hicu_allow_max_smem((const void*)householder_kernel);
  hicu_launch(householder_kernel, 1, 1024, (sm ? bytes : 0) + (size_t)n * sizeof(double2), (cudaStream_t)stream, 
      n, r, (const double2*)V, tol, (double2*)gws, sm, (double2*)refl, (double2*)tau, flags, status_dev, gate);
  return hicu_check_launch("householder_kernel");
}

int hicu_apply_reflectors_gated(int n, int r, const void* refl, const void* tau, const int* flags, int cols,
                                const void* Bin, void* B, void* out32, int p, const int* gate, void* stream) {
  if (n < 1 || r < 0 || cols < 1 || !B || !Bin) return hicu_set_error(HICU_ERR_PARAMETER, "apply_reflectors: bad arguments");
  if (out32 && (p < 1 || cols % p != 0)) return hicu_set_error(HICU_ERR_PARAMETER, "apply_reflectors: bad p");
  if (r >= 1 && n <= 32 * kArPer) {
    const int pairs = (cols + 1) / 2;
    hicu_launch(apply_reflectors_res2_kernel, (pairs + kAr2Warps - 1) / kAr2Warps, kAr2Warps * 32, 0,
                (cudaStream_t)stream, n, r, (const double2*)refl, (const double2*)tau, flags, cols,
                (const double2*)Bin, (double2*)B, (float2*)out32, p ? p : 1, gate);
    return hicu_check_launch("apply_reflectors_res2_kernel");
  }
  int warps = 8;
  while (warps > 1 && (size_t)(warps + kReflChunk) * n * sizeof(double2) > kSmemCap) warps >>= 1;
  const size_t smem = (size_t)(warps + kReflChunk) * n * sizeof(double2);
  if (smem > kSmemCap) return hicu_set_error(HICU_ERR_SIZE, "apply_reflectors: n too large");
  hicu_allow_max_smem((const void*)apply_reflectors_kernel);
  const int blocks = (cols + warps - 1) / warps;
  hicu_launch(apply_reflectors_kernel, blocks, warps * 32, smem, (cudaStream_t)stream, 
      n, r, (const double2*)refl, (const double2*)tau, flags, cols, (const double2*)Bin, (double2*)B, (float2*)out32,
      p ? p : 1, gate);
  return hicu_check_launch("apply_reflectors_kernel");
}

extern "C" int hicu_householder(int n, int r, const void* V, double tol, void* refl, void* tau, int* flags,
                                int* status_dev, void* stream) {
  return hicu_householder_gated(n, r, V, tol, refl, tau, flags, status_dev, nullptr, stream);
}

extern "C" int hicu_apply_reflectors(int n, int r, const void* refl, const void* tau, const int* flags, int cols,
                                     const void* Bin, void* B, void* out32, int p, void* stream) {
  return hicu_apply_reflectors_gated(n, r, refl, tau, flags, cols, Bin, B, out32, p, nullptr, stream);
}

// ---------------------------------------------------------------------------
// SVD coil compression basis (no reference function):
// eigenvectors of the nc x nc coil covariance by the same Jacobi kernel,
// columns sorted by decreasing eigenvalue, phase fixed so the
// largest-magnitude entry (first on ties) is real positive.
// ---------------------------------------------------------------------------
namespace {

__global__ void eye_kernel(int n, double2* __restrict__ I) {
  hicu_pdl_entry();
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x)
    I[e] = cd((e / n) == (e % n) ? 1.0 : 0.0, 0.0);
}

__global__ void coil_phase_kernel(int nc, int nv, const double2* __restrict__ E, const double* __restrict__ evals,
                                  const int* __restrict__ order, double2* __restrict__ basis,
                                  double* __restrict__ evals_out) {
  hicu_pdl_entry();
  const int j = threadIdx.x;
  if (j >= nc) return;
  int best = 0;
  double bm = -1.0;
  for (int i = 0; i < nc; ++i) {
    const double a = abs2d(E[(size_t)i * nc + j]);
    if (a > bm) { bm = a; best = i; }
  }
  const double2 e = E[(size_t)best * nc + j];
  const double mag = sqrt(abs2d(e));
  const double2 ph = mag > 0.0 ? cd(e.x / mag, e.y / mag) : cd(1.0, 0.0);
  if (j < nv) {
    for (int i = 0; i < nc; ++i) basis[(size_t)i * nv + j] = cmulc(ph, E[(size_t)i * nc + j]);  // E / ph
  }
  if (evals_out) evals_out[j] = evals[order[j]];
}

}  // namespace

extern "C" size_t hicu_coil_basis_workspace(int nc) {
  return nystrom_layout(nc, nc, nullptr).bytes + 2 * (size_t)nc * nc * sizeof(double2) + 512;
}

extern "C" int hicu_coil_basis(int nc, int nv, const void* cov, void* basis, double* evals, void* ws,
                               size_t ws_bytes, void* stream) {
  if (nc < 1 || nc > 32 || nv < 1 || nv > nc || !cov || !basis || !ws)
    return hicu_set_error(HICU_ERR_PARAMETER, "coil_basis: bad arguments");
  if (ws_bytes < hicu_coil_basis_workspace(nc)) return hicu_set_error(HICU_ERR_WORKSPACE, "coil_basis: workspace");
  NysWs w = nystrom_layout(nc, nc, (char*)ws);
  char* extra = (char*)ws + ((w.bytes + 255) & ~(size_t)255);
  double2* I = (double2*)extra;
  double2* E = I + (size_t)nc * nc;
  int* status = (int*)(E + (size_t)nc * nc);
  cudaStream_t st = (cudaStream_t)stream;
  int s;
  hicu_launch(eye_kernel, 1, 256, 0, st, nc, I);
  if ((s = hicu_check_launch("eye_kernel"))) return s;
  const size_t bytes = (size_t)nc * nc * sizeof(double2);
  hicu_allow_max_smem((const void*)jacobi_kernel);
  hicu_launch(jacobi_kernel, 1, 1024, bytes, st, nc, (const double2*)cov, w.scratch, true, kMaxSweeps, 1e-15, w.log,
                                        w.nrounds, w.evals, w.order, status);
  if ((s = hicu_check_launch("jacobi_kernel"))) return s;
  // E = I J with columns in descending-eigenvalue order (no scaling)
  hicu_launch(rot_apply_kernel, 1, 32 * 8, (size_t)8 * nc * sizeof(double2), st, nc, nc, nc, I, w.log, w.nrounds, w.evals,
                                                                       w.order, E, nullptr, false);
  if ((s = hicu_check_launch("rot_apply_kernel"))) return s;
  // E columns are already in descending order; identity order for the phase step
  hicu_launch(coil_phase_kernel, 1, 32, 0, st, nc, nv, E, w.evals, w.order, (double2*)basis, evals);
  return hicu_check_launch("coil_phase_kernel");
}
