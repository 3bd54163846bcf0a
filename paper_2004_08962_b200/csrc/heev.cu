// Top-r eigenpairs of a small Hermitian PSD matrix M (l x l, l <= 256) for the
// nullspace step: Householder tridiagonalisation (the zhetd2 recurrence),
// warp-parallel multisection bisection on the real tridiagonal (Sturm
// counts), inverse iteration per eigenvalue, cluster re-orthogonalisation
// and the back-transform through the reflectors.  Replaces the cyclic Jacobi
// sweep in the Nystrom path: O(l^3) work in l sequential steps instead of
// ~10 sweeps x (l-1) rounds of smem-bound rotations.
//
// Used by hicu_nystrom (dense.cu); no reference function (the reference
// gets its singular vectors from LAPACK zgesdd, subspace.py:150).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cooperative_groups.h>

#include "common.cuh"

namespace {

__device__ __forceinline__ double warp_sum_d(double t) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}
__device__ __forceinline__ double2 warp_sum_z(double2 t) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
    t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
  }
  return t;
}

// Householder reduction A = Q T Q^H (lower), one CTA of 1024 threads.
// Outputs d (l), e (l-1), tau (l-1) and the reflectors transposed:
// Vt[k*l + i] = v_k[i] (v_k[k+1] = 1).  A is held with leading dimension
// l+1 so column walks (lanes over rows) are bank-conflict free; the
// matrix-vector product is row-parallel with j-chunk partials in shared memory
// (no per-row shuffle reductions on the sequential critical path).
template <bool SMEM>
__global__ void __launch_bounds__(1024)
hetrd_kernel(int l, const double2* __restrict__ Ain, double2* __restrict__ Aws,
             double* __restrict__ d, double* __restrict__ e, double2* __restrict__ tau,
             double2* __restrict__ Vt) {
  hicu_pdl_entry();
  extern __shared__ double2 sA[];
  double2* A = SMEM ? sA : Aws;
  const int lda = l + 1;
  __shared__ double2 sv[256], sw[256];
  __shared__ double2 part[4][256];
  __shared__ double redd[32];
  __shared__ double2 redz[32];
  __shared__ double2 s_tau, s_scal, s_alpha2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
  for (int q = tid; q < l * l; q += nt) A[(size_t)(q / l) * lda + q % l] = Ain[q];
  for (int q = tid; q < l * l; q += nt) Vt[q] = cd(0.0, 0.0);
  __syncthreads();
  for (int k = 0; k + 1 < l; ++k) {
    const int k1 = k + 1, m = l - k1;
    // ---- column norm of A[k+2:, k] (warp 0, smem partials) and the reflector ----
    if (warp == 0) {
      double t = 0.0;
      for (int i = k + 2 + lane; i < l; i += 32) t += abs2d(A[(size_t)i * lda + k]);
      redd[lane] = t;
      __syncwarp();
      if (lane == 0) {
        double tt = 0.0;
        for (int q = 0; q < 32; ++q) tt += redd[q];
        const double2 alpha = A[(size_t)k1 * lda + k];
        double2 tv = cd(0.0, 0.0), scal = cd(0.0, 0.0);
        double beta;
        if (tt == 0.0 && alpha.y == 0.0) {
          beta = alpha.x;  // H = I
        } else {
          beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + tt), alpha.x);
          const double ib = 1.0 / beta;
          tv = cd((beta - alpha.x) * ib, -alpha.y * ib);
          const double2 den = cd(alpha.x - beta, alpha.y);
          const double idd = 1.0 / abs2d(den);
          scal = cd(den.x * idd, -den.y * idd);  // 1 / (alpha - beta)
        }
        e[k] = beta;
        d[k] = A[(size_t)k * lda + k].x;
        tau[k] = tv;
        s_tau = tv;
        s_scal = scal;
      }
    }
    __syncthreads();
    const double2 tk = s_tau;
    const double2 sc = s_scal;
    for (int i = k1 + tid; i < l; i += nt) {
      const double2 v = (i == k1) ? cd(1.0, 0.0) : cmul(A[(size_t)i * lda + k], sc);
      sv[i] = v;
      Vt[(size_t)k * l + i] = v;
    }
    __syncthreads();
    if (tk.x == 0.0 && tk.y == 0.0) continue;  // uniform
    // ---- y = A22 v: thread (row, chunk), 4 chunks over j ----
    {
      const int nchunk = 4, rows_per = nt / nchunk;  // nt/4 rows per pass
      const int c = tid / rows_per, rr = tid % rows_per;
      const int clen = (m + nchunk - 1) / nchunk;
      const int j0 = k1 + c * clen, j1 = min(l, j0 + clen);
      for (int i = k1 + rr; i < l; i += rows_per) {
        // four independent chains: with A in global memory (l > ~110) each
        // step streams A22 from L2, and one chain kept one load in flight
        double2 a0 = cd(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
        const double2* Ai = A + (size_t)i * lda;
        int j = j0;
        for (; j + 3 < j1; j += 4) {
          const double2 x0 = Ai[j], x1 = Ai[j + 1], x2 = Ai[j + 2], x3 = Ai[j + 3];
          zfma(a0, x0, sv[j]);
          zfma(a1, x1, sv[j + 1]);
          zfma(a2, x2, sv[j + 2]);
          zfma(a3, x3, sv[j + 3]);
        }
        for (; j < j1; ++j) zfma(a0, Ai[j], sv[j]);
        part[c][i] = (a0 + a1) + (a2 + a3);
      }
    }
    __syncthreads();
    // ---- w = tau * y; alpha2 = -tau/2 (w^H v) ----
    {
      double2 pz = cd(0.0, 0.0);
      for (int i = k1 + tid; i < l; i += nt) {
        const double2 y = part[0][i] + part[1][i] + part[2][i] + part[3][i];
        const double2 wv = cmul(tk, y);
        sw[i] = wv;
        zfmac(pz, wv, sv[i]);
      }
      pz = warp_sum_z(pz);
      if (lane == 0) redz[warp] = pz;
    }
    __syncthreads();
    if (tid == 0) {
      double2 dot = cd(0.0, 0.0);
      for (int q = 0; q < (nt >> 5); ++q) dot = dot + redz[q];
      const double2 td = cmul(tk, dot);
      s_alpha2 = cd(-0.5 * td.x, -0.5 * td.y);
    }
    __syncthreads();
    // ---- A22 -= v w'^H + w' v^H with w' = w + alpha2 v (formed on the fly) ----
    const double2 a2 = s_alpha2;
    for (int i = k1 + warp; i < l; i += nt / 32) {
      const double2 vi = sv[i];
      const double2 wi = sw[i] + cmul(a2, vi);
      double2* Ai = A + (size_t)i * lda;
#pragma unroll 4
      for (int j = k1 + lane; j < l; j += 32) {
        const double2 vj = sv[j];
        const double2 wj = sw[j] + cmul(a2, vj);
        Ai[j] = Ai[j] - cmul(vi, conjd(wj)) - cmul(wi, conjd(vj));
      }
    }
    __syncthreads();
  }
  if (tid == 0) d[l - 1] = A[(size_t)(l - 1) * lda + (l - 1)].x;
}

// Householder tridiagonalisation on a thread-block cluster (l in (96, 256]:
// the C3 / C4 / C5 nullspace, l = 150 / 225 / 180).  One cluster of kHcCS
// CTAs holds the matrix in distributed shared memory: row i lives in CTA
// i % kHcCS (cyclic, so the shrinking trailing block stays balanced), at
// most 32 rows x (l + 1) per CTA.  Per step k: the owner of row k forms the
// reflector from conj(row k) (the matrix is Hermitian and both triangles are
// updated) and writes v and tau into every CTA's shared memory; after a
// cluster barrier each CTA forms y = A22 v for its rows, w = tau y, and
// writes its w entries and its w^H v partial into every CTA; after a second
// barrier each CTA updates its rows with the rank-2 term.  v, w, tau and the
// partials are double-buffered by step parity, so a CTA still updating step k
// never sees step k + 1's broadcasts.  Two cluster barriers per step instead
// of the single-CTA kernel's L2 round trips over A22 (hetrd_kernel<false>
// streams the whole trailing block from L2 twice per step).  Same outputs as
// hetrd_kernel: d, e, tau, Vt.
constexpr int kHcCS = 8;
constexpr int kHcThreads = 512;
constexpr int kHcMaxL = 256;

__global__ void __cluster_dims__(kHcCS, 1, 1) __launch_bounds__(kHcThreads, 1)
hetrd_cluster_kernel(int l, const double2* __restrict__ Ain, double* __restrict__ d, double* __restrict__ e,
                     double2* __restrict__ tau, double2* __restrict__ Vt) {
  hicu_pdl_entry();
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  extern __shared__ double2 hcA[];  // [nr][lda]
  __shared__ double2 sv[2][kHcMaxL], sw[2][kHcMaxL];
  __shared__ double2 pdot[2][kHcCS];
  __shared__ double2 s_tau[2], s_scal;
  __shared__ double2 redz[kHcThreads / 32];
  const int lda = l + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = kHcThreads / 32;
  const int nr = (l - cr + kHcCS - 1) / kHcCS;  // rows of this CTA: i = cr + kHcCS * r
  for (int q = tid; q < nr * l; q += kHcThreads) {
    const int r = q / l, j = q - r * l;
    hcA[(size_t)r * lda + j] = Ain[(size_t)(cr + kHcCS * r) * l + j];
  }
  for (int q = cr * kHcThreads + tid; q < l * l; q += kHcCS * kHcThreads) Vt[q] = cd(0.0, 0.0);
  cluster.sync();
  // (a) the owner of row kk forms reflector kk from conj(row kk) and broadcasts v, tau into the
  // buffers of parity kk & 1; called by every thread of the owner CTA (row kk is final and visible)
  auto build_reflector = [&](int kk) {
    const int nb = kk & 1, kk1 = kk + 1, mm = l - kk1;
    const double2* row = hcA + (size_t)(kk / kHcCS) * lda;
    if (warp == 0) {
      double t = 0.0;
      for (int j = kk + 2 + lane; j < l; j += 32) t += abs2d(row[j]);
      t = warp_sum_d(t);
      if (lane == 0) {
        const double2 alpha = conjd(row[kk1]);
        double2 tv = cd(0.0, 0.0), scal = cd(0.0, 0.0);
        double beta;
        if (t == 0.0 && alpha.y == 0.0) {
          beta = alpha.x;  // H = I
        } else {
          beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + t), alpha.x);
          const double ib = 1.0 / beta;
          tv = cd((beta - alpha.x) * ib, -alpha.y * ib);
          const double2 den = cd(alpha.x - beta, alpha.y);
          const double idd = 1.0 / abs2d(den);
          scal = cd(den.x * idd, -den.y * idd);  // 1 / (alpha - beta)
        }
        e[kk] = beta;
        d[kk] = row[kk].x;
        tau[kk] = tv;
        s_scal = scal;
        for (int c = 0; c < kHcCS; ++c) *cluster.map_shared_rank(&s_tau[nb], c) = tv;
      }
    }
    __syncthreads();
    const double2 sc = s_scal;
    for (int q = tid; q < kHcCS * mm; q += kHcThreads) {
      const int c = q / mm, j = kk1 + (q - c * mm);
      const double2 v = j == kk1 ? cd(1.0, 0.0) : cmul(conjd(row[j]), sc);
      *cluster.map_shared_rank(&sv[nb][j], c) = v;
      if (c == 0) Vt[(size_t)kk * l + j] = v;
    }
  };
  // Split cluster barrier: every CTA arrives as soon as it has nothing more to publish for the
  // next step (the next owner: after broadcasting the next reflector) and waits only when it
  // needs that reflector, so the rank-2 update of the other rows runs under the barrier.
  auto arrive = [] { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); };
  auto wait = [] { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); };
  if (l > 1) {
    if (cr == 0) build_reflector(0);
    arrive();
  }
  for (int k = 0; k + 1 < l; ++k) {
    const int buf = k & 1, k1 = k + 1;
    const bool more = k1 + 1 < l;  // reflector k + 1 exists
    wait();                        // v, tau of step k everywhere
    const double2 tk = s_tau[buf];
    if (tk.x == 0.0 && tk.y == 0.0) {  // H = I (uniform over the cluster): nothing to update
      if (more) {
        __syncthreads();  // row k + 1 was last updated by another warp (the wait above orders arrivals only)
        if (cr == k1 % kHcCS) build_reflector(k1);
        arrive();
      }
      continue;
    }
    // ---- (b) y = A22 v for this CTA's rows, w = tau y, broadcast w and w^H v ----
    double2 pz = cd(0.0, 0.0);
    for (int r = warp; r < nr; r += nw) {
      const int i = cr + kHcCS * r;
      if (i < k1) continue;
      const double2* Ai = hcA + (size_t)r * lda;
      double2 a0 = cd(0.0, 0.0), a1 = a0;
      int j = k1 + lane;
      for (; j + 32 < l; j += 64) {
        zfma(a0, Ai[j], sv[buf][j]);
        zfma(a1, Ai[j + 32], sv[buf][j + 32]);
      }
      if (j < l) zfma(a0, Ai[j], sv[buf][j]);
      const double2 y = warp_sum_z(a0 + a1);
      const double2 wv = cmul(tk, y);
      if (lane < kHcCS) *cluster.map_shared_rank(&sw[buf][i], lane) = wv;
      if (lane == 0) zfmac(pz, wv, sv[buf][i]);
    }
    if (lane == 0) redz[warp] = pz;
    __syncthreads();
    if (warp == 0) {
      double2 t = lane < nw ? redz[lane] : cd(0.0, 0.0);
      t = warp_sum_z(t);
      if (lane < kHcCS) *cluster.map_shared_rank(&pdot[buf][cr], lane) = t;
    }
    cluster.sync();  // w and the partials everywhere
    // ---- (c) rank-2 update of this CTA's rows: A22 -= v w'^H + w' v^H, w' = w + alpha2 v ----
    double2 dot = cd(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < kHcCS; ++c) dot = dot + pdot[buf][c];
    const double2 td = cmul(tk, dot);
    const double2 a2 = cd(-0.5 * td.x, -0.5 * td.y);
    // the next pivot row first (one element per thread), then its reflector, then the barrier arrival
    const int rnext = (more && cr == k1 % kHcCS) ? k1 / kHcCS : -1;
    if (more) {
      if (rnext >= 0) {
        const double2 vi = sv[buf][k1];
        const double2 wi = sw[buf][k1] + cmul(a2, vi);
        double2* Ai = hcA + (size_t)rnext * lda;
        for (int j = k1 + tid; j < l; j += kHcThreads) {
          const double2 vj = sv[buf][j];
          const double2 wj = sw[buf][j] + cmul(a2, vj);
          Ai[j] = Ai[j] - cmul(vi, conjd(wj)) - cmul(wi, conjd(vj));
        }
        __syncthreads();
        build_reflector(k1);
      }
      arrive();
    }
    for (int r = warp; r < nr; r += nw) {
      const int i = cr + kHcCS * r;
      if (i < k1 || r == rnext) continue;
      const double2 vi = sv[buf][i];
      const double2 wi = sw[buf][i] + cmul(a2, vi);
      double2* Ai = hcA + (size_t)r * lda;
      for (int j = k1 + lane; j < l; j += 32) {
        const double2 vj = sv[buf][j];
        const double2 wj = sw[buf][j] + cmul(a2, vj);
        Ai[j] = Ai[j] - cmul(vi, conjd(wj)) - cmul(wi, conjd(vj));
      }
    }
  }
  __syncthreads();
  if (cr == (l - 1) % kHcCS && tid == 0) d[l - 1] = hcA[(size_t)((l - 1) / kHcCS) * lda + (l - 1)].x;
  cluster.sync();  // no CTA exits while others may still write into its shared memory
}

// Latency-oriented variant for l <= kHetrd2Max (A resident in shared memory):
// two block barriers per step.  Phase B: warp-per-row matvec y = A22 v with
// batched shuffle reductions (the rows of one warp reduce together so their
// shuffle chains overlap), w = tau y and the w^H v partials.  Phase D: the
// rank-2 update; warp 0 owns the next pivot row k+1 and builds the next
// reflector right after updating it (norm by shuffles, v written into the
// other half of a double-buffered smem vector).  The reflector uses row k
// (A[k][j] = conj(A[j][k]), both triangles are kept).
constexpr int kHetrd2Max = 110;
constexpr int kHetrd2Rows = 8;  // rows per warp in phase B (16 warps x 8 >= kHetrd2Max)

__device__ __forceinline__ void hetrd2_reflector(int l, int k, const double2* A, int lda, int lane, double* d,
                                                 double* e, double2* tau, double2* s_tau, double2* sv_next) {
  // x = column k below the diagonal = conj(row k), alpha = x[k+1]
  double t = 0.0;
  for (int j = k + 2 + lane; j < l; j += 32) t += abs2d(A[(size_t)k * lda + j]);
  t = warp_sum_d(t);
  double2 tv = cd(0.0, 0.0), scal = cd(0.0, 0.0);
  double beta = 0.0;
  if (lane == 0) {
    const double2 alpha = conjd(A[(size_t)k * lda + k + 1]);
    if (t == 0.0 && alpha.y == 0.0) {
      beta = alpha.x;  // H = I
    } else {
      beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + t), alpha.x);
      const double ib = 1.0 / beta;
      tv = cd((beta - alpha.x) * ib, -alpha.y * ib);
      const double2 den = cd(alpha.x - beta, alpha.y);
      const double idd = 1.0 / abs2d(den);
      scal = cd(den.x * idd, -den.y * idd);  // 1 / (alpha - beta)
    }
    e[k] = beta;
    d[k] = A[(size_t)k * lda + k].x;
    tau[k] = tv;
    *s_tau = tv;
  }
  scal.x = __shfl_sync(0xffffffffu, scal.x, 0);
  scal.y = __shfl_sync(0xffffffffu, scal.y, 0);
  for (int j = k + 1 + lane; j < l; j += 32)
    sv_next[j] = (j == k + 1) ? cd(1.0, 0.0) : cmul(conjd(A[(size_t)k * lda + j]), scal);
}

__global__ void __launch_bounds__(512)
hetrd2_kernel(int l, const double2* __restrict__ Ain, double* __restrict__ d, double* __restrict__ e,
              double2* __restrict__ tau, double2* __restrict__ Vt) {
  hicu_pdl_entry();
  extern __shared__ double2 A[];
  const int lda = l + 1;
  __shared__ double2 sv[2][kHetrd2Max + 2], sw[kHetrd2Max + 2];
  __shared__ double2 redz[16];
  __shared__ double2 s_tau[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = 16;
  for (int q = tid; q < l * l; q += 512) A[(size_t)(q / l) * lda + q % l] = Ain[q];
  for (int q = tid; q < l * l; q += 512) Vt[q] = cd(0.0, 0.0);
  __syncthreads();
  if (warp == 0 && l > 1) hetrd2_reflector(l, 0, A, lda, lane, d, e, tau, &s_tau[0], sv[0]);
  __syncthreads();
  for (int k = 0; k + 1 < l; ++k) {
    const int k1 = k + 1, par = k & 1;
    const double2 tk = s_tau[par];
    const bool active = !(tk.x == 0.0 && tk.y == 0.0);
    const double2* v = sv[par];
    // ---- phase B: y = A22 v (warp per row, batched reductions), w = tau y, w^H v ----
    if (active) {
      double2 acc[kHetrd2Rows];
#pragma unroll
      for (int q = 0; q < kHetrd2Rows; ++q) {
        acc[q] = cd(0.0, 0.0);
        const int i = k1 + warp + q * nw;
        if (i < l) {
          const double2* Ai = A + (size_t)i * lda;
          for (int j = k1 + lane; j < l; j += 32) zfma(acc[q], Ai[j], v[j]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < kHetrd2Rows; ++q) {
          acc[q].x += __shfl_xor_sync(0xffffffffu, acc[q].x, o);
          acc[q].y += __shfl_xor_sync(0xffffffffu, acc[q].y, o);
        }
      double2 pdot = cd(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < kHetrd2Rows; ++q) {
        const int i = k1 + warp + q * nw;
        if (i < l) {
          const double2 wi = cmul(tk, acc[q]);
          const double2 vi = v[i];
          zfmac(pdot, wi, vi);
          if (lane == 0) {
            sw[i] = wi;
            Vt[(size_t)k * l + i] = vi;
          }
        }
      }
      if (lane == 0) redz[warp] = pdot;
    }
    __syncthreads();
    // ---- phase D: A22 -= v w'^H + w' v^H, w' = w + alpha2 v; warp 0 then builds the next reflector ----
    double2* vn = sv[par ^ 1];
    if (active) {
      double2 dot = cd(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < nw; ++q) dot = dot + redz[q];
      const double2 td = cmul(tk, dot);
      const double2 a2 = cd(-0.5 * td.x, -0.5 * td.y);
      // warp 0: row k1 only; warps 1..15: rows k1+1.. round-robin
      const int i0 = warp == 0 ? k1 : k1 + warp;
      const int istep = warp == 0 ? l : nw - 1;
      for (int i = i0; i < l; i += istep) {
        const double2 vi = v[i];
        const double2 wi = sw[i] + cmul(a2, vi);
        double2* Ai = A + (size_t)i * lda;
        for (int j = k1 + lane; j < l; j += 32) {
          const double2 vj = v[j];
          const double2 wj = sw[j] + cmul(a2, vj);
          Ai[j] = Ai[j] - cmul(vi, conjd(wj)) - cmul(wi, conjd(vj));
        }
      }
    }
    if (warp == 0 && k1 + 1 < l) {
      __syncwarp();
      hetrd2_reflector(l, k1, A, lda, lane, d, e, tau, &s_tau[par ^ 1], vn);
    }
    __syncthreads();
  }
  if (tid == 0) d[l - 1] = A[(size_t)(l - 1) * lda + (l - 1)].x;
}

// Thread-per-row variant (128 threads, l <= 128, A in shared memory with
// lda = l + 1 rounded up to 1 mod 8 so a warp walking 32 rows of one column
// touches all 32 banks).  Per step: [A] thread j forms v_j, barrier; [B]
// thread i forms y_i = A22[i, :] v (no cross-thread reduction), w_i = tau y_i
// and the w^H v partials, barrier; [D] thread i updates row i,
//   A[i][j] -= v_i conj(w_j) + (w_i + c v_i) conj(v_j),  c = 2 Re(alpha2)
// (the Hermitian rank-2 update with w' = w + alpha2 v folded in), and thread
// 0, which owns the next pivot row, accumulates its norm during the update
// and forms the next reflector; barrier.  Instruction count per step is
// ~20 m per thread with no shuffles on the matvec.
constexpr int kHetrd3Max = 128;

// Reflector scalars for step k of the tridiagonalisation from row k:
// x = conj(A[k][k+1:]), alpha = x[0], tail = |x[1:]|^2.
__device__ __forceinline__ void hetrd3_reflector(int k, double tail, double2 akk1, double dkk, double* d, double* e,
                                                 double2* tau, double2* s_tau, double2* s_sc) {
  const double2 alpha = conjd(akk1);
  double2 tv = cd(0.0, 0.0), scal = cd(0.0, 0.0);
  double beta;
  if (tail == 0.0 && alpha.y == 0.0) {
    beta = alpha.x;  // H = I
  } else {
    beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + tail), alpha.x);
    const double ib = 1.0 / beta;
    tv = cd((beta - alpha.x) * ib, -alpha.y * ib);
    const double2 den = cd(alpha.x - beta, alpha.y);
    const double idd = 1.0 / abs2d(den);
    scal = cd(den.x * idd, -den.y * idd);  // 1 / (alpha - beta)
  }
  e[k] = beta;
  d[k] = dkk;
  tau[k] = tv;
  *s_tau = tv;
  *s_sc = scal;
}

__global__ void __launch_bounds__(128)
hetrd3_kernel(int l, int lda, const double2* __restrict__ Ain, double* __restrict__ d, double* __restrict__ e,
              double2* __restrict__ tau, double2* __restrict__ Vt) {
  hicu_pdl_entry();
  extern __shared__ double2 A[];
  __shared__ double2 sv[kHetrd3Max], sw[kHetrd3Max];
  __shared__ double2 red[4];
  __shared__ double2 s_tau, s_sc;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int q = t; q < l * l; q += 128) A[(size_t)(q / l) * lda + q % l] = Ain[q];
  for (int q = t; q < l * l; q += 128) Vt[q] = cd(0.0, 0.0);
  __syncthreads();
  if (t == 0 && l > 1) {
    double tail = 0.0;
    for (int j = 2; j < l; ++j) tail += abs2d(A[j]);
    hetrd3_reflector(0, tail, A[1], A[0].x, d, e, tau, &s_tau, &s_sc);
  }
  __syncthreads();
  for (int k = 0; k + 1 < l; ++k) {
    const int k1 = k + 1;
    const double2 tk = s_tau, sc = s_sc;
    if (tk.x == 0.0 && tk.y == 0.0) {
      // H = I: the trailing block is unchanged; thread 0 forms the next reflector from row k1
      if (t == 0 && k1 + 1 < l) {
        double tail = 0.0;
        for (int j = k1 + 2; j < l; ++j) tail += abs2d(A[(size_t)k1 * lda + j]);
        hetrd3_reflector(k1, tail, A[(size_t)k1 * lda + k1 + 1], A[(size_t)k1 * lda + k1].x, d, e, tau, &s_tau, &s_sc);
      }
      __syncthreads();
      continue;
    }
    // [A] v_j = (j == k1) ? 1 : conj(A[k][j]) sc
    {
      const int j = k1 + t;
      if (j < l) {
        const double2 vj = (j == k1) ? cd(1.0, 0.0) : cmul(conjd(A[(size_t)k * lda + j]), sc);
        sv[j] = vj;
        Vt[(size_t)k * l + j] = vj;
      }
    }
    __syncthreads();
    // [B] y_i = sum_j A[i][j] v_j (two accumulators), w_i = tau y_i, partial conj(w_i) v_i
    const int i = k1 + t;
    double2 wi = cd(0.0, 0.0), vi = cd(0.0, 0.0);
    {
      double2 pd = cd(0.0, 0.0);
      if (i < l) {
        const double2* Ai = A + (size_t)i * lda;
        double2 a0 = cd(0.0, 0.0), a1 = cd(0.0, 0.0), a2 = cd(0.0, 0.0), a3 = cd(0.0, 0.0);
        int j = k1;
        for (; j + 3 < l; j += 4) {  // four independent chains (DFMA latency ~9 cycles)
          const double2 x0 = Ai[j], x1 = Ai[j + 1], x2 = Ai[j + 2], x3 = Ai[j + 3];
          const double2 y0 = sv[j], y1 = sv[j + 1], y2 = sv[j + 2], y3 = sv[j + 3];
          zfma(a0, x0, y0);
          zfma(a1, x1, y1);
          zfma(a2, x2, y2);
          zfma(a3, x3, y3);
        }
        for (; j < l; ++j) zfma(a0, Ai[j], sv[j]);
        a0 = a0 + a2;
        a1 = a1 + a3;
        wi = cmul(tk, a0 + a1);
        vi = sv[i];
        sw[i] = wi;
        zfmac(pd, wi, vi);
      }
      pd = cd(warp_sum_d(pd.x), warp_sum_d(pd.y));
      if (lane == 0) red[warp] = pd;
    }
    __syncthreads();
    // [D] rank-2 update of row i; thread 0 (row k1) then forms the next reflector
    {
      const double2 dot = red[0] + red[1] + red[2] + red[3];
      const double2 td = cmul(tk, dot);
      const double c = -td.x;  // 2 Re(alpha2), alpha2 = -tau (w^H v) / 2
      if (i < l) {
        const double2 wpi = wi + c * vi;
        double2* Ai = A + (size_t)i * lda;
        double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;  // |row k1|^2 partials (used by thread 0)
        int j = k1;
        for (; j + 3 < l; j += 4) {
          const double2 v0 = sv[j], v1 = sv[j + 1], v2 = sv[j + 2], v3 = sv[j + 3];
          const double2 w0 = sw[j], w1 = sw[j + 1], w2 = sw[j + 2], w3 = sw[j + 3];
          const double2 n0 = Ai[j] - cmul(vi, conjd(w0)) - cmul(wpi, conjd(v0));
          const double2 n1 = Ai[j + 1] - cmul(vi, conjd(w1)) - cmul(wpi, conjd(v1));
          const double2 n2 = Ai[j + 2] - cmul(vi, conjd(w2)) - cmul(wpi, conjd(v2));
          const double2 n3 = Ai[j + 3] - cmul(vi, conjd(w3)) - cmul(wpi, conjd(v3));
          Ai[j] = n0;
          Ai[j + 1] = n1;
          Ai[j + 2] = n2;
          Ai[j + 3] = n3;
          if (j >= k1 + 2) t0 += abs2d(n0);
          if (j + 1 >= k1 + 2) t1 += abs2d(n1);
          t2 += abs2d(n2);
          t3 += abs2d(n3);
        }
        for (; j < l; ++j) {
          const double2 nv = Ai[j] - cmul(vi, conjd(sw[j])) - cmul(wpi, conjd(sv[j]));
          Ai[j] = nv;
          if (j >= k1 + 2) t0 += abs2d(nv);
        }
        const double tail = (t0 + t1) + (t2 + t3);
        if (t == 0 && k1 + 1 < l)
          hetrd3_reflector(k1, tail, Ai[k1 + 1], Ai[k1].x, d, e, tau, &s_tau, &s_sc);
      }
    }
    __syncthreads();
  }
  if (t == 0) d[l - 1] = A[(size_t)(l - 1) * lda + (l - 1)].x;
}

// 512-thread variant: 4 threads per row (thread (row i, quarter q) owns the
// columns j = k1 + q + 4u), up to 128 rows, lda == 4 mod 8 so the 8 lanes of a
// 16-byte shared-memory phase (2 rows x 4 quarters) hit disjoint banks.  The
// reflector vector is formed on the fly from row k (v_j = conj(A[k][j]) sc),
// so a step needs two barriers: [B] matvec partials + 4-lane reduction,
// w_i = tau y_i, w^H v partials; [D] rank-2 update (c = 2 Re(alpha2) folded
// into a per-row factor) while the four owners of row k1 accumulate its tail
// norm, then thread 0 forms the next reflector.
constexpr int kHetrd4Max = 128;

__global__ void __launch_bounds__(512)
hetrd4_kernel(int l, int lda, const double2* __restrict__ Ain, double* __restrict__ d, double* __restrict__ e,
              double2* __restrict__ tau, double2* __restrict__ Vt) {
  hicu_pdl_entry();
  extern __shared__ double2 A[];
  __shared__ double2 sw[kHetrd4Max];
  __shared__ double2 red[16];
  __shared__ double2 s_tau, s_sc;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int qd = t & 3, rowo = t >> 2;  // quarter, row offset

  for (int x = t; x < l * l; x += 512) A[(size_t)(x / l) * lda + x % l] = Ain[x];
  for (int x = t; x < l * l; x += 512) Vt[x] = cd(0.0, 0.0);
  __syncthreads();
  if (t == 0 && l > 1) {
    double tail = 0.0;
    for (int j = 2; j < l; ++j) tail += abs2d(A[j]);
    hetrd3_reflector(0, tail, A[1], A[0].x, d, e, tau, &s_tau, &s_sc);
  }
  __syncthreads();
  for (int k = 0; k + 1 < l; ++k) {
    const int k1 = k + 1;
    const double2 tk = s_tau, sc = s_sc;
    const double2* Ak = A + (size_t)k * lda;
    const int i = k1 + rowo;
    const bool has_row = i < l;
    if (tk.x == 0.0 && tk.y == 0.0) {
      if (t == 0 && k1 + 1 < l) {
        double tail = 0.0;
        for (int j = k1 + 2; j < l; ++j) tail += abs2d(A[(size_t)k1 * lda + j]);
        hetrd3_reflector(k1, tail, A[(size_t)k1 * lda + k1 + 1], A[(size_t)k1 * lda + k1].x, d, e, tau, &s_tau,
                         &s_sc);
      }
      __syncthreads();
      continue;
    }
    // ---- [B] y_i partial over my quarter, 4-lane reduction, w_i, w^H v partials ----
    double2 vi = cd(0.0, 0.0), wi = cd(0.0, 0.0);
    {
      double2 a0 = cd(0.0, 0.0), a1 = cd(0.0, 0.0);
      if (has_row) {
        const double2* Ai = A + (size_t)i * lda;
        int j = k1 + qd;
        for (; j + 4 < l; j += 8) {
          const double2 v0 = (j == k1) ? cd(1.0, 0.0) : cmul(conjd(Ak[j]), sc);
          const double2 v1 = cmul(conjd(Ak[j + 4]), sc);
          zfma(a0, Ai[j], v0);
          zfma(a1, Ai[j + 4], v1);
        }
        if (j < l) {
          const double2 v0 = (j == k1) ? cd(1.0, 0.0) : cmul(conjd(Ak[j]), sc);
          zfma(a0, Ai[j], v0);
        }
        vi = (i == k1) ? cd(1.0, 0.0) : cmul(conjd(Ak[i]), sc);
      }
      double2 y = a0 + a1;
      y.x += __shfl_xor_sync(0xffffffffu, y.x, 1);
      y.y += __shfl_xor_sync(0xffffffffu, y.y, 1);
      y.x += __shfl_xor_sync(0xffffffffu, y.x, 2);
      y.y += __shfl_xor_sync(0xffffffffu, y.y, 2);
      double2 pd = cd(0.0, 0.0);
      if (has_row) {
        wi = cmul(tk, y);
        if (qd == 0) {
          sw[i] = wi;
          Vt[(size_t)k * l + i] = vi;
          zfmac(pd, wi, vi);
        }
      }
      pd = cd(warp_sum_d(pd.x), warp_sum_d(pd.y));
      if (lane == 0) red[warp] = pd;
    }
    __syncthreads();
    // ---- [D] A[i][j] -= v_i conj(w_j) + (w_i + c v_i) conj(v_j) over my quarter ----
    {
      double2 dot = cd(0.0, 0.0);
#pragma unroll
      for (int w = 0; w < 16; ++w) dot = dot + red[w];
      const double c = -cmul(tk, dot).x;  // 2 Re(alpha2), alpha2 = -tau (w^H v) / 2
      double tl0 = 0.0, tl1 = 0.0;
      if (has_row) {
        const double2 wpi = wi + c * vi;
        double2* Ai = A + (size_t)i * lda;
        int j = k1 + qd;
        for (; j + 4 < l; j += 8) {
          const double2 v0 = (j == k1) ? cd(1.0, 0.0) : cmul(conjd(Ak[j]), sc);
          const double2 v1 = cmul(conjd(Ak[j + 4]), sc);
          const double2 n0 = Ai[j] - cmul(vi, conjd(sw[j])) - cmul(wpi, conjd(v0));
          const double2 n1 = Ai[j + 4] - cmul(vi, conjd(sw[j + 4])) - cmul(wpi, conjd(v1));
          Ai[j] = n0;
          Ai[j + 4] = n1;
          if (j >= k1 + 2) tl0 += abs2d(n0);
          tl1 += abs2d(n1);
        }
        if (j < l) {
          const double2 v0 = (j == k1) ? cd(1.0, 0.0) : cmul(conjd(Ak[j]), sc);
          const double2 n0 = Ai[j] - cmul(vi, conjd(sw[j])) - cmul(wpi, conjd(v0));
          Ai[j] = n0;
          if (j >= k1 + 2) tl0 += abs2d(n0);
        }
      }
      if (warp == 0) {  // row k1 = threads 0..3
        double tl = tl0 + tl1;
        tl += __shfl_xor_sync(0xffffffffu, tl, 1);
        tl += __shfl_xor_sync(0xffffffffu, tl, 2);
        if (t == 0 && k1 + 1 < l) {
          const double2* Ar = A + (size_t)k1 * lda;
          hetrd3_reflector(k1, tl, Ar[k1 + 1], Ar[k1].x, d, e, tau, &s_tau, &s_sc);
        }
      }
    }
    __syncthreads();
  }
  if (t == 0) d[l - 1] = A[(size_t)(l - 1) * lda + (l - 1)].x;
}

// Register-resident variant (l <= 96): the full Hermitian matrix lives in
// registers, warp w holding columns 6w..6w+5 and lane t rows t, t+32, t+64
// (18 complex per thread), so no step streams A through shared memory.
// Step k: [R] the warp owning column k (= conj of row k) forms reflector k
// from its registers (one warp reduction) and publishes v; [B] every thread
// forms partial matrix-vector products over its 6 columns for its 3 rows
// (shared partials, no shuffles) and its share of v^H A v; [C] warps 0-2 sum
// the 16 partials per row into w = tau A v; [D] every thread applies the
// rank-2 update to its 18 elements (v and w are zero outside the trailing
// block, so the update needs no masks).  Same reflector scalars as
// hetrd3_reflector; v/w double-buffered by step parity, 3 barriers per step.
constexpr int kHetrd6Max = 96;
#ifndef HICU_H6_WARPS
#define HICU_H6_WARPS 12  // measured per C2 nullspace iteration: 8: 581 us, 12: 580, 16: 616, 24: 765
#endif
constexpr int kH6Warps = HICU_H6_WARPS, kH6Cols = 96 / HICU_H6_WARPS;  // warps x columns = 96; 3 row slots per lane
__device__ long long g_h6_trace[3][6];  // debug (HICU_HETRD_TRACE): thread 0 clocks at steps 10, 40, 70

// reflector k from column k (x = rows lane + 32u of column k, in registers
// of every lane of the calling warp): scalars, v into sv, reflector row of Vt
__device__ __forceinline__ void hetrd6_reflect(int k, int l, int lane, const double2 (&x)[3], double* d, double* e,
                                               double2* tau, double2* Vt, double2* svb, double2* stau,
                                               double2* ssc) {
  const int k1 = k + 1;
  double tl = 0.0;
  double2 alpha = cd(0.0, 0.0), dkk = cd(0.0, 0.0);
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int i = lane + 32 * u;
    tl += (i >= k + 2 && i < l) ? abs2d(x[u]) : 0.0;
    alpha = (i == k1) ? x[u] : alpha;
    dkk = (i == k) ? x[u] : dkk;
  }
  tl = warp_sum_d(tl);
  alpha.x = __shfl_sync(0xffffffffu, alpha.x, k1 & 31);
  alpha.y = __shfl_sync(0xffffffffu, alpha.y, k1 & 31);
  dkk.x = __shfl_sync(0xffffffffu, dkk.x, k & 31);
  if (lane == 0) hetrd3_reflector(k, tl, conjd(alpha), dkk.x, d, e, tau, stau, ssc);
  __syncwarp();
  const double2 tk = *stau, sc = *ssc;
  const bool act = !(tk.x == 0.0 && tk.y == 0.0);
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int i = lane + 32 * u;
    if (i >= kHetrd6Max) continue;
    double2 vi = (i == k1) ? cd(1.0, 0.0) : cmul(x[u], sc);
    const bool on = act && i >= k1 && i < l;
    svb[i] = on ? vi : cd(0.0, 0.0);
    if (on) Vt[(size_t)k * l + i] = vi;
  }
}

__global__ void __launch_bounds__(kH6Warps * 32)
hetrd6_kernel(int l, const double2* __restrict__ Ain, double* __restrict__ d, double* __restrict__ e,
              double2* __restrict__ tau, double2* __restrict__ Vt) {
  hicu_pdl_entry();
  __shared__ double2 sv[2][kHetrd6Max], sw[2][kHetrd6Max];
  __shared__ double2 part[kH6Warps][kHetrd6Max];
  __shared__ double sq[kH6Warps];
  __shared__ double2 s_tau[2], s_sc[2];
  __shared__ double s_c;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  double2 a[3][kH6Cols];
#pragma unroll
  for (int u = 0; u < 3; ++u)
#pragma unroll
    for (int c = 0; c < kH6Cols; ++c) {
      const int i = lane + 32 * u, j = kH6Cols * w + c;
      a[u][c] = (i < l && j < l) ? Ain[(size_t)i * l + j] : cd(0.0, 0.0);
    }
  for (int x = t; x < l * l; x += kH6Warps * 32) Vt[x] = cd(0.0, 0.0);
  __syncthreads();  // Vt zeroed before any reflector row is written
  if (w == 0 && l > 1) {
    double2 x[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) x[u] = a[u][0];
    hetrd6_reflect(0, l, lane, x, d, e, tau, Vt, sv[0], &s_tau[0], &s_sc[0]);
  }
  for (int k = 0; k + 1 < l; ++k) {
    const int k1 = k + 1, par = k & 1;
    const int slot = k == 10 ? 0 : (k == 40 ? 1 : (k == 70 ? 2 : -1));
    if (slot >= 0 && t == 0) g_h6_trace[slot][0] = clock64();
    __syncthreads();  // reflector k published
    if (slot >= 0 && t == 0) g_h6_trace[slot][1] = clock64();
    const double2 tk = s_tau[par];
    // ---- [B] partial A v over my columns for my 3 rows; share of v^H A v ----
    {
      double2 p[3] = {cd(0.0, 0.0), cd(0.0, 0.0), cd(0.0, 0.0)};
      if (kH6Cols * w + kH6Cols > k1) {  // v is zero on the columns < k1
        double2 p2[3] = {cd(0.0, 0.0), cd(0.0, 0.0), cd(0.0, 0.0)};
#pragma unroll
        for (int c = 0; c < kH6Cols; ++c) {
          const double2 vj = sv[par][kH6Cols * w + c];
#pragma unroll
          for (int u = 0; u < 3; ++u)
            if (32 * u + 32 > k1) {  // rows < k1 are never read again
              if (c & 1) zfma(p2[u], a[u][c], vj);
              else zfma(p[u], a[u][c], vj);
            }
        }
#pragma unroll
        for (int u = 0; u < 3; ++u) p[u] = p[u] + p2[u];
      }
      double qv = 0.0;
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int i = lane + 32 * u;
        if (i < kHetrd6Max) {
          part[w][i] = p[u];
          const double2 vi = sv[par][i];
          qv += vi.x * p[u].x + vi.y * p[u].y;  // Re(conj(v_i) p_i)
        }
      }
      qv = warp_sum_d(qv);
      if (lane == 0) sq[w] = qv;
    }
    __syncthreads();
    if (slot >= 0 && t == 0) g_h6_trace[slot][2] = clock64();
    // ---- [C] w_i = tau sum_w part[w][i] (one row per thread) ----
    if (t < kHetrd6Max) {
      double2 y0 = cd(0.0, 0.0), y1 = cd(0.0, 0.0), y2 = cd(0.0, 0.0), y3 = cd(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < kH6Warps; q += 4) {
        y0 = y0 + part[q][t];
        y1 = y1 + part[q + 1][t];
        y2 = y2 + part[q + 2][t];
        y3 = y3 + part[q + 3][t];
      }
      sw[par][t] = (t >= k1 && t < l) ? cmul(tk, (y0 + y1) + (y2 + y3)) : cd(0.0, 0.0);
    }
    if (t == kHetrd6Max) {  // 2 Re(alpha2) = -|tau|^2 v^H A v (fixed-order tree over the warps)
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int q = 0; q < kH6Warps; ++q) s4[q & 3] += sq[q];
      s_c = -(tk.x * tk.x + tk.y * tk.y) * ((s4[0] + s4[1]) + (s4[2] + s4[3]));
    }
    __syncthreads();
    if (slot >= 0 && t == 0) g_h6_trace[slot][3] = clock64();
    // ---- [D] A -= v w^H + (w + c v) v^H on my elements; the owner of column
    //      k+1 keeps its fresh values and forms reflector k+1 right away ----
    {
      const double c = s_c;
      double2 vr[3], wr[3], xn[3];
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int i = lane + 32 * u;
        vr[u] = i < kHetrd6Max ? sv[par][i] : cd(0.0, 0.0);
        const double2 wi = i < kHetrd6Max ? sw[par][i] : cd(0.0, 0.0);
        wr[u] = wi + c * vr[u];  // row factor of the second term: w_i + c v_i
        xn[u] = cd(0.0, 0.0);
      }
      const bool own_next = k1 + 1 < l && w == k1 / kH6Cols;
      if (kH6Cols * w + kH6Cols > k1) {  // v, w are zero outside the trailing block
#pragma unroll
        for (int c2 = 0; c2 < kH6Cols; ++c2) {
          const int j = kH6Cols * w + c2;
          const double2 vj = sv[par][j], wj = sw[par][j];
#pragma unroll
          for (int u = 0; u < 3; ++u) {
            if (32 * u + 32 > k1) {
              // a -= v_i conj(w_j) + wp_i conj(v_j)  (4 FMAs per component)
              double2 x = a[u][c2];
              x.x = fma(-vr[u].x, wj.x, fma(-vr[u].y, wj.y, x.x));
              x.x = fma(-wr[u].x, vj.x, fma(-wr[u].y, vj.y, x.x));
              x.y = fma(-vr[u].y, wj.x, fma(vr[u].x, wj.y, x.y));
              x.y = fma(-wr[u].y, vj.x, fma(wr[u].x, vj.y, x.y));
              a[u][c2] = x;
            }
            if (j == k1) xn[u] = a[u][c2];
          }
        }
      }
      if (own_next) hetrd6_reflect(k1, l, lane, xn, d, e, tau, Vt, sv[par ^ 1], &s_tau[par ^ 1], &s_sc[par ^ 1]);
      if (slot >= 0 && t == 0) g_h6_trace[slot][4] = clock64() + (long long)(a[0][0].x > 1e300);
      if (slot >= 0 && t == 0) g_h6_trace[slot][5] = clock64();
    }
  }
  // d[l-1] = A[l-1][l-1]
#pragma unroll
  for (int u = 0; u < 3; ++u)
#pragma unroll
    for (int c = 0; c < kH6Cols; ++c)
      if (lane + 32 * u == l - 1 && kH6Cols * w + c == l - 1) d[l - 1] = a[u][c].x;
}

// 1/q to ~1e-15 relative: fp32 seed (MUFU) + two Newton steps in fp64
// (the Sturm count only needs the sign of each pivot).  Falls back to an IEEE
// division when q is outside the fp32 exponent range.
__device__ __forceinline__ double fast_rcp(double q) {
  const double aq = fabs(q);
  if (aq < 1e-30 || aq > 1e30) return 1.0 / q;
  double r = (double)__frcp_rn((float)q);
  r = r * (2.0 - q * r);
  r = r * (2.0 - q * r);
  return r;
}

// Sturm count: number of eigenvalues of T (d, e2 = e^2) strictly below x.
__device__ __forceinline__ int sturm_count(int l, const double* d, const double* e2, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int i = 1; i < l; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// Division-free Sturm count: the leading principal minors p_i of T - xI obey
// p_{i+1} = (d_i - x) p_i - e_i^2 p_{i-1}; the number of negative ratios
// q_i = p_i / p_{i-1} (the LDL^T pivots of sturm_count) is the number of
// eigenvalues below x.  Two dependent FMAs per step instead of a division;
// |q_i| < pivmin is mapped to q_i = -pivmin exactly as in sturm_count, and
// the pair (p_i, p_{i-1}) is rescaled by a power of two every 8 steps.
__device__ __forceinline__ int sturm_count_poly(int l, const double* d, const double* e2, double x, double pivmin) {
  double pm = 1.0, p = d[0] - x;
  if (fabs(p) < pivmin) p = -pivmin;
  int cnt = p < 0.0;
  for (int i = 1; i < l; ++i) {
    double pn = (d[i] - x) * p - e2[i - 1] * pm;
    if (fabs(pn) < pivmin * fabs(p)) pn = -pivmin * p;  // q = pn / p = -pivmin
    cnt += (pn < 0.0) != (p < 0.0);
    pm = p;
    p = pn;
    if ((i & 7) == 0) {
      // scale both by 2^-e, e = exponent of max(|p|, |pm|)
      const double m = fmax(fabs(p), fabs(pm));
      const int ex = (int)((__double_as_longlong(m) >> 52) & 0x7ff) - 1023;
      const double sc = __longlong_as_double((long long)(1023 - ex) << 52);
      if (ex > -1000 && ex < 1000) {
        p *= sc;
        pm *= sc;
      }
    }
  }
  return cnt;
}

// One warp per target eigenvalue (j-th largest, j < r): 33-way multisection.
__global__ void stebz_kernel(int l, int r, const double* __restrict__ dg, const double* __restrict__ eg,
                             double* __restrict__ lam) {
  hicu_pdl_entry();
  __shared__ double d[256], e2[256], ea_s[256];
  __shared__ double s_lo, s_hi, s_piv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int i = tid; i < l; i += blockDim.x) {
    d[i] = dg[i];
    const double ei = (i + 1 < l) ? eg[i] : 0.0;
    e2[i] = ei * ei;
    ea_s[i] = (i > 0 ? fabs(eg[i - 1]) : 0.0) + fabs(ei);
  }
  __syncthreads();
  if (warp == 0) {  // Gershgorin bounds: warp-parallel min / max
    double lo = 1e300, hi = -1e300, emax = 0.0;
    for (int i = lane; i < l; i += 32) {
      lo = fmin(lo, d[i] - ea_s[i]);
      hi = fmax(hi, d[i] + ea_s[i]);
      if (i + 1 < l) emax = fmax(emax, e2[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    }
    if (lane == 0) {
      const double nrm = fmax(fabs(lo), fabs(hi));
      s_piv = fmax(2.2e-308, 1e-300 * emax) + 2.2e-308;
      s_lo = lo - 2.2e-16 * nrm * l - 1e-300;
      s_hi = hi + 2.2e-16 * nrm * l + 1e-300;
    }
  }
  __syncthreads();
  const double pivmin = s_piv;
  for (int j = blockIdx.x * nw + warp; j < r; j += gridDim.x * nw) {
    const int k = l - 1 - j;  // ascending index of the j-th largest
    double lo = s_lo, hi = s_hi;
    for (int it = 0; it < 64; ++it) {
      const double w = hi - lo;
      if (w <= 4.4e-16 * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin) break;
      const double x = lo + w * (double)(lane + 1) / 33.0;
      const int c = sturm_count_poly(l, d, e2, x, pivmin);
      const unsigned b = __ballot_sync(0xffffffffu, c >= k + 1);
      if (b == 0u) {
        lo = lo + w * 32.0 / 33.0;
      } else {
        const int f = __ffs(b) - 1;
        const double nhi = lo + w * (double)(f + 1) / 33.0;
        const double nlo = (f == 0) ? lo : lo + w * (double)f / 33.0;
        hi = nhi;
        lo = nlo;
      }
    }
    if (lane == 0) lam[j] = 0.5 * (lo + hi);
  }
}

// Inverse iteration: one thread per eigenvalue; (T - lam I) LU with partial
// pivoting (dgttrf form), 3 solves from a deterministic start vector.  The
// per-thread factors live in shared memory, interleaved by thread
// (element i of thread t at [i*T + t]) so a warp's accesses hit distinct banks.
// z is l x r column-major (z[j*l + i]).
__global__ void stein_kernel(int l, int r, const double* __restrict__ d, const double* __restrict__ e,
                             const double* __restrict__ lam, double* __restrict__ z) {
  hicu_pdl_entry();
  extern __shared__ double sm[];
  __shared__ double sd[256], se[256];
  const int T = blockDim.x, t = threadIdx.x;
  for (int i = t; i < l; i += T) {
    sd[i] = d[i];
    se[i] = (i + 1 < l) ? e[i] : 0.0;
  }
  __syncthreads();
  const int j = blockIdx.x * T + t;
  if (j >= r) return;
  double* dl = sm;                    // multipliers
  double* u0 = dl + (size_t)l * T;    // U diagonal
  double* u1 = u0 + (size_t)l * T;    // U super-diagonal
  double* u2 = u1 + (size_t)l * T;    // U second super-diagonal
  double* x = u2 + (size_t)l * T;     // iterate
  unsigned long long swaps[4] = {0ull, 0ull, 0ull, 0ull};  // row-swap bits (l <= 256)
#define AT(arr, i) arr[(size_t)(i) * T + t]
  const double lj = lam[j];
  double tnorm = 0.0;
  for (int i = 0; i < l; ++i)
    tnorm = fmax(tnorm, fabs(sd[i]) + (i > 0 ? fabs(se[i - 1]) : 0.0) + fabs(se[i]));
  const double tiny = 2.2e-16 * fmax(tnorm, 1e-300);
  // LU of T - lam I with partial pivoting (dgttrf form).  The two entries the
  // next step depends on (u0[i+1], u1[i+1]) are carried in registers, so the
  // recurrence chain holds one division and no shared-memory round trip;
  // the factors are stored for the solves off the chain.
  {
    double u0c = sd[0] - lj, u1c = se[0];
    for (int i = 0; i + 1 < l; ++i) {
      const double sub = se[i];
      double u0n = sd[i + 1] - lj, u1n = se[i + 1];
      if (fabs(u0c) >= fabs(sub)) {
        const double f = (u0c != 0.0) ? sub / u0c : 0.0;
        AT(dl, i) = f;
        AT(u0, i) = u0c;
        AT(u1, i) = u1c;
        AT(u2, i) = 0.0;
        u0n -= f * u1c;
      } else {
        const double f = u0c / sub;
        AT(u0, i) = sub;
        const double tt = u0n;
        u0n = u1c - f * tt;
        AT(u1, i) = tt;
        if (i + 2 < l) {
          AT(u2, i) = u1n;
          u1n = -f * u1n;
        } else {
          AT(u2, i) = 0.0;
        }
        AT(dl, i) = f;
        swaps[i >> 6] |= 1ull << (i & 63);
      }
      u0c = u0n;
      u1c = u1n;
    }
    AT(u0, l - 1) = u0c;
    AT(u1, l - 1) = u1c;
    AT(u2, l - 1) = 0.0;
  }
  for (int i = 0; i < l; ++i) {
    double v = AT(u0, i);
    if (fabs(v) < tiny) v = (v < 0.0 ? -tiny : tiny);
    AT(u0, i) = 1.0 / v;  // store the reciprocal: back substitution multiplies
  }
  unsigned sd0 = 2654435761u * (unsigned)(j + 1);
  for (int i = 0; i < l; ++i) {
    sd0 = sd0 * 1664525u + 1013904223u;
    AT(x, i) = 1.0 + 0.5 * ((double)(sd0 >> 8) / 16777216.0 - 0.5);
  }
  for (int itn = 0; itn < 3; ++itn) {
    // forward (L with row swaps): the running entry is carried in a register
    double c = AT(x, 0);
    for (int i = 0; i + 1 < l; ++i) {
      const double nx = AT(x, i + 1), f = AT(dl, i);
      if ((swaps[i >> 6] >> (i & 63)) & 1ull) {
        AT(x, i) = nx;
        c = c - f * nx;
      } else {
        AT(x, i) = c;
        c = nx - f * c;
      }
    }
    AT(x, l - 1) = c;
    double nrm = 0.0;
    double xp1 = 0.0, xp2 = 0.0;
    for (int i = l - 1; i >= 0; --i) {
      double v = AT(x, i) - AT(u1, i) * xp1 - AT(u2, i) * xp2;
      v = v * AT(u0, i);
      AT(x, i) = v;
      xp2 = xp1;
      xp1 = v;
      nrm += v * v;
    }
    const double inv = 1.0 / sqrt(nrm);
    for (int i = 0; i < l; ++i) AT(x, i) *= inv;
  }
  for (int i = 0; i < l; ++i) z[(size_t)j * l + i] = AT(x, i);
#undef AT
}

// Re-orthogonalise clusters (|lam_i - lam_j| <= ctol * |lam_0|) by CGS2 in
// descending order, then fix a sign convention (largest entry positive).
__global__ void __launch_bounds__(256) cluster_orth_kernel(int l, int r, const double* __restrict__ lam,
                                                           double* __restrict__ z, double ctol) {
  hicu_pdl_entry();
  __shared__ double red[8];
  __shared__ double s_dot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double thr = ctol * fabs(lam[0]);
  for (int j = 1; j < r; ++j) {
    double* zj = z + (size_t)j * l;
    for (int pass = 0; pass < 2; ++pass) {
      bool any = false;
      for (int i = j - 1; i >= 0 && fabs(lam[i] - lam[j]) <= thr; --i) {
        any = true;
        const double* zi = z + (size_t)i * l;
        double t = 0.0;
        for (int q = tid; q < l; q += blockDim.x) t += zi[q] * zj[q];
        t = warp_sum_d(t);
        if (lane == 0) red[warp] = t;
        __syncthreads();
        if (tid == 0) {
          double s = 0.0;
          for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
          s_dot = s;
        }
        __syncthreads();
        const double dt = s_dot;
        for (int q = tid; q < l; q += blockDim.x) zj[q] -= dt * zi[q];
        __syncthreads();
      }
      if (!any) break;
      double t = 0.0;
      for (int q = tid; q < l; q += blockDim.x) t += zj[q] * zj[q];
      t = warp_sum_d(t);
      if (lane == 0) red[warp] = t;
      __syncthreads();
      if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        s_dot = 1.0 / sqrt(s);
      }
      __syncthreads();
      const double inv = s_dot;
      for (int q = tid; q < l; q += blockDim.x) zj[q] *= inv;
      __syncthreads();
    }
  }
}

// F[:, j] = Q z_j with Q = H_0 H_1 ... H_{l-2}: apply H_{l-2} first.
// One CTA owns a group of eigenvectors (one warp each) and streams the
// reflectors through shared memory in chunks, so each reflector is read from
// L2 once per CTA instead of once per warp.  F is l x r row-major (c128).
constexpr int kBtChunk = 16;
__global__ void back_transform_kernel(int l, int r, const double2* __restrict__ Vt, const double2* __restrict__ tau,
                                      const double* __restrict__ z, double2* __restrict__ F) {
  hicu_pdl_entry();
  extern __shared__ double2 sm2[];
  const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* x = sm2 + (size_t)warp * l;
  double2* vs = sm2 + (size_t)warps * l;  // kBtChunk reflectors
  __shared__ double2 ts[kBtChunk];
  const int j = blockIdx.x * warps + warp;
  const bool active = j < r;
  if (active)
    for (int i = lane; i < l; i += 32) x[i] = cd(z[(size_t)j * l + i], 0.0);
  for (int k1 = l - 2; k1 >= 0; k1 -= kBtChunk) {
    const int k0 = max(0, k1 - kBtChunk + 1);
    __syncthreads();
    for (int q = threadIdx.x; q < (k1 - k0 + 1) * l; q += blockDim.x)
      vs[q] = Vt[(size_t)(k0 + q / l) * l + q % l];
    for (int q = threadIdx.x; q <= k1 - k0; q += blockDim.x) ts[q] = tau[k0 + q];
    __syncthreads();
    if (!active) continue;
    for (int k = k1; k >= k0; --k) {
      const double2 tk = ts[k - k0];
      if (tk.x == 0.0 && tk.y == 0.0) continue;
      const double2* v = vs + (size_t)(k - k0) * l;
      double2 dot = cd(0.0, 0.0);
      for (int i = k + 1 + lane; i < l; i += 32) zfmac(dot, v[i], x[i]);
      dot = warp_sum_z(dot);
      const double2 f = cmul(tk, dot);
      for (int i = k + 1 + lane; i < l; i += 32) x[i] = x[i] - cmul(v[i], f);
      __syncwarp();
    }
  }
  if (active)
    for (int i = lane; i < l; i += 32) F[(size_t)i * r + j] = x[i];
}

constexpr int kBtPer = 4;  // l <= 128 for the register-resident back-transform (res2 below)

// Streaming variant: two eigenvectors per warp in registers, reflectors read
// from L2 one step ahead (no per-CTA staging of all l-1 reflectors), the two
// dot products reduced in one interleaved shuffle tree.
constexpr int kBt2Warps = 4;
__global__ void __launch_bounds__(kBt2Warps * 32)
back_transform_res2_kernel(int l, int r, const double2* __restrict__ Vt, const double2* __restrict__ tau,
                           const double* __restrict__ z, double2* __restrict__ F) {
  hicu_pdl_entry();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = 2 * (blockIdx.x * kBt2Warps + warp);
  if (j0 >= r) return;
  const bool two = j0 + 1 < r;
  double2 x0[kBtPer], x1[kBtPer];
#pragma unroll
  for (int u = 0; u < kBtPer; ++u) {
    const int i = lane + 32 * u;
    x0[u] = i < l ? cd(z[(size_t)j0 * l + i], 0.0) : cd(0.0, 0.0);
    x1[u] = (i < l && two) ? cd(z[(size_t)(j0 + 1) * l + i], 0.0) : cd(0.0, 0.0);
  }
  double2 vn[kBtPer];
  auto load_v = [&](int k) {
#pragma unroll
    for (int u = 0; u < kBtPer; ++u) {
      const int i = lane + 32 * u;
      vn[u] = (k >= 0 && i > k && i < l) ? __ldg(Vt + (size_t)k * l + i) : cd(0.0, 0.0);
    }
  };
  load_v(l - 2);
  for (int k = l - 2; k >= 0; --k) {
    double2 vr[kBtPer];
#pragma unroll
    for (int u = 0; u < kBtPer; ++u) vr[u] = vn[u];
    load_v(k - 1);
    const double2 tk = __ldg(tau + k);
    if (tk.x == 0.0 && tk.y == 0.0) continue;
    double2 d = cd(0.0, 0.0), e = cd(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < kBtPer; ++u) {
      zfmac(d, vr[u], x0[u]);
      zfmac(e, vr[u], x1[u]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      d.x += __shfl_xor_sync(0xffffffffu, d.x, o);
      d.y += __shfl_xor_sync(0xffffffffu, d.y, o);
      e.x += __shfl_xor_sync(0xffffffffu, e.x, o);
      e.y += __shfl_xor_sync(0xffffffffu, e.y, o);
    }
    const double2 f = cmul(tk, d), g = cmul(tk, e);
#pragma unroll
    for (int u = 0; u < kBtPer; ++u) {
      x0[u] = x0[u] - cmul(vr[u], f);
      x1[u] = x1[u] - cmul(vr[u], g);
    }
  }
#pragma unroll
  for (int u = 0; u < kBtPer; ++u) {
    const int i = lane + 32 * u;
    if (i >= l) continue;
    F[(size_t)i * r + j0] = x0[u];
    if (two) F[(size_t)i * r + j0 + 1] = x1[u];
  }
}

}  // namespace

size_t hicu_heev_top_workspace(int l, int r) {
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  return al((size_t)l * (l + 1) * sizeof(double2)) * 2 + al((size_t)l * sizeof(double)) * 2 +
         al((size_t)l * sizeof(double2)) + al((size_t)r * sizeof(double)) + al((size_t)l * r * sizeof(double)) +
         al((size_t)5 * l * r * sizeof(double));
}

// Top-r eigenpairs of Hermitian A (l x l c128): lam (r, descending) and
// F (l x r c128, orthonormal eigenvectors).  ws from hicu_heev_top_workspace.
int hicu_heev_top(int l, int r, const double2* A, double* lam, double2* F, void* ws, cudaStream_t st) {
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  char* p = (char*)ws;
  double2* Aws = (double2*)p;   p += al((size_t)l * (l + 1) * sizeof(double2));
  double2* Vt = (double2*)p;    p += al((size_t)l * (l + 1) * sizeof(double2));
  double* d = (double*)p;       p += al((size_t)l * sizeof(double));
  double* e = (double*)p;       p += al((size_t)l * sizeof(double));
  double2* tau = (double2*)p;   p += al((size_t)l * sizeof(double2));
  double* lam_s = (double*)p;   p += al((size_t)r * sizeof(double));
  double* z = (double*)p;       p += al((size_t)l * r * sizeof(double));
  (void)lam_s;
  int s;
  const size_t abytes = (size_t)l * (l + 1) * sizeof(double2);
  const bool sm = abytes <= 180 * 1024;
  if (sm) {
    const int lda3 = ((l + 1 + 6) / 8) * 8 + 1;  // >= l + 1, == 1 mod 8
    const size_t a3 = (size_t)l * lda3 * sizeof(double2);
    const int lda4 = ((l + 1 + 3) / 8) * 8 + 4;  // >= l + 1, == 4 mod 8
    const size_t a4 = (size_t)l * lda4 * sizeof(double2);
    if (l <= kHetrd6Max) {
      hicu_launch(hetrd6_kernel, 1, kH6Warps * 32, 0, st, l, A, d, e, tau, Vt);
    } else if (l <= kHetrd4Max && a4 <= 180 * 1024) {
      hicu_allow_max_smem((const void*)hetrd4_kernel);
      hicu_launch(hetrd4_kernel, 1, 512, a4, st, l, lda4, A, d, e, tau, Vt);
    } else if (l <= kHetrd3Max && a3 <= 180 * 1024) {
      hicu_allow_max_smem((const void*)hetrd3_kernel);
      hicu_launch(hetrd3_kernel, 1, 128, a3, st, l, lda3, A, d, e, tau, Vt);
    } else if (l <= kHetrd2Max) {
      hicu_allow_max_smem((const void*)hetrd2_kernel);
      hicu_launch(hetrd2_kernel, 1, 512, abytes, st, l, A, d, e, tau, Vt);
    } else {
      hicu_allow_max_smem((const void*)hetrd_kernel<true>);
      hicu_launch(hetrd_kernel<true>, 1, 1024, abytes, st, l, A, Aws, d, e, tau, Vt);
    }
  } else if (l <= kHcMaxL) {
    // distributed over a cluster (the matrix does not fit one SM's shared memory)
    const size_t hsm = (size_t)((l + kHcCS - 1) / kHcCS) * (l + 1) * sizeof(double2);
    hicu_allow_max_smem((const void*)hetrd_cluster_kernel);
    hicu_launch(hetrd_cluster_kernel, kHcCS, kHcThreads, hsm, st, l, A, d, e, tau, Vt);
  } else {
    hicu_launch(hetrd_kernel<false>, 1, 1024, 0, st, l, A, Aws, d, e, tau, Vt);
  }
  if ((s = hicu_check_launch("hetrd_kernel"))) return s;
  const int wpb = 1;  // one warp (one eigenvalue) per SM: the Sturm recurrence is a division chain
  hicu_launch(stebz_kernel, (r + wpb - 1) / wpb, wpb * 32, 0, st, l, r, d, e, lam);
  if ((s = hicu_check_launch("stebz_kernel"))) return s;
  {
    // one eigenvalue per CTA: the pivoting branches diverge between eigenvalues
    int T = 1;
    while (T > 1 && (size_t)5 * l * T * sizeof(double) > 200 * 1024) T >>= 1;
    const size_t smem = (size_t)5 * l * T * sizeof(double);
    hicu_allow_max_smem((const void*)stein_kernel);
    hicu_launch(stein_kernel, (r + T - 1) / T, T, smem, st, l, r, d, e, lam, z);
  }
  if ((s = hicu_check_launch("stein_kernel"))) return s;
  hicu_launch(cluster_orth_kernel, 1, 256, 0, st, l, r, lam, z, 1e-9);
  if ((s = hicu_check_launch("cluster_orth_kernel"))) return s;
  if (l <= 32 * kBtPer) {
    const int pairs = (r + 1) / 2;
    hicu_launch(back_transform_res2_kernel, (pairs + kBt2Warps - 1) / kBt2Warps, kBt2Warps * 32, 0, st, l, r, Vt, tau,
                z, F);
    return hicu_check_launch("back_transform_res2_kernel");
  }
  const int bw = 8;
  const size_t smem = ((size_t)bw * l + (size_t)kBtChunk * l) * sizeof(double2);
  hicu_allow_max_smem((const void*)back_transform_kernel);
  hicu_launch(back_transform_kernel, (r + bw - 1) / bw, bw * 32, smem, st, l, r, Vt, tau, z, F);
  return hicu_check_launch("back_transform_kernel");
}

// ---------------------------------------------------------------------------
// Top-r eigenpairs of a Hermitian n x n complex128 matrix (row-major, full
// storage): the dense Cadzow baseline's rank-r truncation (oracle.py:138-141,
// truncated SVD of H == top-r eigenvectors of H^H H).  evals descending, V
// n x r orthonormal columns.
// ---------------------------------------------------------------------------
extern "C" size_t hicu_eigh_top_workspace(int n, int r) {
  if (n < 1 || r < 1 || r > n) return 0;
  return hicu_heev_top_workspace(n, r);
}

extern "C" int hicu_eigh_top(int n, int r, const void* A, double* evals, void* V, void* ws, size_t ws_bytes,
                             void* stream) {
  if (n < 1 || r < 1 || r > n || !A || !evals || !V || !ws)
    return hicu_set_error(HICU_ERR_PARAMETER, "eigh_top: bad arguments");
  if (ws_bytes < hicu_heev_top_workspace(n, r)) return hicu_set_error(HICU_ERR_WORKSPACE, "eigh_top: workspace");
  return hicu_heev_top(n, r, (const double2*)A, evals, (double2*)V, ws, (cudaStream_t)stream);
}
