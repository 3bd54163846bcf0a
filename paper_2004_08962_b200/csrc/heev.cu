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

// Householder reduction A = Q T Q^H (lower), one CTA of 512 threads.
// Outputs d (l), e (l-1), tau (l-1) and the reflectors transposed:
// Vt[k*l + i] = v_k[i] (v_k[k+1] = 1).  A is held with leading dimension
// l+1 so column walks (lanes over rows) are bank-conflict free; the
// matrix-vector product is row-parallel with j-chunk partials in shared memory
// (no per-row shuffle reductions on the sequential critical path).
template <bool SMEM>
__global__ void __launch_bounds__(512)
hetrd_kernel(int l, const double2* __restrict__ Ain, double2* __restrict__ Aws,
             double* __restrict__ d, double* __restrict__ e, double2* __restrict__ tau,
             double2* __restrict__ Vt) {
  extern __shared__ double2 sA[];
  double2* A = SMEM ? sA : Aws;
  const int lda = l + 1;
  __shared__ double2 sv[256], sw[256];
  __shared__ double2 part[4][256];
  __shared__ double redd[32];
  __shared__ double2 redz[16];
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
        double2 acc = cd(0.0, 0.0);
        const double2* Ai = A + (size_t)i * lda;
        for (int j = j0; j < j1; ++j) zfma(acc, Ai[j], sv[j]);
        part[c][i] = acc;
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
      // m <= 255 < nt: at most 8 warps hold non-zero partials
      pz = warp_sum_z(pz);
      if (lane == 0 && warp < 16) redz[warp] = pz;
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

// One warp per target eigenvalue (j-th largest, j < r): 33-way multisection.
__global__ void stebz_kernel(int l, int r, const double* __restrict__ dg, const double* __restrict__ eg,
                             double* __restrict__ lam) {
  __shared__ double d[256], e2[256];
  __shared__ double s_lo, s_hi, s_piv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int i = tid; i < l; i += blockDim.x) {
    d[i] = dg[i];
    e2[i] = (i + 1 < l) ? eg[i] * eg[i] : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    double lo = 1e300, hi = -1e300, emax = 0.0;
    for (int i = 0; i < l; ++i) {
      const double ea = (i > 0 ? fabs(eg[i - 1]) : 0.0) + (i + 1 < l ? fabs(eg[i]) : 0.0);
      lo = fmin(lo, d[i] - ea);
      hi = fmax(hi, d[i] + ea);
      if (i + 1 < l) emax = fmax(emax, e2[i]);
    }
    const double nrm = fmax(fabs(lo), fabs(hi));
    s_piv = fmax(2.2e-308, 1e-300 * emax) + 2.2e-308;
    s_lo = lo - 2.2e-16 * nrm * l - 1e-300;
    s_hi = hi + 2.2e-16 * nrm * l + 1e-300;
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
      const int c = sturm_count(l, d, e2, x, pivmin);
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
  for (int i = 0; i < l; ++i) {
    AT(u0, i) = sd[i] - lj;
    AT(u1, i) = se[i];
    AT(u2, i) = 0.0;
  }
  for (int i = 0; i + 1 < l; ++i) {
    const double sub = se[i];
    const double ui = AT(u0, i);
    if (fabs(ui) >= fabs(sub)) {
      const double f = (ui != 0.0) ? sub / ui : 0.0;
      AT(dl, i) = f;
      AT(u0, i + 1) -= f * AT(u1, i);
    } else {
      const double f = ui / sub;
      AT(u0, i) = sub;
      const double tt = AT(u0, i + 1);
      AT(u0, i + 1) = AT(u1, i) - f * tt;
      AT(u1, i) = tt;
      if (i + 2 < l) {
        AT(u2, i) = AT(u1, i + 1);
        AT(u1, i + 1) = -f * AT(u2, i);
      }
      AT(dl, i) = f;
      swaps[i >> 6] |= 1ull << (i & 63);
    }
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
    for (int i = 0; i + 1 < l; ++i) {
      if ((swaps[i >> 6] >> (i & 63)) & 1ull) {
        const double tt = AT(x, i);
        AT(x, i) = AT(x, i + 1);
        AT(x, i + 1) = tt - AT(dl, i) * AT(x, i);
      } else {
        AT(x, i + 1) -= AT(dl, i) * AT(x, i);
      }
    }
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
    hicu_allow_max_smem((const void*)hetrd_kernel<true>);
    hetrd_kernel<true><<<1, 512, abytes, st>>>(l, A, Aws, d, e, tau, Vt);
  } else {
    hetrd_kernel<false><<<1, 512, 0, st>>>(l, A, Aws, d, e, tau, Vt);
  }
  if ((s = hicu_check_launch("hetrd_kernel"))) return s;
  const int wpb = 8;
  stebz_kernel<<<(r + wpb - 1) / wpb, wpb * 32, 0, st>>>(l, r, d, e, lam);
  if ((s = hicu_check_launch("stebz_kernel"))) return s;
  {
    int T = 32;
    while (T > 1 && (size_t)5 * l * T * sizeof(double) > 200 * 1024) T >>= 1;
    const size_t smem = (size_t)5 * l * T * sizeof(double);
    hicu_allow_max_smem((const void*)stein_kernel);
    stein_kernel<<<(r + T - 1) / T, T, smem, st>>>(l, r, d, e, lam, z);
  }
  if ((s = hicu_check_launch("stein_kernel"))) return s;
  cluster_orth_kernel<<<1, 256, 0, st>>>(l, r, lam, z, 1e-9);
  if ((s = hicu_check_launch("cluster_orth_kernel"))) return s;
  const int bw = 8;
  const size_t smem = ((size_t)bw * l + (size_t)kBtChunk * l) * sizeof(double2);
  hicu_allow_max_smem((const void*)back_transform_kernel);
  back_transform_kernel<<<(r + bw - 1) / bw, bw * 32, smem, st>>>(l, r, Vt, tau, z, F);
  return hicu_check_launch("back_transform_kernel");
}
