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

// Householder reduction A = Q T Q^H (lower), one CTA.  Outputs d (l), e (l-1),
// tau (l-1) and the reflectors transposed: Vt[k*l + i] = v_k[i] (v_k[k+1] = 1).
__global__ void __launch_bounds__(1024)
hetrd_kernel(int l, const double2* __restrict__ Ain, double2* __restrict__ Aws, bool use_smem,
             double* __restrict__ d, double* __restrict__ e, double2* __restrict__ tau,
             double2* __restrict__ Vt) {
  extern __shared__ double2 sA[];
  double2* A = use_smem ? sA : Aws;
  __shared__ double2 sv[256], sw[256];
  __shared__ double2 s_tau, s_scal, s_alpha2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int q = tid; q < l * l; q += blockDim.x) A[q] = Ain[q];
  for (int q = tid; q < l * l; q += blockDim.x) Vt[q] = cd(0.0, 0.0);
  __syncthreads();
  for (int k = 0; k + 1 < l; ++k) {
    if (warp == 0) {
      double t = 0.0;
      for (int i = k + 2 + lane; i < l; i += 32) t += abs2d(A[(size_t)i * l + k]);
      t = warp_sum_d(t);
      if (lane == 0) {
        const double2 alpha = A[(size_t)(k + 1) * l + k];
        double2 tv = cd(0.0, 0.0), scal = cd(0.0, 0.0);
        double beta;
        if (t == 0.0 && alpha.y == 0.0) {
          beta = alpha.x;  // H = I
        } else {
          beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + t), alpha.x);
          tv = cd((beta - alpha.x) / beta, -alpha.y / beta);
          const double2 den = cd(alpha.x - beta, alpha.y);
          const double dd = abs2d(den);
          scal = cd(den.x / dd, -den.y / dd);  // 1 / (alpha - beta)
        }
        e[k] = beta;
        d[k] = A[(size_t)k * l + k].x;
        tau[k] = tv;
        s_tau = tv;
        s_scal = scal;
      }
    }
    __syncthreads();
    const double2 tk = s_tau;
    const double2 sc = s_scal;
    for (int i = k + 1 + tid; i < l; i += blockDim.x) {
      const double2 v = (i == k + 1) ? cd(1.0, 0.0) : cmul(A[(size_t)i * l + k], sc);
      sv[i] = v;
      Vt[(size_t)k * l + i] = v;
    }
    __syncthreads();
    if (tk.x == 0.0 && tk.y == 0.0) continue;  // uniform
    // w = tau * A22 v
    for (int i = k + 1 + warp; i < l; i += nw) {
      double2 acc = cd(0.0, 0.0);
      for (int j = k + 1 + lane; j < l; j += 32) zfma(acc, A[(size_t)i * l + j], sv[j]);
      acc = warp_sum_z(acc);
      if (lane == 0) sw[i] = cmul(tk, acc);
    }
    __syncthreads();
    if (warp == 0) {
      double2 dot = cd(0.0, 0.0);
      for (int i = k + 1 + lane; i < l; i += 32) zfmac(dot, sw[i], sv[i]);
      dot = warp_sum_z(dot);
      if (lane == 0) {
        const double2 td = cmul(tk, dot);
        s_alpha2 = cd(-0.5 * td.x, -0.5 * td.y);
      }
    }
    __syncthreads();
    const double2 a2 = s_alpha2;
    for (int i = k + 1 + tid; i < l; i += blockDim.x) sw[i] = sw[i] + cmul(a2, sv[i]);
    __syncthreads();
    // A22 -= v w^H + w v^H
    for (int i = k + 1 + warp; i < l; i += nw) {
      const double2 vi = sv[i], wi = sw[i];
      for (int j = k + 1 + lane; j < l; j += 32) {
        const double2 vj = sv[j], wj = sw[j];
        double2 a = A[(size_t)i * l + j];
        a = a - cmul(vi, conjd(wj)) - cmul(wi, conjd(vj));
        A[(size_t)i * l + j] = a;
      }
    }
    __syncthreads();
  }
  if (tid == 0) d[l - 1] = A[(size_t)(l - 1) * l + (l - 1)].x;
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
// pivoting (dgttrf form), 4 solves from a deterministic start vector.
// z is l x r column-major (z[j*l + i]); scratch 5*l doubles per thread.
__global__ void stein_kernel(int l, int r, const double* __restrict__ d, const double* __restrict__ e,
                             const double* __restrict__ lam, double* __restrict__ z, double* __restrict__ scratch) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= r) return;
  double* dl = scratch + (size_t)j * 5 * l;  // multipliers
  double* u0 = dl + l;                       // U diagonal
  double* u1 = u0 + l;                       // U super-diagonal
  double* u2 = u1 + l;                       // U second super-diagonal (pivoting fill)
  double* ip = u2 + l;                       // 1.0 when rows i, i+1 were swapped
  const double lj = lam[j];
  double tnorm = 0.0;
  for (int i = 0; i < l; ++i)
    tnorm = fmax(tnorm, fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < l ? fabs(e[i]) : 0.0));
  const double tiny = 2.2e-16 * fmax(tnorm, 1e-300);
  // factor (dgttrf) with sub = super = e
  for (int i = 0; i < l; ++i) {
    u0[i] = d[i] - lj;
    u1[i] = (i + 1 < l) ? e[i] : 0.0;
    u2[i] = 0.0;
    ip[i] = 0.0;
  }
  for (int i = 0; i + 1 < l; ++i) {
    const double sub = e[i];
    if (fabs(u0[i]) >= fabs(sub)) {
      const double f = (u0[i] != 0.0) ? sub / u0[i] : 0.0;
      dl[i] = f;
      u0[i + 1] -= f * u1[i];
    } else {
      // swap rows i and i+1
      const double f = u0[i] / sub;
      u0[i] = sub;
      const double t = u0[i + 1];
      u0[i + 1] = u1[i] - f * t;
      u1[i] = t;
      if (i + 2 < l) {
        u2[i] = u1[i + 1];
        u1[i + 1] = -f * u2[i];
      }
      dl[i] = f;
      ip[i] = 1.0;
    }
  }
  for (int i = 0; i < l; ++i)
    if (fabs(u0[i]) < tiny) u0[i] = (u0[i] < 0.0 ? -tiny : tiny);
  double* x = z + (size_t)j * l;
  // deterministic, eigenvalue-dependent start vector
  unsigned s = 2654435761u * (unsigned)(j + 1);
  for (int i = 0; i < l; ++i) {
    s = s * 1664525u + 1013904223u;
    x[i] = 1.0 + 0.5 * ((double)(s >> 8) / 16777216.0 - 0.5);
  }
  for (int itn = 0; itn < 4; ++itn) {
    // apply L^{-1} (with the recorded row swaps)
    for (int i = 0; i + 1 < l; ++i) {
      if (ip[i] != 0.0) {
        const double t = x[i];
        x[i] = x[i + 1];
        x[i + 1] = t - dl[i] * x[i];
      } else {
        x[i + 1] -= dl[i] * x[i];
      }
    }
    // back substitution with U (3 diagonals)
    for (int i = l - 1; i >= 0; --i) {
      double v = x[i];
      if (i + 1 < l) v -= u1[i] * x[i + 1];
      if (i + 2 < l) v -= u2[i] * x[i + 2];
      x[i] = v / u0[i];
    }
    double nrm = 0.0, mx = 0.0;
    for (int i = 0; i < l; ++i) {
      nrm += x[i] * x[i];
      mx = fmax(mx, fabs(x[i]));
    }
    const double inv = 1.0 / sqrt(nrm);
    for (int i = 0; i < l; ++i) x[i] *= inv;
  }
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
// One warp per eigenvector; F is l x r row-major (c128).
__global__ void back_transform_kernel(int l, int r, const double2* __restrict__ Vt, const double2* __restrict__ tau,
                                      const double* __restrict__ z, double2* __restrict__ F) {
  extern __shared__ double2 sx[];
  const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* x = sx + (size_t)warp * l;
  for (int j = blockIdx.x * warps + warp; j < r; j += gridDim.x * warps) {
    for (int i = lane; i < l; i += 32) x[i] = cd(z[(size_t)j * l + i], 0.0);
    __syncwarp();
    for (int k = l - 2; k >= 0; --k) {
      const double2 tk = tau[k];
      if (tk.x == 0.0 && tk.y == 0.0) continue;
      const double2* v = Vt + (size_t)k * l;
      double2 dot = cd(0.0, 0.0);
      for (int i = k + 1 + lane; i < l; i += 32) zfmac(dot, v[i], x[i]);
      dot = warp_sum_z(dot);
      const double2 f = cmul(tk, dot);
      for (int i = k + 1 + lane; i < l; i += 32) x[i] = x[i] - cmul(v[i], f);
      __syncwarp();
    }
    for (int i = lane; i < l; i += 32) F[(size_t)i * r + j] = x[i];
    __syncwarp();
  }
}

}  // namespace

size_t hicu_heev_top_workspace(int l, int r) {
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  return al((size_t)l * l * sizeof(double2)) * 2 + al((size_t)l * sizeof(double)) * 2 +
         al((size_t)l * sizeof(double2)) + al((size_t)r * sizeof(double)) + al((size_t)l * r * sizeof(double)) +
         al((size_t)5 * l * r * sizeof(double));
}

// Top-r eigenpairs of Hermitian A (l x l c128): lam (r, descending) and
// F (l x r c128, orthonormal eigenvectors).  ws from hicu_heev_top_workspace.
int hicu_heev_top(int l, int r, const double2* A, double* lam, double2* F, void* ws, cudaStream_t st) {
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  char* p = (char*)ws;
  double2* Aws = (double2*)p;   p += al((size_t)l * l * sizeof(double2));
  double2* Vt = (double2*)p;    p += al((size_t)l * l * sizeof(double2));
  double* d = (double*)p;       p += al((size_t)l * sizeof(double));
  double* e = (double*)p;       p += al((size_t)l * sizeof(double));
  double2* tau = (double2*)p;   p += al((size_t)l * sizeof(double2));
  double* lam_s = (double*)p;   p += al((size_t)r * sizeof(double));
  double* z = (double*)p;       p += al((size_t)l * r * sizeof(double));
  double* scratch = (double*)p;
  (void)lam_s;
  int s;
  const size_t abytes = (size_t)l * l * sizeof(double2);
  const bool sm = abytes <= 200 * 1024;
  hicu_allow_max_smem((const void*)hetrd_kernel);
  hetrd_kernel<<<1, 1024, sm ? abytes : 0, st>>>(l, A, Aws, sm, d, e, tau, Vt);
  if ((s = hicu_check_launch("hetrd_kernel"))) return s;
  const int wpb = 8;
  stebz_kernel<<<(r + wpb - 1) / wpb, wpb * 32, 0, st>>>(l, r, d, e, lam);
  if ((s = hicu_check_launch("stebz_kernel"))) return s;
  stein_kernel<<<(r + 63) / 64, 64, 0, st>>>(l, r, d, e, lam, z, scratch);
  if ((s = hicu_check_launch("stein_kernel"))) return s;
  cluster_orth_kernel<<<1, 256, 0, st>>>(l, r, lam, z, 1e-9);
  if ((s = hicu_check_launch("cluster_orth_kernel"))) return s;
  const int bw = 4;
  const size_t smem = (size_t)bw * l * sizeof(double2);
  hicu_allow_max_smem((const void*)back_transform_kernel);
  back_transform_kernel<<<(r + bw - 1) / bw, bw * 32, smem, st>>>(l, r, Vt, tau, z, F);
  return hicu_check_launch("back_transform_kernel");
}
