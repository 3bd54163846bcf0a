// Gram matrix G = H(x)^H H(x) — SIMT reference kernel (fp32 FMA over chunks
// of kFlushRows rows, drained into fp64 register accumulators; fp64 split-K
// reduction).  The drain keeps the fp32 chains short: one split of the C5
// shard spans ~195K rows, where a single fp32 chain measured 1.4e-4 relative
// error against an fp64 Gram (scripts/gram_accuracy.py).  Used for geometries the tcgen05 kernel
// does not cover (general supports, circular axes) and as its cross-check.
//
// No reference function computes G; it equals
// hankel_adjoint_apply(x, hankel_apply(x, I)) (hankel.py:255-391).
#include "common.cuh"

namespace {

constexpr int kTile = 64;    // complex outputs per tile edge
constexpr int kBK = 16;      // rows per smem stage
constexpr int kThreads = 256;
constexpr int kFlushRows = 512;  // fp32 chain length before draining into fp64

struct GramPlan {
  int ntile;       // tiles per edge
  int npairs;      // upper-triangle tile pairs
  int splits;      // split-K factor
  int64_t rows_per_split;
};

GramPlan gram_plan(const DevGeom& g) {
  GramPlan p;
  p.ntile = (g.n + kTile - 1) / kTile;
  p.npairs = p.ntile * (p.ntile + 1) / 2;
  const int target = hicu_sm_count() * 3;
  int splits = (target + p.npairs - 1) / p.npairs;
  int64_t max_splits = (g.s + 255) / 256;
  if (splits > max_splits) splits = (int)max_splits;
  if (splits < 1) splits = 1;
  p.rows_per_split = (g.s + splits - 1) / splits;
  p.splits = (int)((g.s + p.rows_per_split - 1) / p.rows_per_split);
  return p;
}

template <bool CIRC>
__global__ void __launch_bounds__(kThreads, 2)
gram_simt_kernel(DevGeom g, const float2* __restrict__ x, int ntile, int64_t rows_per_split,
                 double2* __restrict__ partials) {
  hicu_pdl_entry();
  __shared__ float2 As[kBK][kTile];
  __shared__ float2 Bs[kBK][kTile];
  __shared__ int64_t rbase[kBK];
  __shared__ int rcc[kBK][HICU_MAX_NDIM];

  // tile pair (ti <= tj) from the linear upper-triangle index
  int t = blockIdx.x, ti = 0;
  while (t >= ntile - ti) { t -= ntile - ti; ++ti; }
  const int tj = ti + t;
  const int split = blockIdx.y;
  const int64_t r0 = (int64_t)split * rows_per_split;
  int64_t r1 = r0 + rows_per_split;
  if (r1 > g.s) r1 = g.s;

  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  // fp64 drain targets in shared memory ([slot][thread], conflict-free), so
  // the fp32 tile keeps the register budget of two CTAs per SM
  extern __shared__ double2 acc64[];
  float2 acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      acc[a][b] = cf(0.f, 0.f);
      acc64[(a * 4 + b) * kThreads + threadIdx.x] = cd(0.0, 0.0);
    }

  // outer blocks of kFlushRows rows, drained into fp64 after each block
  for (int64_t rb = r0; rb < r1; rb += kFlushRows) {
    const int64_t re = rb + kFlushRows < r1 ? rb + kFlushRows : r1;
    for (int64_t rc = rb; rc < re; rc += kBK) {
      if (threadIdx.x < kBK) {
        const int64_t i = rc + threadIdx.x;
        int cc[HICU_MAX_NDIM];
        rbase[threadIdx.x] = (i < r1) ? row_base(g, i, cc) : -1;
        if (CIRC)
          for (int c = 0; c < g.ncirc; ++c) rcc[threadIdx.x][c] = cc[c];
      }
      __syncthreads();
      // 2 * kBK * kTile elements, 8 per thread
#pragma unroll
      for (int e = 0; e < (2 * kBK * kTile) / kThreads; ++e) {
        const int idx = threadIdx.x + e * kThreads;
        const int which = idx / (kBK * kTile);
        const int rem = idx % (kBK * kTile);
        const int row = rem / kTile, col = rem % kTile;
        const int kap = (which == 0 ? ti : tj) * kTile + col;
        float2 v = cf(0.f, 0.f);
        const int64_t b = rbase[row];
        if (b >= 0 && kap < g.n) {
          int64_t addr = b + g.koff[kap];
          if (CIRC) addr += circ_part(g, rcc[row], g.pos + (size_t)kap * g.ndim);
          v = __ldg(x + addr);
        }
        if (which == 0) As[row][col] = v; else Bs[row][col] = v;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kBK; ++kk) {
        float2 a[4], b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[q] = As[kk][ty * 4 + q];
          b[q] = Bs[kk][tx * 4 + q];
        }
#pragma unroll
        for (int qa = 0; qa < 4; ++qa)
#pragma unroll
          for (int qb = 0; qb < 4; ++qb) cfmac(acc[qa][qb], a[qa], b[qb]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        double2& d = acc64[(a * 4 + b) * kThreads + threadIdx.x];
        d = d + cd(acc[a][b].x, acc[a][b].y);
        acc[a][b] = cf(0.f, 0.f);
      }
  }
  double2* out = partials + (size_t)split * g.n * g.n;
#pragma unroll
  for (int qa = 0; qa < 4; ++qa) {
    const int ra = ti * kTile + ty * 4 + qa;
    if (ra >= g.n) continue;
#pragma unroll
    for (int qb = 0; qb < 4; ++qb) {
      const int cb = tj * kTile + tx * 4 + qb;
      if (cb >= g.n) continue;
      out[(size_t)ra * g.n + cb] = acc64[(qa * 4 + qb) * kThreads + threadIdx.x];
    }
  }
}

// G[a][b] (a <= b) = sum over splits in order; G[b][a] = conj.
__global__ void gram_reduce_kernel(int n, int splits, const double2* __restrict__ partials,
                                   double2* __restrict__ G) {
  hicu_pdl_entry();
  const int64_t total = (int64_t)n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(e / n), b = (int)(e % n);
    if (a > b) continue;
    double2 s = cd(0.0, 0.0);
    for (int k = 0; k < splits; ++k) s = s + partials[(size_t)k * total + e];
    if (a == b) {
      G[e] = cd(s.x, 0.0);
    } else {
      G[e] = s;
      G[(size_t)b * n + a] = cd(s.x, -s.y);
    }
  }
}

}  // namespace

size_t hicu_gram_simt_workspace(const DevGeom& g) {
  GramPlan p = gram_plan(g);
  return (size_t)p.splits * g.n * g.n * sizeof(double2);
}

int hicu_gram_simt(const DevGeom& g, const float2* x, double2* G, void* ws, size_t ws_bytes, cudaStream_t st) {
  GramPlan p = gram_plan(g);
  const size_t need = (size_t)p.splits * g.n * g.n * sizeof(double2);
  if (ws_bytes < need) return hicu_set_error(HICU_ERR_WORKSPACE, "gram: workspace too small");
  dim3 grid(p.npairs, p.splits);
  const size_t dsm = (size_t)16 * kThreads * sizeof(double2);
  if (g.ncirc > 0) {
    hicu_allow_max_smem((const void*)gram_simt_kernel<true>);
    hicu_launch(gram_simt_kernel<true>, grid, kThreads, dsm, st, g, x, p.ntile, p.rows_per_split, (double2*)ws);
  } else {
    hicu_allow_max_smem((const void*)gram_simt_kernel<false>);
    hicu_launch(gram_simt_kernel<false>, grid, kThreads, dsm, st, g, x, p.ntile, p.rows_per_split, (double2*)ws);
  }
  int s = hicu_check_launch("gram_simt_kernel");
  if (s) return s;
  int64_t total = (int64_t)g.n * g.n;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  hicu_launch(gram_reduce_kernel, blocks, 256, 0, st, g.n, p.splits, (const double2*)ws, G);
  return hicu_check_launch("gram_reduce_kernel");
}
