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
  __shared__ __align__(16) float2 As[kBK][kTile];
  __shared__ __align__(16) float2 Bs[kBK][kTile];
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

  // Gather of one kBK-row block into registers (8 values per thread); the
  // next block's gather is issued before this block's products so the L2
  // latency overlaps the FMAs (one block at a time left the SM idle between
  // the gather and the products).  Macros, not device lambdas (a lambda
  // capturing shared arrays miscompiled).
  constexpr int kPer = (2 * kBK * kTile) / kThreads;
  float2 pre[kPer];
#define GRAM_SIMT_BASES(rc_)                                                         \
  if (threadIdx.x < kBK) {                                                           \
    const int64_t i_ = (rc_) + threadIdx.x;                                          \
    int cc_[HICU_MAX_NDIM];                                                          \
    rbase[threadIdx.x] = (i_ < r1) ? row_base(g, i_, cc_) : -1;                      \
    if (CIRC)                                                                        \
      for (int c_ = 0; c_ < g.ncirc; ++c_) rcc[threadIdx.x][c_] = cc_[c_];           \
  }
#define GRAM_SIMT_GATHER()                                                           \
  _Pragma("unroll") for (int e = 0; e < kPer; ++e) {                                 \
    const int idx = threadIdx.x + e * kThreads;                                      \
    const int which = idx / (kBK * kTile);                                           \
    const int rem = idx % (kBK * kTile);                                             \
    const int row = rem / kTile, col = rem % kTile;                                  \
    const int kap = (which == 0 ? ti : tj) * kTile + col;                            \
    float2 v = cf(0.f, 0.f);                                                         \
    const int64_t bb = rbase[row];                                                   \
    if (bb >= 0 && kap < g.n) {                                                      \
      int64_t addr = bb + g.koff[kap];                                               \
      if (CIRC) addr += circ_part(g, rcc[row], g.pos + (size_t)kap * g.ndim);        \
      v = __ldg(x + addr);                                                           \
    }                                                                                \
    pre[e] = v;                                                                      \
  }
  if (r0 < r1) {
    GRAM_SIMT_BASES(r0)
    __syncthreads();
    GRAM_SIMT_GATHER()
  }
  int since = 0;
  for (int64_t rc = r0; rc < r1; rc += kBK) {
    __syncthreads();  // previous block's products done with As/Bs and rbase
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int idx = threadIdx.x + e * kThreads;
      const int which = idx / (kBK * kTile);
      const int rem = idx % (kBK * kTile);
      const int row = rem / kTile, col = rem % kTile;
      if (which == 0) As[row][col] = pre[e]; else Bs[row][col] = pre[e];
    }
    if (rc + kBK < r1) GRAM_SIMT_BASES(rc + kBK)
    __syncthreads();
    if (rc + kBK < r1) GRAM_SIMT_GATHER()  // in flight during the products below
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      const float4* ar = reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4* br = reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float4 a01 = ar[0], a23 = ar[1], b01 = br[0], b23 = br[1];
      const float2 a[4] = {cf(a01.x, a01.y), cf(a01.z, a01.w), cf(a23.x, a23.y), cf(a23.z, a23.w)};
      const float2 bq[4] = {cf(b01.x, b01.y), cf(b01.z, b01.w), cf(b23.x, b23.y), cf(b23.z, b23.w)};
#pragma unroll
      for (int qa = 0; qa < 4; ++qa)
#pragma unroll
        for (int qb = 0; qb < 4; ++qb) cfmac(acc[qa][qb], a[qa], bq[qb]);
    }
    since += kBK;
    if (since == kFlushRows || rc + kBK >= r1) {  // drain into fp64 every kFlushRows rows and at the end
      since = 0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          double2& d = acc64[(a * 4 + b) * kThreads + threadIdx.x];
          d = d + cd(acc[a][b].x, acc[a][b].y);
          acc[a][b] = cf(0.f, 0.f);
        }
    }
  }
#undef GRAM_SIMT_GATHER
#undef GRAM_SIMT_BASES
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
