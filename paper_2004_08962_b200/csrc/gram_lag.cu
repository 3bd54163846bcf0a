// Shift-structured Gram G = H^H H of the multi-level Hankel (convolution)
// matrix H(x) (reference analogue:
// hankel_adjoint_apply(x, hankel_apply(x, I)), hankel.py:255-391).
//
// Column (t, c) of H is the k-space window x[i + t, c] for region rows i, so
//   G[(t,c),(t',c')] = sum_{i in R} conj(x[i+t, c]) x[i+t', c']
//                    = sum_{j in R+t} conj(x[j, c]) x[j+d, c'],   d = t' - t.
// Every entry is a "lag-d" coil correlation summed over the shifted box R+t.
// Along each spatial axis the positions of interest [o, o+e+K-1) fall into
// at most 2K-1 classes of equal tap membership (positions p with the same set
// {t : o+t <= p < o+t+e}): K-1 single left-edge positions, one long core
// [o+K-1, o+e) holding every tap, K-1 single right-edge positions (circular
// axes: one class).  So with T[d][cell] = sum over the positions of one cell
// (a product of per-axis classes) of conj(x[j]) x[j+d] (an Nc x Nc block),
//   G[(t,c),(t+d,c')] = sum_{cells containing t} T[d][cell][c][c'].
// Only lags in the lexicographic half-space are formed (G is Hermitian): the
// dense Gram's n(n+1)/2 x s complex MACs (n = taps x coils) become
// ~((2K-1)^d / 2) x Nc^2 x (positions) -- 21x less work for the 5x5x5x8
// kernels of C4/C5, 8x for 5x5x8, 14x for 7x7x10.
//
// Kernels (fp32 FMA products, fp32 per-CTA partials of a few hundred terms,
// fp64 everywhere after; fixed summation order, no atomics: deterministic):
//   lag_core_kernel   the long last-axis core class: lines of k-space staged
//                     in shared memory (coil planes, cp.async double buffer),
//                     one warp per (last-axis lag, coil block), lanes over
//                     positions, an Nc x CB register block of accumulators;
//   lag_edge_kernel   the short last-axis classes (edge positions);
//   lag_reduceU_kernel fixed-order fp64 sums of the chunk partials, folded
//                     over the line-axis classes containing each tap;
//   lag_axis_kernel   the same containment sum over each outer axis;
//   lag_gather_kernel G from the per-(lag, tap) table (Hermitian by construction).
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "tc_common.cuh"

namespace {

constexpr int kMaxL = 3;        // spatial axes (outer axes <= 2)
constexpr int kMaxK = 8;        // kernel extent per spatial axis
constexpr int kMaxCls = 2 * kMaxK - 1;
constexpr int kMaxBlocks = kMaxCls * kMaxCls;
constexpr int kMaxOl = (kMaxCls * kMaxCls + 1) / 2;
constexpr int kCoreThreadsMax = 512;
constexpr int kCoreStages = 4;   // lines in flight (cp.async ring)
constexpr int kEdgeThreads = 256;
constexpr int kLinesPerChunkA = 64;
constexpr int kLinesPerChunkB = 1024;
// tensor-core core class: per line, fp16 hi/lo polyphase operand tiles
// [A_hi 8 KB | A_lo 8 KB | B_hi 16 KB | B_lo 16 KB] (K-major SWIZZLE_64B images)
constexpr int kTcLineBytes = 49152;
constexpr int kTcStages = 4;        // line pairs in flight (48 KB each)
constexpr int kTcPPD = 4;           // line pairs per TMEM accumulation chain (12 MMAs each)
constexpr int kTcEpiWarps = 8;
constexpr int kTcThreads = (2 + kTcEpiWarps) * 32;
constexpr int kTcCols = 80;         // TMEM columns each epilogue thread drains

struct LagParams {
  int L;           // spatial axes
  int perm[kMaxL]; // plan axis a is geometry axis perm[a]; the last plan axis (the "line" axis) is the
                   // spatial axis with the longest core class, so lines are long whatever the layout
  int NC, CB, NCB; // coils, coil rows per warp block, NC / CB
  int64_t N[kMaxL];
  int64_t cstride[kMaxL];  // element (complex) stride of each spatial axis
  int K[kMaxL];
  int circ[kMaxL];
  int ncls[kMaxL];
  int cls_beg[kMaxL][kMaxCls], cls_end[kMaxL][kMaxCls], cls_lo[kMaxL][kMaxCls], cls_hi[kMaxL][kMaxCls];
  int core_cls;    // index of the core class on the last axis (-1: none)
  int NB;          // outer class blocks
  int nol;         // outer lags (half-plane)
  int ol_d[kMaxOl][2];
  int ol_index[kMaxCls][kMaxCls];
  int DZ;          // last-axis lags: dz in [-(K-1), K-1]
  // core kernel
  int GZ, NG;      // lags per CTA, groups
  int CA;          // chunks per (ol, group) summed over blocks
  int chunksA[kMaxBlocks + 1];  // prefix
  int lpcA;
  int64_t P;       // core positions per line
  int64_t c0;      // first core position
  // edge kernel
  int NE;          // non-core last-axis classes
  int edge_cls[kMaxCls];
  int NQ, QB, NQB, LL;
  int CBt;         // chunks per (ol, qblock) summed over blocks
  int chunksB[kMaxBlocks + 1];
  int lpcB;
  int NCL;         // last-axis classes
};

struct LagPlan {
  bool ok = false;
  bool tc = false;  // core class on the tensor cores (lagtc_* kernels)
  LagParams p;
  size_t t_off = 0, a_off = 0, b_off = 0, bytes = 0;
  size_t prep_off = 0, amax_off = 0;  // tensor path: per-line operand tiles, amax partials
  int64_t lines_all = 0;
  int64_t nT = 0;   // complex entries of T
  int64_t nU = 0, nV = 0, nW = 0;  // containment-sum tables (U: line axis, V: + axis 1, W: all axes)
  size_t u_off = 0, v_off = 0, w_off = 0;
  int64_t nA = 0, nB = 0;  // CTAs
  size_t smemA = 0, smemB = 0;
  int threadsA = 0;
};

// coil rows per warp: two Nc x CB blocks of fp32x2 accumulators (CB * Nc <= 20,
// so 16 warps of <= 128 registers fit one SM)
__host__ __device__ constexpr int cb_for(int nc) {
  int best = 1;
  for (int cb = 1; cb <= nc; ++cb)
    if (nc % cb == 0 && cb * nc <= 20) best = cb;
  return best;
}
int choose_cb(int nc) { return cb_for(nc); }

// one k-space position (Nc complex) per shared-memory row, padded to an odd
// number of 16-byte chunks: lanes reading consecutive rows hit distinct banks
__host__ __device__ constexpr int row_bytes(int nc) {
  return 16 * (((nc * 8 + 15) / 16) % 2 ? (nc * 8 + 15) / 16 : (nc * 8 + 15) / 16 + 1);
}

// acc += conj(a) * b with two packed fp32x2 FMAs (FFMA2), both with a
// broadcast scalar operand so no register pair is rebuilt per use:
//   acc += a.x * (b.x, b.y) + a.y * (b.y, -b.x)      (bn = (b.y, -b.x), once per b)
__device__ __forceinline__ float2 cfmac2(float2 acc, float2 a, float2 b, float2 bn) {
  acc = __ffma2_rn(make_float2(a.x, a.x), b, acc);
  return __ffma2_rn(make_float2(a.y, a.y), bn, acc);
}

void axis_classes(int64_t N, int64_t o, int64_t e, int K, bool circ, LagParams& p, int a) {
  if (circ) {
    p.ncls[a] = 1;
    p.cls_beg[a][0] = 0;
    p.cls_end[a][0] = (int)N;
    p.cls_lo[a][0] = 0;
    p.cls_hi[a][0] = K - 1;
    return;
  }
  int nc = 0;
  for (int64_t q = o; q < o + e + K - 1; ++q) {
    const int lo = (int)std::max<int64_t>(0, q - o - e + 1), hi = (int)std::min<int64_t>(K - 1, q - o);
    if (nc > 0 && p.cls_lo[a][nc - 1] == lo && p.cls_hi[a][nc - 1] == hi && p.cls_end[a][nc - 1] == q) {
      p.cls_end[a][nc - 1] = (int)q + 1;
      continue;
    }
    if (nc >= kMaxCls) {
      p.ncls[a] = -1;
      return;
    }
    p.cls_beg[a][nc] = (int)q;
    p.cls_end[a][nc] = (int)q + 1;
    p.cls_lo[a][nc] = lo;
    p.cls_hi[a][nc] = hi;
    ++nc;
  }
  p.ncls[a] = nc;
}

LagPlan make_plan(const DevGeom& g) {
  LagPlan pl;
  LagParams& p = pl.p;
  memset(&p, 0, sizeof(p));
  if (g.nc < 1 || g.nc > 16) return pl;
  const int L = g.ndim - 1;
  if (L < 1 || L > kMaxL) return pl;
  if (g.nsp * g.nc != g.n) return pl;
  p.L = L;
  p.NC = g.nc;
  p.CB = choose_cb(g.nc);
  p.NCB = g.nc / p.CB;
  bool circ[kMaxL] = {false, false, false};
  for (int c = 0; c < g.ncirc; ++c) {
    if (g.circ_axes[c] >= L) return pl;
    circ[g.circ_axes[c]] = true;
  }
  // line axis: the spatial axis with the longest core class (positions of
  // interest minus the 2(K-1) edge positions; the whole axis when circular)
  int line = L - 1;
  int64_t best = -1;
  for (int a = L - 1; a >= 0; --a) {
    const int64_t K = g.kext[a];
    const int64_t core = circ[a] ? g.dims[a] : g.rext[a] - K + 1;
    if (core > best) {
      best = core;
      line = a;
    }
  }
  {
    int k = 0;
    for (int a = 0; a < L; ++a)
      if (a != line) p.perm[k++] = a;
    p.perm[L - 1] = line;
  }
  for (int a = 0; a < L; ++a) {
    const int ga = p.perm[a];
    const int K = (int)g.kext[ga];
    if (K < 1 || K > kMaxK) return pl;
    p.N[a] = g.dims[ga];
    p.cstride[a] = g.stride[ga];
    p.K[a] = K;
    p.circ[a] = circ[ga] ? 1 : 0;
    if (circ[ga] && K > g.dims[ga]) return pl;
    axis_classes(g.dims[ga], g.roff[ga], g.rext[ga], K, circ[ga], p, a);
    if (p.ncls[a] < 1) return pl;
  }
  // outer blocks and lags
  const int la = L - 1;
  p.NB = 1;
  for (int a = 0; a < la; ++a) p.NB *= p.ncls[a];
  const int D0 = la >= 1 ? 2 * p.K[0] - 1 : 1, D1 = la >= 2 ? 2 * p.K[1] - 1 : 1;
  p.nol = 0;
  for (int i = 0; i < kMaxCls; ++i)
    for (int j = 0; j < kMaxCls; ++j) p.ol_index[i][j] = -1;
  for (int i = 0; i < D0; ++i)
    for (int j = 0; j < D1; ++j) {
      const int d0 = la >= 1 ? i - (p.K[0] - 1) : 0, d1 = la >= 2 ? j - (p.K[1] - 1) : 0;
      const bool pos = d0 > 0 || (d0 == 0 && d1 >= 0);
      if (!pos) continue;
      p.ol_d[p.nol][0] = d0;
      p.ol_d[p.nol][1] = d1;
      p.ol_index[i][j] = p.nol;
      ++p.nol;
    }
  const int KL = p.K[la];
  p.DZ = 2 * KL - 1;
  p.NCL = p.ncls[la];
  p.core_cls = -1;
  for (int c = 0; c < p.NCL; ++c)
    if (p.cls_lo[la][c] == 0 && p.cls_hi[la][c] == KL - 1 && p.cls_end[la][c] - p.cls_beg[la][c] >= 1) p.core_cls = c;
  p.NE = 0;
  for (int c = 0; c < p.NCL; ++c)
    if (c != p.core_cls) p.edge_cls[p.NE++] = c;
  auto block_lines = [&](int b) -> int64_t {
    int64_t nl = 1;
    int r = b;
    for (int a = la - 1; a >= 0; --a) {
      const int k = r % p.ncls[a];
      r /= p.ncls[a];
      nl *= p.cls_end[a][k] - p.cls_beg[a][k];
    }
    return nl;
  };
  // tensor-core core class (lagtc_core_kernel): 8 coils, a non-circular line
  // axis of at most 256 positions and at most 9 last-axis lags
  pl.tc = g.nc == 8 && !p.circ[la] && p.K[la] <= 5 && p.N[la] <= 256 && p.core_cls >= 0 &&
          !(g.flags & HICU_GEOM_FORCE_FFMA_LAG);
  // core kernel
  if (p.core_cls >= 0) {
    p.P = p.cls_end[la][p.core_cls] - p.cls_beg[la][p.core_cls];
    p.c0 = p.cls_beg[la][p.core_cls];
    const int wmax = kCoreThreadsMax / 32;
    int gz = std::max(1, wmax / p.NCB);
    p.NG = (p.DZ + gz - 1) / gz;
    p.GZ = (p.DZ + p.NG - 1) / p.NG;
    if (pl.tc) {  // one CTA covers all DZ last-axis lags of its outer lag
      p.NG = 1;
      p.GZ = p.DZ;
    }
    p.lpcA = kLinesPerChunkA;
    p.chunksA[0] = 0;
    for (int b = 0; b < p.NB; ++b)
      p.chunksA[b + 1] = p.chunksA[b] + (int)((block_lines(b) + p.lpcA - 1) / p.lpcA);
    p.CA = p.chunksA[p.NB];
    pl.nA = (int64_t)p.nol * p.NG * p.CA;
    pl.threadsA = 32 * p.GZ * p.NCB;
    pl.smemA = (size_t)kCoreStages * row_bytes(p.NC) * (2 * p.P + p.GZ);
    if (!pl.tc && pl.smemA > (size_t)200 * 1024) return pl;
  }
  // edge kernel
  if (p.NE > 0) {
    p.NQ = p.NE * p.DZ * p.NCB;
    p.QB = std::min(p.NQ, kEdgeThreads);
    p.NQB = (p.NQ + p.QB - 1) / p.QB;
    p.LL = std::max(1, kEdgeThreads / p.QB);
    p.lpcB = kLinesPerChunkB;
    p.chunksB[0] = 0;
    for (int b = 0; b < p.NB; ++b)
      p.chunksB[b + 1] = p.chunksB[b] + (int)((block_lines(b) + p.lpcB - 1) / p.lpcB);
    p.CBt = p.chunksB[p.NB];
    pl.nB = (int64_t)p.nol * p.NQB * p.CBt;
    pl.smemB = (size_t)p.QB * p.CB * p.NC * sizeof(float2);
  }
  pl.nT = 0;  // T is never stored: lag_reduceU folds the line-axis classes directly
  auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
  pl.t_off = 0;
  pl.a_off = 0;
  pl.b_off = pl.a_off + al((size_t)pl.nA * p.GZ * p.NC * p.NC * sizeof(float2));
  pl.bytes = pl.b_off + al((size_t)pl.nB * p.QB * p.CB * p.NC * sizeof(float2));
  {
    const int NC2 = p.NC * p.NC, KL = p.K[la];
    const int K0 = la >= 1 ? p.K[0] : 1, K1 = la >= 2 ? p.K[1] : 1;
    pl.nU = (int64_t)p.nol * p.DZ * p.NB * KL * NC2;
    pl.nV = la >= 2 ? (int64_t)p.nol * p.DZ * p.ncls[0] * K1 * KL * NC2 : 0;
    pl.nW = (int64_t)p.nol * p.DZ * K0 * K1 * KL * NC2;
    pl.u_off = al(pl.bytes);
    pl.v_off = pl.u_off + al(pl.nU * sizeof(double2));
    pl.w_off = pl.v_off + al(pl.nV * sizeof(double2));
    pl.bytes = pl.w_off + al(pl.nW * sizeof(double2));
  }
  if (pl.tc) {
    pl.lines_all = 1;
    for (int a = 0; a < la; ++a) pl.lines_all *= p.N[a];
    pl.amax_off = al(pl.bytes);
    pl.prep_off = pl.amax_off + 4096;
    pl.bytes = pl.prep_off + (size_t)pl.lines_all * kTcLineBytes;
  }
  pl.ok = true;
  return pl;
}

// outer coordinates of line li of block b; returns false when the neighbour
// block (shifted by the outer lag) leaves a non-circular axis
__device__ __forceinline__ void block_ranges(const LagParams& P, int b, int (&beg)[2], int (&len)[2]) {
  const int la = P.L - 1;
  beg[0] = beg[1] = 0;
  len[0] = len[1] = 1;
  int r = b;
  for (int a = la - 1; a >= 0; --a) {
    const int k = r % P.ncls[a];
    r /= P.ncls[a];
    beg[a] = P.cls_beg[a][k];
    len[a] = P.cls_end[a][k] - P.cls_beg[a][k];
  }
}

__device__ __forceinline__ bool neighbour_ok(const LagParams& P, const int (&beg)[2], const int (&len)[2], int ol) {
  const int la = P.L - 1;
  for (int a = 0; a < la; ++a) {
    if (P.circ[a]) continue;
    const int d = P.ol_d[ol][a];
    if (beg[a] + d < 0 || beg[a] + len[a] - 1 + d >= P.N[a]) return false;
  }
  return true;
}

__device__ __forceinline__ void line_offsets(const LagParams& P, const int (&beg)[2], const int (&len)[2], int ol,
                                             int64_t li, int64_t& base, int64_t& nbr) {
  const int la = P.L - 1;
  int64_t q[2];
  if (la == 2) {
    q[0] = li / len[1];
    q[1] = li % len[1];
  } else {
    q[0] = li;
    q[1] = 0;
  }
  base = 0;
  nbr = 0;
  for (int a = 0; a < la; ++a) {
    const int64_t pa = beg[a] + q[a];
    int64_t pn = pa + P.ol_d[ol][a];
    if (P.circ[a]) {
      if (pn < 0) pn += P.N[a];
      if (pn >= P.N[a]) pn -= P.N[a];
    }
    base += pa * P.cstride[a];
    nbr += pn * P.cstride[a];
  }
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}

// Grid: one CTA per (line chunk of a class block) x (outer lag, last-axis lag
// group), the (lag, group) index fastest so CTAs resident together share
// their k-space lines in L2.  Accumulation: acc += conj(a) b for a = base
// position (CB coils of this warp's block), b = neighbour position + dz (all
// Nc coils), as two broadcast-scalar FFMA2 chains per product
//   accR += a.x * (b.x, b.y),  accI += a.y * (b.x, b.y)
//   conj(a) b = (accR.x + accI.y, accR.y - accI.x)
// so no operand pair is swapped or negated in the inner loop.
template <int NC, int CB>
__global__ void __launch_bounds__(kCoreThreadsMax, 1)
lag_core_kernel(const __grid_constant__ LagParams P, const float2* __restrict__ x, float2* __restrict__ part) {
  hicu_pdl_entry();
  constexpr int RB = row_bytes(NC);
  constexpr bool V16 = (NC % 2) == 0;
  extern __shared__ __align__(16) uint8_t lsm[];
  const int64_t bid = blockIdx.x;
  const int nlg = P.nol * P.NG;
  const int rowblk = (int)(bid / nlg);
  const int olg = (int)(bid % nlg);
  const int ol = olg / P.NG, gzi = olg % P.NG;
  int b = 0;
  while (P.chunksA[b + 1] <= rowblk) ++b;
  const int chunk = rowblk - P.chunksA[b];
  const int dz_lo = gzi * P.GZ - (P.K[P.L - 1] - 1);
  const int gz_n = min(P.GZ, P.DZ - gzi * P.GZ);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dzi = warp / P.NCB, cbi = warp % P.NCB;
  float2* out = part + (size_t)bid * P.GZ * NC * NC;
  int beg[2], len[2];
  block_ranges(P, b, beg, len);
  const int64_t nlines = (int64_t)len[0] * len[1];
  const int64_t l0 = (int64_t)chunk * P.lpcA, l1 = min(nlines, l0 + P.lpcA);
  if (!neighbour_ok(P, beg, len, ol)) {
    for (int i = threadIdx.x; i < P.GZ * NC * NC; i += blockDim.x) out[i] = cf(0.f, 0.f);
    return;
  }
  const int la = P.L - 1;
  const int pn = (int)P.P;
  const int nw = pn + P.GZ - 1;               // neighbour rows per buffer
  const int nwa = pn + gz_n - 1;              // neighbour rows the active lags read
  const size_t bufsz = (size_t)(pn + nw) * RB;
  const int64_t NL = P.N[la];
  const int64_t ls = P.cstride[la];  // element stride along the line axis
  auto stage = [&](int64_t li, int buf) {
    int64_t base, nbr;
    line_offsets(P, beg, len, ol, li, base, nbr);
    uint8_t* sb = lsm + (size_t)buf * bufsz;
    uint8_t* sn = sb + (size_t)pn * RB;
    if (V16) {
      constexpr int H = NC / 2;  // 16-byte chunks per position
      for (int e = threadIdx.x; e < pn * H; e += blockDim.x) {
        const int j = e / H, k = e % H;
        cp_async16(sb + j * RB + k * 16, x + base + (P.c0 + j) * ls + 2 * k);
      }
      for (int e = threadIdx.x; e < nwa * H; e += blockDim.x) {
        const int j = e / H, k = e % H;
        int64_t q = P.c0 + dz_lo + j;
        if (P.circ[la]) {
          q %= NL;
          if (q < 0) q += NL;
        }
        cp_async16(sn + j * RB + k * 16, x + nbr + q * ls + 2 * k);
      }
    } else {
      for (int e = threadIdx.x; e < pn * NC; e += blockDim.x) {
        const int j = e / NC, c = e % NC;
        cp_async8(sb + j * RB + c * 8, x + base + (P.c0 + j) * ls + c);
      }
      for (int e = threadIdx.x; e < nwa * NC; e += blockDim.x) {
        const int j = e / NC, c = e % NC;
        int64_t q = P.c0 + dz_lo + j;
        if (P.circ[la]) {
          q %= NL;
          if (q < 0) q += NL;
        }
        cp_async8(sn + j * RB + c * 8, x + nbr + q * ls + c);
      }
    }
  };
  float2 accR[CB][NC], accI[CB][NC];
#pragma unroll
  for (int a = 0; a < CB; ++a)
#pragma unroll
    for (int c = 0; c < NC; ++c) accR[a][c] = accI[a][c] = cf(0.f, 0.f);
  const bool active = dzi < gz_n;
  // ring of kCoreStages line buffers: lines li+1 .. li+kCoreStages-1 are in
  // flight while line li is consumed (one commit group per line, maybe empty)
#pragma unroll
  for (int k = 0; k < kCoreStages - 1; ++k) {
    if (l0 + k < l1) stage(l0 + k, k);
    cp_async_commit();
  }
  for (int64_t li = l0; li < l1; ++li) {
    const int buf = (int)((li - l0) % kCoreStages);
    cp_async_wait<kCoreStages - 2>();
    __syncthreads();
    // refill the buffer consumed in the previous iteration (free after the barrier)
    if (li + kCoreStages - 1 < l1) stage(li + kCoreStages - 1, (int)((li - l0 + kCoreStages - 1) % kCoreStages));
    cp_async_commit();
    if (active) {
      const uint8_t* sb = lsm + (size_t)buf * bufsz + cbi * CB * 8;
      const uint8_t* sn = lsm + (size_t)buf * bufsz + (size_t)pn * RB + dzi * RB;
      for (int j = lane; j < pn; j += 32) {
        float2 a[CB], v[NC];
#pragma unroll
        for (int q = 0; q < CB; ++q) a[q] = *(const float2*)(sb + j * RB + q * 8);
        if (V16) {
#pragma unroll
          for (int k = 0; k < NC / 2; ++k) {
            const float4 w = *(const float4*)(sn + j * RB + k * 16);
            v[2 * k] = make_float2(w.x, w.y);
            v[2 * k + 1] = make_float2(w.z, w.w);
          }
        } else {
#pragma unroll
          for (int c = 0; c < NC; ++c) v[c] = *(const float2*)(sn + j * RB + c * 8);
        }
#pragma unroll
        for (int q = 0; q < CB; ++q)
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            accR[q][c] = __ffma2_rn(make_float2(a[q].x, a[q].x), v[c], accR[q][c]);
            accI[q][c] = __ffma2_rn(make_float2(a[q].y, a[q].y), v[c], accI[q][c]);
          }
      }
    }
  }
  cp_async_wait<0>();
  // conj(a) b, then a fixed-order warp reduction of the lanes' partial sums
#pragma unroll
  for (int q = 0; q < CB; ++q)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      float2 v = make_float2(accR[q][c].x + accI[q][c].y, accR[q][c].y - accI[q][c].x);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
      }
      accR[q][c] = v;
    }
  if (lane == 0 && dzi < P.GZ) {
#pragma unroll
    for (int q = 0; q < CB; ++q)
#pragma unroll
      for (int c = 0; c < NC; ++c)
        out[((size_t)dzi * NC + cbi * CB + q) * NC + c] = active ? accR[q][c] : cf(0.f, 0.f);
  }
}

template <int NC, int CB>
__global__ void __launch_bounds__(kEdgeThreads)
lag_edge_kernel(const __grid_constant__ LagParams P, const float2* __restrict__ x, float2* __restrict__ part) {
  hicu_pdl_entry();
  extern __shared__ __align__(16) float2 esm[];
  const int64_t bid = blockIdx.x;
  const int olq = (int)(bid / P.CBt);
  const int rem = (int)(bid % P.CBt);
  const int ol = olq / P.NQB, qb = olq % P.NQB;
  int b = 0;
  while (P.chunksB[b + 1] <= rem) ++b;
  const int chunk = rem - P.chunksB[b];
  const int tq = threadIdx.x % P.QB, ll = threadIdx.x / P.QB;
  const int q = qb * P.QB + tq;
  const bool qok = q < P.NQ && ll < P.LL;
  const int e = q / (P.DZ * P.NCB), dzi = (q / P.NCB) % P.DZ, cbi = q % P.NCB;
  const int la = P.L - 1;
  const int dz = dzi - (P.K[la] - 1);
  int beg[2], len[2];
  block_ranges(P, b, beg, len);
  const int64_t nlines = (int64_t)len[0] * len[1];
  const int64_t l0 = (int64_t)chunk * P.lpcB, l1 = min(nlines, l0 + P.lpcB);
  const bool ok = neighbour_ok(P, beg, len, ol);
  float2 acc[CB][NC];
#pragma unroll
  for (int a = 0; a < CB; ++a)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[a][c] = cf(0.f, 0.f);
  if (ok && qok) {
    const int cls = P.edge_cls[e];
    const int pb = P.cls_beg[la][cls], pe = P.cls_end[la][cls];
    const int64_t cs = P.cstride[la];
    for (int64_t li = l0 + ll; li < l1; li += P.LL) {
      int64_t base, nbr;
      line_offsets(P, beg, len, ol, li, base, nbr);
      for (int pz = pb; pz < pe; ++pz) {
        const int64_t pn = (int64_t)pz + dz;
        if (pn < 0 || pn >= P.N[la]) continue;
        float2 a[CB];
#pragma unroll
        for (int t = 0; t < CB; ++t) a[t] = x[base + pz * cs + cbi * CB + t];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const float2 v = x[nbr + pn * cs + c];
          const float2 vn = make_float2(v.y, -v.x);
#pragma unroll
          for (int t = 0; t < CB; ++t) acc[t][c] = cfmac2(acc[t][c], a[t], v, vn);
        }
      }
    }
  }
  // fixed-order reduction over the line lanes through shared memory
  float2* red = esm;
  for (int r = 1; r < P.LL; ++r) {
    if (ll == r && qok) {
#pragma unroll
      for (int t = 0; t < CB; ++t)
#pragma unroll
        for (int c = 0; c < NC; ++c) red[((size_t)tq * CB + t) * NC + c] = acc[t][c];
    }
    __syncthreads();
    if (ll == 0 && qok) {
#pragma unroll
      for (int t = 0; t < CB; ++t)
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[t][c] = acc[t][c] + red[((size_t)tq * CB + t) * NC + c];
    }
    __syncthreads();
  }
  if (ll == 0 && qok) {
    float2* out = part + ((size_t)bid * P.QB + tq) * CB * NC;
#pragma unroll
    for (int t = 0; t < CB; ++t)
#pragma unroll
      for (int c = 0; c < NC; ++c) out[t * NC + c] = acc[t][c];
  } else if (ll == 0 && tq < P.QB) {
    float2* out = part + ((size_t)bid * P.QB + tq) * CB * NC;
    for (int i = 0; i < CB * NC; ++i) out[i] = cf(0.f, 0.f);
  }
}

// Containment sums (replace lag_reduce + lag_assemble's per-entry loop over
// every cell that contains the tap: up to (K)^3 = 125 T reads per G entry at
// C4/C5).  G[(t,c),(t+d,c')] = sum over cells containing t of T[d][cell] is
// separable over the axes, so it is formed axis by axis:
//   U[ol][dz][b][tl]        = sum_{line class kl contains tl} T[ol][dz][b][kl]   (lag_reduceU: T never stored)
//   V[ol][dz][k0][t1][tl]   = sum_{k1 contains t1} U[ol][dz][k0*n1+k1][tl]       (two outer axes)
//   W[ol][dz][t0][t1][tl]   = sum_{k0 contains t0} V (or U with one outer axis)
// and the G entries are a gather from W.  Fixed summation order: deterministic.
__global__ void lag_reduceU_kernel(const __grid_constant__ LagParams P, const float2* __restrict__ partA,
                                   const float2* __restrict__ partB, double2* __restrict__ U, int64_t total) {
  hicu_pdl_entry();
  const int NC = P.NC, NC2 = NC * NC, la = P.L - 1, KL = P.K[la];
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int cc = (int)(idx % NC2);
    int64_t r = idx / NC2;
    const int b = (int)(r % P.NB);
    r /= P.NB;
    const int dz = (int)(r % P.DZ);
    const int ol = (int)(r / P.DZ);
    const int c = cc / NC, c2 = cc % NC;
    double2 u[kMaxK];
#pragma unroll
    for (int t = 0; t < kMaxK; ++t) u[t] = cd(0.0, 0.0);
    for (int cls = 0; cls < P.NCL; ++cls) {
      double sx = 0.0, sy = 0.0;
      if (cls == P.core_cls) {
        const int gzi = dz / P.GZ, dzi = dz % P.GZ;
        const int64_t nlg = (int64_t)P.nol * P.NG;
        const int64_t bid0 = (int64_t)P.chunksA[b] * nlg + (int64_t)ol * P.NG + gzi;
        const int nch = P.chunksA[b + 1] - P.chunksA[b];
        // four independent chains (four loads in flight), combined in a fixed order
        double ax[4] = {0.0, 0.0, 0.0, 0.0}, ay[4] = {0.0, 0.0, 0.0, 0.0};
        const float2* pa = partA + (bid0 * P.GZ + dzi) * NC2 + cc;
        const int64_t cst = nlg * P.GZ * NC2;
        int ch = 0;
        for (; ch + 3 < nch; ch += 4) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float2 v = pa[(int64_t)(ch + u) * cst];
            ax[u] += v.x;
            ay[u] += v.y;
          }
        }
        for (; ch < nch; ++ch) {
          const float2 v = pa[(int64_t)ch * cst];
          ax[0] += v.x;
          ay[0] += v.y;
        }
        sx = (ax[0] + ax[1]) + (ax[2] + ax[3]);
        sy = (ay[0] + ay[1]) + (ay[2] + ay[3]);
      } else {
        int e = 0;
        while (e < P.NE && P.edge_cls[e] != cls) ++e;
        const int cbi = c / P.CB, t = c % P.CB;
        const int q = (e * P.DZ + dz) * P.NCB + cbi;
        const int qb = q / P.QB, tq = q % P.QB;
        const int64_t bid0 = ((int64_t)ol * P.NQB + qb) * P.CBt + P.chunksB[b];
        const int nch = P.chunksB[b + 1] - P.chunksB[b];
        for (int ch = 0; ch < nch; ++ch) {
          const float2 v = partB[(((bid0 + ch) * P.QB + tq) * P.CB + t) * NC + c2];
          sx += v.x;
          sy += v.y;
        }
      }
#pragma unroll
      for (int tl = 0; tl < kMaxK; ++tl)
        if (tl < KL && tl >= P.cls_lo[la][cls] && tl <= P.cls_hi[la][cls]) u[tl] = u[tl] + cd(sx, sy);
    }
    double2* o = U + (((int64_t)(ol * P.DZ + dz) * P.NB + b) * KL) * NC2 + cc;
    for (int tl = 0; tl < KL; ++tl) o[(int64_t)tl * NC2] = u[tl];
  }
}

// one outer axis reduction: out[pre][t][post] = sum_{k contains t} in[pre][k][post]
// (pre = (ol, dz) [x k0 for the inner outer axis], post = taps of later axes x NC^2)
__global__ void lag_axis_kernel(const __grid_constant__ LagParams P, int axis, int64_t npre, int nk, int64_t npost,
                                const double2* __restrict__ in, double2* __restrict__ out) {
  hicu_pdl_entry();
  const int K = P.K[axis];
  const int64_t total = npre * K * npost;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t post = idx % npost;
    int64_t r = idx / npost;
    const int t = (int)(r % K);
    const int64_t pre = r / K;
    double sx = 0.0, sy = 0.0;
    const double2* src = in + pre * nk * npost + post;
    for (int k = 0; k < nk; ++k) {
      if (t < P.cls_lo[axis][k] || t > P.cls_hi[axis][k]) continue;
      const double2 v = src[(int64_t)k * npost];
      sx += v.x;
      sy += v.y;
    }
    out[idx] = cd(sx, sy);
  }
}

// G[i][j] = W[ol][dz][t0][t1][tl][c][c'] of the lexicographically non-negative
// lag (mirrored entries: the conjugate); real diagonal.
__global__ void lag_gather_kernel(const __grid_constant__ LagParams P, const double2* __restrict__ W,
                                  const int32_t* __restrict__ pos, int ndim, int n, double2* __restrict__ G) {
  hicu_pdl_entry();
  const int L = P.L, la = L - 1, NC = P.NC;
  const int K0 = la >= 1 ? P.K[0] : 1, K1 = la >= 2 ? P.K[1] : 1, KL = P.K[la];
  const int64_t total = (int64_t)n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    int ti[kMaxL], tj[kMaxL];
    for (int a = 0; a < L; ++a) {
      ti[a] = pos[(size_t)i * ndim + P.perm[a]];
      tj[a] = pos[(size_t)j * ndim + P.perm[a]];
    }
    int ci = pos[(size_t)i * ndim + L], cj = pos[(size_t)j * ndim + L];
    int sgn = 0;
    for (int a = 0; a < L && sgn == 0; ++a) sgn = (tj[a] > ti[a]) - (tj[a] < ti[a]);
    const bool mirror = sgn < 0 || (sgn == 0 && ci > cj);
    int t[kMaxL], d[kMaxL];
    for (int a = 0; a < L; ++a) {
      t[a] = mirror ? tj[a] : ti[a];
      d[a] = mirror ? ti[a] - tj[a] : tj[a] - ti[a];
    }
    const int c = mirror ? cj : ci, c2 = mirror ? ci : cj;
    const int i0 = la >= 1 ? d[0] + P.K[0] - 1 : 0, i1 = la >= 2 ? d[1] + P.K[1] - 1 : 0;
    const int ol = P.ol_index[i0][i1];
    const int dz = d[la] + P.K[la] - 1;
    const int t0 = la >= 1 ? t[0] : 0, t1 = la >= 2 ? t[1] : 0;
    const double2 v =
        W[((((int64_t)(ol * P.DZ + dz) * K0 + t0) * K1 + t1) * KL + t[la]) * NC * NC + (int64_t)c * NC + c2];
    G[idx] = cd(v.x, i == j ? 0.0 : (mirror ? -v.y : v.y));
  }
}

// TMA-staged variant for Nc = 8 (every configuration with 8 coils): each
// line segment arrives as 64-row boxes of [20 floats] from a tensor map over
// [16 floats] rows -- the 4 floats past the row are out of bounds and fill
// with zeros, which yields exactly the padded 80-byte rows above with no
// per-element cp.async (one thread issues 2 x ceil(rows / 64) TMA loads per
// line; completion on one mbarrier per ring buffer).
constexpr int kTmaRows = 64;

__device__ __forceinline__ int tma_boxes(int rows) { return (rows + kTmaRows - 1) / kTmaRows; }

constexpr int kTmaThreadsMax = 416;  // 12 compute warps + the producer: <= 128 registers

template <int CB>
__global__ void __launch_bounds__(kTmaThreadsMax, 1)
lag_core_tma_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ LagParams P,
                    float2* __restrict__ part) {
  // warps 0 .. W-1 compute (W = GZ * NCB), warp W is the TMA producer; ring
  // buffers hand off through full (TMA bytes landed) / empty (W warps done)
  // mbarriers, so compute warps never wait for each other
  constexpr int NC = 8;
  constexpr int RB = 80;
  extern __shared__ __align__(1024) uint8_t tsm[];
  __shared__ __align__(8) uint64_t full[kCoreStages], empty[kCoreStages];
  const int64_t bid = blockIdx.x;
  const int nlg = P.nol * P.NG;
  const int rowblk = (int)(bid / nlg);
  const int olg = (int)(bid % nlg);
  const int ol = olg / P.NG, gzi = olg % P.NG;
  int b = 0;
  while (P.chunksA[b + 1] <= rowblk) ++b;
  const int chunk = rowblk - P.chunksA[b];
  const int la = P.L - 1;
  const int dz_lo = gzi * P.GZ - (P.K[la] - 1);
  const int gz_n = min(P.GZ, P.DZ - gzi * P.GZ);
  const int nwarps = P.GZ * P.NCB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dzi = warp / P.NCB, cbi = warp % P.NCB;
  float2* out = part + (size_t)bid * P.GZ * NC * NC;
  int beg[2], len[2];
  block_ranges(P, b, beg, len);
  const int64_t nlines = (int64_t)len[0] * len[1];
  const int64_t l0 = (int64_t)chunk * P.lpcA, l1 = min(nlines, l0 + P.lpcA);
  if (!neighbour_ok(P, beg, len, ol)) {
    hicu_pdl_entry();
    for (int i = threadIdx.x; i < P.GZ * NC * NC; i += blockDim.x) out[i] = cf(0.f, 0.f);
    return;
  }
  const int pn = (int)P.P;
  const int nwa = pn + gz_n - 1;
  const int rb_base = tma_boxes(pn) * kTmaRows;           // rows reserved for the base segment
  const int rb_nbr = tma_boxes(pn + P.GZ - 1) * kTmaRows;  // and for the neighbour segment
  const size_t bufsz = (size_t)(rb_base + rb_nbr) * RB;
  if (threadIdx.x == 0) {
    for (int k = 0; k < kCoreStages; ++k) {
      tc::mbar_init(&full[k], 1);
      tc::mbar_init(&empty[k], nwarps);
    }
    tc::mbar_init_fence();
  }
  __syncthreads();
  hicu_pdl_entry();
  if (warp == nwarps) {
    // ---------------- TMA producer (one thread) ----------------
    if (lane == 0) {
      const int nbb = tma_boxes(pn), nbn = tma_boxes(nwa);
      const uint32_t bytes = (uint32_t)((nbb + nbn) * kTmaRows * RB);
      for (int64_t li = l0; li < l1; ++li) {
        const int it = (int)(li - l0);
        const int buf = it % kCoreStages;
        if (it >= kCoreStages) tc::mbar_wait(&empty[buf], (uint32_t)(((it / kCoreStages) - 1) & 1));
        int64_t q0 = li, q1 = 0;
        if (la == 2) {
          q0 = li / len[1];
          q1 = li % len[1];
        }
        int cb[2] = {0, 0}, cn[2] = {0, 0};
        for (int a = 0; a < la; ++a) {
          const int pa = beg[a] + (int)(a == 0 ? q0 : q1);
          int pq = pa + P.ol_d[ol][a];
          if (P.circ[a]) {
            if (pq < 0) pq += (int)P.N[a];
            if (pq >= P.N[a]) pq -= (int)P.N[a];
          }
          cb[a] = pa;
          cn[a] = pq;
        }
        uint8_t* sb = tsm + (size_t)buf * bufsz;
        uint8_t* sn = sb + (size_t)rb_base * RB;
        tc::mbar_expect_tx(&full[buf], bytes);
        // tensor dims (floats, line axis, outer axis 1, outer axis 0); a non-circular line axis
        const int o1b = la >= 2 ? cb[1] : 0, o0b = la >= 1 ? cb[0] : 0;
        const int o1n = la >= 2 ? cn[1] : 0, o0n = la >= 1 ? cn[0] : 0;
        for (int k = 0; k < nbb; ++k)
          tc::tma_load_4d(sb + (size_t)k * kTmaRows * RB, &tm, 0, (int)P.c0 + k * kTmaRows, o1b, o0b, &full[buf]);
        for (int k = 0; k < nbn; ++k)
          tc::tma_load_4d(sn + (size_t)k * kTmaRows * RB, &tm, 0, (int)P.c0 + dz_lo + k * kTmaRows, o1n, o0n,
                          &full[buf]);
      }
    }
    return;
  }
  float2 accR[CB][NC], accI[CB][NC];
#pragma unroll
  for (int q = 0; q < CB; ++q)
#pragma unroll
    for (int c = 0; c < NC; ++c) accR[q][c] = accI[q][c] = cf(0.f, 0.f);
  const bool active = dzi < gz_n;
  for (int64_t li = l0; li < l1; ++li) {
    const int it = (int)(li - l0);
    const int buf = it % kCoreStages;
    tc::mbar_wait(&full[buf], (uint32_t)((it / kCoreStages) & 1));
    if (active) {
      const uint8_t* sb = tsm + (size_t)buf * bufsz + cbi * CB * 8;
      const uint8_t* sn = tsm + (size_t)buf * bufsz + (size_t)rb_base * RB + dzi * RB;
      // two positions per iteration: both positions' operands are loaded
      // before either's products (hides the shared-memory latency)
      for (int j0 = lane; j0 < pn; j0 += 64) {
        const int j1 = j0 + 32;
        const bool two = j1 < pn;
        float2 a0[CB], v0[NC], a1[CB], v1[NC];
        if (CB == 2) {  // one 16-byte load per position (conflict-free across lanes; 8-byte loads 2-way conflict)
          const float4 w0 = *(const float4*)(sb + j0 * RB);
          const float4 w1 = two ? *(const float4*)(sb + j1 * RB) : make_float4(0.f, 0.f, 0.f, 0.f);
          a0[0] = make_float2(w0.x, w0.y);
          a0[CB - 1] = make_float2(w0.z, w0.w);
          a1[0] = make_float2(w1.x, w1.y);
          a1[CB - 1] = make_float2(w1.z, w1.w);
        } else {
#pragma unroll
          for (int q = 0; q < CB; ++q) {
            a0[q] = *(const float2*)(sb + j0 * RB + q * 8);
            a1[q] = two ? *(const float2*)(sb + j1 * RB + q * 8) : cf(0.f, 0.f);
          }
        }
#pragma unroll
        for (int k = 0; k < NC / 2; ++k) {
          const float4 w0 = *(const float4*)(sn + j0 * RB + k * 16);
          const float4 w1 = two ? *(const float4*)(sn + j1 * RB + k * 16) : make_float4(0.f, 0.f, 0.f, 0.f);
          v0[2 * k] = make_float2(w0.x, w0.y);
          v0[2 * k + 1] = make_float2(w0.z, w0.w);
          v1[2 * k] = make_float2(w1.x, w1.y);
          v1[2 * k + 1] = make_float2(w1.z, w1.w);
        }
#pragma unroll
        for (int q = 0; q < CB; ++q)
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            accR[q][c] = __ffma2_rn(make_float2(a0[q].x, a0[q].x), v0[c], accR[q][c]);
            accI[q][c] = __ffma2_rn(make_float2(a0[q].y, a0[q].y), v0[c], accI[q][c]);
          }
#pragma unroll
        for (int q = 0; q < CB; ++q)
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            accR[q][c] = __ffma2_rn(make_float2(a1[q].x, a1[q].x), v1[c], accR[q][c]);
            accI[q][c] = __ffma2_rn(make_float2(a1[q].y, a1[q].y), v1[c], accI[q][c]);
          }
      }
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&empty[buf]);
  }
#pragma unroll
  for (int q = 0; q < CB; ++q)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      float2 v = make_float2(accR[q][c].x + accI[q][c].y, accR[q][c].y - accI[q][c].x);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
      }
      accR[q][c] = v;
    }
  if (lane == 0 && dzi < P.GZ) {
#pragma unroll
    for (int q = 0; q < CB; ++q)
#pragma unroll
      for (int c = 0; c < NC; ++c)
        out[((size_t)dzi * NC + cbi * CB + q) * NC + c] = active ? accR[q][c] : cf(0.f, 0.f);
  }
}

// ---------------------------------------------------------------------------
// Tensor-core core class (8 coils, line axis <= 256 positions, K <= 5 along it).
//
// Polyphase form: position j = 8u + v along the line.  For one line pair
// (base line L, neighbour line R = L + outer lag),
//   D[(v,c,p), (s,w,c',q)] = sum_u A[u][(v,c,p)] B_s[u][(w,c',q)]
// with A[u][(v,c,p)] = part p of x_L[8u + v, c] (zero outside the core class)
// and B_s[u][(w,c',q)] = part q of x_R[8u + w - 4 + 8s, c']: M = 8 phases x
// 8 coils x re/im = 128 rows, N = 2 shifts x 8 phases x 16 = 256 columns, K =
// u (32 values: two K = 16 steps).  Entry (v, s, w) is the last-axis lag
// dz = 8s + w - 4 - v, so every row holds all 9 lags |dz| <= 4 in the 144
// consecutive columns [16 v, 16 v + 144), and conj(a) b sums re*re + im*im /
// re*im - im*re of the (p, q) pairs.  Operands: fp16 hi/lo of x s (s a
// power of two from max |x|); products A_hi B_hi + A_hi B_lo + A_lo B_hi
// (22-bit operands, fp32 accumulation in TMEM).  One CTA = one outer lag x
// one chunk of lines of one outer class block (the same grid, partial-sum
// layout and reduce / assemble kernels as the CUDA-core path).  A line
// pair is one 48 KB stage (two bulk copies), 6 MMAs of M128 N256 K16; TMEM
// holds two 256-column accumulators: the MMA warp fills one for kTcPPD pairs
// while the epilogue drains the other into fp32 registers.
// ---------------------------------------------------------------------------


__device__ __forceinline__ float lag_pow2_scale(float amax) {
  if (!(amax > 0.f) || !(amax < 3.0e38f)) return 1.f;
  int e;
  frexpf(amax, &e);
  e = e < -100 ? -100 : (e > 110 ? 110 : e);
  return ldexpf(1.f, 15 - e);
}

__device__ __forceinline__ float lag_amax_reduce(const float* __restrict__ amax, int namax) {
  const int lane = threadIdx.x & 31;
  float m = 0.f;
  for (int i = lane; i < namax; i += 32) m = fmaxf(m, __ldg(amax + i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  return m;
}

__global__ void __launch_bounds__(256) lagtc_amax_kernel(const float4* __restrict__ x, int64_t n4, float* __restrict__ part) {
  hicu_pdl_entry();
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(x + i);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  __shared__ float wm[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t = fmaxf(t, wm[w]);
    part[blockIdx.x] = t;
  }
}

// byte offset of 16-byte chunk ch (halfs 8ch..8ch+7) of row r in a K-major SW64 tile
__device__ __forceinline__ int lag_sw64(int r, int ch) { return r * 64 + ((ch ^ ((r >> 1) & 3)) << 4); }

// One CTA per line (plan order): the line's A (core positions only) and B
// (both shifts) tiles, fp16 hi/lo of x s, in their shared-memory image.
__global__ void __launch_bounds__(256) lagtc_prep_kernel(const __grid_constant__ LagParams P,
                                                         const float2* __restrict__ x, const float* __restrict__ amax,
                                                         int namax, uint8_t* __restrict__ out) {
  hicu_pdl_entry();
  __shared__ __align__(16) __half hs[256][16], lsm[256][16];
  __shared__ float s_sa;
  const int la = P.L - 1;
  const int64_t li = blockIdx.x;
  int64_t base = 0;
  if (la == 2) base = (li / P.N[1]) * P.cstride[0] + (li % P.N[1]) * P.cstride[1];
  else if (la == 1) base = li * P.cstride[0];
  if (threadIdx.x < 32) {
    const float m = lag_amax_reduce(amax, namax);
    if (threadIdx.x == 0) s_sa = lag_pow2_scale(m);
  }
  __syncthreads();
  const float sa = s_sa;
  const int NL = (int)P.N[la];
  const int64_t lst = P.cstride[la];
  for (int e = threadIdx.x; e < 256 * 8; e += 256) {
    const int pos = e >> 3, c = e & 7;
    const float2 v = pos < NL ? __ldg(x + base + pos * lst + c) : make_float2(0.f, 0.f);
    const float xr = v.x * sa, xi = v.y * sa;
    const __half hr = __float2half_rn(xr), hi = __float2half_rn(xi);
    hs[pos][2 * c] = hr;
    hs[pos][2 * c + 1] = hi;
    lsm[pos][2 * c] = __float2half_rn(xr - __half2float(hr));
    lsm[pos][2 * c + 1] = __float2half_rn(xi - __half2float(hi));
  }
  __syncthreads();
  uint8_t* o = out + li * (int64_t)kTcLineBytes;
  const int c0 = (int)P.c0, c1 = (int)(P.c0 + P.P);
  const __half hz = __float2half_rn(0.f);
  // A: rows (v, c, p) = 16 v + 2 c + p, K = u; zero outside the core class
  for (int t = threadIdx.x; t < 128 * 4; t += 256) {
    const int r = t >> 2, ch = t & 3, v = r >> 4, cp = r & 15;
    __align__(16) __half hv[8], lv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int pos = 8 * (8 * ch + k) + v;
      const bool in = pos >= c0 && pos < c1;
      hv[k] = in ? hs[pos][cp] : hz;
      lv[k] = in ? lsm[pos][cp] : hz;
    }
    *reinterpret_cast<uint4*>(o + lag_sw64(r, ch)) = *reinterpret_cast<const uint4*>(hv);
    *reinterpret_cast<uint4*>(o + 8192 + lag_sw64(r, ch)) = *reinterpret_cast<const uint4*>(lv);
  }
  // B: rows (s, w, c', q) = 128 s + 16 w + 2 c' + q at position 8u + w - 4 + 8s
  for (int t = threadIdx.x; t < 256 * 4; t += 256) {
    const int r = t >> 2, ch = t & 3, sh = r >> 7, w = (r >> 4) & 7, cq = r & 15;
    __align__(16) __half hv[8], lv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int pos = 8 * (8 * ch + k) + w - 4 + 8 * sh;
      const bool in = pos >= 0 && pos < NL;
      hv[k] = in ? hs[pos][cq] : hz;
      lv[k] = in ? lsm[pos][cq] : hz;
    }
    *reinterpret_cast<uint4*>(o + 16384 + lag_sw64(r, ch)) = *reinterpret_cast<const uint4*>(hv);
    *reinterpret_cast<uint4*>(o + 32768 + lag_sw64(r, ch)) = *reinterpret_cast<const uint4*>(lv);
  }
}

__device__ __forceinline__ void lag_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ int64_t lag_line_index(const LagParams& P, int p0, int p1) {
  const int la = P.L - 1;
  return la == 2 ? (int64_t)p0 * P.N[1] + p1 : (la == 1 ? (int64_t)p0 : 0);
}

__global__ void __launch_bounds__(kTcThreads, 1)
lagtc_core_kernel(const __grid_constant__ LagParams P, const uint8_t* __restrict__ lines,
                  const float* __restrict__ amax, int namax, float2* __restrict__ part) {
  constexpr int NC = 8;
  extern __shared__ __align__(1024) uint8_t tcs_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)tcs_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[kTcStages], empty[kTcStages], tfull[2], tempty[2];
  __shared__ uint32_t tslot;
  __shared__ float s_inv;
  const int64_t bid = blockIdx.x;
  const int nlg = P.nol * P.NG;
  const int rowblk = (int)(bid / nlg);
  const int ol = (int)(bid % nlg);  // NG == 1
  int b = 0;
  while (P.chunksA[b + 1] <= rowblk) ++b;
  const int chunk = rowblk - P.chunksA[b];
  const int la = P.L - 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float2* out = part + (size_t)bid * P.GZ * NC * NC;
  int beg[2], len[2];
  block_ranges(P, b, beg, len);
  const int64_t nlines = (int64_t)len[0] * len[1];
  const int64_t l0 = (int64_t)chunk * P.lpcA, l1 = min(nlines, l0 + P.lpcA);
  if (!neighbour_ok(P, beg, len, ol)) {
    hicu_pdl_entry();
    for (int i = threadIdx.x; i < P.GZ * NC * NC; i += blockDim.x) out[i] = cf(0.f, 0.f);
    return;
  }
  const int npairs = (int)(l1 - l0);
  const int ngroups = (npairs + kTcPPD - 1) / kTcPPD;
  if (threadIdx.x == 0) {
    for (int k = 0; k < kTcStages; ++k) {
      tc::mbar_init(&full[k], 1);
      tc::mbar_init(&empty[k], 1);
    }
    for (int k = 0; k < 2; ++k) {
      tc::mbar_init(&tfull[k], 1);
      tc::mbar_init(&tempty[k], kTcEpiWarps);
    }
    tc::mbar_init_fence();
  }
  if (warp == 1) tc::tmem_alloc(&tslot, 512);
  hicu_pdl_entry();
  if (warp == 1) {
    const float m = lag_amax_reduce(amax, namax);
    if (lane == 0) {
      const float sa = lag_pow2_scale(m);
      s_inv = 1.f / (sa * sa);
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;

  if (warp == 0) {
    // ---------------- producer: base-line A tiles + neighbour-line B tiles ----------------
    int s = 0;
    uint32_t ph = 0;
    for (int k = 0; k < npairs; ++k) {
      const int64_t li = l0 + k;
      int q0 = (int)li, q1 = 0;
      if (la == 2) {
        q0 = (int)(li / len[1]);
        q1 = (int)(li % len[1]);
      }
      const int pa0 = beg[0] + q0, pa1 = beg[1] + q1;
      int pn0 = pa0 + P.ol_d[ol][0], pn1 = pa1 + P.ol_d[ol][1];
      if (la >= 1 && P.circ[0]) pn0 = pn0 < 0 ? pn0 + (int)P.N[0] : (pn0 >= P.N[0] ? pn0 - (int)P.N[0] : pn0);
      if (la >= 2 && P.circ[1]) pn1 = pn1 < 0 ? pn1 + (int)P.N[1] : (pn1 >= P.N[1] ? pn1 - (int)P.N[1] : pn1);
      const uint8_t* la_src = lines + lag_line_index(P, pa0, pa1) * kTcLineBytes;
      const uint8_t* lb_src = lines + lag_line_index(P, pn0, pn1) * kTcLineBytes + 16384;
      tc::mbar_wait(&empty[s], ph ^ 1);
      if (tc::elect_one()) {
        uint8_t* st = sm + (size_t)s * kTcLineBytes;
        tc::mbar_expect_tx(&full[s], kTcLineBytes);
        lag_bulk(st, la_src, 16384, &full[s]);
        lag_bulk(st + 16384, lb_src, 32768, &full[s]);
      }
      __syncwarp();
      if (++s == kTcStages) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = tc::idesc_f16(128, 256);
    const uint64_t d0 = tc::desc_sw64(tc::smem_u32(sm));
    int s = 0;
    uint32_t ph = 0;
    for (int k = 0; k < npairs; ++k) {
      const int grp = k / kTcPPD, tb = grp & 1;
      const bool first = (k % kTcPPD) == 0;
      if (first) tc::mbar_wait(&tempty[tb], ((grp >> 1) & 1) ^ 1);
      tc::mbar_wait(&full[s], ph);
      tc::fence_after();
      const uint64_t da = d0 + (uint64_t)((s * kTcLineBytes) >> 4);
      const uint64_t dal = da + (8192 >> 4), db = da + (16384 >> 4), dbl = da + (32768 >> 4);
      const uint32_t d = tmem + (uint32_t)(tb * 256);
      if (tc::elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t o = (uint64_t)(ks * 2);  // +32 B: the second K = 16 step of the 64-byte rows
          tc::mma_f16(d, da + o, db + o, idesc, (first && ks == 0) ? 0u : 1u);  // A_hi B_hi
          tc::mma_f16(d, da + o, dbl + o, idesc, 1u);                          // A_hi B_lo
          tc::mma_f16(d, dal + o, db + o, idesc, 1u);                          // A_lo B_hi
        }
        tc::mma_commit(&empty[s]);
        if ((k % kTcPPD) == kTcPPD - 1 || k == npairs - 1) tc::mma_commit(&tfull[tb]);
      }
      __syncwarp();
      if (++s == kTcStages) { s = 0; ph ^= 1; }
    }
  } else {
    // ---------------- epilogue: drain into fp32 registers, reduce at the end ----------------
    const int ew = warp - 2, q = warp & 3, h = ew >> 2;
    const int m = 32 * q + lane;  // TMEM lane = A row (v, c, p)
    const int v = m >> 4;
    const int cbase = 32 * q + kTcCols * h;  // first of this thread's kTcCols columns
    float acc[kTcCols];
#pragma unroll
    for (int i = 0; i < kTcCols; ++i) acc[i] = 0.f;
    for (int grp = 0; grp < ngroups; ++grp) {
      const int tb = grp & 1;
      tc::mbar_wait(&tfull[tb], (grp >> 1) & 1);
      tc::fence_after();
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(tb * 256 + cbase);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t r[5][8];
#pragma unroll
        for (int i = 0; i < 5; ++i) tc::tmem_ld8_nowait(ta + (uint32_t)(8 * (5 * half + i)), r[i]);
        tc::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 5; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[8 * (5 * half + i) + j] += __uint_as_float(r[i][j]);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[tb]);
    }
    // all MMAs are complete (the last tfull): the stage buffers become the
    // reduction table red[row][144] (the row's 9 lags x 16 columns)
    constexpr int RS = 148;
    float* red = reinterpret_cast<float*>(sm);
#pragma unroll
    for (int i = 0; i < kTcCols; ++i) {
      const int cr = cbase + i - 16 * v;
      if (cr >= 0 && cr < 144) red[m * RS + cr] = acc[i];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kTcEpiWarps * 32) : "memory");
    const float inv = s_inv;
    const int et = threadIdx.x - 64;
    for (int o = et; o < 9 * NC * NC; o += kTcEpiWarps * 32) {
      const int dzi = o >> 6, c = (o >> 3) & 7, c2 = o & 7;
      const int col = 16 * dzi + 2 * c2;
      float re = 0.f, im = 0.f;
#pragma unroll
      for (int vv = 0; vv < 8; ++vv) {
        const float* rr = red + (16 * vv + 2 * c) * RS + col;  // row (vv, c, re)
        const float* ri = rr + RS;                             // row (vv, c, im)
        re += rr[0] + ri[1];
        im += rr[1] - ri[0];
      }
      const int pd = dzi - 4 + P.K[la] - 1;  // plan lag index of dz = dzi - 4
      if (pd >= 0 && pd < P.GZ) out[((size_t)pd * NC + c) * NC + c2] = cf(re * inv, im * inv);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

// Edge classes of the tensor-core geometries (8 coils, non-circular line
// axis, K <= 5 along it, N >= 4K - 4 positions per line): one CTA per (outer
// lag, chunk of lpcB lines of one outer class block), 288 threads = (edge
// position e, last-axis lag dz, coil block cbi).  Lines are staged 32 at a
// time in shared memory -- the edge positions of the base lines and the
// positions [0, 2K-2) and [N-2K+2, N) of the neighbour lines, each a row of 8
// coils; consecutive lines of a block row are adjacent in memory, so every
// staging load is a coalesced run of 64-byte rows (the per-thread
// gathers of lag_edge_kernel were latency-bound).  Same partial layout as
// lag_edge_kernel.
constexpr int kE2Lines = 14;   // 2 x 14 staged lines = 69 KB: three CTAs per SM
constexpr int kE2Threads = 288; // most threads of a CTA; launched with the active pairs x NCB rounded up to warps
                                // (224 at 5 taps when the edges touch the array bounds: three CTAs of 96 registers per SM)
constexpr int kE2LS = 8 * 8 + 2, kE2RS = 24 * (8 + 2) + 2;  // float2 per staged line (base edges, neighbour window)

__global__ void __maxnreg__(96)
lag_edge2_kernel(const __grid_constant__ LagParams P, const float2* __restrict__ x, float2* __restrict__ part) {
  hicu_pdl_entry();
  constexpr int NC = 8, CB = 2;
  const int la = P.L - 1;
  const int K = P.K[la];
  const int W = 3 * K - 3;          // neighbour window of one edge group: (K - 1) edges x (2K - 1) lags
  const int NR = 2 * W;             // staged neighbour positions (left and right edge groups)
  const int lo_base = P.cls_beg[la][P.edge_cls[0]] - (K - 1);          // first left edge - (K - 1)
  const int hi_base = P.cls_beg[la][P.edge_cls[K - 1]] - (K - 1);      // first right edge - (K - 1)
  const int NL = (int)P.N[la];
  extern __shared__ __align__(16) uint8_t e2sm[];
  // Two staging buffers of kE2Lines lines each.  Per line: the base line's edge positions [8][NC] and the
  // neighbour window [24][NC + 2] -- rows padded to 5 16-byte chunks (80 B) so the 8 rows a warp reads at
  // once (its 8 lags) fall on distinct banks; both line strides are an odd number of chunks (staging
  // stores).  The next sub-chunk's lines are in flight (cp.async) while this one is multiplied.
  constexpr int LS = kE2LS, RS = kE2RS, RW = NC + 2, BUF = kE2Lines * (kE2LS + kE2RS);
  float2* sbuf = reinterpret_cast<float2*>(e2sm);
  __shared__ int64_t sbase[2][kE2Lines], snbr[2][kE2Lines];
  const int bidx = blockIdx.x;
  const int ol = bidx / P.CBt;
  const int chunk = bidx % P.CBt;  // global chunk id over blocks
  int b = 0;
  while (P.chunksB[b + 1] <= chunk) ++b;
  const int ch = chunk - P.chunksB[b];
  int beg[2], len[2];
  block_ranges(P, b, beg, len);
  const int64_t nlines = (int64_t)len[0] * len[1];
  const int64_t l0 = (int64_t)ch * P.lpcB, l1 = min(nlines, l0 + P.lpcB);
  const bool ok = neighbour_ok(P, beg, len, ol);
  const int t = threadIdx.x, nthr = blockDim.x;
  // Output slot q = (e * DZ + dz) * NCB + cbi.  An (edge position, lag) pair whose neighbour
  // position falls outside the line contributes nothing (28 % of the pairs for 5 taps), so the
  // threads are dealt the ACTIVE pairs in slot order: the products fill the first warps densely
  // and the remaining warps only stage (they also write the zero partials of the inactive slots).
  auto pair_pr = [&](int pair) { return P.cls_beg[la][P.edge_cls[pair / P.DZ]] + pair % P.DZ - (K - 1); };
  const int npairs = P.NE * P.DZ;
  __shared__ int s_pairs[kE2Threads], s_nact;  // the active pairs in slot order (built by warp 0)
  if (t < 32) {
    int base = 0;
    for (int r0 = 0; r0 < npairs; r0 += 32) {
      const int pair = r0 + t;
      const int prp = pair < npairs ? pair_pr(pair) : -1;
      const bool a = prp >= 0 && prp < NL;
      const unsigned m = __ballot_sync(0xffffffffu, a);
      if (a) s_pairs[base + __popc(m & ((1u << t) - 1u))] = pair;
      base += __popc(m);
    }
    if (t == 0) s_nact = base;
  }
  __syncthreads();
  const int q = (t / P.NCB < s_nact) ? s_pairs[t / P.NCB] * P.NCB + t % P.NCB : -1;
  const bool qok = q >= 0;
  const int qq = qok ? q : 0;
  const int e = qq / (P.DZ * P.NCB), dzi = (qq / P.NCB) % P.DZ, cbi = qq % P.NCB;
  const int dz = dzi - (K - 1);
  const int pe = P.cls_beg[la][P.edge_cls[e]];
  const int pr = pe + dz;
  const bool act = ok && qok;
  const int ridx = e < K - 1 ? pr - lo_base : W + pr - hi_base;
  float2 accR[CB][NC], accI[CB][NC];
#pragma unroll
  for (int a = 0; a < CB; ++a)
#pragma unroll
    for (int c = 0; c < NC; ++c) accR[a][c] = accI[a][c] = cf(0.f, 0.f);
  const int64_t ls = P.cstride[la];
  if (ok && l0 < l1) {
    auto offsets = [&](int64_t lb, int bf) {
      if (lb + t < l1 && t < kE2Lines) line_offsets(P, beg, len, ol, lb + t, sbase[bf][t], snbr[bf][t]);
    };
    // 16-byte pieces; consecutive threads -> the pieces of one position row across consecutive lines
    // (adjacent 64-byte rows in memory)
    auto issue = [&](int64_t lb, int bf) {
      const int nl = (int)min((int64_t)kE2Lines, l1 - lb);
      float2* sL = sbuf + (size_t)bf * BUF;
      float2* sR = sL + kE2Lines * LS;
      const int per = 4 * nl;
      for (int i = t; i < (P.NE + NR) * per; i += nthr) {
        const int r = i / per, rem = i - r * per, j = rem >> 2, pc4 = rem & 3;
        if (r < P.NE) {
          const int pos = P.cls_beg[la][P.edge_cls[r]];
          cp_async16(reinterpret_cast<float4*>(sL + j * LS + r * NC) + pc4,
                     reinterpret_cast<const float4*>(x + sbase[bf][j] + pos * ls) + pc4);
        } else {
          const int k = r - P.NE;
          const int pos = k < W ? lo_base + k : hi_base + k - W;
          float4* dst = reinterpret_cast<float4*>(sR + j * RS + k * RW) + pc4;
          if (pos >= 0 && pos < NL) cp_async16(dst, reinterpret_cast<const float4*>(x + snbr[bf][j] + pos * ls) + pc4);
          else *dst = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    offsets(l0, 0);
    __syncthreads();
    issue(l0, 0);
    int it = 0;
    for (int64_t lb = l0; lb < l1; lb += kE2Lines, ++it) {
      const int bf = it & 1;
      const int64_t nx = lb + kE2Lines;
      const int nl = (int)min((int64_t)kE2Lines, l1 - lb);
      if (nx < l1) offsets(nx, bf ^ 1);
      __syncthreads();  // the next offsets are visible; the other buffer's reads (previous sub-chunk) are done
      if (nx < l1) {
        issue(nx, bf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();  // this sub-chunk has landed for every thread
      if (act) {
        const float2* sL = sbuf + (size_t)bf * BUF;
        const float2* sR = sL + kE2Lines * LS;
        for (int j = 0; j < nl; ++j) {
          float2 a[CB], bv[NC];
#pragma unroll
          for (int u = 0; u < CB; ++u) a[u] = sL[j * LS + e * NC + cbi * CB + u];
#pragma unroll
          for (int c = 0; c < NC; ++c) bv[c] = sR[j * RS + ridx * RW + c];
#pragma unroll
          for (int u = 0; u < CB; ++u)
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              accR[u][c] = __ffma2_rn(make_float2(a[u].x, a[u].x), bv[c], accR[u][c]);
              accI[u][c] = __ffma2_rn(make_float2(a[u].y, a[u].y), bv[c], accI[u][c]);
            }
        }
      }
    }
  }
  // conj(a) b = (accR.x + accI.y, accR.y - accI.x); lag_edge_kernel's partial layout
  auto slot = [&](int qs) {
    const int qb = qs / P.QB, tq = qs % P.QB;
    return part + ((((size_t)ol * P.NQB + qb) * P.CBt + chunk) * P.QB + tq) * CB * NC;
  };
  if (act) {
    float2* out = slot(q);
#pragma unroll
    for (int u = 0; u < CB; ++u)
#pragma unroll
      for (int c = 0; c < NC; ++c) out[u * NC + c] = cf(accR[u][c].x + accI[u][c].y, accR[u][c].y - accI[u][c].x);
  }
  // zero partials: every slot when the neighbour block does not exist, else the inactive pairs' slots
  for (int qs = t; qs < P.NQ; qs += nthr) {
    const int prs = pair_pr(qs / P.NCB);
    if (ok && prs >= 0 && prs < NL) continue;
    float2* out = slot(qs);
    for (int i = 0; i < CB * NC; ++i) out[i] = cf(0.f, 0.f);
  }
}

typedef CUresult (*LagEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

LagEncodeFn lag_encode() {
  static LagEncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (LagEncodeFn)p;
    else
      cudaGetLastError();
  }
  return fn;
}

// Tensor map for the TMA core kernel: dims (16 floats, line axis, outer axis
// 1, outer axis 0) in plan order with the array's byte strides; boxes of
// 20 floats x 64 rows (the 4 extra floats are out of bounds: zero padding).
bool lag_tmap(CUtensorMap* tm, const LagParams& P, const float2* x) {
  LagEncodeFn enc = lag_encode();
  if (!enc) return false;
  const int la = P.L - 1;
  cuuint64_t dims[4] = {16, (cuuint64_t)P.N[la], (cuuint64_t)(la >= 2 ? P.N[1] : 1), (cuuint64_t)(la >= 1 ? P.N[0] : 1)};
  cuuint64_t strides[3] = {(cuuint64_t)P.cstride[la] * 8, la >= 2 ? (cuuint64_t)P.cstride[1] * 8 : dims[1] * 64,
                           la >= 1 ? (cuuint64_t)P.cstride[0] * 8 : dims[1] * dims[2] * 64};
  cuuint32_t box[4] = {20, (cuuint32_t)kTmaRows, 1, 1}, es[4] = {1, 1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float2*>(x), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NC>
int launch_nc(const LagPlan& pl, const float2* x, void* ws, cudaStream_t st) {
  constexpr int CB = cb_for(NC);
  const LagParams& P = pl.p;
  if (P.CB != CB) return hicu_set_error(HICU_ERR_PARAMETER, "gram_lag: coil block mismatch");
  float2* partA = (float2*)((char*)ws + pl.a_off);
  float2* partB = (float2*)((char*)ws + pl.b_off);
  int s;
  if (pl.nA > 0 && pl.tc) {
    // tensor-core core class: amax of x, per-line operand tiles, then the MMA kernel
    float* am = (float*)((char*)ws + pl.amax_off);
    uint8_t* lines = (uint8_t*)ws + pl.prep_off;
    int64_t n4 = pl.lines_all * P.N[P.L - 1] * NC / 2;  // float4 count of the k-space array
    const int namax = (int)std::min<int64_t>(2 * hicu_sm_count(), std::max<int64_t>(1, (n4 + 255) / 256));
    hicu_launch(lagtc_amax_kernel, namax, 256, 0, st, (const float4*)x, n4, am);
    if ((s = hicu_check_launch("lagtc_amax_kernel"))) return s;
    hicu_launch(lagtc_prep_kernel, (unsigned)pl.lines_all, 256, 0, st, P, x, (const float*)am, namax, lines);
    if ((s = hicu_check_launch("lagtc_prep_kernel"))) return s;
    const size_t smem = (size_t)kTcStages * kTcLineBytes + 1024;
    hicu_allow_max_smem((const void*)lagtc_core_kernel);
    hicu_launch(lagtc_core_kernel, (unsigned)pl.nA, kTcThreads, smem, st, P, (const uint8_t*)lines, (const float*)am,
                namax, partA);
    if ((s = hicu_check_launch("lagtc_core_kernel"))) return s;
  } else if (pl.nA > 0) {
    bool done = false;
    if constexpr (NC == 8) {
      const int la = P.L - 1;
      CUtensorMap tm;
      const int rows = ((int)P.P + kTmaRows - 1) / kTmaRows * kTmaRows +
                       ((int)P.P + P.GZ - 1 + kTmaRows - 1) / kTmaRows * kTmaRows;
      const size_t smem = (size_t)kCoreStages * rows * 80 + 1024;
      if (!P.circ[la] && smem <= (size_t)200 * 1024 && pl.threadsA + 32 <= kTmaThreadsMax && lag_tmap(&tm, P, x)) {
        hicu_allow_max_smem((const void*)lag_core_tma_kernel<CB>);
        hicu_launch(lag_core_tma_kernel<CB>, (unsigned)pl.nA, pl.threadsA + 32, smem, st, tm, P, partA);
        if ((s = hicu_check_launch("lag_core_tma_kernel"))) return s;
        done = true;
      }
    }
    if (!done) {
      hicu_allow_max_smem((const void*)lag_core_kernel<NC, CB>);
      hicu_launch(lag_core_kernel<NC, CB>, (unsigned)pl.nA, pl.threadsA, pl.smemA, st, P, x, partA);
      if ((s = hicu_check_launch("lag_core_kernel"))) return s;
    }
  }
  int e2_active = 0;  // (edge position, lag) pairs whose neighbour position lies inside the line
  {
    const int la = P.L - 1;
    for (int e = 0; e < P.NE; ++e)
      for (int dzi = 0; dzi < P.DZ; ++dzi) {
        const int pr = P.cls_beg[la][P.edge_cls[e]] + dzi - (P.K[la] - 1);
        if (pr >= 0 && pr < (int)P.N[la]) ++e2_active;
      }
  }
  const int e2_threads = max(64, (e2_active * P.NCB + 31) / 32 * 32);
  if (pl.nB > 0 && pl.tc && e2_threads <= kE2Threads && P.NQ <= kE2Threads && P.NE == 2 * (P.K[P.L - 1] - 1)) {
    hicu_allow_max_smem((const void*)lag_edge2_kernel);
    hicu_launch(lag_edge2_kernel, (unsigned)(P.nol * P.CBt), e2_threads, (size_t)2 * kE2Lines * (kE2LS + kE2RS) * 8, st, P, x,
                partB);
    if ((s = hicu_check_launch("lag_edge2_kernel"))) return s;
  } else if (pl.nB > 0) {
    hicu_allow_max_smem((const void*)lag_edge_kernel<NC, CB>);
    hicu_launch(lag_edge_kernel<NC, CB>, (unsigned)pl.nB, kEdgeThreads, pl.smemB, st, P, x, partB);
    if ((s = hicu_check_launch("lag_edge_kernel"))) return s;
  }
  return HICU_OK;
}

}  // namespace

bool hicu_gram_lag_supported(const DevGeom& g) {
  if (!(g.nc >= 1 && g.nc <= 8) && g.nc != 10 && g.nc != 12 && g.nc != 16) return false;
  return make_plan(g).ok;
}

// fp32 flops the lag kernels execute (8 per complex MAC: core + edge
// products of the lines whose neighbour block is in range)
double hicu_gram_lag_flops(const DevGeom& g) {
  LagPlan pl = make_plan(g);
  if (!pl.ok) return 0.0;
  const LagParams& P = pl.p;
  const int la = P.L - 1;
  double lines_pos = 0.0;
  for (int ol = 0; ol < P.nol; ++ol)
    for (int b = 0; b < P.NB; ++b) {
      int r = b, ok = 1;
      double nl = 1.0;
      for (int a = la - 1; a >= 0; --a) {
        const int k = r % P.ncls[a];
        r /= P.ncls[a];
        const int beg = P.cls_beg[a][k], len = P.cls_end[a][k] - P.cls_beg[a][k];
        const int d = P.ol_d[ol][a];
        if (!P.circ[a] && (beg + d < 0 || beg + len - 1 + d >= P.N[a])) ok = 0;
        nl *= len;
      }
      if (!ok) continue;
      double pos = P.core_cls >= 0 ? (double)P.P * P.DZ : 0.0;
      for (int e = 0; e < P.NE; ++e) {
        const int c = P.edge_cls[e];
        for (int pz = P.cls_beg[la][c]; pz < P.cls_end[la][c]; ++pz)
          for (int dz = -(P.K[la] - 1); dz <= P.K[la] - 1; ++dz)
            if (pz + dz >= 0 && pz + dz < P.N[la]) pos += 1.0;
      }
      lines_pos += nl * pos;
    }
  return lines_pos * P.NC * P.NC * 8.0;
}

bool hicu_gram_lag_tc(const DevGeom& g) {
  LagPlan pl = make_plan(g);
  return pl.ok && pl.tc;
}

size_t hicu_gram_lag_workspace(const DevGeom& g) {
  LagPlan pl = make_plan(g);
  return pl.ok ? pl.bytes : 0;
}

int hicu_gram_lag(const DevGeom& g, const float2* x, double2* G, void* ws, size_t ws_bytes, cudaStream_t st) {
  LagPlan pl = make_plan(g);
  if (!pl.ok) return hicu_set_error(HICU_ERR_PARAMETER, "gram_lag: unsupported geometry");
  if (ws_bytes < pl.bytes) return hicu_set_error(HICU_ERR_WORKSPACE, "gram_lag: workspace too small");
  int s;
  switch (g.nc) {
    case 1: s = launch_nc<1>(pl, x, ws, st); break;
    case 2: s = launch_nc<2>(pl, x, ws, st); break;
    case 3: s = launch_nc<3>(pl, x, ws, st); break;
    case 4: s = launch_nc<4>(pl, x, ws, st); break;
    case 5: s = launch_nc<5>(pl, x, ws, st); break;
    case 6: s = launch_nc<6>(pl, x, ws, st); break;
    case 7: s = launch_nc<7>(pl, x, ws, st); break;
    case 8: s = launch_nc<8>(pl, x, ws, st); break;
    case 10: s = launch_nc<10>(pl, x, ws, st); break;
    case 12: s = launch_nc<12>(pl, x, ws, st); break;
    case 16: s = launch_nc<16>(pl, x, ws, st); break;
    default: return hicu_set_error(HICU_ERR_PARAMETER, "gram_lag: coil count");
  }
  if (s) return s;
  const float2* partA = (const float2*)((char*)ws + pl.a_off);
  const float2* partB = (const float2*)((char*)ws + pl.b_off);
  const LagParams& P = pl.p;
  const int la = P.L - 1, NC2 = P.NC * P.NC, KL = P.K[la];
  double2* U = (double2*)((char*)ws + pl.u_off);
  double2* V = (double2*)((char*)ws + pl.v_off);
  double2* W = (double2*)((char*)ws + pl.w_off);
  auto blocks_for = [](int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, (int64_t)hicu_sm_count() * 16); };
  {
    const int64_t nU = pl.nU / NC2 * NC2;
    hicu_launch(lag_reduceU_kernel, blocks_for(nU), 256, 0, st, P, partA, partB, U, (int64_t)P.nol * P.DZ * P.NB * NC2);
    if ((s = hicu_check_launch("lag_reduceU_kernel"))) return s;
  }
  const int64_t od = (int64_t)P.nol * P.DZ;
  if (la == 2) {  // axis 1: U[od][k0][k1][tl] -> V[od][k0][t1][tl]
    hicu_launch(lag_axis_kernel, blocks_for(pl.nV), 256, 0, st, P, 1, od * P.ncls[0], P.ncls[1], (int64_t)KL * NC2,
                (const double2*)U, V);
    if ((s = hicu_check_launch("lag_axis_kernel"))) return s;
    hicu_launch(lag_axis_kernel, blocks_for(pl.nW), 256, 0, st, P, 0, od, P.ncls[0], (int64_t)P.K[1] * KL * NC2,
                (const double2*)V, W);
    if ((s = hicu_check_launch("lag_axis_kernel"))) return s;
  } else if (la == 1) {  // axis 0: U[od][k0][tl] -> W[od][t0][tl]
    hicu_launch(lag_axis_kernel, blocks_for(pl.nW), 256, 0, st, P, 0, od, P.ncls[0], (int64_t)KL * NC2,
                (const double2*)U, W);
    if ((s = hicu_check_launch("lag_axis_kernel"))) return s;
  } else {
    W = U;  // one spatial axis: NB = 1
  }
  const int64_t total = (int64_t)g.n * g.n;
  hicu_launch(lag_gather_kernel, blocks_for(total), 256, 0, st, P, (const double2*)W, g.pos, g.ndim, g.n, G);
  return hicu_check_launch("lag_gather_kernel");
}
