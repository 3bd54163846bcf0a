// Hankel convolution u = H(y) Q~ and its transpose (the k-space scatter
// g = H^H(u) Q~^H) on the 5th-generation tensor cores: tcgen05 kind::f16 with
// fp16 hi/lo splits under a power-of-two scale (FP32-grade accuracy: 22
// significant bits per operand, the precision of a 3xTF32 split), TMEM
// accumulators.
//
// Reference: hankel.py:255-322 (hankel_apply), hankel.py:394-440
// (kspace_adjoint_scatter), solver.py:335-351 (objective / ELS terms, DC).
//
// Scope: coil-separable support with Nc = 8 coils, p = 8 JL columns, no
// circular axes, 1..3 spatial axes, kernel last-axis extent nb <= 8.  One
// spatial position of the k-space array is a row of 16 floats (8 complex
// coils) and a row of u is also 16 floats (8 complex columns): one K = 16
// step of a kind::f16 MMA, a 32-byte SWIZZLE_32B K-major operand row.
//
// Shift-GEMM formulation.  For every kernel "prefix" a (all spatial axes but
// the last) one MMA multiplies a 128-row tile of one k-space line by the
// stacked operators of ALL last-axis taps b:
//   D[m, b, :] = A_a[m, :] . B_{a,b}^T      (N = 16 * nb per precision term)
// accumulated over a in TMEM.  Output row i then needs D[i + b, b, :] (conv)
// or D[i - b, b, :] (scatter): the shift moves to the epilogue, which stages
// D in a shared-memory window that carries nb - 1 rows from one tile to the
// next along the line.
//
// Split products: A_hi [B_hi; B_lo] (one MMA, N = 32 nb) plus A_lo B_hi
// (N = 16 nb, accumulated into the A_hi B_hi columns); the dropped lo*lo term
// is ~2^-22 relative.  A scale: max |A| from amax_kernel partials (the kernel
// launched just before); B scale: in the image trailer.  The epilogue
// multiplies by 1 / (s_A s_B), a power of two (exact).
//
// Why fp16 and not 3xTF32 (measured, scripts/tc_unit_f16.cu and the per-role
// cycle counters of HICU_CONV_TC_DEBUG=32): with TMA-staged fp32 A tiles, raw
// fp32 hi and converter-written lo, a stage (one prefix group) moved ~68 KB
// through shared memory (TMA write, converter read + write, MMA operand
// reads of 4 tf32 MMAs) -- ~530 cycles at 128 B/clk, the kernel's real
// limit.  fp16 operands halve the MMA operand bytes and the MMA count (one
// K = 16 step instead of two K = 8), and the converter warps now load A rows
// straight from global memory into registers (kPrefetch stages ahead), so
// an fp32 A tile never touches shared memory: ~32 KB per stage.
//
// Epilogues are fused: conv writes u and the objective partial |u|^2; the ELS
// variant never stores w = H(g)Q~ and accumulates Re<w,u>, |w|^2; the scatter
// applies hard / soft data consistency to every k-space position (positions
// no tap reaches get the DC term only) and accumulates the four DC partial
// sums (same meaning as ops.cu:scatter_coil_kernel).  Partial sums are per
// CTA in fixed order (deterministic).
//
// Warp roles (448 threads, one persistent CTA per SM, whole lines per CTA):
// warp 0 B-image producer (streamed mode), warp 1 TMEM owner + MMA issuer,
// warps 2-5 A converters (global -> registers -> fp16 hi/lo tiles), warps
// 6-13 epilogue (TMEM lane quarter = warp % 4).
#include <cuda.h>
#include <stdlib.h>

#include <cuda_fp16.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "tc_common.cuh"

namespace {

constexpr int kTileM = 128;
constexpr int kAmaxSlot = 512;             // entries of a producer's max partials (consumers read all of them)
constexpr int kMaxNb = 8;                  // last-axis kernel extent
constexpr int kMaxGroups = 64;             // kernel prefixes (product of the other spatial extents)
constexpr int kMaxTaps = 128;              // spatial taps
constexpr int kMaxStages = 16;
constexpr int kEpiWarps = 8;  // two warps per TMEM lane quarter, each owning 8 of the 16 output floats
constexpr int kThreads = (2 + kEpiWarps) * 32;
constexpr int kSmemBudget = 220 * 1024;    // conservative dynamic shared memory budget (sm_100a opt-in 227 KB)

// Operand geometry per complex row width CW (coils == JL columns: 8 for
// C1/C2/C4/C5, 10 for C3).  A row carries KA = 2 CW real components; its
// split form is [KP fp16 hi | KP fp16 lo] with KP = KA rounded up to K = 16
// steps (zero padded); a tap contributes NO = 2 CW output columns.
template <int CW>
struct Cw {
  static constexpr int KA = 2 * CW;
  static constexpr int NO = 2 * CW;
  static constexpr int KP = (KA + 15) / 16 * 16;  // halfs per hi (lo) part
  static constexpr int KS = KP / 16;               // K = 16 steps per part
  static constexpr int RB = 4 * KP;                // split row bytes: 64 (SW64) or 128 (SW128)
  static constexpr int ATILE = kTileM * RB;        // one 128-row A tile
  static constexpr int GPS = CW == 8 ? 5 : 1;      // prefix groups per pipeline stage (one TMA box; CW 10: 6 MMAs per group already)
  static constexpr int ASTAGE = GPS * ATILE;
  static constexpr int BROW = 2 * KP;              // B image row bytes: 32 (SW32) or 64 (SW64)
  static constexpr int NH = NO / 2;                // output floats per epilogue thread (two per row)
  static constexpr int CH = CW / 2;                // coils per epilogue thread (scatter)
  static constexpr int WROW = NO + 4;              // window row floats (+16 B: conflict-free rows)
  static constexpr bool CAT = CW == 8;             // A_hi [B_hi; B_lo] in one MMA (N = 2 ntot = 32 nb <= 256)
  static constexpr int WIN_FLOATS = (kTileM + kMaxNb - 1) * WROW + kMaxNb * (kMaxNb - 1) * NO;
};

// byte offset of (row r, 16-byte chunk ch) in a K-major swizzled tile with
// rows of RBY bytes (SW32 / SW64 / SW128: the swizzle is on absolute address
// bits; every operand buffer is 1024-byte aligned)
template <int RBY>
__host__ __device__ __forceinline__ int swz(int r, int ch) {
  if (RBY == 32) return r * 32 + ((ch ^ ((r >> 2) & 1)) << 4);
  if (RBY == 64) return r * 64 + ((ch ^ ((r >> 1) & 3)) << 4);
  return r * 128 + ((ch ^ (r & 7)) << 4);
}

template <int RBY>
__device__ __forceinline__ uint64_t desc_swz(uint32_t saddr) {
  if (RBY == 32) return tc::desc_sw32(saddr);
  if (RBY == 64) return tc::desc_sw64(saddr);
  return tc::desc_sw128(saddr);
}

struct CtParams {
  int L;                  // spatial axes (1..3)
  int nsp;                // spatial taps
  int ndim;               // geometry rank (pos stride per support entry)
  int nb;                 // kernel extent along the last (tile) axis
  int ng;                 // kernel prefixes
  int kpre[2];            // kernel extents of the prefix axes
  int stages;
  int tbuf_stride;        // TMEM columns between the two accumulator buffers (0: one buffer)
  int nacc;               // accumulator sets per tile (prefix groups dealt round-robin; shortens chains)
  int stage_bytes;        // two A tiles (+ the two prefix groups' B images when streamed)
  int dc_mode;
  float lam;
  int nparts_total;       // entries of `parts` (per value) the ABI promised
  int chunks;             // tiles per line
  int nlines;
  int ldim[2];            // line extents of the prefix axes (conv: rext, scatter: dims)
  int ext_last;           // conv: rext (output rows per line); scatter: dims (positions per line)
  int roff[3];
  int rext[3];
  int64_t ostride[2];     // output strides (rows / positions) of the prefix axes
  int debug;              // experiment bits (HICU_CONV_TC_DEBUG): 1 no MMA, 2 no B copy, 4 no A load/convert,
                          // 8 no TMEM drain, 32 per-role cycle counters, 64 no converter proxy fence
  const uint8_t* bimg;    // B images (fp16 hi/lo, ng groups + scale trailer), bulk-copied in
  int bimg_early;         // 1: bimg was written >= 2 kernels earlier, copy it before the grid-dependency wait
  int perm[3];            // kernel spatial axis k is geometry axis perm[k]; k = L-1 is the tile ("line") axis
  int64_t lstride;        // output stride (rows / positions) along the line axis
  const float* amax;      // max |A component| partials (amax_kernel) -> the A scale
  int namax;
  float* amax_out;        // optional: per-CTA max |output component| (conv: u, scatter: g), zero-filled to kAmaxSlot
  int k1;                 // extent of the innermost prefix axis (pairs of groups never straddle it)
  int abox;               // bytes of one stage's A box (GPS tiles, one when L == 1)
  int ntot;               // MMA N of one precision block: round16(NO nb)
  int cat;                // 1: A_hi [B_hi; B_lo] in one MMA (2 ntot <= 256), else separate hi / lo MMAs
  // three-line tiles (conv_tri_kernel): a tile computes output lines i, i+1, i+2 along the inner prefix axis
  int tri;                // 1: B images in the three-line layout (per outer prefix: hi block, lo block)
  int ko;                 // outer prefix extent (1 when L == 2)
  int ntri;               // three-line groups along the inner line axis
  int sd;                 // input lines per stage (k1 + 2: one TMA box)
};

__device__ __forceinline__ void decode_line(const CtParams& P, int line, int (&lc)[2]) {
  lc[0] = lc[1] = 0;
  if (P.L == 3) {
    lc[1] = line % P.ldim[1];
    lc[0] = line / P.ldim[1];
  } else if (P.L == 2) {
    lc[0] = line;
  }
}

// Scatter: prefix group g reaches k-space line lc iff the u line lc - roff - a exists.
template <int MODE>
__device__ __forceinline__ bool group_valid(const CtParams& P, const int (&ga)[kMaxGroups][2], int g,
                                            const int (&lc)[2]) {
  if (MODE < 2) return true;
  bool ok = true;
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    if (d < P.L - 1) {
      const int r = lc[d] - P.roff[d] - ga[g][d];
      ok = ok && r >= 0 && r < P.rext[d];
    }
  }
  return ok;
}

// bitmask of the prefix groups that reach line lc (all groups for the conv)
template <int MODE>
__device__ __forceinline__ uint64_t line_groups(const CtParams& P, const int (&ga)[kMaxGroups][2], const int (&lc)[2]) {
  if (MODE < 2) return P.ng >= 64 ? ~0ull : ((1ull << P.ng) - 1ull);
  uint64_t m = 0;
  for (int g = 0; g < P.ng; ++g)
    if (group_valid<MODE>(P, ga, g, lc)) m |= 1ull << g;
  return m;
}

template <int MODE>
__device__ __forceinline__ bool line_active(const CtParams& P, const int (&ga)[kMaxGroups][2], const int (&lc)[2]) {
  if (MODE < 2) return true;
  for (int g = 0; g < P.ng; ++g)
    if (group_valid<MODE>(P, ga, g, lc)) return true;
  return false;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory"); }

// DC inputs of one k-space position (the CH coils of one epilogue thread):
// loaded before the tile's accumulators are ready, so the global-load
// latency overlaps the MMAs
template <int CH>
struct DcIn {
  uint8_t mk[CH];
  float2 y[CH], x[CH];
};

template <int CH>
__device__ __forceinline__ DcIn<CH> dc_load(const CtParams& P, size_t e0, int h, const uint8_t* __restrict__ mask,
                                            const float2* __restrict__ y, const float2* __restrict__ x0) {
  const size_t e = e0 + (size_t)CH * h;
  DcIn<CH> d;
  if (CH == 4) {
    const uint32_t mm = P.dc_mode != 2 ? __ldg(reinterpret_cast<const uint32_t*>(mask + e)) : 0u;
#pragma unroll
    for (int c = 0; c < CH; ++c) d.mk[c] = (uint8_t)(mm >> (8 * c));
  } else {
#pragma unroll
    for (int c = 0; c < CH; ++c) d.mk[c] = P.dc_mode != 2 ? __ldg(mask + e + c) : (uint8_t)0;
  }
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    d.y[c] = d.x[c] = make_float2(0.f, 0.f);
    if (P.dc_mode == 1) {
      d.y[c] = __ldg(y + e + c);
      d.x[c] = __ldg(x0 + e + c);
    }
  }
  return d;
}

// Scatter epilogue for one k-space position, the CH coils of this thread:
// data consistency + the four partial sums (|g|^2, |res|^2, <g,res>, |g|^2
// on observed); returns max |g component| written.
template <int CH>
__device__ __forceinline__ float scatter_store(const CtParams& P, size_t e0, int h, const float (&v)[2 * CH],
                                               const DcIn<CH>& d, float2* __restrict__ gout, double (&acc)[4]) {
  float mx = 0.f;
  const size_t e = e0 + (size_t)CH * h;
  float a[2 * CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const bool on = P.dc_mode != 2 && d.mk[c] == 1;
    float ar = v[2 * c], ai = v[2 * c + 1];
    if (P.dc_mode == 0) {
      if (on) ar = ai = 0.f;
    } else if (P.dc_mode == 1) {
      const float rr = on ? d.y[c].x - d.x[c].x : 0.f, ri = on ? d.y[c].y - d.x[c].y : 0.f;
      acc[1] += (double)rr * rr + (double)ri * ri;
      ar = ar + P.lam * rr;
      ai = ai + P.lam * ri;
      if (on) {
        acc[2] += (double)ar * rr + (double)ai * ri;
        acc[3] += (double)ar * ar + (double)ai * ai;
      }
    }
    acc[0] += (double)ar * ar + (double)ai * ai;
    a[2 * c] = ar;
    a[2 * c + 1] = ai;
    mx = fmaxf(mx, fmaxf(fabsf(ar), fabsf(ai)));
  }
  if (CH == 4) {
    float4* gp = reinterpret_cast<float4*>(gout + e);
    gp[0] = make_float4(a[0], a[1], a[2], a[3]);
    gp[1] = make_float4(a[4], a[5], a[6], a[7]);
  } else {
#pragma unroll
    for (int c = 0; c < CH; ++c) gout[e + c] = make_float2(a[2 * c], a[2 * c + 1]);
  }
  return mx;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

// fp16 hi/lo split with a power-of-two scale s: x s = hi + lo with
// hi = rn(x s) and lo = rn(x s - hi) (the residual is exact in fp32), i.e. 22
// significant bits -- the precision of the 3xTF32 split -- as long as x s
// stays inside fp16's range: s maps max |x| into [2^14, 2^15).  Values below
// 2^-24 / s lose relative precision, but their absolute error (< 2^-25 / s =
// 2^-40 max |x|) is far below fp32 rounding of the sums they enter.
__host__ __device__ __forceinline__ float pow2_scale(float amax) {
  if (!(amax > 0.f) || !(amax < 3.0e38f)) return 1.f;
  int e;
  frexpf(amax, &e);  // amax = m 2^e, m in [0.5, 1)
  e = e < -100 ? -100 : (e > 110 ? 110 : e);
  return ldexpf(1.f, 15 - e);
}

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// B images of all prefix groups, fp16: prefix g at base + g * gbytes; rows
// b NO + n (hi block) and ntot + b NO + n (lo block), K = the operand's real
// components (zero padded to KP), scaled by sb.
template <int MODE, int CW>
__device__ __forceinline__ void bimage_put(uint8_t* base, const CtParams& P, const int (&spos)[kMaxTaps][3], int e,
                                           float2 q, uint32_t gbytes, float sb) {
  using T = Cw<CW>;
  const int L = P.L;
  const int sp = e / (CW * CW), c = (e / CW) % CW, j = e % CW;
  const int g = L == 1 ? 0 : (L == 2 ? spos[sp][0] : spos[sp][0] * P.kpre[1] + spos[sp][1]);
  const int b = spos[sp][L - 1];
  uint8_t* gb = base + (size_t)g * gbytes;
  if (P.tri) {
    // three-line layout: per outer prefix go a hi block then a lo block of k1
    // images each (inner prefix ga1 at image k1 - 1 - ga1 for the conv, ga1
    // for the scatter), so an MMA's B rows for output slots t_lo..t_hi are
    // consecutive images; an image's lo rows sit k1 images after its hi rows
    const int go = L == 3 ? spos[sp][0] : 0, ga1 = L == 3 ? spos[sp][1] : spos[sp][0];
    const int k1 = L == 3 ? P.kpre[1] : P.kpre[0];
    const int idx = MODE < 2 ? k1 - 1 - ga1 : ga1;
    gb = base + (size_t)go * gbytes * k1 + (size_t)idx * P.ntot * T::BROW;
  }
#pragma unroll
  for (int tp = 0; tp < 2; ++tp)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      int n, k;
      float v;
      if (MODE < 2) {  // n = 2j + t', k = 2c + t: u_j = sum_c y_c q_cj
        n = 2 * j + tp;
        k = 2 * c + t;
        v = tp == 0 ? (t == 0 ? q.x : -q.y) : (t == 0 ? q.y : q.x);
      } else {  // n = 2c + t', k = 2j + t: g_c = sum_j conj(q_cj) u_j
        n = 2 * c + tp;
        k = 2 * j + t;
        v = tp == 0 ? (t == 0 ? q.x : q.y) : (t == 0 ? -q.y : q.x);
      }
      const float x = v * sb;
      const __half hi = __float2half_rn(x);
      const __half lo = __float2half_rn(x - __half2float(hi));
      const int rh = b * T::NO + n;
      const int rl = P.tri ? (L == 3 ? P.kpre[1] : P.kpre[0]) * P.ntot + rh : P.ntot + rh;  // tri: lo block k1 images on
      *reinterpret_cast<__half*>(gb + swz<T::BROW>(rh, k >> 3) + (k & 7) * 2) = hi;
      *reinterpret_cast<__half*>(gb + swz<T::BROW>(rl, k >> 3) + (k & 7) * 2) = lo;
    }
}

// NH consecutive TMEM columns of this thread's lane (8 or 10), without the wait
template <int NH>
__device__ __forceinline__ void tmem_ld_row(uint32_t taddr, uint32_t (&r)[NH]) {
  uint32_t a[8];
  tc::tmem_ld8_nowait(taddr, a);
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = a[i];
  if (NH > 8) {
    uint32_t b2[2];
    tc::tmem_ld2_nowait(taddr + 8, b2);
    r[8 % NH] = b2[0];
    r[9 % NH] = b2[1];
  }
}

// MODE 0: conv forward (u, obj); 1: conv ELS (Re<w,u>, |w|^2); 2: scatter + DC.
// BS: B images streamed per stage (they do not fit next to the pipeline).
template <int MODE, bool BS, int CW>
__global__ void __launch_bounds__(kThreads, 1)
conv_tc_kernel(const __grid_constant__ CUtensorMap tmap, const CtParams P, float2* __restrict__ out,
               const float2* __restrict__ uin, const uint8_t* __restrict__ mask, const float2* __restrict__ y,
               const float2* __restrict__ x0, double* __restrict__ parts) {
  constexpr int NV = MODE == 0 ? 1 : (MODE == 1 ? 2 : 4);
  using T = Cw<CW>;
  constexpr int NH = T::NH, CH = T::CH, NO = T::NO, WROW = T::WROW;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int nb = P.nb, ng = P.ng, L = P.L, S = P.stages;
  const uint32_t gbytes = 2u * (uint32_t)P.ntot * T::BROW;  // B image of one prefix: hi and lo blocks
  uint8_t* sB = smem;
  uint8_t* sStage = sB + (BS ? 0 : (size_t)ng * gbytes);
  const int stb = P.stage_bytes;
  float* sWin = reinterpret_cast<float*>(sStage + (size_t)S * stb);  // per-tap window + carries
  // tempty[buffer * 3 + set]: the epilogue has drained that accumulator set
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], tfull[2], tempty[6];
  __shared__ __align__(8) uint64_t bres;
  __shared__ uint32_t tslot;
  __shared__ int ga[kMaxGroups][2];
  __shared__ double red[kEpiWarps][NV];
  __shared__ float s_scale[2];  // A scale, 1 / (A scale x B scale)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // debug bit 32: per-role cycle counters (waits vs work), written to `out` (conv forward only)
  __shared__ long long pc[12];
  const bool pf = (P.debug & 32) != 0;
  if (threadIdx.x < 12) pc[threadIdx.x] = 0;

  // ---- prologue part 1 (before the grid-dependency wait): static data and
  // barrier/TMEM setup, overlapping the previous kernel ----
  if (threadIdx.x < ng) {
    const int g = threadIdx.x;
    ga[g][0] = L == 2 ? g : (L == 3 ? g / P.kpre[1] : 0);
    ga[g][1] = L == 3 ? g % P.kpre[1] : 0;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) tc::mbar_init(&tfull[b], 1);
    for (int b = 0; b < 6; ++b) tc::mbar_init(&tempty[b], kEpiWarps);  // one arrival per epilogue warp
    tc::mbar_init(&bres, 1);
    tc::mbar_init_fence();
    if (!BS && P.bimg_early) {  // the images are older than the previous kernel: fetch them now
      tc::mbar_expect_tx(&bres, (uint32_t)ng * gbytes);
      bulk_g2s(sB, P.bimg, (uint32_t)ng * gbytes, &bres);
    }
  }
  if (warp == 1) tc::tmem_alloc(&tslot, 512);
  // ---- prologue part 2: inputs written by the previous kernels ----
  hicu_pdl_entry();
  if (!BS && !P.bimg_early && threadIdx.x == 0) {
    tc::mbar_expect_tx(&bres, (uint32_t)ng * gbytes);
    bulk_g2s(sB, P.bimg, (uint32_t)ng * gbytes, &bres);
  }
  if (warp == 1) {
    float m = 0.f;
    for (int i = lane; i < P.namax; i += 32) m = fmaxf(m, __ldg(P.amax + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      const float sa = pow2_scale(m);
      const float sb = *reinterpret_cast<const float*>(P.bimg + (size_t)ng * gbytes);
      s_scale[0] = sa;
      s_scale[1] = 1.f / (sa * sb);
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  const int nbuf = P.tbuf_stride > 0 ? 2 : 1;
  if (pf && threadIdx.x == 0) pc[8] = clock64();

  if (warp == 0) {
    // ---------------- TMA producer: two prefix groups' A tiles per stage (+ their B images when streamed) ----------------
    // warp-uniform loop (loop state in uniform registers); one elected lane issues.
    // Groups g and g + 1 of one pair are adjacent lines along tensor dimension
    // 2 (conv: c2 and c2 + 1; scatter: c2 and c2 - 1), so one TMA box of depth
    // 2 loads both (scatter: tile 0 = group g + 1).
    int s = 0;
    uint32_t ph = 0;
    for (int line = blockIdx.x; line < P.nlines; line += gridDim.x) {
     int lc[2];
     decode_line(P, line, lc);
     const uint64_t gm = line_groups<MODE>(P, ga, lc);
     for (int c = 0; c < P.chunks; ++c)
     for (int g = 0, t1 = 0; g < ng; ) {
      const int cnt = min(T::GPS, P.k1 - t1);  // a stage's groups never straddle the outer prefix axis
      const int g0 = g;
      g += cnt;
      t1 += cnt;
      if (t1 >= P.k1) t1 = 0;
      if (!((gm >> g0) & ((1ull << cnt) - 1ull))) continue;
      const long long t0p = (pf && lane == 0) ? clock64() : 0;
      tc::mbar_wait(&empty[s], ph ^ 1);
      if (pf && lane == 0) pc[0] += clock64() - t0p;
      // tensor coordinate 1 = line axis, 2 = axis L-2, 3 = axis L-3
      int c1, c2 = 0, c3 = 0;
      if (MODE < 2) {
        c1 = P.roff[L - 1] + c * kTileM;
        if (L == 2) c2 = P.roff[0] + lc[0] + ga[g0][0];
        if (L == 3) {
          c2 = P.roff[1] + lc[1] + ga[g0][1];
          c3 = P.roff[0] + lc[0] + ga[g0][0];
        }
      } else {
        c1 = c * kTileM;
        if (L == 2) c2 = lc[0] - P.roff[0] - ga[g0][0];
        if (L == 3) {
          c2 = lc[1] - P.roff[1] - ga[g0][1];
          c3 = lc[0] - P.roff[0] - ga[g0][0];
        }
        c2 -= cnt - 1;  // the box starts at the last group's line
      }
      if (tc::elect_one()) {
        if (P.debug & 2) {
          tc::mbar_arrive(&full[s]);
        } else {
          uint8_t* dst = sStage + (size_t)s * stb;
          tc::mbar_expect_tx(&full[s], (uint32_t)P.abox + (BS ? (uint32_t)cnt * gbytes : 0u));
          tc::tma_load_4d(dst, &tmap, 0, c1, c2, c3, &full[s]);
          if (BS) {
            for (int j = 0; j < cnt; ++j)
              bulk_g2s(dst + T::ASTAGE + j * gbytes, P.bimg + (size_t)(g0 + j) * gbytes, gbytes, &full[s]);
          }
        }
      }
      __syncwarp();
      if (++s == S) { s = 0; ph ^= 1; }
     }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // warp-uniform loop; one elected lane (always lane 0: the warp is
    // converged) issues the MMAs and the commits that track them
    if (!BS) tc::mbar_wait(&bres, 0);  // resident B images landed (async proxy, no fence needed)
    const uint32_t idesc_cat = tc::idesc_f16(kTileM, 2 * P.ntot), idesc_hi = tc::idesc_f16(kTileM, P.ntot);
    // descriptors advance by address >> 4 in their low 14 bits (shared-memory addresses < 256 KB)
    const uint64_t dstage0 = desc_swz<T::RB>(tc::smem_u32(sStage)), dimg0 = desc_swz<T::BROW>(tc::smem_u32(sB));
    const uint64_t dstageb0 = desc_swz<T::BROW>(tc::smem_u32(sStage));  // streamed B images
    const uint32_t blo16 = ((uint32_t)P.ntot * T::BROW) >> 4;  // the B image's lo block
    const uint32_t stb16 = (uint32_t)stb >> 4, g16 = gbytes >> 4;
    int s = 0, tb = 0;
    uint32_t ph = 0, tph = 0;
    for (int line = blockIdx.x; line < P.nlines; line += gridDim.x) {
      int lc[2];
      decode_line(P, line, lc);
      const uint64_t gm = line_groups<MODE>(P, ga, lc);
      if (!gm) continue;
      for (int c = 0; c < P.chunks; ++c) {
        const uint32_t d0 = tmem + (uint32_t)(tb * P.tbuf_stride);
        int vi = 0, set = 0;  // valid-group index within the tile; accumulator set = vi % nacc (kept incrementally)
        for (int g = 0, t1 = 0; g < ng; ) {
          const int cnt = min(T::GPS, P.k1 - t1);
          const int g0 = g;
          g += cnt;
          t1 += cnt;
          if (t1 >= P.k1) t1 = 0;
          const uint32_t pv = (uint32_t)((gm >> g0) & ((1ull << cnt) - 1ull));  // valid groups of the stage
          if (!pv) continue;
          const long long t0r = (pf && lane == 0) ? clock64() : 0;
          tc::mbar_wait(&full[s], ph);  // A tiles (+ streamed B images) landed
          if (pf && lane == 0) pc[3] += clock64() - t0r;
          const uint64_t dst = dstage0 + (uint64_t)(s * stb16);
#pragma unroll
          for (int j = 0; j < T::GPS; ++j) {
            if (!((pv >> j) & 1u)) continue;
            if (vi < P.nacc) {  // first use of this accumulator set in the tile: drained by the epilogue?
              const long long t0m = (pf && lane == 0) ? clock64() : 0;
              tc::mbar_wait(&tempty[tb * 3 + set], tph ^ 1);
              if (pf && lane == 0) pc[4] += clock64() - t0m;
            }
            tc::fence_after();
            // tile of group g0 + j: conv j, scatter cnt - 1 - j (its lines run backwards)
            const int tile = MODE == 2 ? cnt - 1 - j : j;
            const uint64_t da = dst + (uint64_t)((tile * T::ATILE) >> 4);
            const uint64_t db = BS ? dstageb0 + (uint64_t)(s * stb16) + (uint64_t)((T::ASTAGE + j * (int)gbytes) >> 4)
                                   : dimg0 + (uint64_t)((g0 + j) * g16);
            const uint32_t d = d0 + (uint32_t)(set * (T::CAT ? 2 : 1) * P.ntot);
            const uint32_t acc = vi >= P.nacc ? 1u : 0u;
            ++vi;
            if (++set == P.nacc) set = 0;
            if (tc::elect_one()) {
              if (!(P.debug & 1)) {
                // A row [hi KP | lo KP]: hi K step ks at +32 ks bytes, lo at +2 KP + 32 ks; B K step at +32 ks
#pragma unroll
                for (int ks = 0; ks < T::KS; ++ks) {
                  const uint64_t ah = da + (uint64_t)(2 * ks), al = da + (uint64_t)((2 * T::KP + 32 * ks) >> 4);
                  const uint64_t bk = db + (uint64_t)(2 * ks);
                  if constexpr (T::CAT) {
                    tc::mma_f16(d, ah, bk, idesc_cat, ks == 0 ? acc : 1u);  // A_hi [B_hi; B_lo]
                    tc::mma_f16(d, al, bk, idesc_hi, 1);                    // + A_lo B_hi
                  } else {
                    tc::mma_f16(d, ah, bk, idesc_hi, ks == 0 ? acc : 1u);   // A_hi B_hi
                    tc::mma_f16(d, ah, bk + blo16, idesc_hi, 1);            // + A_hi B_lo
                    tc::mma_f16(d, al, bk, idesc_hi, 1);                    // + A_lo B_hi
                  }
                }
              }
            }
            __syncwarp();
          }
          const long long t0i = (pf && lane == 0) ? clock64() : 0;
          if (tc::elect_one()) tc::mma_commit(&empty[s]);
          __syncwarp();
          if (pf && lane == 0) pc[5] += clock64() - t0i;
          if (++s == S) { s = 0; ph ^= 1; }
        }
        if (tc::elect_one()) tc::mma_commit(&tfull[tb]);
        __syncwarp();
        if (nbuf == 2) {
          tb ^= 1;
          if (tb == 0) tph ^= 1;
        } else {
          tph ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue ----------------
    // 8 warps: warp w reads TMEM lane quarter q = w & 3 (A-tile rows 32q..)
    // and owns output floats [8h, 8h + 8) of every row (h = column half).
    const int ew = warp - 2;
    const int q = warp & 3, h = ew >> 2;
    const int m = 32 * q + lane;  // TMEM lane = A-tile row
    const int et = threadIdx.x - 64;  // epilogue thread index 0..255
    const float inv = s_scale[1];
    // per-tap window: rows 0..nb-2 = the tap's rows carried from the previous
    // tile, rows nb-1+m = this tile's D[m, b, :] (WROW floats per row)
    float* tapbuf = sWin;
    float* carry = sWin + (kTileM + kMaxNb - 1) * WROW;  // [b][nb-1][NO]
    double acc_v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc_v[i] = 0.0;
    float omax = 0.f;  // max |output component| of this thread (producer max partials)
    int tb = 0;
    uint32_t tph = 0;
    for (int line = blockIdx.x; line < P.nlines; line += gridDim.x) {
      int lc[2];
      decode_line(P, line, lc);
      int64_t obase = 0;
      if (L >= 2) obase += (int64_t)lc[0] * P.ostride[0];
      if (L >= 3) obase += (int64_t)lc[1] * P.ostride[1];
      const uint64_t gm = line_groups<MODE>(P, ga, lc);
      const bool active = gm != 0;
      const int nvalid = __popcll(gm);
      if (active) {
        // carried rows start at zero (u rows before the line / k-space before the region)
        for (int i = et; i < nb * (kMaxNb - 1) * NO; i += kEpiWarps * 32) carry[i] = 0.f;
        epi_bar();
        for (int c = 0; c < P.chunks; ++c) {
          // this tile's epilogue inputs from global memory, loaded before the accumulators are ready
          DcIn<CH> din{};
          float2 upre[CH];
#pragma unroll
          for (int i = 0; i < CH; ++i) upre[i] = make_float2(0.f, 0.f);
          if (MODE == 2) {
            const int x = P.roff[L - 1] + c * kTileM + m;
            if (x < P.ext_last) din = dc_load<CH>(P, (size_t)(obase + (int64_t)x * P.lstride) * CW, h, mask, y, x0);
          } else if (MODE == 1) {
            const int i_out = c * kTileM - (nb - 1) + m;
            if (i_out >= 0 && i_out < P.ext_last) {
              const float2* up = uin + (size_t)(obase + (int64_t)i_out * P.lstride) * CW + CH * h;
              if (CH == 4) {
                const float4 a0 = __ldg(reinterpret_cast<const float4*>(up)), a1 = __ldg(reinterpret_cast<const float4*>(up) + 1);
                upre[0] = make_float2(a0.x, a0.y);
                upre[1] = make_float2(a0.z, a0.w);
                upre[2 % CH] = make_float2(a1.x, a1.y);
                upre[3 % CH] = make_float2(a1.z, a1.w);
              } else {
#pragma unroll
                for (int i = 0; i < CH; ++i) upre[i] = __ldg(up + i);
              }
            }
          }
          long long t0e = (pf && et == 0) ? clock64() : 0;
          tc::mbar_wait(&tfull[tb], tph);
          if (pf && et == 0) {
            const long long t1e = clock64();
            pc[6] += t1e - t0e;
            t0e = t1e;
          }
          tc::fence_after();
          const uint32_t t0 = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(tb * P.tbuf_stride) + (uint32_t)(NH * h);
          const int nsets = min(P.nacc, nvalid);
          const int scols = (T::CAT ? 2 : 1) * P.ntot;  // TMEM columns of one accumulator set
          // drain set by set into registers; each set is released to the MMA
          // warp as soon as it is read (the next tile's groups start on set 0)
          float f[kMaxNb][NH];
#pragma unroll
          for (int b = 0; b < kMaxNb; ++b)
#pragma unroll
            for (int i = 0; i < NH; ++i) f[b][i] = 0.f;
          for (int a = 0; a < P.nacc; ++a) {
            if (a < nsets && !(P.debug & 8)) {
              const uint32_t ta = t0 + (uint32_t)(a * scols);
              if constexpr (NH == 8 && T::CAT) {
                // two taps in flight per wait (A_hi B_hi + A_lo B_hi, and A_hi B_lo columns)
#pragma unroll
                for (int b = 0; b < kMaxNb; b += 2) {
                  if (b < nb) {
                    uint32_t v0[2][8], v1[2][8];
                    tc::tmem_ld8_nowait(ta + (uint32_t)(NO * b), v0[0]);
                    tc::tmem_ld8_nowait(ta + (uint32_t)(P.ntot + NO * b), v1[0]);
                    if (b + 1 < nb) {
                      tc::tmem_ld8_nowait(ta + (uint32_t)(NO * b + NO), v0[1]);
                      tc::tmem_ld8_nowait(ta + (uint32_t)(P.ntot + NO * b + NO), v1[1]);
                    }
                    tc::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < NH; ++i) f[b][i] += __uint_as_float(v0[0][i]) + __uint_as_float(v1[0][i]);
                    if (b + 1 < nb) {
#pragma unroll
                      for (int i = 0; i < NH; ++i) f[b + 1][i] += __uint_as_float(v0[1][i]) + __uint_as_float(v1[1][i]);
                    }
                  }
                }
              } else {
#pragma unroll
              for (int b = 0; b < kMaxNb; ++b) {
                if (b < nb) {
                  // hi block (A_hi B_hi + A_lo B_hi [+ A_hi B_lo when separate]) and, when
                  // concatenated, the A_hi B_lo block ntot columns further
                  uint32_t v0[NH], v1[NH];
                  tmem_ld_row<NH>(ta + (uint32_t)(b * NO), v0);
                  if constexpr (T::CAT) tmem_ld_row<NH>(ta + (uint32_t)(P.ntot + b * NO), v1);
                  tc::tmem_wait_ld();
#pragma unroll
                  for (int i = 0; i < NH; ++i) f[b][i] += __uint_as_float(v0[i]) + (T::CAT ? __uint_as_float(v1[i]) : 0.f);
                }
              }
              }
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[tb * 3 + a]);
          }
          if (pf && et == 0) {
            const long long t1e = clock64();
            pc[7] += t1e - t0e;
            t0e = t1e;
          }
          if (nbuf == 2) {
            tb ^= 1;
            if (tb == 0) tph ^= 1;
          } else {
            tph ^= 1;
          }
          // shifted sums, one tap at a time: conv row m takes D[m + b - (nb-1), b]
          // (window row m + b), scatter row m takes D[m - b, b] (window row nb-1+m-b)
          float v[NH];
#pragma unroll
          for (int i = 0; i < NH; ++i) v[i] = 0.f;
          constexpr int NQ4 = NO / 4;  // float4 pieces per window row
#pragma unroll
          for (int b = 0; b < kMaxNb; ++b) {
            if (b < nb) {
              if (et < (nb - 1) * NQ4) {
                const int r = et / NQ4, kk = et - r * NQ4;
                reinterpret_cast<float4*>(tapbuf + r * WROW)[kk] =
                    reinterpret_cast<const float4*>(carry + (b * (kMaxNb - 1) + r) * NO)[kk];
              }
              const int w = MODE < 2 ? m + b : nb - 1 + m - b;
              if (NH % 4 == 0) {  // 16-byte window traffic
                float4* w4 = reinterpret_cast<float4*>(tapbuf + (nb - 1 + m) * WROW + NH * h);
#pragma unroll
                for (int i = 0; i < NH / 4; ++i)
                  w4[i] = make_float4(f[b][4 * i] * inv, f[b][4 * i + 1] * inv, f[b][4 * i + 2] * inv,
                                      f[b][4 * i + 3] * inv);
                epi_bar();
                const float4* r4 = reinterpret_cast<const float4*>(tapbuf + w * WROW + NH * h);
#pragma unroll
                for (int i = 0; i < NH / 4; ++i) {
                  const float4 t4 = r4[i];
                  v[4 * i] += t4.x;
                  v[4 * i + 1] += t4.y;
                  v[4 * i + 2] += t4.z;
                  v[4 * i + 3] += t4.w;
                }
              } else {
                float2* w2 = reinterpret_cast<float2*>(tapbuf + (nb - 1 + m) * WROW + NH * h);
#pragma unroll
                for (int i = 0; i < NH / 2; ++i) w2[i] = make_float2(f[b][2 * i] * inv, f[b][2 * i + 1] * inv);
                epi_bar();
                const float2* r2 = reinterpret_cast<const float2*>(tapbuf + w * WROW + NH * h);
#pragma unroll
                for (int i = 0; i < NH / 2; ++i) {
                  const float2 t2 = r2[i];
                  v[2 * i] += t2.x;
                  v[2 * i + 1] += t2.y;
                }
              }
              if (et < (nb - 1) * NQ4) {  // this tap's last nb - 1 rows carry into the next tile
                const int r = et / NQ4, kk = et - r * NQ4;
                reinterpret_cast<float4*>(carry + (b * (kMaxNb - 1) + r) * NO)[kk] =
                    reinterpret_cast<const float4*>(tapbuf + (kTileM + r) * WROW)[kk];
              }
              epi_bar();
            }
          }
          if (pf && et == 0) {
            const long long t1e = clock64();
            pc[10] += t1e - t0e;
            t0e = t1e;
          }
          if (MODE < 2) {
            const int i_out = c * kTileM - (nb - 1) + m;
            if (i_out < 0 || i_out >= P.ext_last) continue;
            const int64_t idx = obase + (int64_t)i_out * P.lstride;
            if (MODE == 0) {
              float2* up = out + (size_t)idx * CW + CH * h;
              if (!pf) {  // counter mode keeps `out` for its records
                if (CH == 4) {
                  reinterpret_cast<float4*>(up)[0] = make_float4(v[0], v[1], v[2], v[3]);
                  reinterpret_cast<float4*>(up)[1] = make_float4(v[4], v[5], v[6], v[7 % NH]);
                } else {
#pragma unroll
                  for (int i = 0; i < CH; ++i) up[i] = make_float2(v[2 * i], v[2 * i + 1]);
                }
              }
              double s0 = 0.0, s1 = 0.0;
#pragma unroll
              for (int i = 0; i < NH; i += 2) {
                s0 += (double)v[i] * v[i];
                s1 += (double)v[i + 1] * v[i + 1];
                omax = fmaxf(omax, fmaxf(fabsf(v[i]), fabsf(v[i + 1])));
              }
              acc_v[0] += s0 + s1;
            } else {
              double d0 = 0.0, d1 = 0.0, n0 = 0.0, n1 = 0.0;
#pragma unroll
              for (int i = 0; i < CH; ++i) {
                const float2 uu = upre[i];
                if (i & 1) d1 += (double)v[2 * i] * uu.x + (double)v[2 * i + 1] * uu.y;
                else d0 += (double)v[2 * i] * uu.x + (double)v[2 * i + 1] * uu.y;
              }
#pragma unroll
              for (int i = 0; i < NH; i += 2) {
                n0 += (double)v[i] * v[i];
                n1 += (double)v[i + 1] * v[i + 1];
              }
              acc_v[0] += d0 + d1;
              acc_v[NV - 1] += n0 + n1;
            }
          } else {
            const int x = P.roff[L - 1] + c * kTileM + m;
            if (x >= P.ext_last) continue;
            double a4[4] = {0, 0, 0, 0};
            omax = fmaxf(omax, scatter_store<CH>(P, (size_t)(obase + (int64_t)x * P.lstride) * CW, h, v, din, out, a4));
#pragma unroll
            for (int i = 0; i < NV; ++i) acc_v[i] += a4[i > 3 ? 3 : i];
          }
        }
      }
      if (MODE == 2) {
        // positions no tile covers: DC term only
        const int x_lo = active ? P.roff[L - 1] : 0;
        const int x_hi = active ? P.roff[L - 1] + P.chunks * kTileM : 0;
        float vz[NH];
#pragma unroll
        for (int i = 0; i < NH; ++i) vz[i] = 0.f;
        for (int x = m; x < P.ext_last; x += kTileM) {
          if (x >= x_lo && x < x_hi) continue;
          double a4[4] = {0, 0, 0, 0};
          const size_t e0 = (size_t)(obase + (int64_t)x * P.lstride) * CW;
          omax = fmaxf(omax, scatter_store<CH>(P, e0, h, vz, dc_load<CH>(P, e0, h, mask, y, x0), out, a4));
#pragma unroll
          for (int i = 0; i < NV; ++i) acc_v[i] += a4[i > 3 ? 3 : i];
        }
      }
    }
    // fixed-order reduction over the 256 epilogue threads
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double t = warp_sum_d(acc_v[i]);
      if (lane == 0) red[ew][i] = t;
    }
    epi_bar();
    if (ew == 0 && lane < NV) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < kEpiWarps; ++w) t += red[w][lane];
      parts[(size_t)blockIdx.x * NV + lane] = t;
    }
    if (blockIdx.x == 0)
      for (int i = et + (int)gridDim.x * NV; i < P.nparts_total * NV; i += kEpiWarps * 32) parts[i] = 0.0;
    if (P.amax_out) {  // this CTA's max |output|; CTA 0 zero-fills the slot past the grid
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) omax = fmaxf(omax, __shfl_xor_sync(0xffffffffu, omax, o));
      __shared__ float wmx[kEpiWarps];
      if (lane == 0) wmx[ew] = omax;
      epi_bar();
      if (et == 0) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < kEpiWarps; ++w) t = fmaxf(t, wmx[w]);
        P.amax_out[blockIdx.x] = t;
      }
      if (blockIdx.x == 0)
        for (int i = (int)gridDim.x + et; i < kAmaxSlot; i += kEpiWarps * 32) P.amax_out[i] = 0.f;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (pf && threadIdx.x == 0) pc[9] = clock64();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
  if (pf && threadIdx.x == 0 && MODE != 1) {
    pc[9] -= pc[8];
    long long* o = reinterpret_cast<long long*>(out) + (size_t)blockIdx.x * 12;
    for (int i = 0; i < 12; ++i) o[i] = pc[i];
  }
}

// ---------------------------------------------------------------------------
// Three-line tiles (8 coils, p = 8, last-axis extent nb <= 5, 2-3 spatial axes).
//
// A kind::f16 MMA costs ~175 cycles whatever its N <= 256
// (scripts/tc_rate2.cu), so the one-line tile above, whose MMAs have N = 160
// (A_hi [B_hi; B_lo]) and N = 80 (A_lo B_hi), runs the tensor pipe at ~half
// its rate.  Here a tile computes THREE adjacent output lines i, i+1, i+2
// along the inner prefix axis.  An input line j (of the k1 + 2 that feed the
// three) serves output slot t through inner prefix j - t (conv) or
// t + k1 - 1 - j (scatter); with the prefix images of one outer prefix stored
// as consecutive images (descending / ascending), the B rows of all valid
// slots are one contiguous block, so each input line costs three MMAs of
// N = 80 (#valid slots) <= 240: A_hi B_hi, A_hi B_lo, A_lo B_hi, all into the
// slots' own columns.  Per three output lines: ko (k1 + 2) 3 MMAs instead of
// 3 ko k1 2 (C5: 105 instead of 150), and each input line is staged once per
// three outputs instead of once per output.
//
// Pipeline: a stage = one outer prefix go: a depth-(k1 + 2) TMA box of input
// lines + that prefix's hi / lo image blocks (bulk copy).  Each stage's MMAs
// accumulate into one of two TMEM sets (240 columns, alternating), reset by
// an MMA against a zero B block, and are drained by the epilogue as soon as
// they complete (chains of <= 3 k1 + 1 MMAs, as short as the one-line
// kernel's).  The epilogue sums the stages in fp32 registers per slot, then
// runs the one-line kernel's per-tap shift window, carries and fused
// objective / ELS / data-consistency epilogues for each slot.
constexpr int kTriNb = 5;

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
conv_tri_kernel(const __grid_constant__ CUtensorMap tmap, const CtParams P, float2* __restrict__ out,
                const float2* __restrict__ uin, const uint8_t* __restrict__ mask, const float2* __restrict__ y,
                const float2* __restrict__ x0, double* __restrict__ parts) {
  constexpr int CW = 8;
  constexpr int NV = MODE == 0 ? 1 : (MODE == 1 ? 2 : 4);
  using T = Cw<CW>;
  constexpr int NH = T::NH, CH = T::CH, NO = T::NO, WROW = T::WROW;
  constexpr int CARRY = kMaxNb * (kMaxNb - 1) * NO;  // carry floats of one slot
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int nb = P.nb, L = P.L, S = P.stages, sd = P.sd, ko = P.ko;
  const int k1 = L == 3 ? P.kpre[1] : P.kpre[0];
  const int nob = P.ntot;  // columns of one output slot (NO nb)
  const uint32_t hblk = (uint32_t)k1 * nob * T::BROW;  // one outer prefix's hi (or lo) image block
  const uint32_t abox = (uint32_t)sd * T::ATILE;
  const int stb = P.stage_bytes;
  uint8_t* sZero = smem;  // 3 nob zero B rows: the per-stage accumulator reset
  uint8_t* sStage = smem + 8192;
  float* sWin = reinterpret_cast<float*>(sStage + (size_t)S * stb);
  float* tapbuf = sWin;
  float* carry = sWin + (kTileM + kMaxNb - 1) * WROW;  // [slot][b][nb-1][NO]
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], tfull[2], tempty[2];
  __shared__ uint32_t tslot;
  __shared__ double red[kEpiWarps][NV];
  __shared__ float s_scale[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int inner_ext = P.ldim[L - 2];
  // debug bit 32: per-role cycle counters, written to `out` (conv forward only; same slots as conv_tc_kernel)
  __shared__ long long pc[12];
  const bool pf = (P.debug & 32) != 0;
  if (threadIdx.x < 12) pc[threadIdx.x] = 0;
  const int nunits = (L == 3 ? P.ldim[0] : 1) * P.ntri;

  for (int i = threadIdx.x; i < 8192 / 16; i += kThreads) reinterpret_cast<float4*>(sZero)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  tc::fence_proxy_async();  // the zero block is an MMA operand (async proxy)
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], kEpiWarps);
    }
    tc::mbar_init_fence();
  }
  if (warp == 1) tc::tmem_alloc(&tslot, 512);
  hicu_pdl_entry();
  if (warp == 1) {
    float m = 0.f;
    for (int i = lane; i < P.namax; i += 32) m = fmaxf(m, __ldg(P.amax + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      const float sa = pow2_scale(m);
      const float sb = *reinterpret_cast<const float*>(P.bimg + (size_t)P.ng * 2u * nob * T::BROW);
      s_scale[0] = sa;
      s_scale[1] = 1.f / (sa * sb);
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  if (pf && threadIdx.x == 0) pc[8] = clock64();

  if (warp == 0) {
    // ---------------- TMA producer: per stage the k1 + 2 input lines of one outer prefix + its image blocks ----------------
    int s = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int lo0 = L == 3 ? u / P.ntri : 0, lin0 = 3 * (u % P.ntri);
      for (int c = 0; c < P.chunks; ++c)
        for (int go = 0; go < ko; ++go) {
          const long long t0p = (pf && lane == 0) ? clock64() : 0;
          tc::mbar_wait(&empty[s], ph ^ 1);
          if (pf && lane == 0) pc[0] += clock64() - t0p;
          const int c1 = MODE < 2 ? P.roff[L - 1] + c * kTileM : c * kTileM;
          const int c2 = MODE < 2 ? P.roff[L - 2] + lin0 : lin0 - P.roff[L - 2] - (k1 - 1);
          const int c3 = L == 3 ? (MODE < 2 ? P.roff[0] + lo0 + go : lo0 - P.roff[0] - go) : 0;
          if (tc::elect_one()) {
            uint8_t* dst = sStage + (size_t)s * stb;
            tc::mbar_expect_tx(&full[s], abox + 2u * hblk);
            tc::tma_load_4d(dst, &tmap, 0, c1, c2, c3, &full[s]);
            bulk_g2s(dst + abox, P.bimg + (size_t)go * 2u * hblk, 2u * hblk, &full[s]);
          }
          __syncwarp();
          if (++s == S) { s = 0; ph ^= 1; }
        }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint64_t dstage0 = desc_swz<T::RB>(tc::smem_u32(sStage));
    const uint64_t dimg0 = desc_swz<T::BROW>(tc::smem_u32(sStage + abox));
    const uint64_t dzero = desc_swz<T::BROW>(tc::smem_u32(sZero));
    const uint32_t idesc3 = tc::idesc_f16(kTileM, 3 * nob);
    const uint32_t stb16 = (uint32_t)stb >> 4, img16 = ((uint32_t)nob * T::BROW) >> 4, lo16 = hblk >> 4;
    int s = 0;
    uint32_t ph = 0, tcnt = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x)
      for (int c = 0; c < P.chunks; ++c) {
        // one TMEM set per tile, alternating: the next tile's MMAs run while the epilogue drains this one
        const uint32_t set = tcnt & 1u, tp = (tcnt >> 1) & 1u;
        const uint32_t d = tmem + set * 256u;
        for (int go = 0; go < ko; ++go) {
          const long long t0r = (pf && lane == 0) ? clock64() : 0;
          tc::mbar_wait(&full[s], ph);
          const long long t1r = (pf && lane == 0) ? clock64() : 0;
          if (pf && lane == 0) pc[3] += t1r - t0r;
          if (go == 0) tc::mbar_wait(&tempty[set], tp ^ 1u);  // the epilogue drained this set's previous tile
          if (pf && lane == 0) pc[4] += clock64() - t1r;
          tc::fence_after();
          if (tc::elect_one()) {
            const uint64_t da = dstage0 + (uint64_t)(s * stb16);
            const uint64_t db = dimg0 + (uint64_t)(s * stb16);
            if (go == 0) tc::mma_f16(d, da, dzero, idesc3, 0u);  // reset the set's 3 nob columns
            for (int j = 0; j < sd; ++j) {
              const int t_lo = max(0, j - k1 + 1), t_hi = min(2, j);
              if (t_lo > t_hi) continue;
              const uint32_t idesc = tc::idesc_f16(kTileM, (t_hi - t_lo + 1) * nob);
              const uint64_t ah = da + (uint64_t)((j * T::ATILE) >> 4), al = ah + 2u;  // lo half: +32 B of the row
              const uint64_t bh = db + (uint64_t)((t_lo + k1 - 1 - j) * img16), bl = bh + lo16;
              const uint32_t dd = d + (uint32_t)(t_lo * nob);
              tc::mma_f16(dd, ah, bh, idesc, 1u);  // A_hi B_hi
              tc::mma_f16(dd, ah, bl, idesc, 1u);  // A_hi B_lo
              tc::mma_f16(dd, al, bh, idesc, 1u);  // A_lo B_hi
            }
            tc::mma_commit(&empty[s]);
            if (go == ko - 1) tc::mma_commit(&tfull[set]);
          }
          __syncwarp();
          if (++s == S) { s = 0; ph ^= 1; }
        }
        ++tcnt;
      }
  } else {
    // ---------------- epilogue ----------------
    const int ew = warp - 2;
    const int q = warp & 3, h = ew >> 2;
    const int m = 32 * q + lane;
    const int et = threadIdx.x - 64;
    const float inv = s_scale[1];
    constexpr int NQ4 = NO / 4;
    double acc_v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc_v[i] = 0.0;
    float omax = 0.f;
    uint32_t tcnt = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int lo0 = L == 3 ? u / P.ntri : 0, lin0 = 3 * (u % P.ntri);
      for (int i = et; i < 3 * CARRY; i += kEpiWarps * 32) carry[i] = 0.f;
      epi_bar();
      for (int c = 0; c < P.chunks; ++c) {
        const uint32_t set = tcnt & 1u, tp = (tcnt >> 1) & 1u;
        {
          const long long t0e = (pf && et == 0) ? clock64() : 0;
          tc::mbar_wait(&tfull[set], tp);
          if (pf && et == 0) pc[6] += clock64() - t0e;
        }
        tc::fence_after();
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + set * 256u + (uint32_t)(NH * h);
        const long long t0w = (pf && et == 0) ? clock64() : 0;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int inner = lin0 + t;
          if (inner >= inner_ext) continue;  // uniform: the partial group at the end of the inner axis
          const int64_t obase = L == 3 ? (int64_t)lo0 * P.ostride[0] + (int64_t)inner * P.ostride[1]
                                       : (int64_t)inner * P.ostride[0];
          float* cy = carry + t * CARRY;
          // this slot's accumulators (nb taps x NH floats of this thread's row)
          float f[kTriNb][NH];
          {
            uint32_t v0[kTriNb][NH];
#pragma unroll
            for (int b = 0; b < kTriNb; ++b)
              if (b < nb) tc::tmem_ld8_nowait(ta + (uint32_t)(t * nob + b * NO), v0[b]);
            tc::tmem_wait_ld();
#pragma unroll
            for (int b = 0; b < kTriNb; ++b)
#pragma unroll
              for (int i = 0; i < NH; ++i) f[b][i] = __uint_as_float(v0[b][i]);
          }
          // this slot's epilogue inputs from global memory
          DcIn<CH> din{};
          float2 upre[CH];
#pragma unroll
          for (int i = 0; i < CH; ++i) upre[i] = make_float2(0.f, 0.f);
          if (MODE == 2) {
            const int x = P.roff[L - 1] + c * kTileM + m;
            if (x < P.ext_last) din = dc_load<CH>(P, (size_t)(obase + (int64_t)x * P.lstride) * CW, h, mask, y, x0);
          } else if (MODE == 1) {
            const int i_out = c * kTileM - (nb - 1) + m;
            if (i_out >= 0 && i_out < P.ext_last) {
              const float4* up = reinterpret_cast<const float4*>(uin + (size_t)(obase + (int64_t)i_out * P.lstride) * CW + CH * h);
              const float4 a0 = __ldg(up), a1 = __ldg(up + 1);
              upre[0] = make_float2(a0.x, a0.y);
              upre[1] = make_float2(a0.z, a0.w);
              upre[2] = make_float2(a1.x, a1.y);
              upre[3] = make_float2(a1.z, a1.w);
            }
          }
          // shifted sums, one tap at a time (as in conv_tc_kernel)
          float v[NH];
#pragma unroll
          for (int i = 0; i < NH; ++i) v[i] = 0.f;
#pragma unroll
          for (int b = 0; b < kTriNb; ++b) {
            if (b < nb) {
              if (et < (nb - 1) * NQ4) {
                const int r = et / NQ4, kk = et - r * NQ4;
                reinterpret_cast<float4*>(tapbuf + r * WROW)[kk] =
                    reinterpret_cast<const float4*>(cy + (b * (kMaxNb - 1) + r) * NO)[kk];
              }
              const int w = MODE < 2 ? m + b : nb - 1 + m - b;
              float4* w4 = reinterpret_cast<float4*>(tapbuf + (nb - 1 + m) * WROW + NH * h);
              w4[0] = make_float4(f[b][0] * inv, f[b][1] * inv, f[b][2] * inv, f[b][3] * inv);
              w4[1] = make_float4(f[b][4] * inv, f[b][5] * inv, f[b][6] * inv, f[b][7] * inv);
              epi_bar();
              const float4* r4 = reinterpret_cast<const float4*>(tapbuf + w * WROW + NH * h);
              const float4 t0 = r4[0], t1 = r4[1];
              v[0] += t0.x; v[1] += t0.y; v[2] += t0.z; v[3] += t0.w;
              v[4] += t1.x; v[5] += t1.y; v[6] += t1.z; v[7] += t1.w;
              if (et < (nb - 1) * NQ4) {
                const int r = et / NQ4, kk = et - r * NQ4;
                reinterpret_cast<float4*>(cy + (b * (kMaxNb - 1) + r) * NO)[kk] =
                    reinterpret_cast<const float4*>(tapbuf + (kTileM + r) * WROW)[kk];
              }
              epi_bar();
            }
          }
          if (MODE < 2) {
            const int i_out = c * kTileM - (nb - 1) + m;
            if (i_out < 0 || i_out >= P.ext_last) continue;
            const int64_t idx = obase + (int64_t)i_out * P.lstride;
            if (MODE == 0) {
              float4* up = reinterpret_cast<float4*>(out + (size_t)idx * CW + CH * h);
              if (!pf) {  // counter mode keeps `out` for its records
                up[0] = make_float4(v[0], v[1], v[2], v[3]);
                up[1] = make_float4(v[4], v[5], v[6], v[7]);
              }
              double s0 = 0.0, s1 = 0.0;
#pragma unroll
              for (int i = 0; i < NH; i += 2) {
                s0 += (double)v[i] * v[i];
                s1 += (double)v[i + 1] * v[i + 1];
                omax = fmaxf(omax, fmaxf(fabsf(v[i]), fabsf(v[i + 1])));
              }
              acc_v[0] += s0 + s1;
            } else {
              double d0 = 0.0, d1 = 0.0, n0 = 0.0, n1 = 0.0;
#pragma unroll
              for (int i = 0; i < CH; ++i) {
                const float2 uu = upre[i];
                if (i & 1) d1 += (double)v[2 * i] * uu.x + (double)v[2 * i + 1] * uu.y;
                else d0 += (double)v[2 * i] * uu.x + (double)v[2 * i + 1] * uu.y;
              }
#pragma unroll
              for (int i = 0; i < NH; i += 2) {
                n0 += (double)v[i] * v[i];
                n1 += (double)v[i + 1] * v[i + 1];
              }
              acc_v[0] += d0 + d1;
              acc_v[NV - 1] += n0 + n1;
            }
          } else {
            const int x = P.roff[L - 1] + c * kTileM + m;
            if (x >= P.ext_last) continue;
            double a4[4] = {0, 0, 0, 0};
            omax = fmaxf(omax, scatter_store<CH>(P, (size_t)(obase + (int64_t)x * P.lstride) * CW, h, v, din, out, a4));
#pragma unroll
            for (int i = 0; i < NV; ++i) acc_v[i] += a4[i > 3 ? 3 : i];
          }
        }
        if (pf && et == 0) pc[10] += clock64() - t0w;
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[set]);  // all three slots read
        ++tcnt;
      }
      if (MODE == 2) {
        // positions no tile covers (before the region's reach / past the last tile): DC term only
        const int x_lo = P.roff[L - 1], x_hi = P.roff[L - 1] + P.chunks * kTileM;
        float vz[NH];
#pragma unroll
        for (int i = 0; i < NH; ++i) vz[i] = 0.f;
        for (int t = 0; t < 3; ++t) {
          const int inner = lin0 + t;
          if (inner >= inner_ext) break;
          const int64_t obase = L == 3 ? (int64_t)lo0 * P.ostride[0] + (int64_t)inner * P.ostride[1]
                                       : (int64_t)inner * P.ostride[0];
          for (int x = m; x < P.ext_last; x += kTileM) {
            if (x >= x_lo && x < x_hi) continue;
            double a4[4] = {0, 0, 0, 0};
            const size_t e0 = (size_t)(obase + (int64_t)x * P.lstride) * CW;
            omax = fmaxf(omax, scatter_store<CH>(P, e0, h, vz, dc_load<CH>(P, e0, h, mask, y, x0), out, a4));
#pragma unroll
            for (int i = 0; i < NV; ++i) acc_v[i] += a4[i > 3 ? 3 : i];
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double t = warp_sum_d(acc_v[i]);
      if (lane == 0) red[ew][i] = t;
    }
    epi_bar();
    if (ew == 0 && lane < NV) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < kEpiWarps; ++w) t += red[w][lane];
      parts[(size_t)blockIdx.x * NV + lane] = t;
    }
    if (blockIdx.x == 0)
      for (int i = et + (int)gridDim.x * NV; i < P.nparts_total * NV; i += kEpiWarps * 32) parts[i] = 0.0;
    if (P.amax_out) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) omax = fmaxf(omax, __shfl_xor_sync(0xffffffffu, omax, o));
      __shared__ float wmx[kEpiWarps];
      if (lane == 0) wmx[ew] = omax;
      epi_bar();
      if (et == 0) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < kEpiWarps; ++w) t = fmaxf(t, wmx[w]);
        P.amax_out[blockIdx.x] = t;
      }
      if (blockIdx.x == 0)
        for (int i = (int)gridDim.x + et; i < kAmaxSlot; i += kEpiWarps * 32) P.amax_out[i] = 0.f;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (pf && threadIdx.x == 0) pc[9] = clock64();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
  if (pf && threadIdx.x == 0 && MODE == 0) {
    pc[9] -= pc[8];
    long long* o = reinterpret_cast<long long*>(out) + (size_t)blockIdx.x * 12;
    for (int i = 0; i < 12; ++i) o[i] = pc[i];
  }
}

// B images (fp16 hi/lo, scaled) for one Q~, written once to global memory so
// each conv CTA copies them with one bulk copy; the power-of-two scale sits
// in a trailer after the ng images.  One CTA per image.
template <int MODE, int CW>
__global__ void __launch_bounds__(kThreads) conv_bimage_kernel(const CtParams P, const int32_t* __restrict__ pos,
                                                               const float2* __restrict__ qt_all, size_t qt_stride,
                                                               uint8_t* __restrict__ img_all, size_t img_stride,
                                                               int img_off) {
  hicu_pdl_entry();
  __shared__ int spos[kMaxTaps][3];
  __shared__ float wmax[kThreads / 32];
  const int L = P.L;
  const uint32_t gbytes = 2u * (uint32_t)P.ntot * Cw<CW>::BROW;
  uint8_t* img = img_all + (size_t)(2 * blockIdx.x + img_off) * img_stride;
  const float2* qt = qt_all + (size_t)blockIdx.x * qt_stride;
  for (int t = threadIdx.x; t < P.nsp * L; t += kThreads)
    spos[t / L][t % L] = __ldg(pos + (size_t)(t / L) * CW * P.ndim + P.perm[t % L]);
  const int nq = P.nsp * CW * CW;
  float m = 0.f;
  for (int e = threadIdx.x; e < nq; e += kThreads) {
    const float2 q = __ldg(qt + e);
    m = fmaxf(m, fmaxf(fabsf(q.x), fabsf(q.y)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
  float4* z = reinterpret_cast<float4*>(img);
  for (int i = threadIdx.x; i < P.ng * (int)gbytes / 16; i += kThreads) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();  // zeroing and the max before the image entries
  float mm = 0.f;
  for (int w = 0; w < kThreads / 32; ++w) mm = fmaxf(mm, wmax[w]);
  const float sb = pow2_scale(mm);
  for (int e = threadIdx.x; e < nq; e += kThreads) bimage_put<MODE, CW>(img, P, spos, e, __ldg(qt + e), gbytes, sb);
  if (threadIdx.x == 0) *reinterpret_cast<float*>(img + (size_t)P.ng * gbytes) = sb;
}

// A operand split: each row of 16 floats -> 64 bytes [16 fp16 hi | 16 fp16 lo]
// of x s_A (s_A from the amax partials of the kernel launched just before),
// written in the conv's axis order (line axis fastest), so that every
// 128-row TMA box of the conv is one contiguous 8 KB block (a box along a
// slow axis of the natural layout gathers 128 rows a whole plane apart, and
// the TMA unit then paces the pipeline).  The conv's MMAs read hi as K step
// 0 and lo as K step 1 of the same 64-byte operand rows.  One row per thread.
struct SplitParams {
  int L;
  int64_t ext[3];   // natural (C-order) extents of the spatial axes
  int perm[3];      // kernel axis k = natural axis perm[k]; perm[L-1] is the line axis (fastest in the output)
  int64_t istr[3];  // input (natural C-order) row stride of natural axis a
};

// 4 floats x s -> 4 fp16 hi + 4 fp16 lo halves (8 bytes each)
__device__ __forceinline__ void split4(float4 v, float sa, uint2& hi, uint2& lo) {
  const float x0 = v.x * sa, x1 = v.y * sa, x2 = v.z * sa, x3 = v.w * sa;
  const __half2 h01 = __floats2half2_rn(x0, x1), h23 = __floats2half2_rn(x2, x3);
  const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
  hi = make_uint2(h2u(h01), h2u(h23));
  lo = make_uint2(h2u(__floats2half2_rn(x0 - f01.x, x1 - f01.y)), h2u(__floats2half2_rn(x2 - f23.x, x3 - f23.y)));
}

__device__ __forceinline__ float split_scale(const float* __restrict__ amax, int namax) {
  float m = 0.f;
  for (int i = threadIdx.x; i < namax; i += 32) m = fmaxf(m, __ldg(amax + i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  return pow2_scale(m);
}

template <int CW>
__global__ void __launch_bounds__(256) split_kernel(const float4* __restrict__ x, int64_t rows, const SplitParams sp,
                                                    const float* __restrict__ amax, int namax, uint4* __restrict__ out) {
  using T = Cw<CW>;
  constexpr int QR = T::KA / 4, QP = T::KP / 4;  // float4 pieces per input row; 8-byte pieces per half
  hicu_pdl_entry();
  __shared__ float s_sa;
  if (threadIdx.x < 32) {
    const float m = split_scale(amax, namax);
    if (threadIdx.x == 0) s_sa = m;
  }
  __syncthreads();
  const float sa = s_sa;
  // threads walk OUTPUT rows (consecutive threads write consecutive rows:
  // coalesced stores); each reads its whole input row
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < rows; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = o, r = 0;
    for (int k = sp.L - 1; k >= 0; --k) {
      const int a = sp.perm[k];
      const int64_t ca = t % sp.ext[a];
      t /= sp.ext[a];
      r += ca * sp.istr[a];
    }
    uint2 hw[QP], lw[QP];
#pragma unroll
    for (int k = 0; k < QP; ++k) {
      if (k < QR) split4(__ldg(x + r * QR + k), sa, hw[k], lw[k]);
      else hw[k] = lw[k] = make_uint2(0u, 0u);
    }
    uint4* po = out + o * (T::RB / 16);
#pragma unroll
    for (int k = 0; k < QP / 2; ++k) {
      po[k] = make_uint4(hw[2 * k].x, hw[2 * k].y, hw[2 * k + 1].x, hw[2 * k + 1].y);
      po[QP / 2 + k] = make_uint4(lw[2 * k].x, lw[2 * k].y, lw[2 * k + 1].x, lw[2 * k + 1].y);
    }
  }
}

// The same split as a batched tiled transpose, for a line axis that is not
// the array's fastest: the natural array is [A][Lx][B] rows (Lx = line
// axis), the output [A][B][Lx].  A kTT x TB tile of rows is read as runs of
// TB contiguous rows and written as runs of kTT contiguous rows, so both
// directions are coalesced (the row-per-thread split_kernel reads rows a
// plane apart).  Grid (ceil(B/TB), ceil(Lx/kTT), A), 256 threads.
constexpr int kTT = 32;
template <int CW>
struct TT {
  static constexpr int TB = Cw<CW>::RB == 64 ? 8 : 4;        // B rows per tile (16 KB of shared memory)
  static constexpr int PITCH = kTT * Cw<CW>::RB + 32;         // bytes per tile b-row (+32: fewer store conflicts)
  static constexpr int SMEM = TB * PITCH;
};

template <int CW>
__global__ void __launch_bounds__(256) split_t_kernel(const float4* __restrict__ x, int64_t Lx, int64_t B,
                                                      const float* __restrict__ amax, int namax,
                                                      uint4* __restrict__ out) {
  using T = Cw<CW>;
  constexpr int QR = T::KA / 4, QP = T::KP / 4, TB = TT<CW>::TB, PITCH = TT<CW>::PITCH;
  hicu_pdl_entry();
  extern __shared__ __align__(16) uint8_t tt[];
  __shared__ float s_sa;
  if (threadIdx.x < 32) {
    const float m = split_scale(amax, namax);
    if (threadIdx.x == 0) s_sa = m;
  }
  __syncthreads();
  const float sa = s_sa;
  const int64_t b0 = (int64_t)blockIdx.x * TB, l0 = (int64_t)blockIdx.y * kTT, a = blockIdx.z;
  // read: piece i -> (lx_l, b_l, pc): runs of TB rows along B (pads written as zeros)
  for (int i = threadIdx.x; i < kTT * TB * QP; i += 256) {
    const int pc = i % QP, b_l = (i / QP) % TB, lx_l = i / (QP * TB);
    const int64_t lx = l0 + lx_l, b = b0 + b_l;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (pc < QR && lx < Lx && b < B) v = __ldg(x + ((a * Lx + lx) * B + b) * QR + pc);
    uint2 hi, lo;
    split4(v, sa, hi, lo);
    uint8_t* row = tt + b_l * PITCH + lx_l * T::RB;
    *reinterpret_cast<uint2*>(row + pc * 8) = hi;
    *reinterpret_cast<uint2*>(row + 2 * T::KP + pc * 8) = lo;
  }
  __syncthreads();
  // write: piece i -> (b_l, lx_l, chunk): runs of kTT rows along Lx
  constexpr int NCH = T::RB / 16;
  for (int i = threadIdx.x; i < kTT * TB * NCH; i += 256) {
    const int ch = i % NCH, lx_l = (i / NCH) % kTT, b_l = i / (NCH * kTT);
    const int64_t lx = l0 + lx_l, b = b0 + b_l;
    if (lx < Lx && b < B)
      out[((a * B + b) * Lx + lx) * NCH + ch] = *reinterpret_cast<const uint4*>(tt + b_l * PITCH + lx_l * T::RB + ch * 16);
  }
}

// max |component| partials of an fp32 array (the A-operand scale of the next conv)
__global__ void __launch_bounds__(256) amax_kernel(const float4* __restrict__ x, int64_t n4, float* __restrict__ part) {
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

thread_local const uint8_t* t_bimg = nullptr;
thread_local int t_bimg_early = 0;
thread_local const float* t_amax_in = nullptr;  // the A operand's max partials, written by its producer
thread_local float* t_amax_out = nullptr;       // where this launch's epilogue writes its output's max partials

// Per-(device, stream) scratch: amax partials and the B images of calls that
// arrive without prebuilt ones.  Kernels on one stream run in order, so one
// buffer per stream is race-free; it only grows.
uint8_t* stream_scratch(cudaStream_t st, size_t bytes) {
  struct Entry {
    int dev;
    cudaStream_t st;
    uint8_t* p;
    size_t n;
  };
  static std::mutex mu;
  static std::vector<Entry> entries;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : entries)
    if (e.dev == dev && e.st == st) {
      if (e.n >= bytes) return e.p;
      cudaStreamSynchronize(st);
      cudaFree(e.p);
      e.p = nullptr;
      if (cudaMalloc(&e.p, bytes) != cudaSuccess) {
        cudaGetLastError();
        e.n = 0;
        return nullptr;
      }
      e.n = bytes;
      return e.p;
    }
  uint8_t* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  entries.push_back({dev, st, p, bytes});
  return p;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
    else
      cudaGetLastError();
  }
  return fn;
}

// 4-D map over a row-major [ext[0], .., ext[L-1], 16 floats] array seen in
// the kernel's axis order: dims (16, ext[perm[L-1]], ext[perm[L-2]],
// ext[perm[L-3]]) with the array's own strides (any spatial axis can be the
// tile axis), 128-row x 16-float boxes (one per stage), no swizzle (only the converter warps
// read the fp32 tile: linear 16-byte reads), zero fill out of bounds.
int make_tmap(CUtensorMap* tm, const void* base, int L, const int64_t* ext, const int* perm, int cw, int depth) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return hicu_set_error(HICU_ERR_CUDA, "conv_tc: cuTensorMapEncodeTiled unavailable");
  // the split array is stored in kernel axis order: line axis perm[L-1] fastest; rows of
  // [KP hi | KP lo] fp16 (64 B: SWIZZLE_64B, 128 B: SWIZZLE_128B)
  const int kp = cw == 8 ? 16 : 32, rb = 4 * kp, gps = cw == 8 ? Cw<8>::GPS : Cw<10>::GPS;
  cuuint64_t dims[4] = {(cuuint64_t)(2 * kp), (cuuint64_t)ext[perm[L - 1]], (cuuint64_t)(L >= 2 ? ext[perm[L - 2]] : 1),
                        (cuuint64_t)(L >= 3 ? ext[perm[L - 3]] : 1)};
  cuuint64_t strides[3] = {(cuuint64_t)rb, rb * dims[1], rb * dims[1] * dims[2]};
  // depth GPS along dimension 2: a stage's prefix groups are adjacent lines
  cuuint32_t box[4] = {(cuuint32_t)(2 * kp), (cuuint32_t)kTileM, (cuuint32_t)(L >= 2 ? (depth > 0 ? depth : gps) : 1), 1},
             es[4] = {1, 1, 1, 1};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return hicu_set_error(HICU_ERR_CUDA, "conv_tc: cuTensorMapEncodeTiled failed");
  return HICU_OK;
}

// Tensor maps depend only on (pointer, extents, axis order): a small
// per-thread cache keeps cuTensorMapEncodeTiled off the per-launch path.
int cached_tmap(CUtensorMap* tm, const void* base, int L, const int64_t* ext, const int* perm, int cw, int depth) {
  struct Entry {
    const void* base;
    int L, cw, depth;
    int64_t ext[3];
    int perm[3];
    CUtensorMap map;
  };
  static thread_local Entry cache[16];
  static thread_local int used = 0, next = 0;
  for (int i = 0; i < used; ++i) {
    const Entry& e = cache[i];
    bool same = e.base == base && e.L == L && e.cw == cw && e.depth == depth;
    for (int d = 0; d < L && same; ++d) same = e.ext[d] == ext[d] && e.perm[d] == perm[d];
    if (same) {
      *tm = e.map;
      return HICU_OK;
    }
  }
  const int st = make_tmap(tm, base, L, ext, perm, cw, depth);
  if (st) return st;
  Entry& e = cache[next];
  e.base = base;
  e.L = L;
  e.cw = cw;
  e.depth = depth;
  for (int d = 0; d < 3; ++d) {
    e.ext[d] = d < L ? ext[d] : 0;
    e.perm[d] = d < L ? perm[d] : 0;
  }
  e.map = *tm;
  next = (next + 1) % 16;
  if (used < 16) ++used;
  return HICU_OK;
}

// Per-(device, stream) producer max slots (3 x kAmaxSlot floats), never
// reallocated: a slot written by one call is read by a later call.
float* stream_amax_slots(cudaStream_t st) {
  struct Entry {
    int dev;
    cudaStream_t st;
    float* p;
  };
  static std::mutex mu;
  static std::vector<Entry> entries;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : entries)
    if (e.dev == dev && e.st == st) return e.p;
  float* p = nullptr;
  if (cudaMalloc(&p, 3 * kAmaxSlot * sizeof(float)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  entries.push_back({dev, st, p});
  return p;
}

// Tile ("line") axis: the spatial axis that minimises the 128-row tiles the
// kernel walks, lines x ceil((extent + nb - 1) / 128): a k-space volume
// whose last axis is short (C4: 25 frames -> one 20 %-full tile per line) is
// tiled along a long axis instead (C4: x; C5: readout, 252 + 4 = 256 rows =
// two full tiles instead of 160-row lines in two tiles).
void choose_perm(const DevGeom& g, int MODE, int (&perm)[3]) {
  const int L = g.ndim - 1;
  const int64_t* lext = MODE < 2 ? g.rext : g.dims;
  int best = L - 1;
  double best_tiles = 1e300;
  for (int a = L - 1; a >= 0; --a) {
    // the original last axis, or any axis with >= 2 taps (a 1-tap tile axis would
    // chain every tap's MMA into one TMEM accumulator: fp32 rounding grows)
    if (g.kext[a] > kMaxNb || (a != L - 1 && g.kext[a] < 2)) continue;
    int64_t ng = 1;
    for (int b = 0; b < L; ++b)
      if (b != a) ng *= g.kext[b];
    if (ng > kMaxGroups) continue;
    double lines = 1.0;
    for (int b = 0; b < L; ++b)
      if (b != a) lines *= (double)lext[b];
    const double tiles = lines * (double)((g.rext[a] + g.kext[a] - 1 + kTileM - 1) / kTileM);
    if (tiles < best_tiles) {
      best_tiles = tiles;
      best = a;
    }
  }
  int k = 0;
  for (int a = 0; a < L; ++a)
    if (a != best) perm[k++] = a;
  perm[L - 1] = best;
  for (int d = L; d < 3; ++d) perm[d] = d;
}

// HICU_CONV_TC_TRI=0 keeps the one-line tiles (A/B measurement of the three-line kernel)
bool tri_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HICU_CONV_TC_TRI");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}

struct Shape {
  int L, nb, ng, kpre[2];
  int cw;            // complex row width (8 or 10)
  int ntot, cat;     // MMA N of one precision block; A_hi [B_hi; B_lo] in one MMA
  size_t gbytes;     // B image bytes of one prefix (hi + lo blocks)
  int bstream;       // B images copied per stage (they do not fit resident)
  size_t stage;      // bytes per pipeline stage
  size_t fixed;      // resident B images + window + alignment slack
  int tri;           // three-line tiles (conv_tri_kernel) and their B-image layout
  int sd;            // tri: input lines per stage (k1 + 2)
  size_t tstage, tfixed;  // tri: bytes per stage, fixed bytes (zero block + window + 3 carries + slack)
};

template <int CW>
bool shape_cw(const DevGeom& g, Shape* sh, const int* perm) {
  using T = Cw<CW>;
  const int L = g.ndim - 1;
  int ng = 1;
  for (int d = 0; d < L; ++d)
    if (g.kext[d] < 1) return false;
  for (int d = 0; d < L - 1; ++d) ng *= (int)g.kext[perm[d]];
  const int nb = (int)g.kext[perm[L - 1]];
  if (nb > kMaxNb || ng > kMaxGroups) return false;
  const int ntot = (T::NO * nb + 15) / 16 * 16;
  if (ntot > 256) return false;
  sh->L = L;
  sh->nb = nb;
  sh->ng = ng;
  sh->kpre[0] = L >= 2 ? (int)g.kext[perm[0]] : 1;
  sh->kpre[1] = L >= 3 ? (int)g.kext[perm[1]] : 1;
  sh->cw = CW;
  sh->ntot = ntot;
  sh->cat = T::CAT ? 1 : 0;
  if (T::CAT && 2 * ntot > 256) return false;
  sh->gbytes = (size_t)2 * ntot * T::BROW;
  const size_t win = ((size_t)T::WIN_FLOATS * 4 + 1023) & ~(size_t)1023;
  // resident B images when they fit next to >= 3 stages, else the stage groups' images per stage
  const size_t res_fixed = (size_t)ng * sh->gbytes + win + 1024;
  if (res_fixed + 3 * (size_t)T::ASTAGE <= (size_t)kSmemBudget) {
    sh->bstream = 0;
    sh->stage = T::ASTAGE;
    sh->fixed = res_fixed;
  } else {
    sh->bstream = 1;
    sh->stage = T::ASTAGE + T::GPS * sh->gbytes;
    sh->fixed = win + 1024;
  }
  // three-line tiles: 8 coils, 3 slots x 16 nb <= 256 MMA columns, a
  // depth-(k1 + 2) box of input lines per stage, >= 2 stages
  sh->tri = 0;
  if (CW == 8 && L >= 2 && nb <= kTriNb && !(tri_disabled())) {
    const int k1 = L == 3 ? sh->kpre[1] : sh->kpre[0];
    sh->sd = k1 + 2;
    const size_t twin = ((size_t)((kTileM + kMaxNb - 1) * T::WROW + 3 * kMaxNb * (kMaxNb - 1) * T::NO) * 4 + 1023) &
                        ~(size_t)1023;
    sh->tfixed = 8192 + twin + 1024;
    sh->tstage = ((size_t)sh->sd * T::ATILE + 2 * (size_t)k1 * ntot * T::BROW + 1023) & ~(size_t)1023;
    if (sh->sd <= 8 && sh->tfixed + 2 * sh->tstage <= (size_t)kSmemBudget) sh->tri = 1;
  }
  return sh->fixed + 3 * sh->stage <= (size_t)kSmemBudget;
}

bool shape_of(const DevGeom& g, int p, Shape* sh, const int* perm) {
  const int L = g.ndim - 1;
  if (g.ncirc != 0 || L < 1 || L > 3 || g.nsp < 1 || g.nsp > kMaxTaps) return false;
  if (g.nc == 8 && p == 8 && g.kext[L] == 8) return shape_cw<8>(g, sh, perm);
  if (g.nc == 10 && p == 10 && g.kext[L] == 10) return shape_cw<10>(g, sh, perm);
  return false;
}

// bytes of one B image set (ng fp16 group images + the scale trailer)
size_t image_bytes(const Shape& sh) { return (size_t)sh.ng * sh.gbytes + 256; }

template <int MODE, bool BS, int CW>
int launch_bs(const Shape& sh, CtParams P, const CUtensorMap& tm, float2* out, const float2* uin, const uint8_t* mask,
              const float2* y, const float2* x0, double* parts, int64_t lines, int nparts_total, cudaStream_t st) {
  // dynamic shared memory available to this instantiation on the current
  // device (the opt-in attribute is per device: hicu_allow_max_smem raises it
  // once per (kernel, device) and is called on every launch; the derived
  // budget is cached per device id and published after the attribute is set,
  // so a concurrent first launch from another host thread cannot race it)
  constexpr int kMaxDev = 64;
  static std::atomic<size_t> avail_a[kMaxDev];
  int dev = 0;
  cudaGetDevice(&dev);
  hicu_allow_max_smem((const void*)conv_tc_kernel<MODE, BS, CW>);
  size_t avail = (dev >= 0 && dev < kMaxDev) ? avail_a[dev].load(std::memory_order_acquire) : 0;
  if (!avail) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)conv_tc_kernel<MODE, BS, CW>);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    avail = (size_t)optin - fa.sharedSizeBytes;
    if (dev >= 0 && dev < kMaxDev) avail_a[dev].store(avail, std::memory_order_release);
  }
  if (avail < sh.fixed + 3 * sh.stage) return hicu_set_error(HICU_ERR_SIZE, "conv_tc: shared memory");
  P.stages = (int)((avail - sh.fixed) / sh.stage);
  if (P.stages > kMaxStages) P.stages = kMaxStages;
  const size_t smem = sh.fixed + (size_t)P.stages * sh.stage;
  int64_t grid = lines;
  if (grid > hicu_sm_count()) grid = hicu_sm_count();
  if (grid > nparts_total) grid = nparts_total;
  if (grid < 1) grid = 1;
  hicu_launch(conv_tc_kernel<MODE, BS, CW>, (int)grid, kThreads, smem, st, tm, P, out, uin, mask, y, x0, parts);
  return hicu_check_launch("conv_tc_kernel");
}

template <int MODE>
int launch_tri(const Shape& sh, CtParams P, const CUtensorMap& tm, float2* out, const float2* uin, const uint8_t* mask,
               const float2* y, const float2* x0, double* parts, int nparts_total, cudaStream_t st) {
  constexpr int kMaxDev = 64;
  static std::atomic<size_t> avail_a[kMaxDev];
  int dev = 0;
  cudaGetDevice(&dev);
  hicu_allow_max_smem((const void*)conv_tri_kernel<MODE>);
  size_t avail = (dev >= 0 && dev < kMaxDev) ? avail_a[dev].load(std::memory_order_acquire) : 0;
  if (!avail) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)conv_tri_kernel<MODE>);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    avail = (size_t)optin - fa.sharedSizeBytes;
    if (dev >= 0 && dev < kMaxDev) avail_a[dev].store(avail, std::memory_order_release);
  }
  if (avail < sh.tfixed + 2 * sh.tstage) return hicu_set_error(HICU_ERR_SIZE, "conv_tc: shared memory (three-line tiles)");
  P.stage_bytes = (int)sh.tstage;
  P.stages = (int)std::min<size_t>(kMaxStages, (avail - sh.tfixed) / sh.tstage);
  const size_t smem = sh.tfixed + (size_t)P.stages * sh.tstage;
  P.ntri = (P.ldim[P.L - 2] + 2) / 3;
  const int64_t units = (int64_t)(P.L == 3 ? P.ldim[0] : 1) * P.ntri;
  int64_t grid = std::min<int64_t>(units, hicu_sm_count());
  if (grid > nparts_total) grid = nparts_total;
  if (grid < 1) grid = 1;
  hicu_launch(conv_tri_kernel<MODE>, (int)grid, kThreads, smem, st, tm, P, out, uin, mask, y, x0, parts);
  return hicu_check_launch("conv_tri_kernel");
}

void fill_shape_params(CtParams& P, const DevGeom& g, const Shape& sh, const int (&perm)[3]) {
  P.tri = sh.tri;
  P.ko = sh.L == 3 ? sh.kpre[0] : 1;
  P.sd = sh.sd;
  P.ntot = sh.ntot;
  P.cat = sh.cat;
  for (int d = 0; d < 3; ++d) P.perm[d] = perm[d];
  P.L = sh.L;
  P.nsp = g.nsp;
  P.ndim = g.ndim;
  P.nb = sh.nb;
  P.ng = sh.ng;
  P.kpre[0] = sh.kpre[0];
  P.kpre[1] = sh.kpre[1];
}

template <int MODE>
int build_image(const DevGeom& g, const Shape& sh, const int (&perm)[3], const float2* qt_all, int G, uint8_t* img,
                size_t ib, int img_off, cudaStream_t st) {
  CtParams P{};
  fill_shape_params(P, g, sh, perm);
  const size_t qs = (size_t)g.nsp * sh.cw * sh.cw;
  if (sh.cw == 8)
    hicu_launch(conv_bimage_kernel<MODE, 8>, G, kThreads, 0, st, P, g.pos, qt_all, qs, img, ib, img_off);
  else
    hicu_launch(conv_bimage_kernel<MODE, 10>, G, kThreads, 0, st, P, g.pos, qt_all, qs, img, ib, img_off);
  return hicu_check_launch("conv_bimage_kernel");
}

template <int MODE, int CW>
int launch_cw(const DevGeom& g, const Shape& sh, const int (&perm)[3], const uint8_t* bimg, int bimg_early,
              const float* amax_in, float* amax_out, const float2* asrc, const float2* qt, float2* out,
              const float2* uin, const uint8_t* mask, const float2* y, const float2* x0, int dc_mode, float lam,
              double* parts, int nparts_total, cudaStream_t st) {
  using T = Cw<CW>;
  const int L = sh.L;
  CtParams P{};
  fill_shape_params(P, g, sh, perm);
  // accumulator sets: chains of at most ~18 MMAs per TMEM accumulator (the
  // tensor core's fp32 accumulation error grows with the chain length)
  const int mpp = T::KS * (sh.cat ? 2 : 3);  // MMAs per prefix
  const int scols = (sh.cat ? 2 : 1) * sh.ntot;  // TMEM columns of one accumulator set
  P.nacc = std::min(3, std::max(1, (mpp * sh.ng + 17) / 18));
  if (P.nacc * scols > 512) P.nacc = 512 / scols;
  P.tbuf_stride = 2 * P.nacc * scols <= 512 ? 256 : 0;  // double-buffered tiles when two fit
  P.dc_mode = dc_mode;
  P.lam = lam;
  P.nparts_total = nparts_total;
  {
    static int dbg = -1;
    if (dbg < 0) {
      const char* e = getenv("HICU_CONV_TC_DEBUG");
      dbg = e ? atoi(e) : 0;
    }
    P.debug = dbg;
  }
  for (int d = 0; d < L; ++d) {
    P.roff[d] = (int)g.roff[perm[d]];
    P.rext[d] = (int)g.rext[perm[d]];
  }
  // lines run over the region (conv) or k-space (scatter); output strides in
  // rows of u (region-major, geometry axis order) or k-space positions
  const int64_t* lext = MODE < 2 ? g.rext : g.dims;
  int64_t ostr[3] = {1, 1, 1};
  {
    int64_t s = 1;
    for (int a = L - 1; a >= 0; --a) {
      ostr[a] = s;
      s *= lext[a];
    }
  }
  P.ext_last = (int)lext[perm[L - 1]];
  P.chunks = (int)((g.rext[perm[L - 1]] + sh.nb - 1 + kTileM - 1) / kTileM);
  P.lstride = ostr[perm[L - 1]];
  int64_t lines = 1;
  for (int d = 0; d < L - 1; ++d) {
    P.ldim[d] = (int)lext[perm[d]];
    P.ostride[d] = ostr[perm[d]];
    lines *= lext[perm[d]];
  }
  if (lines > (int64_t)1 << 30) return hicu_set_error(HICU_ERR_SIZE, "conv_tc: too many lines");
  P.nlines = (int)lines;
  // A operand: k-space array (conv, extents dims) or u (scatter, extents rext),
  // split into fp16 hi|lo rows (the TMA source) in this stream's scratch
  const int64_t* aext = MODE < 2 ? g.dims : g.rext;
  int64_t arows = 1;
  for (int a = 0; a < L; ++a) arows *= aext[a];
  const int64_t a4n = arows * (T::KA / 4);  // float4 count of the A operand
  const int namax = (int)std::min<int64_t>(2 * hicu_sm_count(), std::max<int64_t>(1, (a4n + 255) / 256));
  const size_t ib = image_bytes(sh);
  const size_t split_off = 4096, img_off = split_off + (((size_t)arows * T::RB + 1023) & ~(size_t)1023);
  uint8_t* scr = stream_scratch(st, img_off + (bimg ? 0 : ib));
  if (!scr) return hicu_set_error(HICU_ERR_CUDA, "conv_tc: scratch allocation failed");
  CUtensorMap tm;
  int s = cached_tmap(&tm, scr + split_off, L, aext, perm, CW, sh.tri ? sh.sd : 0);
  if (s) return s;
  if (!bimg) {
    s = build_image<MODE>(g, sh, perm, qt, 1, scr + img_off, 0, 0, st);
    if (s) return s;
    bimg = scr + img_off;
  }
  bimg_early = 1;  // the amax and split kernels always run between the image and this launch
  const float* amax = reinterpret_cast<const float*>(scr);
  int namax_used = namax;
  if (amax_in) {  // the producer of the A operand wrote its max partials: no amax pass
    amax = amax_in;
    namax_used = kAmaxSlot;
  } else {
    hicu_launch(amax_kernel, namax, 256, 0, st, reinterpret_cast<const float4*>(asrc), a4n,
                reinterpret_cast<float*>(scr));
    if ((s = hicu_check_launch("amax_kernel"))) return s;
  }
  {
    SplitParams sp{};
    sp.L = L;
    for (int a = 0; a < L; ++a) {
      sp.ext[a] = aext[a];
      sp.perm[a] = perm[a];
    }
    int64_t st2 = 1;  // natural row strides of the input
    for (int a = L - 1; a >= 0; --a) {
      sp.istr[a] = st2;
      st2 *= aext[a];
    }
    const int la = perm[L - 1];  // the line axis (natural index)
    int64_t A = 1, B = 1;
    for (int a = 0; a < la; ++a) A *= aext[a];
    for (int a = la + 1; a < L; ++a) B *= aext[a];
    const int64_t Lx = aext[la];
    constexpr int TB = TT<CW>::TB;
    if (B >= TB && A <= 65535 && (Lx + kTT - 1) / kTT <= 65535) {
      hicu_allow_max_smem((const void*)split_t_kernel<CW>);
      const dim3 grid((unsigned)((B + TB - 1) / TB), (unsigned)((Lx + kTT - 1) / kTT), (unsigned)A);
      hicu_launch(split_t_kernel<CW>, grid, 256, (size_t)TT<CW>::SMEM, st, reinterpret_cast<const float4*>(asrc), Lx,
                  B, amax, namax_used, reinterpret_cast<uint4*>(scr + split_off));
      if ((s = hicu_check_launch("split_t_kernel"))) return s;
    } else {
      const int sb = (int)std::min<int64_t>(8 * hicu_sm_count(), std::max<int64_t>(1, (arows + 255) / 256));
      hicu_launch(split_kernel<CW>, sb, 256, 0, st, reinterpret_cast<const float4*>(asrc), arows, sp,
                  amax, namax_used, reinterpret_cast<uint4*>(scr + split_off));
      if ((s = hicu_check_launch("split_kernel"))) return s;
    }
  }
  P.amax = amax;
  P.namax = namax_used;
  P.amax_out = amax_out;
  P.stage_bytes = (int)sh.stage;
  P.k1 = L == 3 ? sh.kpre[1] : sh.ng;
  P.abox = L >= 2 ? T::ASTAGE : T::ATILE;
  P.bimg = bimg;
  P.bimg_early = bimg_early;
  if (sh.tri) return launch_tri<MODE>(sh, P, tm, out, uin, mask, y, x0, parts, nparts_total, st);
  if (sh.bstream)
    return launch_bs<MODE, true, CW>(sh, P, tm, out, uin, mask, y, x0, parts, lines, nparts_total, st);
  return launch_bs<MODE, false, CW>(sh, P, tm, out, uin, mask, y, x0, parts, lines, nparts_total, st);
}

template <int MODE>
int launch(const DevGeom& g, const float2* asrc, const float2* qt, float2* out, const float2* uin, const uint8_t* mask,
           const float2* y, const float2* x0, int dc_mode, float lam, double* parts, int nparts_total,
           cudaStream_t st) {
  // the hints are consumed by this launch whatever happens below (an early
  // error return must not leave them set for an unrelated later call)
  const uint8_t* bimg = t_bimg;
  const int bimg_early = t_bimg_early;
  t_bimg = nullptr;
  const float* amax_in = t_amax_in;
  float* amax_out = t_amax_out;
  t_amax_in = nullptr;
  t_amax_out = nullptr;
  int perm[3];
  choose_perm(g, MODE, perm);
  Shape sh;
  if (!shape_of(g, g.nc, &sh, perm))
    return hicu_set_error(HICU_ERR_SHAPE, "conv_tc: geometry outside the tensor-core scope");
  if (sh.cw == 8)
    return launch_cw<MODE, 8>(g, sh, perm, bimg, bimg_early, amax_in, amax_out, asrc, qt, out, uin, mask, y, x0,
                              dc_mode, lam, parts, nparts_total, st);
  return launch_cw<MODE, 10>(g, sh, perm, bimg, bimg_early, amax_in, amax_out, asrc, qt, out, uin, mask, y, x0,
                             dc_mode, lam, parts, nparts_total, st);
}

}  // namespace

bool hicu_conv_tc_supported(const DevGeom& g, int p) {
  Shape sh;
  int p0[3], p2[3];
  choose_perm(g, 0, p0);
  choose_perm(g, 2, p2);
  return shape_of(g, p, &sh, p0) && shape_of(g, p, &sh, p2);
}

size_t hicu_conv_tc_bimage_bytes(const DevGeom& g, int p) {
  Shape sh, sh2;
  int p0[3], p2[3];
  choose_perm(g, 0, p0);
  choose_perm(g, 2, p2);
  if (!shape_of(g, p, &sh, p0) || !shape_of(g, p, &sh2, p2)) return 0;
  return std::max(image_bytes(sh), image_bytes(sh2));
}

// images for steps j < G: (j, conv/ELS layout) at img + 2j * ib, (j, scatter) at img + (2j+1) * ib
int hicu_conv_tc_build_bimages(const DevGeom& g, const float2* qt_all, int p, int G, uint8_t* img, size_t ib,
                               cudaStream_t st) {
  for (int mode = 0; mode <= 2; mode += 2) {
    // each image in the axis order its convolution launch will choose
    int perm[3];
    choose_perm(g, mode, perm);
    Shape sh;
    if (!shape_of(g, p, &sh, perm)) return hicu_set_error(HICU_ERR_SHAPE, "conv_tc: no B image");
    const int s = mode == 0 ? build_image<0>(g, sh, perm, qt_all, G, img, ib, 0, st)
                            : build_image<2>(g, sh, perm, qt_all, G, img, ib, 1, st);
    if (s) return s;
  }
  return HICU_OK;
}

// the next conv_tc launch on this host thread takes its A-operand scale from
// the max partials `in` (kAmaxSlot floats written by the operand's producer)
// instead of an amax pass, and writes its output's max partials to `out`
void hicu_conv_tc_amax_hint(const float* in, float* out) {
  t_amax_in = in;
  t_amax_out = out;
}

float* hicu_conv_tc_amax_slots(cudaStream_t st) { return stream_amax_slots(st); }

// the next conv_tc launch on this host thread copies its B image from `img`
// (early: the image was written at least two kernels before that launch)
void hicu_conv_tc_bimage_hint(const void* img, int early) {
  t_bimg = (const uint8_t*)img;
  t_bimg_early = early;
}

int hicu_conv_tc(const DevGeom& g, const float2* y, const float2* qt, float2* u, double* parts, int mode,
                 int nparts_total, cudaStream_t st) {
  if (mode == 0)
    return launch<0>(g, y, qt, u, nullptr, nullptr, nullptr, nullptr, 2, 0.f, parts, nparts_total, st);
  return launch<1>(g, y, qt, nullptr, u, nullptr, nullptr, nullptr, 2, 0.f, parts, nparts_total, st);
}

int hicu_scatter_tc(const DevGeom& g, const float2* qt, const float2* u, const uint8_t* mask, const float2* y,
                    const float2* x0, int dc_mode, float lam, float2* gout, double* parts, int nparts_total,
                    cudaStream_t st) {
  return launch<2>(g, u, qt, gout, nullptr, mask, y, x0, dc_mode, lam, parts, nparts_total, st);
}
