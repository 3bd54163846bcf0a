// Hankel convolution u = H(y) Q~ and its transpose (the k-space scatter
// g = H^H(u) Q~^H) on the 5th-generation tensor cores: tcgen05 kind::tf32 with
// a 3xTF32 split (FP32-grade accuracy), TMA-staged operands, TMEM accumulators.
//
// Reference: hankel.py:255-322 (hankel_apply), hankel.py:394-440
// (kspace_adjoint_scatter), solver.py:335-351 (objective / ELS terms, DC).
//
// Formulation (coil-separable support, Nc = 8 coils, p = 8 JL columns).  A
// spatial tap of the k-space array is one 64-byte row of 16 floats (8 complex
// coils), and a row of u is also 16 floats (8 complex columns), so both
// operands are natively K-major with 64-byte rows -- exactly the SWIZZLE_64B
// canonical layout a TMA box of [8 rows x 16 floats] produces.
//   conv:    D[m, :] = sum_taps A_tap[m, :] B_tap^T,  A_tap = y rows (m + tap),
//            B_tap = real embedding of Q~[tap, :, :] (16 x 16)
//   scatter: D[m, :] = sum_taps A_tap[m, :] B_tap^T,  A_tap = u rows (m - tap),
//            B_tap = real embedding of conj(Q~[tap, :, :])^T
// with M = 128 consecutive positions along the last spatial axis (one tile),
// N = 16, K = 16 per tap (two K=8 MMA steps).
//
// Hankel reuse: taps that share their prefix (all spatial axes but the last)
// read the same k-space line, shifted by b rows.  One TMA load of
// 128 + spread rows serves every tap b of that group; the MMA descriptor start
// address is shifted by b * 64 bytes (the swizzle is on absolute address bits,
// scripts/tc_unit2.cu).  Each k-space element is fetched once per prefix tap
// (5x for a 5x5 kernel) instead of once per tap (25x).
//
// 3xTF32: x = hi + lo; D += A_hi B_hi + A_hi B_lo + A_lo B_hi.  The B images
// (all taps, hi and lo) are built once per CTA in shared memory; A boxes are
// split in place by converter warps after TMA lands them.
//
// Epilogues are fused: conv writes u and the objective partial sum |u|^2;
// the ELS variant never stores w = H(g)Q~ and accumulates Re<w,u>, |w|^2; the
// scatter applies hard / soft data consistency and accumulates the four DC
// partial sums (same meaning as ops.cu:scatter_coil_kernel).  Partial sums are
// per CTA in fixed order (deterministic).
//
// Warp roles (320 threads, one persistent CTA per SM): warp 0 TMA producer,
// warp 1 TMEM owner + MMA issuer, warps 2-5 hi/lo converters, warps 6-9
// epilogue (TMEM lane quarter = warp % 4).  Two accumulator sets alternate so
// the epilogue of tile t overlaps the MMAs of tile t + 1.
//
// Accumulation accuracy: the tensor core's fp32 accumulator loses about half
// an ulp per chained MMA (measured: 3.2e-6 relative with all 150 MMAs of a
// 5x5 tile in one accumulator).  Taps are therefore dealt round-robin to
// kAcc = 8 accumulators (16 TMEM columns each) that the epilogue sums.
#include <cuda.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace {

constexpr int kTileM = 128;
constexpr int kMaxTaps = 48;
constexpr int kMaxGroups = 48;
constexpr int kMaxSpread = 32;                       // last-axis tap spread per group
constexpr int kBoxRows = 8;                          // one SW64 atom per TMA box
constexpr int kStageRows = kTileM + kMaxSpread;      // 160
constexpr int kHalfBytes = kStageRows * 64;          // 10240 (hi or lo)
constexpr int kStageBytes = 2 * kHalfBytes;          // 20480
constexpr int kMaxStages = 8;
constexpr int kThreads = 320;
constexpr int kTapBytes = 2048;                      // B image per tap (hi 1 KB + lo 1 KB)
constexpr int kAcc = 4;                              // TMEM accumulator sets per tile (taps round-robin)

struct CtParams {
  int L;                  // spatial axes (1..3)
  int nsp;                // spatial taps
  int ndim;               // geometry rank (pos stride per support entry)
  int stages;
  int dc_mode;
  float lam;
  int nparts_total;       // entries of `parts` (per value) the ABI promised
  int chunks;             // tiles per line
  int ntiles;
  int ldim[2];            // line extents of the prefix axes (conv: rext, scatter: dims)
  int ext_last;           // valid columns along the last axis (conv: rext, scatter: dims)
  int roff[3];
  int rext[3];
  int64_t ostride[2];     // output strides (rows / positions) of the prefix axes
  int debug;              // experiment bits (HICU_CONV_TC_DEBUG): 1 no MMA, 2 no TMA, 4 no convert, 8 no B build
};

struct GroupTable {
  int n;
  int a[kMaxGroups][2];
  int first[kMaxGroups], cnt[kMaxGroups], minb[kMaxGroups], maxb[kMaxGroups];
  short tap_sp[kMaxTaps], tap_b[kMaxTaps];
};

__device__ __forceinline__ void decode_tile(const CtParams& P, int tile, int (&lc)[2], int& chunk) {
  chunk = tile % P.chunks;
  int line = tile / P.chunks;
  lc[0] = lc[1] = 0;
  if (P.L == 3) {
    lc[1] = line % P.ldim[1];
    lc[0] = line / P.ldim[1];
  } else if (P.L == 2) {
    lc[0] = line;
  }
}

template <int MODE>
__device__ __forceinline__ bool group_valid(const CtParams& P, const GroupTable& G, int gi, const int (&lc)[2]) {
  if (MODE < 2) return true;
  bool ok = true;
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    if (d < P.L - 1) {
      const int r = lc[d] - P.roff[d] - G.a[gi][d];
      ok = ok && r >= 0 && r < P.rext[d];
    }
  }
  return ok;
}

template <int MODE>
__device__ __forceinline__ int active_taps(const CtParams& P, const GroupTable& G, const int (&lc)[2]) {
  if (MODE < 2) return P.nsp;
  int n = 0;
  for (int gi = 0; gi < G.n; ++gi)
    if (group_valid<MODE>(P, G, gi, lc)) n += G.cnt[gi];
  return n;
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// MODE 0: conv forward (u, obj); 1: conv ELS (Re<w,u>, |w|^2); 2: scatter + DC.
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
conv_tc_kernel(const __grid_constant__ CUtensorMap tmap64, const __grid_constant__ CUtensorMap tmap8, const CtParams P, const int32_t* __restrict__ pos,
               const float2* __restrict__ qt, float2* __restrict__ out, const float2* __restrict__ uin,
               const uint8_t* __restrict__ mask, const float2* __restrict__ y, const float2* __restrict__ x0,
               double* __restrict__ parts) {
  constexpr int NV = MODE == 0 ? 1 : (MODE == 1 ? 2 : 4);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sB = smem;
  uint8_t* sStage = smem + (size_t)P.nsp * kTapBytes;
  __shared__ __align__(8) uint64_t full[kMaxStages], ready[kMaxStages], empty[kMaxStages], tfull[2], tempty[2];
  __shared__ uint32_t tslot;
  __shared__ GroupTable G;
  __shared__ double red[4][NV];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = P.L, S = P.stages;
  __shared__ uint64_t trace[12];
  const bool tr = (P.debug & 16) != 0;
  if (P.debug & 512) return;
  if (tr && threadIdx.x == 0) trace[0] = gtimer();

  __shared__ int spos[kMaxTaps][3];
  __shared__ int sstart[kMaxTaps];
  // Issue every global load of the prologue up front: support positions and
  // this thread's Q~ entries (one complex value -> a 2x2 block of the real
  // embedding, hi and lo).
  constexpr int kQPer = (kMaxTaps * 64 + kThreads - 1) / kThreads;
  float2 qv[kQPer];
  const int nq = (P.debug & 8) ? 0 : P.nsp * 64;
#pragma unroll
  for (int u = 0; u < kQPer; ++u) {
    const int e = threadIdx.x + u * kThreads;
    qv[u] = e < nq ? __ldg(qt + e) : make_float2(0.f, 0.f);
  }
  for (int t = threadIdx.x; t < ((P.debug & 1024) ? 0 : P.nsp * L); t += kThreads)
    spos[t / L][t % L] = __ldg(pos + (size_t)(t / L) * 8 * P.ndim + t % L);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&ready[s], 128);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 128);
    }
    tc::mbar_init_fence();
  }
  if (warp == 1 && !(P.debug & 256)) tc::tmem_alloc(&tslot, 512);
  __syncthreads();
  // Tap groups (parallel): a group is a maximal run of consecutive taps with
  // the same prefix and the same last-axis window b / (kMaxSpread + 1), so its
  // spread is <= kMaxSpread.  Support positions come sorted (C order), which
  // makes every prefix one group per window.
  if (threadIdx.x < P.nsp) {
    const int sp = threadIdx.x;
    const int b = spos[sp][L - 1];
    bool st = sp == 0;
    if (!st) {
      st = b / (kMaxSpread + 1) != spos[sp - 1][L - 1] / (kMaxSpread + 1);
      if (L >= 2) st = st || spos[sp][0] != spos[sp - 1][0];
      if (L >= 3) st = st || spos[sp][1] != spos[sp - 1][1];
    }
    sstart[sp] = st ? 1 : 0;
    G.tap_sp[sp] = (short)sp;
    G.tap_b[sp] = (short)b;
  }
  __syncthreads();
  if (!(P.debug & 128) && threadIdx.x < P.nsp && sstart[threadIdx.x]) {
    const int sp = threadIdx.x;
    int gi = 0;
    for (int j = 1; j <= sp; ++j) gi += sstart[j];
    int e = sp + 1;
    int lo = spos[sp][L - 1], hi = lo;
    while (e < P.nsp && !sstart[e]) {
      lo = min(lo, spos[e][L - 1]);
      hi = max(hi, spos[e][L - 1]);
      ++e;
    }
    G.a[gi][0] = L >= 2 ? spos[sp][0] : 0;
    G.a[gi][1] = L >= 3 ? spos[sp][1] : 0;
    G.first[gi] = sp;
    G.cnt[gi] = e - sp;
    G.minb[gi] = lo;
    G.maxb[gi] = hi;
    if (e == P.nsp) G.n = gi + 1;
  }
  if (P.debug & 32) {  // experiment: dump the tap-group table into `out` and stop
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
      int* o = reinterpret_cast<int*>(out);
      o[0] = G.n;
      for (int gi = 0; gi < min(G.n, kMaxGroups); ++gi) {
        o[1 + 6 * gi] = G.first[gi];
        o[2 + 6 * gi] = G.cnt[gi];
        o[3 + 6 * gi] = G.minb[gi];
        o[4 + 6 * gi] = G.maxb[gi];
        o[5 + 6 * gi] = G.a[gi][0];
        o[6 + 6 * gi] = G.a[gi][1];
      }
    }
    __syncthreads();
    if (warp == 1 && !(P.debug & 256)) tc::tmem_dealloc(tslot, 512);
    return;
  }
  // B images of every tap: rows 0-15 hi, rows 16-31 lo (one N = 32 operand),
  // rows of 64 B, SW64 swizzle on absolute address bits.
#pragma unroll
  for (int u = 0; u < kQPer; ++u) {
    const int e = threadIdx.x + u * kThreads;
    if (e >= nq) break;
    const int sp = e >> 6, c = (e >> 3) & 7, j = e & 7;
    const float2 q = qv[u];
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
        const float hi = tc::tf32_rna(v), lo = tc::tf32_rna(v - hi);
        const uint32_t off = (uint32_t)sp * kTapBytes + n * 64 + ((((k >> 2) ^ ((n >> 1) & 3))) << 4) + (k & 3) * 4;
        *reinterpret_cast<float*>(sB + off) = hi;
        *reinterpret_cast<float*>(sB + off + 1024) = lo;
      }
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  if (tr && threadIdx.x == 0) trace[1] = gtimer();

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
        int lc[2], chunk;
        decode_tile(P, tile, lc, chunk);
        for (int gi = 0; gi < G.n; ++gi) {
          if (!group_valid<MODE>(P, G, gi, lc)) continue;
          const int nbox = (kTileM + G.maxb[gi] - G.minb[gi] + kBoxRows - 1) / kBoxRows;
          tc::mbar_wait(&empty[s], ph ^ 1);
          if (P.debug & 2) {
            tc::mbar_arrive(&full[s]);
            if (++s == S) { s = 0; ph ^= 1; }
            continue;
          }
          tc::mbar_expect_tx(&full[s], (uint32_t)nbox * kBoxRows * 64);
          int c[4] = {0, 0, 0, 0};
          // tensor coordinate 1 = last spatial axis, 2 = axis L-2, 3 = axis L-3
          if (MODE < 2) {
            c[1] = P.roff[L - 1] + chunk * kTileM + G.minb[gi];
            if (L == 2) c[2] = P.roff[0] + lc[0] + G.a[gi][0];
            if (L == 3) {
              c[2] = P.roff[1] + lc[1] + G.a[gi][1];
              c[3] = P.roff[0] + lc[0] + G.a[gi][0];
            }
          } else {
            c[1] = chunk * kTileM - P.roff[L - 1] - G.maxb[gi];
            if (L == 2) c[2] = lc[0] - P.roff[0] - G.a[gi][0];
            if (L == 3) {
              c[2] = lc[1] - P.roff[1] - G.a[gi][1];
              c[3] = lc[0] - P.roff[0] - G.a[gi][0];
            }
          }
          uint8_t* dst = sStage + (size_t)s * kStageBytes;
          if (tr && tile == (int)blockIdx.x && gi == 0) trace[2] = gtimer();
          // 64-row boxes, then 8-row boxes for the remainder (TMA cost is per instruction)
          int r0 = 0;
          for (; r0 + 64 <= nbox * kBoxRows; r0 += 64)
            tc::tma_load_4d(dst + r0 * 64, &tmap64, 0, c[1] + r0, c[2], c[3], &full[s]);
          for (; r0 < nbox * kBoxRows; r0 += kBoxRows)
            tc::tma_load_4d(dst + r0 * 64, &tmap8, 0, c[1] + r0, c[2], c[3], &full[s]);
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc32 = tc::idesc_tf32(kTileM, 32), idesc16 = tc::idesc_tf32(kTileM, 16);
      const uint32_t bbase = tc::smem_u32(sB);
      int s = 0, tb = 0;
      uint32_t ph = 0, tph = 0;
      for (int tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
        int lc[2], chunk;
        decode_tile(P, tile, lc, chunk);
        if (active_taps<MODE>(P, G, lc) == 0) continue;
        tc::mbar_wait(&tempty[tb], tph ^ 1);
        tc::fence_after();
        const uint32_t dcol = tmem + (uint32_t)tb * 256;
        int ti = 0;  // active tap index within the tile -> accumulator set ti % kAcc
        for (int gi = 0; gi < G.n; ++gi) {
          if (!group_valid<MODE>(P, G, gi, lc)) continue;
          tc::mbar_wait(&ready[s], ph);
          tc::fence_after();
          if (tr && tile == (int)blockIdx.x && gi == 0) trace[4] = gtimer();
          const uint32_t ahi = tc::smem_u32(sStage + (size_t)s * kStageBytes), alo = ahi + kHalfBytes;
          for (int t = G.first[gi]; t < G.first[gi] + G.cnt[gi]; ++t, ++ti) {
            const int b = G.tap_b[t];
            const uint32_t rows = (uint32_t)(MODE < 2 ? b - G.minb[gi] : G.maxb[gi] - b);
            const uint32_t bcat = bbase + (uint32_t)G.tap_sp[t] * kTapBytes;  // [B_hi; B_lo], N = 32
            const uint32_t d = dcol + (uint32_t)(ti % kAcc) * 48;               // cols 0-31: A_hi [B_hi;B_lo], 32-47: A_lo B_hi
            uint32_t acc = ti >= kAcc ? 1u : 0u;
            if (P.debug & 1) continue;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint32_t ao = rows * 64 + ks * 32;
              tc::mma_tf32(d, tc::desc_sw64(ahi + ao), tc::desc_sw64(bcat + ks * 32), idesc32, acc);
              tc::mma_tf32(d + 32, tc::desc_sw64(alo + ao), tc::desc_sw64(bcat + ks * 32), idesc16, acc);
              acc = 1;
            }
          }
          tc::mma_commit(&empty[s]);
          if (++s == S) { s = 0; ph ^= 1; }
        }
        tc::mma_commit(&tfull[tb]);
        if (tr && tile == (int)blockIdx.x) trace[5] = gtimer();
        tb ^= 1;
        if (tb == 0) tph ^= 1;
      }
    }
    __syncwarp();
  } else if (warp < 6) {
    // ---------------- hi/lo converters ----------------
    const int ct = threadIdx.x - 64;
    int s = 0;
    uint32_t ph = 0;
    for (int tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
      int lc[2], chunk;
      decode_tile(P, tile, lc, chunk);
      for (int gi = 0; gi < G.n; ++gi) {
        if (!group_valid<MODE>(P, G, gi, lc)) continue;
        const int nbox = (kTileM + G.maxb[gi] - G.minb[gi] + kBoxRows - 1) / kBoxRows;
        tc::mbar_wait(&full[s], ph);
        if (tr && ct == 0 && tile == (int)blockIdx.x && gi == 0) trace[3] = gtimer();
        float4* hi4 = reinterpret_cast<float4*>(sStage + (size_t)s * kStageBytes);
        float4* lo4 = reinterpret_cast<float4*>(sStage + (size_t)s * kStageBytes + kHalfBytes);
        for (int i = ct; i < ((P.debug & 4) ? 0 : nbox * kBoxRows * 4); i += 128) {
          const float4 v = hi4[i];
          float4 h, l;
          h.x = tc::tf32_rna(v.x); l.x = tc::tf32_rna(v.x - h.x);
          h.y = tc::tf32_rna(v.y); l.y = tc::tf32_rna(v.y - h.y);
          h.z = tc::tf32_rna(v.z); l.z = tc::tf32_rna(v.z - h.z);
          h.w = tc::tf32_rna(v.w); l.w = tc::tf32_rna(v.w - h.w);
          hi4[i] = h;
          lo4[i] = l;
        }
        tc::fence_proxy_async();
        tc::mbar_arrive(&ready[s]);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue ----------------
    const int q = warp & 3;
    const int m = 32 * q + lane;
    double acc_v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc_v[i] = 0.0;
    int tb = 0;
    uint32_t tph = 0;
    for (int tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
      int lc[2], chunk;
      decode_tile(P, tile, lc, chunk);
      float v[16];
      const int nact = active_taps<MODE>(P, G, lc);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = 0.f;
      if (nact > 0) {
        tc::mbar_wait(&tfull[tb], tph);
        tc::fence_after();
        if (tr && threadIdx.x == 192 && tile == (int)blockIdx.x) trace[6] = gtimer();
        const uint32_t t0 = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)tb * 256;
        for (int k = 0; k < min(nact, kAcc); ++k) {
#pragma unroll
          for (int h = 0; h < 3; ++h) {
            float w[16];
            tc::tmem_ld16(t0 + (uint32_t)(k * 48 + h * 16), w);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += w[i];
          }
        }
        tc::fence_before();
        tc::mbar_arrive(&tempty[tb]);
        tb ^= 1;
        if (tb == 0) tph ^= 1;
      }
      const int col = chunk * kTileM + m;
      if (col >= P.ext_last) continue;
      int64_t idx = col;
      if (L >= 2) idx += (int64_t)lc[0] * P.ostride[0];
      if (L >= 3) idx += (int64_t)lc[1] * P.ostride[1];
      if (MODE == 0) {
        float4* up = reinterpret_cast<float4*>(out + (size_t)idx * 8);
#pragma unroll
        for (int i = 0; i < 4; ++i) up[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc_v[0] += (double)v[i] * v[i];
      } else if (MODE == 1) {
        const float4* up = reinterpret_cast<const float4*>(uin + (size_t)idx * 8);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 uu = up[i];
          acc_v[0] += (double)v[4 * i] * uu.x + (double)v[4 * i + 1] * uu.y + (double)v[4 * i + 2] * uu.z +
                      (double)v[4 * i + 3] * uu.w;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) acc_v[NV - 1] += (double)v[i] * v[i];
      } else {
        const size_t e0 = (size_t)idx * 8;
        uint8_t mk[8];
        if (P.dc_mode != 2) {
          const uint2 mm = *reinterpret_cast<const uint2*>(mask + e0);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            mk[c] = (uint8_t)(mm.x >> (8 * c));
            mk[4 + c] = (uint8_t)(mm.y >> (8 * c));
          }
        }
        float4* gp = reinterpret_cast<float4*>(out + e0);
#pragma unroll
        for (int c2 = 0; c2 < 4; ++c2) {
          float a[4] = {v[4 * c2], v[4 * c2 + 1], v[4 * c2 + 2], v[4 * c2 + 3]};
          float4 yy = make_float4(0.f, 0.f, 0.f, 0.f), xx = yy;
          if (P.dc_mode == 1) {
            yy = reinterpret_cast<const float4*>(y + e0)[c2];
            xx = reinterpret_cast<const float4*>(x0 + e0)[c2];
          }
          const float yv[4] = {yy.x, yy.y, yy.z, yy.w}, xv[4] = {xx.x, xx.y, xx.z, xx.w};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const bool on = P.dc_mode != 2 && mk[2 * c2 + h] == 1;
            float ar = a[2 * h], ai = a[2 * h + 1];
            if (P.dc_mode == 0) {
              if (on) ar = ai = 0.f;
            } else if (P.dc_mode == 1) {
              const float rr = on ? yv[2 * h] - xv[2 * h] : 0.f, ri = on ? yv[2 * h + 1] - xv[2 * h + 1] : 0.f;
              acc_v[1] += (double)rr * rr + (double)ri * ri;
              ar = ar + P.lam * rr;
              ai = ai + P.lam * ri;
              if (on) {
                acc_v[2] += (double)ar * rr + (double)ai * ri;
                acc_v[3] += (double)ar * ar + (double)ai * ai;
              }
            }
            acc_v[0] += (double)ar * ar + (double)ai * ai;
            a[2 * h] = ar;
            a[2 * h + 1] = ai;
          }
          gp[c2] = make_float4(a[0], a[1], a[2], a[3]);
        }
      }
    }
    if (tr && threadIdx.x == 192) trace[7] = gtimer();
    // fixed-order reduction over the 128 epilogue threads
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double t = warp_sum_d(acc_v[i]);
      if (lane == 0) red[q][i] = t;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (warp == 6 && lane < NV) {
      const double t = red[0][lane] + red[1][lane] + red[2][lane] + red[3][lane];
      parts[(size_t)blockIdx.x * NV + lane] = t;
    }
    if (blockIdx.x == 0)
      for (int i = threadIdx.x - 192 + (int)gridDim.x * NV; i < P.nparts_total * NV; i += 128) parts[i] = 0.0;
  }
  if (tr && threadIdx.x == 192) trace[8] = gtimer();
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
  if (tr && threadIdx.x == 0 && MODE == 0) {
    trace[9] = gtimer();
    uint64_t* o = reinterpret_cast<uint64_t*>(out) + (size_t)blockIdx.x * 12;
    for (int i = 0; i < 10; ++i) o[i] = trace[i];
  }
}

// The driver entry point is resolved at run time through cudart so the
// library loads (and its exports can be checked) on hosts without a driver.
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

int make_tmap(CUtensorMap* tm, const void* base, int L, const int64_t* ext, int box_rows) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return hicu_set_error(HICU_ERR_CUDA, "conv_tc: cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {16, (cuuint64_t)ext[L - 1], (cuuint64_t)(L >= 2 ? ext[L - 2] : 1),
                        (cuuint64_t)(L >= 3 ? ext[L - 3] : 1)};
  cuuint64_t strides[3] = {64, 64 * dims[1], 64 * dims[1] * dims[2]};
  cuuint32_t box[4] = {16, (cuuint32_t)box_rows, 1, 1}, es[4] = {1, 1, 1, 1};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return hicu_set_error(HICU_ERR_CUDA, "conv_tc: cuTensorMapEncodeTiled failed");
  return HICU_OK;
}

// Tensor maps depend only on (pointer, extents): a small per-thread cache
// keeps cuTensorMapEncodeTiled off the per-launch path of the stage driver.
int cached_tmap(CUtensorMap* tm, const void* base, int L, const int64_t* ext, int box_rows) {
  struct Entry {
    const void* base;
    int L, box_rows;
    int64_t ext[3];
    CUtensorMap map;
  };
  static thread_local Entry cache[16];
  static thread_local int used = 0, next = 0;
  for (int i = 0; i < used; ++i) {
    const Entry& e = cache[i];
    if (e.base == base && e.L == L && e.box_rows == box_rows && e.ext[0] == ext[0] && (L < 2 || e.ext[1] == ext[1]) &&
        (L < 3 || e.ext[2] == ext[2])) {
      *tm = e.map;
      return HICU_OK;
    }
  }
  const int st = make_tmap(tm, base, L, ext, box_rows);
  if (st) return st;
  Entry& e = cache[next];
  e.base = base;
  e.L = L;
  e.box_rows = box_rows;
  for (int d = 0; d < 3; ++d) e.ext[d] = d < L ? ext[d] : 0;
  e.map = *tm;
  next = (next + 1) % 16;
  if (used < 16) ++used;
  return HICU_OK;
}

template <int MODE>
int launch(const DevGeom& g, const void* tsrc, const float2* qt, float2* out, const float2* uin, const uint8_t* mask,
           const float2* y, const float2* x0, int dc_mode, float lam, double* parts, int nparts_total,
           cudaStream_t st) {
  const int L = g.ndim - 1;
  CtParams P{};
  P.L = L;
  P.nsp = g.nsp;
  P.ndim = g.ndim;
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
    P.roff[d] = (int)g.roff[d];
    P.rext[d] = (int)g.rext[d];
  }
  const int64_t* lext = MODE < 2 ? g.rext : g.dims;  // tile lines run over the region (conv) or k-space (scatter)
  P.ext_last = (int)lext[L - 1];
  P.chunks = (P.ext_last + kTileM - 1) / kTileM;
  int64_t lines = 1;
  for (int d = 0; d < L - 1; ++d) {
    P.ldim[d] = (int)lext[d];
    lines *= lext[d];
  }
  int64_t str = P.ext_last;
  for (int d = L - 2; d >= 0; --d) {
    P.ostride[d] = str;
    str *= lext[d];
  }
  if (lines * P.chunks > (int64_t)1 << 30) return hicu_set_error(HICU_ERR_SIZE, "conv_tc: too many tiles");
  P.ntiles = (int)(lines * P.chunks);
  // TMA source: k-space array (conv, extents dims) or u (scatter, extents rext).
  CUtensorMap tm64, tm8;
  int s = cached_tmap(&tm64, tsrc, L, MODE < 2 ? g.dims : g.rext, 64);
  if (!s) s = cached_tmap(&tm8, tsrc, L, MODE < 2 ? g.dims : g.rext, kBoxRows);
  if (s) return s;
  // Shared-memory budget per kernel instantiation (queried once).
  static size_t avail = 0;
  if (!avail) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)conv_tc_kernel<MODE>);
    int optin = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    avail = (size_t)optin - fa.sharedSizeBytes;
    hicu_allow_max_smem((const void*)conv_tc_kernel<MODE>);
  }
  const size_t fixed = (size_t)g.nsp * kTapBytes + 1024;
  if (avail < fixed + 2 * kStageBytes) return hicu_set_error(HICU_ERR_SIZE, "conv_tc: shared memory");
  P.stages = (int)((avail - fixed) / kStageBytes);
  if (P.stages > kMaxStages) P.stages = kMaxStages;
  const size_t smem = fixed + (size_t)P.stages * kStageBytes;
  int64_t grid = P.ntiles;
  if (grid > hicu_sm_count()) grid = hicu_sm_count();
  if (grid > nparts_total) grid = nparts_total;
  if (grid < 1) grid = 1;
  conv_tc_kernel<MODE><<<(int)grid, kThreads, smem, st>>>(tm64, tm8, P, g.pos, qt, out, uin, mask, y, x0, parts);
  return hicu_check_launch("conv_tc_kernel");
}

}  // namespace

bool hicu_conv_tc_supported(const DevGeom& g, int p) {
  const int L = g.ndim - 1;
  return g.nc == 8 && p == 8 && g.ncirc == 0 && L >= 1 && L <= 3 && g.nsp >= 1 && g.nsp <= kMaxTaps;
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
