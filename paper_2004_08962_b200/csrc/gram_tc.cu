// Gram matrix G = H(x)^H H(x) on the 5th-generation tensor cores (tcgen05,
// kind::tf32, 3xTF32 split for FP32-grade accuracy), implicit im2col.
//
// Real embedding: H_real (s x 2n) holds, for region row i and kernel column
// kappa = tap*Nc + c, the floats (re, im) of X[i + pos(kappa)].  For a
// coil-separable support the 2*Nc = 16 floats of one spatial tap are
// contiguous in k-space, so G_real = H_real^T H_real is a GEMM over rows i
// (K) whose M/N operands are tap columns:
//   D[mu, nu] += sum_i A[mu, i] B[nu, i],  A = H_real[:, M tile]^T, B = H_real[:, N tile]^T
// G[k1,k2] = (G_rr + G_ii) + i (G_ri - G_ir) is assembled in fp64 by the
// split-K reduction kernel (only tile pairs holding k1 <= k2 are computed).
//
// 3xTF32: x = hi + lo, hi = rna_tf32(x); D += A_hi B_hi + A_hi B_lo + A_lo B_hi.
//
// Accumulation accuracy: tcgen05 fp32 accumulation loses precision in
// proportion to the number of MMAs chained into one accumulator (measured on
// C2: 1.5e-5 relative after ~650 chained MMAs, 1.5e-6 after ~50).  Each CTA
// therefore alternates two TMEM accumulators (256 columns each) in chains of
// kChain k-blocks; 16 epilogue warps drain a finished chain with tcgen05.ld
// and add it into fp32 registers (round-to-nearest) while the tensor core
// fills the other buffer.
//
// Operands are staged K-major (canonical no-swizzle core matrices, LBO 128 B,
// SBO 256 B): MN-major tf32 operands returned all-zero results on this part
// in a unit test (scripts/tc_unit.cu).  Producer warps gather the 16 floats x
// 16 rows of every tap of the tile, split hi/lo on the fly and write 16-byte
// K-major chunks.
//
// Warp roles (800 threads): warps 0-7 producers, warp 8 TMEM owner + MMA
// issuer (one lane), warps 9-24 epilogue (TMEM lane quarter = warp % 4,
// 64-column group = (warp - 9) / 4).
//
// Scope: coil-separable support with Nc = 8 (16 floats per tap), no circular
// axes, <= 3 spatial axes, 8..128 spatial taps.  Other geometries use the SIMT
// kernel (gram_simt.cu).
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace {

constexpr int kBK = 16;           // rows (K) per pipeline stage: 2 MMA k-steps of 8
constexpr int kMT = 8;            // taps per M tile  (M = 128 real columns)
constexpr int kNT = 16;           // taps per N tile  (N <= 256 real columns)
#ifndef HICU_GRAM_CHAIN
#define HICU_GRAM_CHAIN 8  // 4: 1.15e-6 -> 6.4e-7 vs fp64 at C2, 2.4e-6 -> 2.2e-6 at the C5 shard, 6 % slower there
#endif
constexpr int kChain = HICU_GRAM_CHAIN;  // k-blocks per TMEM accumulation chain
#ifndef HICU_GRAM_PROD_WARPS
#define HICU_GRAM_PROD_WARPS 8  // 6: 26.0 ms, 4: 41.0 ms, 12: 23.7 ms at the C5 shard (8: 23.6 ms)
#endif
constexpr int kProdWarps = HICU_GRAM_PROD_WARPS;
constexpr int kProducers = kProdWarps * 32;
constexpr int kEpiWarps = 16;
constexpr int kThreads = (kProdWarps + 1 + kEpiWarps) * 32;
constexpr int kMaxStages = 6;
constexpr int kPartCols = 256;
constexpr int kMaxPairs = 160;

struct TcParams {
  int T;                 // spatial taps
  int nsp;               // spatial axes (1..3)
  int64_t rext[3];       // region extents per spatial axis (last = K-contiguous)
  int64_t roff[3];
  int64_t fstride[3];    // float strides of the spatial axes in the k-space array
  int64_t nkb_line;      // k-blocks per region line
  int64_t nkb;           // total k-blocks
  int64_t kb_per_split;
  int npairs;
  int stages;
  unsigned char pair_m[kMaxPairs], pair_n[kMaxPairs];  // tile pair -> (m tile, n tile)
};

struct PairTable {
  short v[16 * 8];  // [m tile][n tile] -> pair index or -1
};

__host__ __device__ __forceinline__ int64_t hmin64(int64_t a, int64_t b) { return a < b ? a : b; }

__host__ __device__ __forceinline__ int mtile_first_tap(int m, int T) {
  const int f = m * kMT;
  return (f + kMT > T) ? T - kMT : f;  // last tile shifted back so it stays full
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major no-swizzle descriptor: core matrix = 8 MN rows x 16 B, LBO = next 4 K, SBO = next 8 MN rows.
__device__ __forceinline__ uint64_t make_desc_kmajor(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm100)
  return d;                // layout type 0: no swizzle
}

// Instruction descriptor: kind::tf32, fp32 accumulate, A and B K-major.
__device__ __forceinline__ uint32_t make_idesc_tf32(int M, int N) {
  uint32_t d = 0;
  d |= 1u << 4;   // D format F32
  d |= 2u << 7;   // A format TF32
  d |= 2u << 10;  // B format TF32
  d |= (uint32_t)(N >> 3) << 17;
  d |= (uint32_t)(M >> 4) << 24;
  return d;
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16_raw(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

#ifndef HICU_GRAM_PREFETCH
#define HICU_GRAM_PREFETCH 0  // 1: next stage's gathers issued before this stage's stores (spills at 72 regs)
#endif
constexpr int kTasks = (kNT + kMT) * 64 / kProducers;  // gather tasks per producer thread and stage

// Region-line walker for the producer: the k-block -> (line, chunk) ->
// float offset decomposition is done once per CTA with divisions and then
// advanced incrementally (64-bit division per k-block cost ~100 producer
// instructions of ~430 per k-block in an ncu source profile).
struct GramCursor {
  int64_t base;     // float offset of the chunk's first row
  int valid;        // rows of the chunk inside the region line
  int chunk;        // chunk index within the line
  int64_t c[3];     // line coordinates (axes 0..L-1)
};

__device__ __forceinline__ void cursor_valid(const TcParams& p, GramCursor& cu) {
  const int L = p.nsp - 1;
  cu.valid = (int)hmin64(kBK, p.rext[L] - (int64_t)cu.chunk * kBK);
}

__device__ __forceinline__ void cursor_init(const TcParams& p, int64_t kb, GramCursor& cu) {
  const int L = p.nsp - 1;
  int64_t line = kb / p.nkb_line;
  cu.chunk = (int)(kb % p.nkb_line);
  cu.base = (p.roff[L] + (int64_t)cu.chunk * kBK) * 16;
  for (int d = L - 1; d >= 0; --d) {
    cu.c[d] = line % p.rext[d];
    line /= p.rext[d];
    cu.base += (p.roff[d] + cu.c[d]) * p.fstride[d];
  }
  cursor_valid(p, cu);
}

__device__ __forceinline__ void cursor_next(const TcParams& p, GramCursor& cu) {
  const int L = p.nsp - 1;
  if (++cu.chunk < p.nkb_line) {
    cu.base += kBK * 16;
  } else {
    cu.base -= (int64_t)(cu.chunk - 1) * kBK * 16;  // back to the line start
    cu.chunk = 0;
    for (int d = L - 1; d >= 0; --d) {  // odometer over the line coordinates
      if (++cu.c[d] < p.rext[d]) {
        cu.base += p.fstride[d];
        break;
      }
      cu.base -= (p.rext[d] - 1) * p.fstride[d];
      cu.c[d] = 0;
    }
  }
  cursor_valid(p, cu);
}

// Loads of one k-block for this producer thread: task it covers float
// j = t % 16 of tap q = t / 64 for the 4 rows of quad (t / 16) % 4
// (t = tid + it * kProducers); toff[it] = tap offset + j + 64 quad, or -1.
__device__ __forceinline__ void gram_gather(const float* __restrict__ x, const GramCursor& cu,
                                            const int (&toff)[kTasks], float (&v)[kTasks][4]) {
  const float* xb = x + cu.base;
#pragma unroll
  for (int it = 0; it < kTasks; ++it) {
    const int quad = ((threadIdx.x + it * kProducers) >> 4) & 3;
#pragma unroll
    for (int r = 0; r < 4; ++r)
      v[it][r] = (toff[it] >= 0 && quad * 4 + r < cu.valid) ? __ldg(xb + toff[it] + r * 16) : 0.f;
  }
}

// Stage layout (per hi/lo half): for k-step ks (8 rows), tap q of the list,
// MN row j (0..15), row k: ks*list*512 + (2q + j/8)*256 + ((k%8)/4)*128 + (j%8)*16 + (k%4)*4.
__global__ void __launch_bounds__(kThreads, 1)
gram_tc_kernel(const float* __restrict__ x, TcParams p, const int* __restrict__ tap_off, float* __restrict__ part) {
  hicu_pdl_entry();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[kMaxStages], empty_bar[kMaxStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = blockIdx.x, split = blockIdx.y;
  const int T = p.T;
  const int m0 = mtile_first_tap(p.pair_m[pair], T);
  const int n0 = p.pair_n[pair] * kNT;
  const int NT = min(kNT, T - n0);
  const bool a_inside = (m0 >= n0) && (m0 + kMT <= n0 + NT);
  const int list = NT + (a_inside ? 0 : kMT);
  const int a_off = a_inside ? (m0 - n0) : NT;
  const uint32_t half_bytes = (uint32_t)(list * 2 * 512);
  const uint32_t stage_bytes = 2 * half_bytes;
  const int64_t kb0 = (int64_t)split * p.kb_per_split;
  const int64_t kb1 = hmin64(p.nkb, kb0 + p.kb_per_split);
  const int nkb = (int)(kb1 > kb0 ? kb1 - kb0 : 0);
  const int nchains = (nkb + kChain - 1) / kChain;
  const int S = p.stages;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], kProducers);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kProdWarps) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp < kProdWarps) {
    // ---------------- producers: gather, split hi/lo, K-major stores ----------------
    // All kTasks x 4 loads of a stage are issued together, and the next
    // stage's loads are issued before this stage is converted and stored, so
    // each producer thread keeps ~2 stages of L2 gathers in flight (one stage
    // at a time with 8 loads in flight left the tensor pipe at ~22 %).
    const int tid = threadIdx.x;
    const int ntask = list * 64;
    int toff[kTasks];
#pragma unroll
    for (int it = 0; it < kTasks; ++it) {
      const int t = tid + it * kProducers;
      const int q = t >> 6;
      const int tap = (q < NT) ? n0 + q : m0 + (q - NT);
      toff[it] = t < ntask ? tap_off[tap] + (t & 15) + ((t >> 4) & 3) * 64 : -1;
    }
    GramCursor cu;
    if (kb0 < kb1) cursor_init(p, kb0, cu);
    float va[kTasks][4];
#if HICU_GRAM_PREFETCH
    float vb[kTasks][4];
    if (kb0 < kb1) gram_gather(x, cu, toff, va);
#endif
    int s = 0;
    uint32_t ph = 0;
    for (int64_t kb = kb0; kb < kb1; ++kb) {
#if HICU_GRAM_PREFETCH
      mbar_wait(&empty_bar[s], ph ^ 1);
      if (kb + 1 < kb1) {
        cursor_next(p, cu);
        gram_gather(x, cu, toff, vb);
      }
#elif defined(HICU_GRAM_EXP_NOPROD)  // experiment: no gathers (stages carry stale data)
      cursor_next(p, cu);
      mbar_wait(&empty_bar[s], ph ^ 1);
      mbar_arrive(&full_bar[s]);
      if (++s == S) { s = 0; ph ^= 1; }
      continue;
#else
      gram_gather(x, cu, toff, va);
      cursor_next(p, cu);
      mbar_wait(&empty_bar[s], ph ^ 1);
#endif
      uint8_t* sb = smem + (size_t)s * stage_bytes;
#pragma unroll
      for (int it = 0; it < kTasks; ++it) {
        const int t = tid + it * kProducers;
        if (t < ntask) {
          const int j = t & 15;
          const int quad = (t >> 4) & 3;
          const int q = t >> 6;
          float h[4], l[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            uint32_t hb;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(va[it][r]));
            h[r] = __uint_as_float(hb);
            l[r] = va[it][r] - h[r];
          }
          const int ks = quad >> 1, kq = quad & 1;
          const uint32_t off = (uint32_t)ks * list * 512 + (uint32_t)(2 * q + (j >> 3)) * 256 + (uint32_t)kq * 128 +
                               (uint32_t)(j & 7) * 16;
          *(float4*)(sb + off) = make_float4(h[0], h[1], h[2], h[3]);
          *(float4*)(sb + half_bytes + off) = make_float4(l[0], l[1], l[2], l[3]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&full_bar[s]);
#if HICU_GRAM_PREFETCH
#pragma unroll
      for (int it = 0; it < kTasks; ++it)
#pragma unroll
        for (int r = 0; r < 4; ++r) va[it][r] = vb[it][r];
#endif
      if (++s == S) { s = 0; ph ^= 1; }
    }
  } else if (warp == kProdWarps) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = make_idesc_tf32(128, 16 * NT);
    int s = 0;
    uint32_t ph = 0;
    int chunk = (int)(kb0 % p.nkb_line);  // advanced per k-block (no 64-bit modulo in the issue loop)
    const int64_t lastlen = p.rext[p.nsp - 1];
    for (int c = 0; c < nchains; ++c) {
      const int b = c & 1;
      mbar_wait(&tempty[b], ((c >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dcol = tmem + (uint32_t)(256 * b);
      bool first = true;
      const int j1 = min(nkb, (c + 1) * kChain);
      for (int j = c * kChain; j < j1; ++j) {
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        const int valid = (int)hmin64(kBK, lastlen - (int64_t)chunk * kBK);
        if (++chunk == p.nkb_line) chunk = 0;
        const int nks = (valid + 7) / 8;
        if (lane == 0) {
          const uint32_t sbase = smem_u32(smem + (size_t)s * stage_bytes);
          for (int ks = 0; ks < nks; ++ks) {
            const uint32_t kbase = sbase + (uint32_t)ks * list * 512;
            const uint64_t a_hi = make_desc_kmajor(kbase + (uint32_t)a_off * 512);
            const uint64_t a_lo = make_desc_kmajor(kbase + half_bytes + (uint32_t)a_off * 512);
            const uint64_t b_hi = make_desc_kmajor(kbase);
            const uint64_t b_lo = make_desc_kmajor(kbase + half_bytes);
#ifndef HICU_GRAM_EXP_NOMMA  // experiment: pipeline without the tensor-core work
            umma_tf32(dcol, a_hi, b_hi, idesc, first ? 0u : 1u);
            umma_tf32(dcol, a_hi, b_lo, idesc, 1u);
            umma_tf32(dcol, a_lo, b_hi, idesc, 1u);
#endif
            first = false;
          }
          umma_commit(&empty_bar[s]);
        }
        __syncwarp();
        if (++s == S) { s = 0; ph ^= 1; }
      }
      if (lane == 0) umma_commit(&tfull[b]);
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: drain chains into fp32 registers ----------------
    const int ew = warp - (kProdWarps + 1);
    const int q4 = warp & 3;  // TMEM lane quarter
    const int grp = ew >> 2;  // 64-column group
    const int row = 32 * q4 + lane;
    const int c0 = 64 * grp;
    const int ncols = max(0, min(64, 16 * NT - c0));
    float acc[64];
#pragma unroll
    for (int q = 0; q < 64; ++q) acc[q] = 0.f;
    for (int c = 0; c < nchains; ++c) {
      const int b = c & 1;
      mbar_wait(&tfull[b], (c >> 1) & 1);
      tc_fence_after();
      if (ncols > 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t r[16];
          tmem_ld16_raw(tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)(256 * b + c0 + 16 * i), r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int q = 0; q < 16; ++q) acc[16 * i + q] += __uint_as_float(r[q]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
    float* dst = part + ((size_t)pair * gridDim.y + split) * 128 * kPartCols + (size_t)row * kPartCols + c0;
#pragma unroll
    for (int q = 0; q < 64; q += 4)
      if (q < ncols) *(float4*)(dst + q) = make_float4(acc[q], acc[q + 1], acc[q + 2], acc[q + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kProdWarps) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------------------
// TMA-fed variant (gram_tc2_kernel).  A planar copy Xt[f][position] of the
// k-space (f = the 16 floats of one spatial position: 8 coils x re/im) makes
// every tap's operand tile K-major along positions, so the producer is one
// TMA box [16 positions x 16 floats] (SWIZZLE_64B, 1 KB) per tap per k-block
// instead of 4 warps of scalar gathers.  Converter warps write A_lo =
// rna(x - trunc(x)) next to the raw tile (the tensor core reads the raw fp32
// container as trunc(x) = A_hi) and zero the K columns past the region line.
// MMA issue, chained TMEM accumulators, epilogue and the split-K reduction are
// those of gram_tc_kernel.
// Warp roles (704 threads): warp 0 TMA producer, warp 1 TMEM owner + MMA
// issuer, warps 2-5 converters, warps 6-21 epilogue.
constexpr int kEpi0v2 = 6;
constexpr int kThreads2 = (kEpi0v2 + kEpiWarps) * 32;
constexpr int kMaxTaps2 = 128;

// Blocked planar copies of the k-space for the TMA producer.  Copy b (one per
// last-axis kernel offset, b < kext_last <= kMaxShift) is shifted by
// sigma_b = (roff_last + b) mod 16 positions and stored as
//   Xt_b[line][blk][f][t] = X[line][16 blk + t + sigma_b][f]   (0 past the line)
// so the operand box of any tap, chunk and line is one contiguous 1 KB block
// [16 f rows x 16 positions]: K-major SWIZZLE_64B, one 16-byte aligned TMA op.
constexpr int kMaxShift = 8;
struct TmapSet {
  CUtensorMap m[kMaxShift];
};

__global__ void gram_planar_kernel(int64_t nlines, int dlast, int nblk, int nshift, int roff_last,
                                   const float* __restrict__ x, float* __restrict__ xt) {
  hicu_pdl_entry();
  // one thread per (line, blk, f, t) of one copy; t fastest (coalesced writes)
  const int64_t per_copy = nlines * nblk * 256;
  const int64_t total = per_copy * nshift;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / per_copy);
    int64_t r = e % per_copy;
    const int t = (int)(r & 15), f = (int)((r >> 4) & 15);
    r >>= 8;
    const int blk = (int)(r % nblk);
    const int64_t line = r / nblk;
    const int sig = (roff_last + b) & 15;
    const int pos = 16 * blk + t + sig;
    xt[e] = pos < dlast ? __ldg(x + ((size_t)line * dlast + pos) * 16 + f) : 0.f;
  }
}

__global__ void __launch_bounds__(kThreads2, 1)
gram_tc2_kernel(const __grid_constant__ TmapSet tms, TcParams p, const int32_t* __restrict__ pos, int ndim,
                float* __restrict__ part, int dbg, const float* __restrict__ xt, int64_t copy_floats, int nblk,
                int d3, int cpasync) {
  hicu_pdl_entry();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[kMaxStages], ready_bar[kMaxStages], empty_bar[kMaxStages], tfull[2],
      tempty[2];
  __shared__ uint32_t tmem_slot;
  __shared__ int tap_c[kMaxTaps2][3];  // per tap: last-axis offset, prefix offsets
  __shared__ int64_t tap_term[kNT + kMT];  // cp.async producer: per-tile source offsets
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = blockIdx.x, split = blockIdx.y;
  const int T = p.T;
  const int L = p.nsp;  // spatial axes
  const int m0 = mtile_first_tap(p.pair_m[pair], T);
  const int n0 = p.pair_n[pair] * kNT;
  const int NT = min(kNT, T - n0);
  const bool a_inside = (m0 >= n0) && (m0 + kMT <= n0 + NT);
  const int list = NT + (a_inside ? 0 : kMT);
  const int a_off = a_inside ? (m0 - n0) : NT;
  const uint32_t half_bytes = (uint32_t)(list * 1024);
  const uint32_t stage_bytes = 2 * half_bytes;
  const int64_t kb0 = (int64_t)split * p.kb_per_split;
  const int64_t kb1 = hmin64(p.nkb, kb0 + p.kb_per_split);
  const int nkb = (int)(kb1 > kb0 ? kb1 - kb0 : 0);
  const int nchains = (nkb + kChain - 1) / kChain;
  const int S = p.stages;

  for (int t = threadIdx.x; t < T * L; t += blockDim.x) {
    const int tp = t / L, d = t % L;
    const int v = __ldg(pos + (size_t)tp * 8 * ndim + d);
    if (d == L - 1) tap_c[tp][0] = v;
    else tap_c[tp][1 + d] = v;
  }
  __syncthreads();
  // cp.async producer: per-tile source offset (floats) independent of the line
  if (cpasync && threadIdx.x < list) {
    const int q = threadIdx.x;
    const int tap = (q < NT) ? n0 + q : m0 + (q - NT);
    const int bsh = tap_c[tap][0];
    int64_t tt = ((int)p.roff[L - 1] + bsh) >> 4;
    if (L == 2) tt += (int64_t)tap_c[tap][1] * nblk;
    if (L == 3) tt += ((int64_t)tap_c[tap][1] * d3 + tap_c[tap][2]) * nblk;
    tap_term[q] = (int64_t)bsh * copy_floats + tt * 256;
  }
  if (threadIdx.x == 0) {
    for (int st = 0; st < S; ++st) {
      mbar_init(&full_bar[st], cpasync ? 32 : 1);
      mbar_init(&ready_bar[st], 128);
      mbar_init(&empty_bar[st], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0 && cpasync) {
    // ---------------- cp.async producer (all 32 lanes) ----------------
    // Each operand tile is a contiguous 1 KB block [16 f rows x 16 positions]
    // of the planar copy; lanes issue its 64 16-byte chunks with cp.async
    // into the SW64-swizzled K-major layout (chunk u of row f lands at
    // 16 (u ^ ((f >> 1) & 3))) and arm the stage's full barrier with
    // cp.async.mbarrier.arrive (no thread waits for the data: the producer
    // runs up to S stages ahead, each stage ~24 KB in flight).
    int st = 0;
    uint32_t ph = 0;
    for (int64_t kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&empty_bar[st], ph ^ 1);
      const int64_t line = kb / p.nkb_line;
      const int chunk = (int)(kb % p.nkb_line);
      int lc[2] = {0, 0};
      {
        int64_t rem = line;
        for (int d = L - 2; d >= 0; --d) {
          lc[d] = (int)(rem % p.rext[d]);
          rem /= p.rext[d];
        }
      }
      const uint32_t sb = smem_u32(smem + (size_t)st * stage_bytes);
      // lane covers rows f = lane / 4 and f + 8 of every tile, chunk u = lane % 4;
      // source block = line term (line, chunk) + per-tile term (tap_term)
      const int f0 = lane >> 2, u = lane & 3;
      const uint32_t d0 = (uint32_t)f0 * 64 + (uint32_t)((u ^ ((f0 >> 1) & 3)) << 4);
      const uint32_t d1 = (uint32_t)(f0 + 8) * 64 + (uint32_t)((u ^ (((f0 + 8) >> 1) & 3)) << 4);
      int64_t lt = chunk;
      if (L == 2) lt += (int64_t)((int)p.roff[0] + lc[0]) * nblk;
      if (L == 3) lt += ((int64_t)((int)p.roff[0] + lc[0]) * d3 + ((int)p.roff[1] + lc[1])) * nblk;
      const float* srcl = xt + lt * 256 + f0 * 16 + u * 4;
#pragma unroll 4
      for (int q = 0; q < list; ++q) {
        const float* src = srcl + tap_term[q];
        const uint32_t dst = sb + (uint32_t)q * 1024;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + d0), "l"(src) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + d1), "l"(src + 128) : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full_bar[st])) : "memory");
      if (++st == S) { st = 0; ph ^= 1; }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int64_t kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty_bar[st], ph ^ 1);
        const int64_t line = kb / p.nkb_line;
        const int chunk = (int)(kb % p.nkb_line);
        int lc[2] = {0, 0};
        {
          int64_t rem = line;
          for (int d = L - 2; d >= 0; --d) {
            lc[d] = (int)(rem % p.rext[d]);
            rem /= p.rext[d];
          }
        }
        if (dbg & 2) {
          mbar_arrive(&full_bar[st]);
          if (++st == S) { st = 0; ph ^= 1; }
          continue;
        }
        tc::mbar_expect_tx(&full_bar[st], half_bytes);
        uint8_t* sb = smem + (size_t)st * stage_bytes;
        for (int q = 0; q < list; ++q) {
          const int tap = (q < NT) ? n0 + q : m0 + (q - NT);
          // copy b = last-axis offset of the tap; block = (roff + b + 16 chunk - sigma_b) / 16
          const int bsh = tap_c[tap][0];
          const int pstart = (int)p.roff[L - 1] + bsh + chunk * kBK;
          const int blk = (pstart - (pstart & 15)) >> 4;
          int c3 = 0, c4 = 0;
          if (L == 2) c3 = (int)p.roff[0] + lc[0] + tap_c[tap][1];
          if (L == 3) {
            c3 = (int)p.roff[1] + lc[1] + tap_c[tap][2];
            c4 = (int)p.roff[0] + lc[0] + tap_c[tap][1];
          }
          tc::tma_load_5d(sb + (size_t)q * 1024, &tms.m[(dbg & 16) ? 0 : bsh], 0, 0, blk, c3, c4, &full_bar[st]);
        }
        if (++st == S) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = make_idesc_tf32(128, 16 * NT);
    int st = 0;
    uint32_t ph = 0;
    for (int c = 0; c < nchains; ++c) {
      const int b = c & 1;
      mbar_wait(&tempty[b], ((c >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dcol = tmem + (uint32_t)(256 * b);
      bool first = true;
      const int j1 = min(nkb, (c + 1) * kChain);
      for (int j = c * kChain; j < j1; ++j) {
        const int64_t kb = kb0 + j;
        mbar_wait(&ready_bar[st], ph);
        tc_fence_after();
        const int chunk = (int)(kb % p.nkb_line);
        const int valid = (int)hmin64(kBK, p.rext[L - 1] - (int64_t)chunk * kBK);
        const int nks = (valid + 7) / 8;
        if (lane == 0) {
          const uint32_t sbase = smem_u32(smem + (size_t)st * stage_bytes);
          for (int ks = 0; ks < ((dbg & 1) ? 0 : nks); ++ks) {
            const uint32_t kofs = (uint32_t)ks * 32;
            const uint64_t a_hi = tc::desc_sw64(sbase + (uint32_t)a_off * 1024 + kofs);
            const uint64_t a_lo = tc::desc_sw64(sbase + half_bytes + (uint32_t)a_off * 1024 + kofs);
            const uint64_t b_hi = tc::desc_sw64(sbase + kofs);
            const uint64_t b_lo = tc::desc_sw64(sbase + half_bytes + kofs);
            umma_tf32(dcol, a_hi, b_hi, idesc, first ? 0u : 1u);
            umma_tf32(dcol, a_hi, b_lo, idesc, 1u);
            umma_tf32(dcol, a_lo, b_hi, idesc, 1u);
            first = false;
          }
          umma_commit(&empty_bar[st]);
        }
        __syncwarp();
        if (++st == S) { st = 0; ph ^= 1; }
      }
      if (lane == 0) umma_commit(&tfull[b]);
      __syncwarp();
    }
  } else if (warp < kEpi0v2) {
    // ---------------- converters: A_lo and line-tail zeroing ----------------
    const int ct = threadIdx.x - 64;
    int st = 0;
    uint32_t ph = 0;
    for (int64_t kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&full_bar[st], ph);
      const int chunk = (int)(kb % p.nkb_line);
      const int valid = (int)hmin64(kBK, p.rext[L - 1] - (int64_t)chunk * kBK);
      uint8_t* sb = smem + (size_t)st * stage_bytes;
      float4* raw4 = reinterpret_cast<float4*>(sb);
      float4* lo4 = reinterpret_cast<float4*>(sb + half_bytes);
      // float4 slot s: box q = s / 64, row f = (s % 64) / 4, physical 16-B chunk u = s % 4;
      // logical K = 4 * (u ^ ((row byte address >> 7) & 3)) + e
      for (int sidx = ct; sidx < ((dbg & 4) ? 0 : list * 64); sidx += 128) {
        float4 v = raw4[sidx];
        if (valid < kBK) {
          const int f = (sidx & 63) >> 2, u = sidx & 3;
          const int k4 = 4 * (u ^ ((f >> 1) & 3));
          if (k4 + 0 >= valid) v.x = 0.f;
          if (k4 + 1 >= valid) v.y = 0.f;
          if (k4 + 2 >= valid) v.z = 0.f;
          if (k4 + 3 >= valid) v.w = 0.f;
          raw4[sidx] = v;
        }
        lo4[sidx] = make_float4(tc::tf32_lo(v.x), tc::tf32_lo(v.y), tc::tf32_lo(v.z), tc::tf32_lo(v.w));
      }
      tc::fence_proxy_async();
      mbar_arrive(&ready_bar[st]);
      if (++st == S) { st = 0; ph ^= 1; }
    }
  } else {
    // ---------------- epilogue: drain chains into fp32 registers ----------------
    const int ew = warp - kEpi0v2;
    const int q4 = warp & 3;  // TMEM lane quarter
    const int grp = ew >> 2;  // 64-column group
    const int row = 32 * q4 + lane;
    const int c0 = 64 * grp;
    const int ncols = max(0, min(64, 16 * NT - c0));
    float acc[64];
#pragma unroll
    for (int q = 0; q < 64; ++q) acc[q] = 0.f;
    for (int c = 0; c < nchains; ++c) {
      const int b = c & 1;
      mbar_wait(&tfull[b], (c >> 1) & 1);
      tc_fence_after();
      if (ncols > 0 && !(dbg & 8)) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t r[16];
          tmem_ld16_raw(tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)(256 * b + c0 + 16 * i), r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int q = 0; q < 16; ++q) acc[16 * i + q] += __uint_as_float(r[q]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
    float* dst = part + ((size_t)pair * gridDim.y + split) * 128 * kPartCols + (size_t)row * kPartCols + c0;
#pragma unroll
    for (int q = 0; q < 64; q += 4)
      if (q < ncols) *(float4*)(dst + q) = make_float4(acc[q], acc[q + 1], acc[q + 2], acc[q + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------------------
// Cluster-multicast variant (gram_tc3_kernel).  The np tile pairs of one
// split-K slice run as one thread-block cluster (np <= 8): every CTA needs the
// same k-space rows, only different taps, so each k-block's T tap tiles
// ([16 f x 16 positions], 1 KB, from the planar copies) are loaded ONCE per
// cluster -- CTA r issues tiles r, r + np, ... with TMA multicast into all np
// CTAs -- instead of 24 gathered tiles per CTA.  That divides the L2 traffic
// by ~np and the per-CTA TMA issue by ~np (a 1 KB op costs ~68 cycles, so 24
// per k-block outran the MMA).  Stage s is refilled only when every CTA of the
// cluster has consumed it: the MMA warp's tcgen05.commit multicasts its
// arrival to the empty barrier of all np CTAs.  Converters (A_lo split, line
// tail zeroing), MMA chains, epilogue and reduction are those of gram_tc2.
__device__ __forceinline__ void tma_load_5d_mc(void* dst, const void* tmap, int c0, int c1, int c2, int c3, int c4,
                                               uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
      "%3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__global__ void __launch_bounds__(kThreads2, 1)
gram_tc3_kernel(const __grid_constant__ TmapSet tms, TcParams p, const int32_t* __restrict__ pos, int ndim,
                float* __restrict__ part, int dbg) {
  hicu_pdl_entry();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[kMaxStages], ready_bar[kMaxStages], empty_bar[kMaxStages], tfull[2],
      tempty[2];
  __shared__ uint32_t tmem_slot;
  __shared__ int tap_c[kMaxTaps2][3];  // per tap: last-axis offset, prefix offsets
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = blockIdx.x, split = blockIdx.y;
  const int np = p.npairs;  // == cluster size
  const unsigned rank = hicu_cluster_rank();
  const uint16_t mask = (uint16_t)((1u << np) - 1u);
  const int T = p.T;
  const int L = p.nsp;  // spatial axes
  const int m0 = mtile_first_tap(p.pair_m[pair], T);
  const int n0 = p.pair_n[pair] * kNT;
  const int NT = min(kNT, T - n0);
  const uint32_t half_bytes = (uint32_t)(T * 1024);
  const uint32_t stage_bytes = 2 * half_bytes;
  const int64_t kb0 = (int64_t)split * p.kb_per_split;
  const int64_t kb1 = hmin64(p.nkb, kb0 + p.kb_per_split);
  const int nkb = (int)(kb1 > kb0 ? kb1 - kb0 : 0);
  const int nchains = (nkb + kChain - 1) / kChain;
  const int S = p.stages;

  for (int t = threadIdx.x; t < T * L; t += blockDim.x) {
    const int tp = t / L, d = t % L;
    const int v = __ldg(pos + (size_t)tp * 8 * ndim + d);
    if (d == L - 1) tap_c[tp][0] = v;
    else tap_c[tp][1 + d] = v;
  }
  if (threadIdx.x == 0) {
    for (int st = 0; st < S; ++st) {
      mbar_init(&full_bar[st], 1);
      mbar_init(&ready_bar[st], 128);
      mbar_init(&empty_bar[st], np);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  // every CTA's barriers are initialised before any peer multicasts into them
  hicu_cluster_arrive();
  hicu_cluster_wait();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // ---------------- TMA multicast producer ----------------
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int64_t kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty_bar[st], ph ^ 1);  // all np CTAs released this stage
        const int64_t line = kb / p.nkb_line;
        const int chunk = (int)(kb % p.nkb_line);
        int lc[2] = {0, 0};
        {
          int64_t rem = line;
          for (int d = L - 2; d >= 0; --d) {
            lc[d] = (int)(rem % p.rext[d]);
            rem /= p.rext[d];
          }
        }
        tc::mbar_expect_tx(&full_bar[st], half_bytes);  // all T tiles land here, from all issuers
        uint8_t* sb = smem + (size_t)st * stage_bytes;
        for (int q = (int)rank; q < T; q += np) {
          const int bsh = tap_c[q][0];
          const int pstart = (int)p.roff[L - 1] + bsh + chunk * kBK;
          const int blk = (pstart - (pstart & 15)) >> 4;
          int c3 = 0, c4 = 0;
          if (L == 2) c3 = (int)p.roff[0] + lc[0] + tap_c[q][1];
          if (L == 3) {
            c3 = (int)p.roff[1] + lc[1] + tap_c[q][2];
            c4 = (int)p.roff[0] + lc[0] + tap_c[q][1];
          }
          tma_load_5d_mc(sb + (size_t)q * 1024, &tms.m[bsh], 0, 0, blk, c3, c4, &full_bar[st], mask);
        }
        if (++st == S) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = make_idesc_tf32(128, 16 * NT);
    int st = 0;
    uint32_t ph = 0;
    for (int c = 0; c < nchains; ++c) {
      const int b = c & 1;
      mbar_wait(&tempty[b], ((c >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dcol = tmem + (uint32_t)(256 * b);
      bool first = true;
      const int j1 = min(nkb, (c + 1) * kChain);
      for (int j = c * kChain; j < j1; ++j) {
        const int64_t kb = kb0 + j;
        mbar_wait(&ready_bar[st], ph);
        tc_fence_after();
        const int chunk = (int)(kb % p.nkb_line);
        const int valid = (int)hmin64(kBK, p.rext[L - 1] - (int64_t)chunk * kBK);
        const int nks = (valid + 7) / 8;
        if (lane == 0) {
          const uint32_t sbase = smem_u32(smem + (size_t)st * stage_bytes);
          for (int ks = 0; ks < ((dbg & 1) ? 0 : nks); ++ks) {
            const uint32_t kofs = (uint32_t)ks * 32;
            const uint64_t a_hi = tc::desc_sw64(sbase + (uint32_t)m0 * 1024 + kofs);
            const uint64_t a_lo = tc::desc_sw64(sbase + half_bytes + (uint32_t)m0 * 1024 + kofs);
            const uint64_t b_hi = tc::desc_sw64(sbase + (uint32_t)n0 * 1024 + kofs);
            const uint64_t b_lo = tc::desc_sw64(sbase + half_bytes + (uint32_t)n0 * 1024 + kofs);
            umma_tf32(dcol, a_hi, b_hi, idesc, first ? 0u : 1u);
            umma_tf32(dcol, a_hi, b_lo, idesc, 1u);
            umma_tf32(dcol, a_lo, b_hi, idesc, 1u);
            first = false;
          }
          umma_commit_mc(&empty_bar[st], mask);
        }
        __syncwarp();
        if (++st == S) { st = 0; ph ^= 1; }
      }
      if (lane == 0) umma_commit(&tfull[b]);
      __syncwarp();
    }
  } else if (warp < kEpi0v2) {
    // ---------------- converters: A_lo and line-tail zeroing (all T tiles) ----------------
    const int ct = threadIdx.x - 64;
    int st = 0;
    uint32_t ph = 0;
    for (int64_t kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&full_bar[st], ph);
      const int chunk = (int)(kb % p.nkb_line);
      const int valid = (int)hmin64(kBK, p.rext[L - 1] - (int64_t)chunk * kBK);
      uint8_t* sb = smem + (size_t)st * stage_bytes;
      float4* raw4 = reinterpret_cast<float4*>(sb);
      float4* lo4 = reinterpret_cast<float4*>(sb + half_bytes);
      for (int sidx = ct; sidx < ((dbg & 4) ? 0 : T * 64); sidx += 128) {
        float4 v = raw4[sidx];
        if (valid < kBK) {
          const int f = (sidx & 63) >> 2, u = sidx & 3;
          const int k4 = 4 * (u ^ ((f >> 1) & 3));
          if (k4 + 0 >= valid) v.x = 0.f;
          if (k4 + 1 >= valid) v.y = 0.f;
          if (k4 + 2 >= valid) v.z = 0.f;
          if (k4 + 3 >= valid) v.w = 0.f;
          raw4[sidx] = v;
        }
        lo4[sidx] = make_float4(tc::tf32_lo(v.x), tc::tf32_lo(v.y), tc::tf32_lo(v.z), tc::tf32_lo(v.w));
      }
      tc::fence_proxy_async();
      mbar_arrive(&ready_bar[st]);
      if (++st == S) { st = 0; ph ^= 1; }
    }
  } else {
    // ---------------- epilogue: drain chains into fp32 registers ----------------
    const int ew = warp - kEpi0v2;
    const int q4 = warp & 3;  // TMEM lane quarter
    const int grp = ew >> 2;  // 64-column group
    const int row = 32 * q4 + lane;
    const int c0 = 64 * grp;
    const int ncols = max(0, min(64, 16 * NT - c0));
    float acc[64];
#pragma unroll
    for (int q = 0; q < 64; ++q) acc[q] = 0.f;
    for (int c = 0; c < nchains; ++c) {
      const int b = c & 1;
      mbar_wait(&tfull[b], (c >> 1) & 1);
      tc_fence_after();
      if (ncols > 0 && !(dbg & 8)) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t r[16];
          tmem_ld16_raw(tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)(256 * b + c0 + 16 * i), r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int q = 0; q < 16; ++q) acc[16 * i + q] += __uint_as_float(r[q]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
    float* dst = part + ((size_t)pair * gridDim.y + split) * 128 * kPartCols + (size_t)row * kPartCols + c0;
#pragma unroll
    for (int q = 0; q < 64; q += 4)
      if (q < ncols) *(float4*)(dst + q) = make_float4(acc[q], acc[q + 1], acc[q + 2], acc[q + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
  // no CTA leaves while a peer may still multicast into it or arrive on its barriers
  hicu_cluster_arrive();
  hicu_cluster_wait();
}

// G[k1][k2] (k1 <= k2) from the real partials: (rr + ii) + i (ri - ir), summed
// over splits in fp64 in a fixed order; mirrored conjugate below the diagonal.
__global__ void gram_tc_reduce_kernel(int n, int nc, int T, int splits, PairTable pt, int ntn,
                                      const float* __restrict__ part, double2* __restrict__ G) {
  hicu_pdl_entry();
  const int64_t total = (int64_t)n * n;
  const size_t blk = (size_t)128 * kPartCols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int k1 = (int)(e / n), k2 = (int)(e % n);
    if (k1 > k2) continue;
    const int t1 = k1 / nc, c1 = k1 % nc, t2 = k2 / nc, c2 = k2 % nc;
    int mt = t1 / kMT;
    while (mtile_first_tap(mt, T) > t1) --mt;  // first tile containing t1
    const int lt1 = t1 - mtile_first_tap(mt, T);
    const int nt = t2 / kNT, lt2 = t2 - nt * kNT;
    const int pr = pt.v[mt * ntn + nt];
    const int mu = (lt1 * nc + c1) * 2, nu = (lt2 * nc + c2) * 2;
    double rr = 0.0, ii = 0.0, ri = 0.0, ir = 0.0;
    for (int sp = 0; sp < splits; ++sp) {
      const float* b = part + ((size_t)pr * splits + sp) * blk;
      rr += b[(size_t)mu * kPartCols + nu];
      ri += b[(size_t)mu * kPartCols + nu + 1];
      ir += b[(size_t)(mu + 1) * kPartCols + nu];
      ii += b[(size_t)(mu + 1) * kPartCols + nu + 1];
    }
    const double gr = rr + ii, gi = ri - ir;
    if (k1 == k2) {
      G[e] = cd(gr, 0.0);
    } else {
      G[e] = cd(gr, gi);
      G[(size_t)k2 * n + k1] = cd(gr, -gi);
    }
  }
}

// per tap: flat float offset of its coil-0 sample relative to the row base (= 2*koff)
__global__ void tc_tap_table_kernel(int T, int nc, const int64_t* __restrict__ koff, int* __restrict__ out) {
  hicu_pdl_entry();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T) out[t] = (int)(2 * koff[(size_t)t * nc]);
}

struct TcPlan {
  bool ok = false;
  TcParams p;
  PairTable pt;
  int splits = 0;
  int mtiles = 0, ntiles = 0;
  size_t part_bytes = 0, smem_bytes = 0;
};

TcPlan tc_plan(const DevGeom& g) {
  TcPlan pl;
  if (g.nc != 8 || g.ncirc != 0) return pl;
  const int nsp = g.ndim - 1;
  if (nsp < 1 || nsp > 3) return pl;
  const int T = g.nsp;
  if (T < kMT || T > 128) return pl;
  TcParams& p = pl.p;
  p.T = T;
  p.nsp = nsp;
  for (int d = 0; d < 3; ++d) {
    p.rext[d] = d < nsp ? g.rext[d] : 1;
    p.roff[d] = d < nsp ? g.roff[d] : 0;
    p.fstride[d] = d < nsp ? 2 * g.stride[d] : 0;
  }
  const int64_t rl = p.rext[nsp - 1];
  p.nkb_line = (rl + kBK - 1) / kBK;
  int64_t lines = 1;
  for (int d = 0; d < nsp - 1; ++d) lines *= p.rext[d];
  p.nkb = lines * p.nkb_line;
  pl.mtiles = (T + kMT - 1) / kMT;
  pl.ntiles = (T + kNT - 1) / kNT;
  int np = 0;
  for (int m = 0; m < pl.mtiles; ++m)
    for (int nn = 0; nn < pl.ntiles; ++nn) {
      const int mf = mtile_first_tap(m, T), nl = min(T, (nn + 1) * kNT) - 1;
      pl.pt.v[m * pl.ntiles + nn] = -1;
      if (mf <= nl) {  // the tile holds some k1 <= k2 entries
        if (np >= kMaxPairs) return pl;
        p.pair_m[np] = (unsigned char)m;
        p.pair_n[np] = (unsigned char)nn;
        pl.pt.v[m * pl.ntiles + nn] = (short)np++;
      }
    }
  p.npairs = np;
  // one wave: np * splits <= SM count (one CTA per SM at ~200 KB of shared
  // memory; a 149th CTA would double the kernel time)
  int splits = hicu_sm_count() / np;
  if (splits > p.nkb) splits = (int)p.nkb;
  if (splits < 1) splits = 1;
  p.kb_per_split = (p.nkb + splits - 1) / splits;
  pl.splits = (int)((p.nkb + p.kb_per_split - 1) / p.kb_per_split);
  const size_t stage_bytes = (size_t)(kNT + kMT) * 2 * 1024;
  int stages = (int)((200 * 1024) / stage_bytes);
  if (stages > kMaxStages) stages = kMaxStages;
  if (stages < 2) return pl;
  p.stages = stages;
  pl.smem_bytes = stages * stage_bytes + 1024;
  pl.part_bytes = (size_t)np * pl.splits * 128 * kPartCols * sizeof(float);
  pl.ok = true;
  return pl;
}

typedef CUresult (*GramEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

GramEncodeFn gram_encode() {
  static GramEncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (GramEncodeFn)f;
    else
      cudaGetLastError();
  }
  return fn;
}

// The gather-producer kernel is the default.  The TMA-fed variant is opt-in
// (HICU_GRAM_TMA=1): with K-major tf32 operands one TMA op carries a 1 KB
// [16 f x 16 positions] tile, and a 1 KB op costs ~68 cycles of TMA issue on
// this part (scripts/tma_rate.cu: 68 / 100 / 131 cycles for 1 / 4 / 8 KB), so
// the 24 ops per 16-row k-block outrun the ~768 MMA cycles they feed
// (measured 512 us vs 359 us at C2 full).
bool use_tma_gram() {
  static int v = -1;
  if (v < 0) v = getenv("HICU_GRAM_TMA") ? 1 : 0;
  return v == 1;
}
// cluster-multicast planar variant (HICU_GRAM_MC=1 while it is being measured)
bool use_mc_gram() {
  static int v = -1;
  if (v < 0) v = getenv("HICU_GRAM_MC") ? 1 : 0;
  return v == 1;
}
// cp.async-fed planar variant (HICU_GRAM_CPASYNC=1 while it is being measured)
bool use_cpasync_gram() {
  static int v = -1;
  if (v < 0) v = getenv("HICU_GRAM_CPASYNC") ? 1 : 0;
  return v == 1;
}

size_t planar_bytes(const DevGeom& g) {
  const int L = g.ndim - 1;
  if (!(use_tma_gram() || use_cpasync_gram() || use_mc_gram()) || L < 1 || g.kext[L - 1] < 1) return 0;
  int64_t nlines = 1;
  for (int d = 0; d < L - 1; ++d) nlines *= g.dims[d];
  const int64_t nblk = (g.dims[L - 1] + 15) / 16 + 1;
  return (((size_t)nlines * nblk * 256 * g.kext[L - 1] * sizeof(float)) + 255) & ~(size_t)255;
}

}  // namespace

bool hicu_gram_tc_supported(const DevGeom& g) { return tc_plan(g).ok; }

size_t hicu_gram_tc_workspace(const DevGeom& g) {
  TcPlan pl = tc_plan(g);
  if (!pl.ok) return 0;
  return pl.part_bytes + 4096 + planar_bytes(g);
}

int hicu_gram_tc(const DevGeom& g, const float2* x, double2* G, void* ws, size_t ws_bytes, cudaStream_t st) {
  TcPlan pl = tc_plan(g);
  if (!pl.ok) return hicu_set_error(HICU_ERR_PARAMETER, "gram_tc: unsupported geometry");
  if (ws_bytes < hicu_gram_tc_workspace(g)) return hicu_set_error(HICU_ERR_WORKSPACE, "gram_tc: workspace");
  float* part = (float*)ws;
  int* toff = (int*)((char*)ws + pl.part_bytes);
  float* xt = (float*)((char*)ws + pl.part_bytes + 4096);
  int s;
  dim3 grid(pl.p.npairs, pl.splits);
  int red_splits = pl.splits;
  GramEncodeFn enc = gram_encode();
  const int Lg = g.ndim - 1;
  if ((use_tma_gram() || use_cpasync_gram() || use_mc_gram()) && enc && g.kext[Lg - 1] >= 1 && g.kext[Lg - 1] <= kMaxShift) {
    const int L = g.ndim - 1;
    const int dlast = (int)g.dims[L - 1];
    const int nblk = (dlast + 15) / 16 + 1;
    const int nshift = (int)g.kext[L - 1];
    int64_t nlines = 1;
    for (int d = 0; d < L - 1; ++d) nlines *= g.dims[d];
    {
      const int64_t total = nlines * nblk * 256 * nshift;
      const int blocks = (int)hmin64((total + 255) / 256, (int64_t)hicu_sm_count() * 16);
      hicu_launch(gram_planar_kernel, blocks, 256, 0, st, nlines, dlast, nblk, nshift, (int)g.roff[L - 1], (const float*)x,
                                                 xt);
      if ((s = hicu_check_launch("gram_planar_kernel"))) return s;
    }
    TmapSet tms;
    cuuint64_t dims[5] = {16, 16, (cuuint64_t)nblk, (cuuint64_t)(L >= 2 ? g.dims[L - 2] : 1),
                          (cuuint64_t)(L >= 3 ? g.dims[L - 3] : 1)};
    cuuint64_t strides[4] = {64, 1024, (cuuint64_t)1024 * nblk, (cuuint64_t)1024 * nblk * dims[3]};
    cuuint32_t box[5] = {16, 16, 1, 1, 1}, es[5] = {1, 1, 1, 1, 1};
    const size_t copy_floats = (size_t)nlines * nblk * 256;
    for (int b = 0; b < nshift; ++b)
      if (enc(&tms.m[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, xt + (size_t)b * copy_floats, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return hicu_set_error(HICU_ERR_CUDA, "gram_tc: cuTensorMapEncodeTiled failed");
    hicu_allow_max_smem((const void*)gram_tc2_kernel);
    static int dbg = -1;
    if (dbg < 0) dbg = getenv("HICU_GRAM_DEBUG") ? atoi(getenv("HICU_GRAM_DEBUG")) : 0;
    if (use_mc_gram() && pl.p.npairs <= 8 && pl.p.T <= kMaxTaps2) {
      // all T tiles per stage: restage the plan for the wider stage
      TcParams p3 = pl.p;
      const size_t sb3 = (size_t)2 * pl.p.T * 1024;
      int st3 = (int)((200 * 1024) / sb3);
      if (st3 > kMaxStages) st3 = kMaxStages;
      if (st3 < 2) return hicu_set_error(HICU_ERR_SIZE, "gram_tc3: shared memory");
      p3.stages = st3;
      hicu_allow_max_smem((const void*)gram_tc3_kernel);
      // one wave of clusters: a cluster of np CTAs needs np SMs of one GPC,
      // so fewer clusters than SMs / np can be resident at once
      static int cap = -1, cap_np = -1;
      if (cap < 0 || cap_np != pl.p.npairs) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = kThreads2;
        cfg.dynamicSmemBytes = st3 * sb3 + 1024;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = pl.p.npairs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, (const void*)gram_tc3_kernel, &cfg) != cudaSuccess || nc < 1) nc = 1;
        cap = nc;
        cap_np = pl.p.npairs;
      }
      int sp3 = (int)hmin64(pl.splits, cap);
      p3.kb_per_split = (p3.nkb + sp3 - 1) / sp3;
      sp3 = (int)((p3.nkb + p3.kb_per_split - 1) / p3.kb_per_split);
      red_splits = sp3;
      const dim3 grid3(pl.p.npairs, sp3);
      if (getenv("HICU_GRAM_MC_INFO"))
        fprintf(stderr, "gram_tc3: grid %d x %d, cluster %d, stages %d, max active clusters %d\n", grid3.x, grid3.y,
                pl.p.npairs, st3, cap);
      hicu_launch_cluster(gram_tc3_kernel, grid3, kThreads2, st3 * sb3 + 1024, st, pl.p.npairs, tms, p3, g.pos, g.ndim,
                          part, dbg);
      if ((s = hicu_check_launch("gram_tc3_kernel"))) return s;
    } else {
      hicu_launch(gram_tc2_kernel, grid, kThreads2, pl.smem_bytes, st, tms, pl.p, g.pos, g.ndim, part, dbg,
                  (const float*)xt, (int64_t)copy_floats, nblk, (int)dims[3], use_cpasync_gram() ? 1 : 0);
    }
    if ((s = hicu_check_launch("gram_tc2_kernel"))) return s;
  } else {
    hicu_launch(tc_tap_table_kernel, (g.nsp + 127) / 128, 128, 0, st, g.nsp, g.nc, g.koff, toff);
    if ((s = hicu_check_launch("tc_tap_table_kernel"))) return s;
    hicu_allow_max_smem((const void*)gram_tc_kernel);
    hicu_launch(gram_tc_kernel, grid, kThreads, pl.smem_bytes, st, (const float*)x, pl.p, toff, part);
    if ((s = hicu_check_launch("gram_tc_kernel"))) return s;
  }
  const int64_t total = (int64_t)g.n * g.n;
  const int rb = (int)hmin64((total + 255) / 256, 1184);
  hicu_launch(gram_tc_reduce_kernel, rb, 256, 0, st, g.n, g.nc, pl.p.T, red_splits, pl.pt, pl.ntiles, part, G);
  return hicu_check_launch("gram_tc_reduce_kernel");
}
