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

}  // namespace

bool hicu_gram_tc_supported(const DevGeom& g) { return tc_plan(g).ok; }

size_t hicu_gram_tc_workspace(const DevGeom& g) {
  TcPlan pl = tc_plan(g);
  if (!pl.ok) return 0;
  return pl.part_bytes + 4096;
}

int hicu_gram_tc(const DevGeom& g, const float2* x, double2* G, void* ws, size_t ws_bytes, cudaStream_t st) {
  TcPlan pl = tc_plan(g);
  if (!pl.ok) return hicu_set_error(HICU_ERR_PARAMETER, "gram_tc: unsupported geometry");
  if (ws_bytes < hicu_gram_tc_workspace(g)) return hicu_set_error(HICU_ERR_WORKSPACE, "gram_tc: workspace");
  float* part = (float*)ws;
  int* toff = (int*)((char*)ws + pl.part_bytes);
  int s;
  dim3 grid(pl.p.npairs, pl.splits);
  hicu_launch(tc_tap_table_kernel, (g.nsp + 127) / 128, 128, 0, st, g.nsp, g.nc, g.koff, toff);
  if ((s = hicu_check_launch("tc_tap_table_kernel"))) return s;
  hicu_allow_max_smem((const void*)gram_tc_kernel);
  hicu_launch(gram_tc_kernel, grid, kThreads, pl.smem_bytes, st, (const float*)x, pl.p, toff, part);
  if ((s = hicu_check_launch("gram_tc_kernel"))) return s;
  const int64_t total = (int64_t)g.n * g.n;
  const int rb = (int)hmin64((total + 255) / 256, 1184);
  hicu_launch(gram_tc_reduce_kernel, rb, 256, 0, st, g.n, g.nc, pl.p.T, pl.splits, pl.pt, pl.ntiles, part, G);
  return hicu_check_launch("gram_tc_reduce_kernel");
}
