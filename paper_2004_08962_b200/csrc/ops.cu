// Gradient-step kernels: forward convolution (u = H(y) Q~) with the fused
// objective reduction, the ELS convolution (w = H(g) Q~ never stored) with
// fused <w,u> / |w|^2 reductions, the gather-form k-space adjoint (col2im)
// with the data-consistency epilogue, and the device-side step update.
//
// Reference: hankel.py:255-322 (hankel_apply), :394-440
// (kspace_adjoint_scatter), :473-558 (objective_and_gradient,
// exact_line_search), solver.py:333-376 (the inlined inner loop).
//
// SIMT fp32 arithmetic with fp64 reductions; one thread per output row
// (conv) or per k-space sample (scatter).  Grid sizes are fixed functions of
// the geometry so partial counts, and hence results, are deterministic.
#include "common.cuh"

bool hicu_conv_tc_supported(const DevGeom& g, int p);
size_t hicu_conv_tc_bimage_bytes(const DevGeom& g, int p);
int hicu_conv_tc_build_bimages(const DevGeom& g, const float2* qt_all, int p, int G, uint8_t* img, size_t ib,
                               cudaStream_t st);
void hicu_conv_tc_bimage_hint(const void* img, int early);
void hicu_conv_tc_amax_hint(const float* in, float* out);
float* hicu_conv_tc_amax_slots(cudaStream_t st);
int hicu_conv_tc(const DevGeom& g, const float2* y, const float2* qt, float2* u, double* parts, int mode,
                 int nparts_total, cudaStream_t st);
int hicu_scatter_tc(const DevGeom& g, const float2* qt, const float2* u, const uint8_t* mask, const float2* y,
                    const float2* x0, int dc_mode, float lam, float2* gout, double* parts, int nparts_total,
                    cudaStream_t st);

namespace {

constexpr int kConvThreads = 256;
constexpr int kScatterThreads = 256;

// At least one block per SM: the tcgen05 kernels (conv_tc.cu) run one
// persistent CTA per SM and write one partial per CTA into the same buffer.
int conv_blocks(int64_t s) {
  int64_t b = (s + kConvThreads - 1) / kConvThreads;
  int64_t cap = (int64_t)hicu_sm_count() * 8;
  if (b > cap) b = cap;
  if (b < hicu_sm_count()) b = hicu_sm_count();
  return (int)b;
}

int scatter_blocks(int64_t N) {
  int64_t b = (N + kScatterThreads - 1) / kScatterThreads;
  int64_t cap = (int64_t)hicu_sm_count() * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

// MODE 0: u = H(y) qt, store u, part = sum |u|^2
// MODE 1: w = H(y) qt, part = (sum Re(conj(w) u), sum |w|^2)
template <int PMAX, bool CIRC, int MODE>
__global__ void __launch_bounds__(kConvThreads)
conv_kernel(DevGeom g, const float2* __restrict__ y, const float2* __restrict__ qt, int p,
            float2* __restrict__ u, double* __restrict__ parts) {
  hicu_pdl_entry();
  extern __shared__ unsigned char smem_raw[];
  float2* sq = reinterpret_cast<float2*>(smem_raw);                       // n * PMAX
  int64_t* skoff = reinterpret_cast<int64_t*>(sq + (size_t)g.n * PMAX);   // n
  int32_t* spos = reinterpret_cast<int32_t*>(skoff + g.n);                 // n * ndim (CIRC only)
  for (int t = threadIdx.x; t < g.n * PMAX; t += blockDim.x) {
    int k = t / PMAX, j = t % PMAX;
    sq[t] = (j < p) ? qt[(size_t)k * p + j] : cf(0.f, 0.f);
  }
  for (int t = threadIdx.x; t < g.n; t += blockDim.x) skoff[t] = g.koff[t];
  if (CIRC)
    for (int t = threadIdx.x; t < g.n * g.ndim; t += blockDim.x) spos[t] = g.pos[t];
  __syncthreads();

  double a0 = 0.0, a1 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.s;
       i += (int64_t)gridDim.x * blockDim.x) {
    int cc[HICU_MAX_NDIM];
    const int64_t base = row_base(g, i, cc);
    float2 acc[PMAX];
#pragma unroll
    for (int j = 0; j < PMAX; ++j) acc[j] = cf(0.f, 0.f);
    for (int k = 0; k < g.n; ++k) {
      int64_t addr = base + skoff[k];
      if (CIRC) addr += circ_part(g, cc, spos + (size_t)k * g.ndim);
      const float2 v = __ldg(y + addr);
      const float2* qk = sq + (size_t)k * PMAX;
#pragma unroll
      for (int j = 0; j < PMAX; ++j) cfma(acc[j], v, qk[j]);
    }
    if (MODE == 0) {
      float2* ui = u + (size_t)i * p;
#pragma unroll
      for (int j = 0; j < PMAX; ++j) {
        if (j < p) {
          ui[j] = acc[j];
          a0 += (double)acc[j].x * acc[j].x + (double)acc[j].y * acc[j].y;
        }
      }
    } else {
      const float2* ui = u + (size_t)i * p;
#pragma unroll
      for (int j = 0; j < PMAX; ++j) {
        if (j < p) {
          const float2 uv = ui[j];
          a0 += (double)acc[j].x * uv.x + (double)acc[j].y * uv.y;
          a1 += (double)acc[j].x * acc[j].x + (double)acc[j].y * acc[j].y;
        }
      }
    }
  }
  if (MODE == 0) {
    double v[1] = {a0};
    block_reduce_store<1>(v, parts + blockIdx.x);
  } else {
    double v[2] = {a0, a1};
    block_reduce_store<2>(v, parts + 2 * (size_t)blockIdx.x);
  }
}

// Gather-form adjoint: g[m] = sum_{kappa,k: m - kappa in region} conj(qt[kappa,k]) u[m-kappa, k]
// followed by data consistency; parts = (|g|^2, |res|^2, Re<Mg,res>, |Mg|^2).
template <int PMAX, bool CIRC>
__global__ void __launch_bounds__(kScatterThreads)
scatter_kernel(DevGeom g, const float2* __restrict__ qt, int p, const float2* __restrict__ u,
               const uint8_t* __restrict__ mask, const float2* __restrict__ y,
               const float2* __restrict__ x0, int dc_mode, float lam, float2* __restrict__ gout,
               double* __restrict__ parts) {
  hicu_pdl_entry();
  extern __shared__ unsigned char smem_raw[];
  float2* sq = reinterpret_cast<float2*>(smem_raw);                        // n * PMAX (conj)
  int32_t* spos = reinterpret_cast<int32_t*>(sq + (size_t)g.n * PMAX);      // n * ndim
  int64_t* srow = reinterpret_cast<int64_t*>(spos + (((size_t)g.n * g.ndim + 1) & ~(size_t)1));  // n
  for (int t = threadIdx.x; t < g.n * PMAX; t += blockDim.x) {
    int k = t / PMAX, j = t % PMAX;
    float2 q = (j < p) ? qt[(size_t)k * p + j] : cf(0.f, 0.f);
    sq[t] = cf(q.x, -q.y);
  }
  for (int t = threadIdx.x; t < g.n * g.ndim; t += blockDim.x) spos[t] = g.pos[t];
  __syncthreads();
  // row-index offset of each tap over the non-circular axes
  for (int t = threadIdx.x; t < g.n; t += blockDim.x) {
    int64_t o = 0;
    for (int d = 0, ci = 0; d < g.ndim; ++d) {
      if (ci < g.ncirc && g.circ_axes[ci] == d) { ++ci; continue; }
      o += (int64_t)spos[(size_t)t * g.ndim + d] * g.rstride[d];
    }
    srow[t] = o;
  }
  __syncthreads();

  double a_g = 0.0, a_res = 0.0, a_num = 0.0, a_den = 0.0;
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < g.N;
       m += (int64_t)gridDim.x * blockDim.x) {
    int64_t mc[HICU_MAX_NDIM];
    int64_t rem = m;
    for (int d = g.ndim - 1; d >= 0; --d) {
      mc[d] = rem % g.dims[d];
      rem /= g.dims[d];
    }
    // row index of (m - kappa) excluding the tap offset, over non-circular axes
    int64_t rbase = 0;
    for (int d = 0, ci = 0; d < g.ndim; ++d) {
      if (ci < g.ncirc && g.circ_axes[ci] == d) { ++ci; continue; }
      rbase += (mc[d] - g.roff[d]) * g.rstride[d];
    }
    float2 acc = cf(0.f, 0.f);
    for (int k = 0; k < g.n; ++k) {
      const int32_t* pk = spos + (size_t)k * g.ndim;
      bool ok = true;
      int64_t ci_row = 0;
      for (int d = 0, ci = 0; d < g.ndim; ++d) {
        if (ci < g.ncirc && g.circ_axes[ci] == d) {
          int64_t r = mc[d] - pk[d];
          if (r < 0) r += g.dims[d];
          ci_row += r * g.rstride[d];
          ++ci;
        } else {
          int64_t r = mc[d] - g.roff[d] - pk[d];
          ok = ok && (r >= 0) && (r < g.rext[d]);
        }
      }
      if (!ok) continue;
      const int64_t row = rbase - srow[k] + ci_row;
      const float2* ur = u + (size_t)row * p;
      const float2* qk = sq + (size_t)k * PMAX;
#pragma unroll
      for (int j = 0; j < PMAX; ++j)
        if (j < p) cfma(acc, qk[j], ur[j]);
    }
    const bool on = (dc_mode != 2) && mask[m] == 1;
    if (dc_mode == 0) {
      if (on) acc = cf(0.f, 0.f);
    } else if (dc_mode == 1) {
      float2 res = on ? (y[m] - x0[m]) : cf(0.f, 0.f);
      a_res += (double)res.x * res.x + (double)res.y * res.y;
      acc = acc + lam * res;
      if (on) {
        a_num += (double)acc.x * res.x + (double)acc.y * res.y;
        a_den += (double)acc.x * acc.x + (double)acc.y * acc.y;
      }
    }
    a_g += (double)acc.x * acc.x + (double)acc.y * acc.y;
    gout[m] = acc;
  }
  double v[4] = {a_g, a_res, a_num, a_den};
  block_reduce_store<4>(v, parts + 4 * (size_t)blockIdx.x);
}

// Seven warps reduce the seven per-step sums in parallel, every partial
// loaded before any add (one L2 round trip instead of a chain); the
// summation order (lane j sums j, j+32, ... then a fixed xor tree) is that of
// warp_sum_parts, so the results are bit-identical to the serial form.
constexpr int kUpdMaxPer = 32;  // partials per lane (n <= 1024)
__device__ __forceinline__ double warp_sum_batched(const double* __restrict__ parts, int np, int stride, int off) {
  const int lane = threadIdx.x & 31;
  double v[kUpdMaxPer];
#pragma unroll
  for (int k = 0; k < kUpdMaxPer; ++k) {
    const int j = lane + 32 * k;
    v[k] = j < np ? __ldg(parts + (size_t)j * stride + off) : 0.0;
  }
  double t = 0.0;
#pragma unroll
  for (int k = 0; k < kUpdMaxPer; ++k)
    if (lane + 32 * k < np) t += v[k];
  for (int j = lane + 32 * kUpdMaxPer; j < np; j += 32) t += parts[(size_t)j * stride + off];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// this CTA's max |y component| into amax_out[blockIdx.x] (the next
// convolution's operand scale); CTA 0 zero-fills the slot past the grid
__device__ __forceinline__ void update_amax_store(float mx, float* __restrict__ amax_out) {
  if (!amax_out) return;
  __shared__ float wm[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmaxf(t, wm[w]);
    amax_out[blockIdx.x] = t;
  }
  if (blockIdx.x == 0)
    for (int i = (int)gridDim.x + threadIdx.x; i < 512; i += blockDim.x) amax_out[i] = 0.f;
}

__global__ void __launch_bounds__(256)
update_kernel(int64_t N, float2* __restrict__ y, const float2* __restrict__ gdir,
              const double* __restrict__ obj_parts, int n_obj,
              const double* __restrict__ dc_parts, int n_dc,
              const double* __restrict__ els_parts, int n_els, int dc_mode, double lam,
              double* __restrict__ rec, bool vec, float* __restrict__ amax_out) {
  hicu_pdl_entry();
  __shared__ double s_eta;
  __shared__ int s_skip;
  __shared__ double sums[7];
  const int warp = threadIdx.x >> 5;
  if (warp < 7) {
    double t;
    switch (warp) {
      case 0: t = warp_sum_batched(obj_parts, n_obj, 1, 0); break;
      case 1: t = warp_sum_batched(dc_parts, n_dc, 4, 0); break;
      case 2: t = warp_sum_batched(dc_parts, n_dc, 4, 1); break;
      case 3: t = warp_sum_batched(dc_parts, n_dc, 4, 2); break;
      case 4: t = warp_sum_batched(dc_parts, n_dc, 4, 3); break;
      case 5: t = warp_sum_batched(els_parts, n_els, 2, 0); break;
      default: t = warp_sum_batched(els_parts, n_els, 2, 1); break;
    }
    if ((threadIdx.x & 31) == 0) sums[warp] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double obj_c = sums[0], gn2 = sums[1], res2 = sums[2], snum = sums[3], sden = sums[4];
    double obj = obj_c, num = sums[5], den = sums[6];
    if (dc_mode == 1) {
      obj += lam * res2;
      num += lam * snum;
      den += lam * sden;
    }
    // solver.py:347: the ELS convolution only runs when any(g); H(0) == 0
    // exactly, so num = den = 0 falls out when g vanishes.
    const bool degenerate = !(den > 0.0);
    const double eta = degenerate ? 0.0 : num / den;
    s_eta = eta;
    s_skip = degenerate ? 1 : 0;
    if (blockIdx.x == 0) {
      rec[HICU_REC_OBJ] = obj;
      rec[HICU_REC_NUM] = num;
      rec[HICU_REC_DEN] = den;
      rec[HICU_REC_ETA] = eta;
      rec[HICU_REC_OBJ_AFTER] = degenerate ? obj : obj - num * num / den;
      rec[HICU_REC_GNORM2] = gn2;
      rec[HICU_REC_DEGENERATE] = degenerate ? 1.0 : 0.0;
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      rec[7] = (double)tt;
    }
  }
  __syncthreads();
  if (s_skip && !amax_out) return;
  const float eta = s_skip ? 0.f : (float)s_eta;  // (a skipped step still reports max |y|)
  float mx = 0.f;
  if (!vec) {  // operands not 16-byte aligned
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < N; m += (int64_t)gridDim.x * blockDim.x) {
      const float2 gv = gdir[m];
      float2 yv = y[m];
      yv.x = fmaf(-eta, gv.x, yv.x);
      yv.y = fmaf(-eta, gv.y, yv.y);
      y[m] = yv;
      mx = fmaxf(mx, fmaxf(fabsf(yv.x), fabsf(yv.y)));
    }
    update_amax_store(mx, amax_out);
    return;
  }
  // two complex elements per thread per pass (16-byte accesses)
  const int64_t N2 = N >> 1;
  float4* y4 = reinterpret_cast<float4*>(y);
  const float4* g4 = reinterpret_cast<const float4*>(gdir);
  // four 16-byte pairs in flight per thread (memory-level parallelism)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t m0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m0 < N2; m0 += 4 * stride) {
    float4 gv[4], yv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t m = m0 + u * stride;
      if (m < N2) {
        gv[u] = g4[m];
        yv[u] = y4[m];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t m = m0 + u * stride;
      if (m < N2) {
        yv[u].x = fmaf(-eta, gv[u].x, yv[u].x);
        yv[u].y = fmaf(-eta, gv[u].y, yv[u].y);
        yv[u].z = fmaf(-eta, gv[u].z, yv[u].z);
        yv[u].w = fmaf(-eta, gv[u].w, yv[u].w);
        y4[m] = yv[u];
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(yv[u].x), fabsf(yv[u].y)), fmaxf(fabsf(yv[u].z), fabsf(yv[u].w))));
      }
    }
  }
  if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const float2 gv = gdir[N - 1];
    float2 yv = y[N - 1];
    yv.x = fmaf(-eta, gv.x, yv.x);
    yv.y = fmaf(-eta, gv.y, yv.y);
    y[N - 1] = yv;
    mx = fmaxf(mx, fmaxf(fabsf(yv.x), fabsf(yv.y)));
  }
  update_amax_store(mx, amax_out);
}

__global__ void ser_kernel(int64_t N, const float2* __restrict__ ref, const float2* __restrict__ y,
                           double* __restrict__ parts) {
  hicu_pdl_entry();
  double e = 0.0, r = 0.0;
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < N;
       m += (int64_t)gridDim.x * blockDim.x) {
    const float2 a = ref[m], b = y[m];
    const double dx = (double)a.x - b.x, dy = (double)a.y - b.y;
    e += dx * dx + dy * dy;
    r += (double)a.x * a.x + (double)a.y * a.y;
  }
  double v[2] = {e, r};
  block_reduce_store<2>(v, parts + 2 * (size_t)blockIdx.x);
}


// ---------------------------------------------------------------------------
// Coil-structured fast paths (DevGeom.nc > 0: kappa = sp*Nc + c, one coil row
// in the region).  Conv: one thread per region row, Nc coils loaded as
// float4 pairs per spatial tap.  Scatter: one thread per SPATIAL k-space
// location accumulating all Nc coils, so each valid spatial tap costs one
// u-row load reused Nc times (the generic kernel tests every (spatial, coil)
// tap pair per coil).
// ---------------------------------------------------------------------------
template <int PMAX, int NCMAX, bool CIRC, int MODE>
__global__ void __launch_bounds__(kConvThreads)
conv_coil_kernel(DevGeom g, const float2* __restrict__ y, const float2* __restrict__ qt, int p,
                 float2* __restrict__ u, double* __restrict__ parts) {
  hicu_pdl_entry();
  extern __shared__ unsigned char smem_raw[];
  const int nc = g.nc, nsp = g.nsp;
  float2* sq = reinterpret_cast<float2*>(smem_raw);                          // n * PMAX
  int64_t* skoff = reinterpret_cast<int64_t*>(sq + (size_t)g.n * PMAX);      // nsp
  int32_t* spos = reinterpret_cast<int32_t*>(skoff + nsp);                    // nsp * ndim
  for (int t = threadIdx.x; t < g.n * PMAX; t += blockDim.x) {
    const int k = t / PMAX, j = t % PMAX;
    sq[t] = (j < p) ? qt[(size_t)k * p + j] : cf(0.f, 0.f);
  }
  for (int t = threadIdx.x; t < nsp; t += blockDim.x) skoff[t] = g.koff[(size_t)t * nc];
  if (CIRC)
    for (int t = threadIdx.x; t < nsp * g.ndim; t += blockDim.x)
      spos[t] = g.pos[(size_t)(t / g.ndim) * nc * g.ndim + t % g.ndim];
  __syncthreads();
  const bool vec2 = (nc % 2) == 0;
  double a0 = 0.0, a1 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.s; i += (int64_t)gridDim.x * blockDim.x) {
    int cc[HICU_MAX_NDIM];
    const int64_t base = row_base(g, i, cc);
    float2 acc[PMAX];
#pragma unroll
    for (int j = 0; j < PMAX; ++j) acc[j] = cf(0.f, 0.f);
    for (int sp = 0; sp < nsp; ++sp) {
      int64_t addr = base + skoff[sp];
      if (CIRC) addr += circ_part(g, cc, spos + (size_t)sp * g.ndim);
      const float2* qsp = sq + (size_t)sp * nc * PMAX;
      if (vec2) {
        const float4* yp = reinterpret_cast<const float4*>(y + addr);
#pragma unroll 4
        for (int c2 = 0; c2 < nc / 2; ++c2) {
          const float4 v = __ldg(yp + c2);
          const float2 v0 = cf(v.x, v.y), v1 = cf(v.z, v.w);
          const float2* q0 = qsp + (size_t)(2 * c2) * PMAX;
#pragma unroll
          for (int j = 0; j < PMAX; ++j) {
            cfma(acc[j], v0, q0[j]);
            cfma(acc[j], v1, q0[PMAX + j]);
          }
        }
      } else {
        for (int c = 0; c < nc; ++c) {
          const float2 v = __ldg(y + addr + c);
          const float2* q0 = qsp + (size_t)c * PMAX;
#pragma unroll
          for (int j = 0; j < PMAX; ++j) cfma(acc[j], v, q0[j]);
        }
      }
    }
    float2* ui = u + (size_t)i * p;
#pragma unroll
    for (int j = 0; j < PMAX; ++j) {
      if (j < p) {
        if (MODE == 0) {
          ui[j] = acc[j];
          a0 += (double)acc[j].x * acc[j].x + (double)acc[j].y * acc[j].y;
        } else {
          const float2 uv = ui[j];
          a0 += (double)acc[j].x * uv.x + (double)acc[j].y * uv.y;
          a1 += (double)acc[j].x * acc[j].x + (double)acc[j].y * acc[j].y;
        }
      }
    }
  }
  if (MODE == 0) {
    double v[1] = {a0};
    block_reduce_store<1>(v, parts + blockIdx.x);
  } else {
    double v[2] = {a0, a1};
    block_reduce_store<2>(v, parts + 2 * (size_t)blockIdx.x);
  }
}

template <int PMAX, int NCMAX, bool CIRC>
__global__ void __launch_bounds__(128)
scatter_coil_kernel(DevGeom g, const float2* __restrict__ qt, int p, const float2* __restrict__ u,
                    const uint8_t* __restrict__ mask, const float2* __restrict__ y,
                    const float2* __restrict__ x0, int dc_mode, float lam, float2* __restrict__ gout,
                    double* __restrict__ parts) {
  hicu_pdl_entry();
  extern __shared__ unsigned char smem_raw[];
  const int nc = g.nc, nsp = g.nsp, L = g.ndim - 1;
  float2* sq = reinterpret_cast<float2*>(smem_raw);                           // n * PMAX, conj
  int64_t* srow = reinterpret_cast<int64_t*>(sq + (size_t)g.n * PMAX);        // nsp
  int32_t* spos = reinterpret_cast<int32_t*>(srow + nsp);                      // nsp * L
  for (int t = threadIdx.x; t < g.n * PMAX; t += blockDim.x) {
    const int k = t / PMAX, j = t % PMAX;
    const float2 q = (j < p) ? qt[(size_t)k * p + j] : cf(0.f, 0.f);
    sq[t] = cf(q.x, -q.y);
  }
  for (int t = threadIdx.x; t < nsp * L; t += blockDim.x)
    spos[t] = g.pos[(size_t)(t / L) * nc * g.ndim + t % L];
  __syncthreads();
  for (int t = threadIdx.x; t < nsp; t += blockDim.x) {
    int64_t o = 0;
    for (int d = 0, ci = 0; d < L; ++d) {
      if (ci < g.ncirc && g.circ_axes[ci] == d) { ++ci; continue; }
      o += (int64_t)spos[(size_t)t * L + d] * g.rstride[d];
    }
    srow[t] = o;
  }
  __syncthreads();
  const int64_t Ns = g.N / nc;
  double a_g = 0.0, a_res = 0.0, a_num = 0.0, a_den = 0.0;
  for (int64_t ms = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ms < Ns; ms += (int64_t)gridDim.x * blockDim.x) {
    int64_t mc[HICU_MAX_NDIM];
    int64_t rem = ms;
    for (int d = L - 1; d >= 0; --d) {
      mc[d] = rem % g.dims[d];
      rem /= g.dims[d];
    }
    int64_t rbase = 0;
    for (int d = 0, ci = 0; d < L; ++d) {
      if (ci < g.ncirc && g.circ_axes[ci] == d) { ++ci; continue; }
      rbase += (mc[d] - g.roff[d]) * g.rstride[d];
    }
    float2 acc[NCMAX];
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) acc[c] = cf(0.f, 0.f);
    for (int sp = 0; sp < nsp; ++sp) {
      const int32_t* pk = spos + (size_t)sp * L;
      bool ok = true;
      int64_t crow = 0;
      for (int d = 0, ci = 0; d < L; ++d) {
        if (CIRC && ci < g.ncirc && g.circ_axes[ci] == d) {
          int64_t r = mc[d] - pk[d];
          if (r < 0) r += g.dims[d];
          crow += r * g.rstride[d];
          ++ci;
        } else {
          const int64_t r = mc[d] - g.roff[d] - pk[d];
          ok = ok && (r >= 0) && (r < g.rext[d]);
        }
      }
      if (!ok) continue;
      const float2* ur = u + (size_t)(rbase - srow[sp] + crow) * p;
      float2 uk[PMAX];
#pragma unroll
      for (int j = 0; j < PMAX; ++j) uk[j] = (j < p) ? __ldg(ur + j) : cf(0.f, 0.f);
      const float2* qsp = sq + (size_t)sp * nc * PMAX;
#pragma unroll
      for (int c = 0; c < NCMAX; ++c) {
        if (c < nc) {
#pragma unroll
          for (int j = 0; j < PMAX; ++j) cfma(acc[c], qsp[c * PMAX + j], uk[j]);
        }
      }
    }
    const int64_t m0 = ms * nc;
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) {
      if (c >= nc) break;
      const int64_t m = m0 + c;
      float2 a = acc[c];
      const bool on = (dc_mode != 2) && mask[m] == 1;
      if (dc_mode == 0) {
        if (on) a = cf(0.f, 0.f);
      } else if (dc_mode == 1) {
        const float2 res = on ? (y[m] - x0[m]) : cf(0.f, 0.f);
        a_res += (double)res.x * res.x + (double)res.y * res.y;
        a = a + lam * res;
        if (on) {
          a_num += (double)a.x * res.x + (double)a.y * res.y;
          a_den += (double)a.x * a.x + (double)a.y * a.y;
        }
      }
      a_g += (double)a.x * a.x + (double)a.y * a.y;
      gout[m] = a;
    }
  }
  double v[4] = {a_g, a_res, a_num, a_den};
  block_reduce_store<4>(v, parts + 4 * (size_t)blockIdx.x);
}

template <int PMAX, int NCMAX>
int launch_conv_coil(const DevGeom& g, const float2* y, const float2* qt, int p, float2* u, double* parts, int mode,
                     cudaStream_t st) {
  const int blocks = conv_blocks(g.s);
  const bool circ = g.ncirc > 0;
  const size_t smem = (size_t)g.n * PMAX * sizeof(float2) + (size_t)g.nsp * sizeof(int64_t) +
                      (circ ? (size_t)g.nsp * g.ndim * sizeof(int32_t) : 0);
  if (smem > 200 * 1024) return hicu_set_error(HICU_ERR_SIZE, "conv: n*p too large for shared memory");
#define HICU_LAUNCH_CONVC(C, M)                                                 \
  do {                                                                          \
    auto kfn = conv_coil_kernel<PMAX, NCMAX, C, M>;                             \
    hicu_allow_max_smem((const void*)kfn);                                      \
    hicu_launch(kfn, blocks, kConvThreads, smem, st, g, y, qt, p, u, parts);             \
  } while (0)
  if (circ) {
    if (mode == 0) HICU_LAUNCH_CONVC(true, 0); else HICU_LAUNCH_CONVC(true, 1);
  } else {
    if (mode == 0) HICU_LAUNCH_CONVC(false, 0); else HICU_LAUNCH_CONVC(false, 1);
  }
#undef HICU_LAUNCH_CONVC
  return hicu_check_launch("conv_coil_kernel");
}

int scatter_coil_blocks(int64_t Ns) {
  int64_t b = (Ns + 127) / 128;
  int64_t cap = (int64_t)hicu_sm_count() * 16;
  if (b > cap) b = cap;
  if (b < hicu_sm_count()) b = hicu_sm_count();
  return (int)b;
}

template <int PMAX, int NCMAX>
int launch_scatter_coil(const DevGeom& g, const float2* qt, int p, const float2* u, const uint8_t* mask,
                        const float2* y, const float2* x0, int dc_mode, float lam, float2* gout, double* parts,
                        cudaStream_t st) {
  const int blocks = scatter_coil_blocks(g.N / g.nc);
  const size_t smem = (size_t)g.n * PMAX * sizeof(float2) + (size_t)g.nsp * sizeof(int64_t) +
                      (size_t)g.nsp * (g.ndim - 1) * sizeof(int32_t);
  if (smem > 200 * 1024) return hicu_set_error(HICU_ERR_SIZE, "scatter: n*p too large for shared memory");
  if (g.ncirc > 0) {
    auto kfn = scatter_coil_kernel<PMAX, NCMAX, true>;
    hicu_allow_max_smem((const void*)kfn);
    hicu_launch(kfn, blocks, 128, smem, st, g, qt, p, u, mask, y, x0, dc_mode, lam, gout, parts);
  } else {
    auto kfn = scatter_coil_kernel<PMAX, NCMAX, false>;
    hicu_allow_max_smem((const void*)kfn);
    hicu_launch(kfn, blocks, 128, smem, st, g, qt, p, u, mask, y, x0, dc_mode, lam, gout, parts);
  }
  return hicu_check_launch("scatter_coil_kernel");
}

template <int PMAX>
int conv_coil_dispatch(const DevGeom& g, const float2* y, const float2* qt, int p, float2* u, double* parts, int mode,
                       cudaStream_t st) {
  if (g.nc <= 8) return launch_conv_coil<PMAX, 8>(g, y, qt, p, u, parts, mode, st);
  if (g.nc <= 10) return launch_conv_coil<PMAX, 10>(g, y, qt, p, u, parts, mode, st);  // C3: 16 -> 10 coils
  if (g.nc <= 16) return launch_conv_coil<PMAX, 16>(g, y, qt, p, u, parts, mode, st);
  return launch_conv_coil<PMAX, 32>(g, y, qt, p, u, parts, mode, st);
}

template <int PMAX>
int scatter_coil_dispatch(const DevGeom& g, const float2* qt, int p, const float2* u, const uint8_t* mask,
                          const float2* y, const float2* x0, int dc_mode, float lam, float2* gout, double* parts,
                          cudaStream_t st) {
  if (g.nc <= 8) return launch_scatter_coil<PMAX, 8>(g, qt, p, u, mask, y, x0, dc_mode, lam, gout, parts, st);
  if (g.nc <= 10) return launch_scatter_coil<PMAX, 10>(g, qt, p, u, mask, y, x0, dc_mode, lam, gout, parts, st);
  if (g.nc <= 16) return launch_scatter_coil<PMAX, 16>(g, qt, p, u, mask, y, x0, dc_mode, lam, gout, parts, st);
  return launch_scatter_coil<PMAX, 32>(g, qt, p, u, mask, y, x0, dc_mode, lam, gout, parts, st);
}

template <int PMAX>
int launch_conv(const DevGeom& g, const float2* y, const float2* qt, int p, float2* u, double* parts,
                int mode, cudaStream_t st) {
  const int blocks = conv_blocks(g.s);
  const bool circ = g.ncirc > 0;
  size_t smem = (size_t)g.n * PMAX * sizeof(float2) + (size_t)g.n * sizeof(int64_t) +
                (circ ? (size_t)g.n * g.ndim * sizeof(int32_t) : 0);
  if (smem > 200 * 1024) return hicu_set_error(HICU_ERR_SIZE, "conv: n*p too large for shared memory");
#define HICU_LAUNCH_CONV(C, M)                                                                    \
  do {                                                                                            \
    auto kfn = conv_kernel<PMAX, C, M>;                                                           \
    hicu_allow_max_smem((const void*)kfn);            \
    hicu_launch(kfn, blocks, kConvThreads, smem, st, g, y, qt, p, u, parts);                               \
  } while (0)
  if (circ) {
    if (mode == 0) HICU_LAUNCH_CONV(true, 0); else HICU_LAUNCH_CONV(true, 1);
  } else {
    if (mode == 0) HICU_LAUNCH_CONV(false, 0); else HICU_LAUNCH_CONV(false, 1);
  }
#undef HICU_LAUNCH_CONV
  return hicu_check_launch("conv_kernel");
}

int conv_dispatch(const hicu_geom* hg, const void* y, const void* qt, int p, const void* u_in, void* u_out,
                  double* parts, int mode, void* stream) {
  if (!hg || !y || !qt || !parts || p < 1) return hicu_set_error(HICU_ERR_PARAMETER, "conv: bad arguments");
  if (p > 32) return hicu_set_error(HICU_ERR_PARAMETER, "conv: p > 32 not supported");
  DevGeom g;
  int st = hicu_make_devgeom(hg, &g);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  float2* u = mode == 0 ? (float2*)u_out : (float2*)u_in;
  if (!u) return hicu_set_error(HICU_ERR_PARAMETER, "conv: null u");
  if (!(hg->flags & HICU_GEOM_FORCE_SIMT_CONV) && hicu_conv_tc_supported(g, p))
    return hicu_conv_tc(g, (const float2*)y, (const float2*)qt, u, parts, mode, conv_blocks(g.s), s);
  if (g.nc > 0) {
    if (p <= 4) return conv_coil_dispatch<4>(g, (const float2*)y, (const float2*)qt, p, u, parts, mode, s);
    if (p <= 8) return conv_coil_dispatch<8>(g, (const float2*)y, (const float2*)qt, p, u, parts, mode, s);
    // exact fit for C3's p = 10 (the 16-wide instantiation spent 60 % more FMAs on zero columns)
    if (p <= 10) return conv_coil_dispatch<10>(g, (const float2*)y, (const float2*)qt, p, u, parts, mode, s);
    if (p <= 16) return conv_coil_dispatch<16>(g, (const float2*)y, (const float2*)qt, p, u, parts, mode, s);
    // the paper's full-stage compression p = 4 Nc: 32 columns for 8 coils
    return conv_coil_dispatch<32>(g, (const float2*)y, (const float2*)qt, p, u, parts, mode, s);
  }
  if (p <= 4) return launch_conv<4>(g, (const float2*)y, (const float2*)qt, p, u, parts, mode, s);
  if (p <= 8) return launch_conv<8>(g, (const float2*)y, (const float2*)qt, p, u, parts, mode, s);
  if (p <= 10) return launch_conv<10>(g, (const float2*)y, (const float2*)qt, p, u, parts, mode, s);
  if (p <= 16) return launch_conv<16>(g, (const float2*)y, (const float2*)qt, p, u, parts, mode, s);
  return launch_conv<32>(g, (const float2*)y, (const float2*)qt, p, u, parts, mode, s);
}

template <int PMAX>
int launch_scatter(const DevGeom& g, const float2* qt, int p, const float2* u, const uint8_t* mask,
                   const float2* y, const float2* x0, int dc_mode, float lam, float2* gout, double* parts,
                   cudaStream_t st) {
  const int blocks = scatter_blocks(g.N);
  size_t smem = (size_t)g.n * PMAX * sizeof(float2) +
                (((size_t)g.n * g.ndim + 1) & ~(size_t)1) * sizeof(int32_t) + (size_t)g.n * sizeof(int64_t);
  if (smem > 200 * 1024) return hicu_set_error(HICU_ERR_SIZE, "scatter: n*p too large for shared memory");
  if (g.ncirc > 0) {
    auto kfn = scatter_kernel<PMAX, true>;
    hicu_allow_max_smem((const void*)kfn);
    hicu_launch(kfn, blocks, kScatterThreads, smem, st, g, qt, p, u, mask, y, x0, dc_mode, lam, gout, parts);
  } else {
    auto kfn = scatter_kernel<PMAX, false>;
    hicu_allow_max_smem((const void*)kfn);
    hicu_launch(kfn, blocks, kScatterThreads, smem, st, g, qt, p, u, mask, y, x0, dc_mode, lam, gout, parts);
  }
  return hicu_check_launch("scatter_kernel");
}

}  // namespace

extern "C" int hicu_conv_uses_tensor_cores(const hicu_geom* hg, int p) {
  DevGeom g;
  if (!hg || hicu_make_devgeom(hg, &g)) return 0;
  return !(hg->flags & HICU_GEOM_FORCE_SIMT_CONV) && hicu_conv_tc_supported(g, p) ? 1 : 0;
}

extern "C" int hicu_conv_nparts(const hicu_geom* hg) {
  DevGeom g;
  if (hicu_make_devgeom(hg, &g)) return -1;
  return conv_blocks(g.s);
}

extern "C" int hicu_scatter_nparts(const hicu_geom* hg) {
  DevGeom g;
  if (hicu_make_devgeom(hg, &g)) return -1;
  return g.nc > 0 ? scatter_coil_blocks(g.N / g.nc) : scatter_blocks(g.N);
}

extern "C" int hicu_conv_fwd(const hicu_geom* g, const void* y, const void* qt, int p, void* u,
                             double* obj_parts, void* stream) {
  return conv_dispatch(g, y, qt, p, nullptr, u, obj_parts, 0, stream);
}

extern "C" int hicu_conv_els(const hicu_geom* g, const void* gdir, const void* qt, int p, const void* u,
                             double* numden_parts, void* stream) {
  return conv_dispatch(g, gdir, qt, p, u, nullptr, numden_parts, 1, stream);
}

extern "C" int hicu_scatter_dc(const hicu_geom* hg, const void* qt, int p, const void* u, const uint8_t* mask,
                               const void* y, const void* x0, int dc_mode, double lam, void* gout,
                               double* dc_parts, void* stream) {
  if (!hg || !qt || !u || (!mask && dc_mode != 2) || !gout || !dc_parts || p < 1)
    return hicu_set_error(HICU_ERR_PARAMETER, "scatter: bad arguments");
  if (p > 32) return hicu_set_error(HICU_ERR_PARAMETER, "scatter: p > 32 not supported");
  if (dc_mode < 0 || dc_mode > 2) return hicu_set_error(HICU_ERR_SHAPE, "scatter: unknown dc mode");
  if (dc_mode == 1 && (!y || !x0)) return hicu_set_error(HICU_ERR_SHAPE, "soft data consistency requires x0");
  DevGeom g;
  int st = hicu_make_devgeom(hg, &g);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  auto q = (const float2*)qt;
  auto uu = (const float2*)u;
  if (g.nc > 0 && !(hg->flags & HICU_GEOM_FORCE_SIMT_CONV) && hicu_conv_tc_supported(g, p))
    return hicu_scatter_tc(g, q, uu, mask, (const float2*)y, (const float2*)x0, dc_mode, (float)lam, (float2*)gout,
                           dc_parts, scatter_coil_blocks(g.N / g.nc), s);
  if (g.nc > 0) {
    auto yy = (const float2*)y;
    auto xx = (const float2*)x0;
    if (p <= 4) return scatter_coil_dispatch<4>(g, q, p, uu, mask, yy, xx, dc_mode, (float)lam, (float2*)gout, dc_parts, s);
    if (p <= 8) return scatter_coil_dispatch<8>(g, q, p, uu, mask, yy, xx, dc_mode, (float)lam, (float2*)gout, dc_parts, s);
    if (p <= 10) return scatter_coil_dispatch<10>(g, q, p, uu, mask, yy, xx, dc_mode, (float)lam, (float2*)gout, dc_parts, s);
    if (p <= 16) return scatter_coil_dispatch<16>(g, q, p, uu, mask, yy, xx, dc_mode, (float)lam, (float2*)gout, dc_parts, s);
    return scatter_coil_dispatch<32>(g, q, p, uu, mask, yy, xx, dc_mode, (float)lam, (float2*)gout, dc_parts, s);
  }
  if (p <= 4)
    return launch_scatter<4>(g, q, p, uu, mask, (const float2*)y, (const float2*)x0, dc_mode, (float)lam,
                             (float2*)gout, dc_parts, s);
  if (p <= 8)
    return launch_scatter<8>(g, q, p, uu, mask, (const float2*)y, (const float2*)x0, dc_mode, (float)lam,
                             (float2*)gout, dc_parts, s);
  if (p <= 16)
    return launch_scatter<16>(g, q, p, uu, mask, (const float2*)y, (const float2*)x0, dc_mode, (float)lam,
                              (float2*)gout, dc_parts, s);
  return launch_scatter<32>(g, q, p, uu, mask, (const float2*)y, (const float2*)x0, dc_mode, (float)lam,
                            (float2*)gout, dc_parts, s);
}

int hicu_step_update_amax(int64_t N, void* y, const void* gdir, const double* obj_parts, int n_obj,
                          const double* dc_parts, int n_dc, const double* els_parts, int n_els, int dc_mode,
                          double lam, double* rec, float* amax_out, void* stream);

extern "C" int hicu_step_update(int64_t N, void* y, const void* gdir, const double* obj_parts, int n_obj,
                                const double* dc_parts, int n_dc, const double* els_parts, int n_els,
                                int dc_mode, double lam, double* rec, void* stream) {
  return hicu_step_update_amax(N, y, gdir, obj_parts, n_obj, dc_parts, n_dc, els_parts, n_els, dc_mode, lam, rec,
                               nullptr, stream);
}

// hicu_step_update that also writes the per-CTA max |y| partials (<= 512)
// the next convolution takes its operand scale from (engine.cu)
int hicu_step_update_amax(int64_t N, void* y, const void* gdir, const double* obj_parts, int n_obj,
                          const double* dc_parts, int n_dc, const double* els_parts, int n_els, int dc_mode,
                          double lam, double* rec, float* amax_out, void* stream) {
  if (!y || !gdir || !obj_parts || !dc_parts || !els_parts || !rec || N < 1)
    return hicu_set_error(HICU_ERR_PARAMETER, "update: bad arguments");
  int64_t b = (N / 2 + 255) / 256;
  int64_t cap = (int64_t)hicu_sm_count() * 2;  // fewer blocks: each re-reads the partials
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  const bool vec = (((uintptr_t)y | (uintptr_t)gdir) & 15) == 0;
  hicu_launch(update_kernel, (int)b, 256, 0, (cudaStream_t)stream, N, (float2*)y, (const float2*)gdir, obj_parts, n_obj,
                                                           dc_parts, n_dc, els_parts, n_els, dc_mode, lam, rec, vec,
                                                           amax_out);
  return hicu_check_launch("update_kernel");
}

__global__ void timestamp_kernel(double* out) {
  hicu_pdl_entry();
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = (double)t;
}

int ser_blocks(int64_t N) {
  int64_t b = (N + 255) / 256;
  int64_t cap = (int64_t)hicu_sm_count() * 2;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

extern "C" int hicu_timestamp(double* out, void* stream) {
  if (!out) return hicu_set_error(HICU_ERR_PARAMETER, "timestamp: null");
  hicu_launch(timestamp_kernel, 1, 1, 0, (cudaStream_t)stream, out);
  return hicu_check_launch("timestamp_kernel");
}

extern "C" int hicu_ser_nparts(int64_t N) { return ser_blocks(N); }

extern "C" int hicu_ser_parts(int64_t N, const void* ref, const void* y, double* parts, int* nparts_out,
                              void* stream) {
  if (!ref || !y || !parts || N < 1) return hicu_set_error(HICU_ERR_PARAMETER, "ser: bad arguments");
  const int b = ser_blocks(N);
  if (nparts_out) *nparts_out = b;
  hicu_launch(ser_kernel, b, 256, 0, (cudaStream_t)stream, N, (const float2*)ref, (const float2*)y, parts);
  return hicu_check_launch("ser_kernel");
}

// ---------------------------------------------------------------------------
// Kernel-slot adjoint out[kappa, j] = sum_i conj(X[i+kappa]) u[i, j]
// (hankel_adjoint_apply, hankel.py:325-391).  Not on the solver's hot path
// (the Gram replaces it); provided for the operator-level API.
// ---------------------------------------------------------------------------
namespace {
template <bool CIRC>
__global__ void conv_adj_kernel(DevGeom g, const float2* __restrict__ x, const float2* __restrict__ u, int k,
                                double2* __restrict__ out) {
  hicu_pdl_entry();
  const int kap = blockIdx.x;
  const int j = blockIdx.y;
  const int32_t* pk = g.pos + (size_t)kap * g.ndim;
  double ax = 0.0, ay = 0.0;
  for (int64_t i = threadIdx.x; i < g.s; i += blockDim.x) {
    int cc[HICU_MAX_NDIM];
    int64_t addr = row_base(g, i, cc) + g.koff[kap];
    if (CIRC) addr += circ_part(g, cc, pk);
    const float2 xv = x[addr], uv = u[(size_t)i * k + j];
    ax += (double)xv.x * uv.x + (double)xv.y * uv.y;
    ay += (double)xv.x * uv.y - (double)xv.y * uv.x;
  }
  double v[2] = {ax, ay};
  __shared__ double res[2];
  block_reduce_store<2>(v, res);
  __syncthreads();
  if (threadIdx.x == 0) out[(size_t)kap * k + j] = cd(res[0], res[1]);
}
}  // namespace

extern "C" int hicu_conv_adj(const hicu_geom* hg, const void* x, const void* u, int k, void* out, void* stream) {
  if (!hg || !x || !u || !out || k < 1) return hicu_set_error(HICU_ERR_PARAMETER, "conv_adj: bad arguments");
  DevGeom g;
  int st = hicu_make_devgeom(hg, &g);
  if (st) return st;
  dim3 grid(g.n, k);
  if (g.ncirc > 0)
    hicu_launch(conv_adj_kernel<true>, grid, 256, 0, (cudaStream_t)stream, g, (const float2*)x, (const float2*)u, k,
                                                                  (double2*)out);
  else
    hicu_launch(conv_adj_kernel<false>, grid, 256, 0, (cudaStream_t)stream, g, (const float2*)x, (const float2*)u, k,
                                                                   (double2*)out);
  return hicu_check_launch("conv_adj_kernel");
}

// Soft-DC line-search terms for the operator-level API (hankel.py:546-550):
// parts[3b] = Re<Mg, res>, [3b+1] = |Mg|^2, [3b+2] = |res|^2, res = M(y - x0).
namespace {
__global__ void soft_terms_kernel(int64_t N, const float2* __restrict__ g, const float2* __restrict__ y,
                                  const float2* __restrict__ x0, const uint8_t* __restrict__ mask,
                                  double* __restrict__ parts) {
  hicu_pdl_entry();
  double a = 0.0, b = 0.0, c = 0.0;
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < N; m += (int64_t)gridDim.x * blockDim.x) {
    if (mask[m] != 1) continue;
    const float2 gv = g[m];
    const float2 res = y[m] - x0[m];
    a += (double)gv.x * res.x + (double)gv.y * res.y;
    b += (double)gv.x * gv.x + (double)gv.y * gv.y;
    c += (double)res.x * res.x + (double)res.y * res.y;
  }
  double v[3] = {a, b, c};
  block_reduce_store<3>(v, parts + 3 * (size_t)blockIdx.x);
}
}  // namespace

extern "C" int hicu_soft_terms(int64_t N, const void* g, const void* y, const void* x0, const uint8_t* mask,
                               double* parts, int* nparts_out, void* stream) {
  if (!g || !y || !x0 || !mask || !parts || N < 1) return hicu_set_error(HICU_ERR_PARAMETER, "soft_terms: bad args");
  const int b = ser_blocks(N);
  if (nparts_out) *nparts_out = b;
  hicu_launch(soft_terms_kernel, b, 256, 0, (cudaStream_t)stream, N, (const float2*)g, (const float2*)y, (const float2*)x0,
                                                         mask, parts);
  return hicu_check_launch("soft_terms_kernel");
}

// ---------------------------------------------------------------------------
// Split form of the step update for the halo-sharded path (one volume over
// several GPUs): the partial sums are reduced locally to 7 raw scalars, the
// caller all-reduces them across ranks, and every rank applies the same eta.
// sums7 = [obj_conv, ||g||^2, ||res||^2, Re<Mg,res>, ||Mg||^2, num_conv, den_conv]
// ---------------------------------------------------------------------------
namespace {
__global__ void step_reduce_kernel(const double* __restrict__ obj_parts, int n_obj, const double* __restrict__ dc_parts,
                                   int n_dc, const double* __restrict__ els_parts, int n_els,
                                   double* __restrict__ sums7) {
  hicu_pdl_entry();
  const double obj_c = warp_sum_parts(obj_parts, n_obj, 1, 0);
  const double gn2 = warp_sum_parts(dc_parts, n_dc, 4, 0);
  const double res2 = warp_sum_parts(dc_parts, n_dc, 4, 1);
  const double snum = warp_sum_parts(dc_parts, n_dc, 4, 2);
  const double sden = warp_sum_parts(dc_parts, n_dc, 4, 3);
  const double num_c = warp_sum_parts(els_parts, n_els, 2, 0);
  const double den_c = warp_sum_parts(els_parts, n_els, 2, 1);
  if (threadIdx.x == 0) {
    sums7[0] = obj_c;
    sums7[1] = gn2;
    sums7[2] = res2;
    sums7[3] = snum;
    sums7[4] = sden;
    sums7[5] = num_c;
    sums7[6] = den_c;
  }
}

__global__ void step_apply_kernel(int64_t N, float2* __restrict__ y, const float2* __restrict__ gdir,
                                  const double* __restrict__ sums7, int dc_mode, double lam, double* __restrict__ rec) {
  hicu_pdl_entry();
  double obj = sums7[0], num = sums7[5], den = sums7[6];
  if (dc_mode == 1) {
    obj += lam * sums7[2];
    num += lam * sums7[3];
    den += lam * sums7[4];
  }
  const bool degenerate = !(den > 0.0);
  const double eta = degenerate ? 0.0 : num / den;
  if (blockIdx.x == 0 && threadIdx.x == 0 && rec) {
    rec[HICU_REC_OBJ] = obj;
    rec[HICU_REC_NUM] = num;
    rec[HICU_REC_DEN] = den;
    rec[HICU_REC_ETA] = eta;
    rec[HICU_REC_OBJ_AFTER] = degenerate ? obj : obj - num * num / den;
    rec[HICU_REC_GNORM2] = sums7[1];
    rec[HICU_REC_DEGENERATE] = degenerate ? 1.0 : 0.0;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    rec[7] = (double)t;
  }
  if (degenerate) return;
  const float e = (float)eta;
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < N; m += (int64_t)gridDim.x * blockDim.x) {
    const float2 gv = gdir[m];
    float2 yv = y[m];
    yv.x = fmaf(-e, gv.x, yv.x);
    yv.y = fmaf(-e, gv.y, yv.y);
    y[m] = yv;
  }
}

// data consistency on a contiguous range of samples, with the partial sums
// (||g||^2, ||res||^2, Re<Mg,res>, ||Mg||^2) of scatter_kernel's epilogue
__global__ void dc_apply_kernel(int64_t n, float2* __restrict__ g, const uint8_t* __restrict__ mask,
                                const float2* __restrict__ y, const float2* __restrict__ x0, int dc_mode, float lam,
                                double* __restrict__ parts) {
  hicu_pdl_entry();
  double a_g = 0.0, a_res = 0.0, a_num = 0.0, a_den = 0.0;
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x) {
    float2 acc = g[m];
    const uint8_t mk = mask[m];
    const bool on = (mk & 1) != 0;
    const bool cnt = (mk & 2) == 0;  // bit 1: a halo copy of another rank's plane, not summed
    if (dc_mode == 0) {
      if (on) acc = cf(0.f, 0.f);
    } else {
      const float2 res = on ? (y[m] - x0[m]) : cf(0.f, 0.f);
      if (cnt) a_res += (double)res.x * res.x + (double)res.y * res.y;
      acc = acc + lam * res;
      if (on && cnt) {
        a_num += (double)acc.x * res.x + (double)acc.y * res.y;
        a_den += (double)acc.x * acc.x + (double)acc.y * acc.y;
      }
    }
    if (cnt) a_g += (double)acc.x * acc.x + (double)acc.y * acc.y;
    g[m] = acc;
  }
  double v[4] = {a_g, a_res, a_num, a_den};
  block_reduce_store<4>(v, parts + 4 * (size_t)blockIdx.x);
}
}  // namespace

extern "C" int hicu_step_reduce(const double* obj_parts, int n_obj, const double* dc_parts, int n_dc,
                                const double* els_parts, int n_els, double* sums7, void* stream) {
  if (!obj_parts || !dc_parts || !els_parts || !sums7) return hicu_set_error(HICU_ERR_PARAMETER, "step_reduce: null");
  hicu_launch(step_reduce_kernel, 1, 32, 0, (cudaStream_t)stream, obj_parts, n_obj, dc_parts, n_dc, els_parts, n_els, sums7);
  return hicu_check_launch("step_reduce_kernel");
}

extern "C" int hicu_step_apply(int64_t N, void* y, const void* gdir, const double* sums7, int dc_mode, double lam,
                               double* rec, void* stream) {
  if (!y || !gdir || !sums7 || N < 1) return hicu_set_error(HICU_ERR_PARAMETER, "step_apply: bad arguments");
  int64_t b = (N + 255) / 256;
  const int64_t cap = (int64_t)hicu_sm_count() * 4;
  if (b > cap) b = cap;
  hicu_launch(step_apply_kernel, (int)b, 256, 0, (cudaStream_t)stream, N, (float2*)y, (const float2*)gdir, sums7, dc_mode,
                                                               lam, rec);
  return hicu_check_launch("step_apply_kernel");
}

extern "C" int hicu_dc_nparts(int64_t n) { return ser_blocks(n); }

extern "C" int hicu_dc_apply(int64_t n, void* g, const uint8_t* mask, const void* y, const void* x0, int dc_mode,
                             double lam, double* parts, void* stream) {
  if (!g || !mask || !parts || n < 1) return hicu_set_error(HICU_ERR_PARAMETER, "dc_apply: bad arguments");
  if (dc_mode == 1 && (!y || !x0)) return hicu_set_error(HICU_ERR_SHAPE, "soft data consistency requires x0");
  hicu_launch(dc_apply_kernel, ser_blocks(n), 256, 0, (cudaStream_t)stream, n, (float2*)g, mask, (const float2*)y,
                                                                   (const float2*)x0, dc_mode, (float)lam, parts);
  return hicu_check_launch("dc_apply_kernel");
}

// Stage-driver helpers: build the tcgen05 B images of the G per-step Q~ once
// (conv/ELS and scatter layouts) into `ws`; returns the bytes per image, or 0
// when the geometry does not run the resident tensor-core path or ws is short.
size_t hicu_conv_images_prepare(const hicu_geom* hg, const void* qt_all, int p, int G, void* ws, size_t ws_bytes,
                                void* stream) {
  if (!hg || !qt_all || !ws || G < 1) return 0;
  if (hg->flags & HICU_GEOM_FORCE_SIMT_CONV) return 0;
  DevGeom g;
  if (hicu_make_devgeom(hg, &g)) return 0;
  if (g.nc <= 0 || !hicu_conv_tc_supported(g, p)) return 0;
  const size_t ib = hicu_conv_tc_bimage_bytes(g, p);
  if (!ib || 2 * (size_t)G * ib > ws_bytes) return 0;
  if (hicu_conv_tc_build_bimages(g, (const float2*)qt_all, p, G, (uint8_t*)ws, ib, (cudaStream_t)stream)) return 0;
  return ib;
}

void hicu_conv_image_hint(const void* img, int early) { hicu_conv_tc_bimage_hint(img, early); }
void hicu_conv_amax_hint(const float* in, float* out) { hicu_conv_tc_amax_hint(in, out); }
float* hicu_conv_amax_slots(void* stream) { return hicu_conv_tc_amax_slots((cudaStream_t)stream); }
