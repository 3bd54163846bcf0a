#include <stdlib.h>
// C-ABI glue: error reporting, geometry validation, device queries and the
// Gram dispatch.  See include/hicu_b200.h for the contract.
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"

size_t hicu_gram_simt_workspace(const DevGeom& g);
bool hicu_gram_tc_supported(const DevGeom& g);
size_t hicu_gram_tc_workspace(const DevGeom& g);
int hicu_gram_tc(const DevGeom& g, const float2* x, double2* G, void* ws, size_t ws_bytes, cudaStream_t st);
int hicu_gram_simt(const DevGeom& g, const float2* x, double2* G, void* ws, size_t ws_bytes, cudaStream_t st);

#include <atomic>

namespace {
thread_local char g_last_error[512] = "";
std::atomic<long long> g_launches{0};
}

int hicu_check_launch(const char* where) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return hicu_check_cuda(cudaGetLastError(), where);
}

extern "C" long long hicu_launch_count(void) { return g_launches.load(); }

int hicu_set_error(int code, const char* msg) {
  snprintf(g_last_error, sizeof(g_last_error), "%s", msg ? msg : "");
  return code;
}

int hicu_check_cuda(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return HICU_OK;
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", where, cudaGetErrorString(e));
  return HICU_ERR_CUDA;
}

bool hicu_pdl_enabled() {
  static int v = -1;
  if (v < 0) v = getenv("HICU_NO_PDL") ? 0 : 1;
  return v == 1;
}

int hicu_sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

void hicu_allow_max_smem(const void* func) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({func, dev})) return;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (optin <= 0) optin = 227 * 1024;
  cudaFuncAttributes attr;
  size_t static_smem = 0;
  if (cudaFuncGetAttributes(&attr, func) == cudaSuccess) static_smem = attr.sharedSizeBytes;
  cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)static_smem);
  (void)cudaGetLastError();  // never leave a sticky error for the caller's launch check
  done.insert({func, dev});
}

int hicu_make_devgeom(const hicu_geom* g, DevGeom* out) {
  if (!g) return hicu_set_error(HICU_ERR_PARAMETER, "null geometry");
  if (g->ndim < 1 || g->ndim > HICU_MAX_NDIM) return hicu_set_error(HICU_ERR_SHAPE, "ndim out of range");
  if (g->n < 1) return hicu_set_error(HICU_ERR_SHAPE, "kernel support is empty");
  if (!g->pos || !g->koff) return hicu_set_error(HICU_ERR_PARAMETER, "null support tables");
  DevGeom d;
  memset(&d, 0, sizeof(d));
  d.ndim = g->ndim;
  d.n = g->n;
  d.flags = g->flags;
  d.pos = g->pos;
  d.koff = g->koff;
  int64_t st = 1;
  for (int a = g->ndim - 1; a >= 0; --a) {
    if (g->dims[a] < 1 || g->rext[a] < 1 || g->roff[a] < 0) return hicu_set_error(HICU_ERR_SHAPE, "invalid region");
    d.dims[a] = g->dims[a];
    d.stride[a] = st;
    st *= g->dims[a];
  }
  d.N = st;
  int64_t rs = 1;
  for (int a = g->ndim - 1; a >= 0; --a) {
    d.roff[a] = g->roff[a];
    d.rext[a] = g->rext[a];
    d.rstride[a] = rs;
    rs *= g->rext[a];
  }
  d.s = rs;
  d.ncirc = 0;
  for (int a = 0; a < g->ndim; ++a) {
    if (g->circular & (1u << a)) {
      if (g->roff[a] != 0 || g->rext[a] != g->dims[a])
        return hicu_set_error(HICU_ERR_SHAPE, "circular axis must span the full extent with offset 0");
      d.circ_axes[d.ncirc++] = a;
    }
  }
  d.nc = 0;
  d.nsp = 0;
  for (int a = 0; a < HICU_MAX_NDIM; ++a) d.kext[a] = a < g->ndim ? g->kext[a] : 0;
  {
    const int L = g->ndim - 1;
    const int64_t ncl = g->dims[L];
    if ((g->flags & HICU_GEOM_COIL_SEPARABLE) && L >= 1 && !(g->circular & (1u << L)) && g->rext[L] == 1 &&
        g->roff[L] == 0 && ncl <= 32 && g->n % ncl == 0) {
      d.nc = (int)ncl;
      d.nsp = g->n / (int)ncl;
    }
  }
  *out = d;
  return HICU_OK;
}

extern "C" int hicu_abi_version(void) { return 2; }

extern "C" const char* hicu_last_error(void) { return g_last_error; }

extern "C" const char* hicu_status_string(int status) {
  switch (status) {
    case HICU_OK: return "ok";
    case HICU_ERR_SHAPE: return "ShapeError";
    case HICU_ERR_PARAMETER: return "ParameterError";
    case HICU_ERR_DEGENERATE_INPUT: return "DegenerateInputError";
    case HICU_ERR_DEGENERATE_DIRECTION: return "DegenerateDirectionError";
    case HICU_ERR_SIZE: return "SizeError";
    case HICU_ERR_CONFIG: return "ConfigError";
    case HICU_ERR_ARRAY_FORMAT: return "ArrayFormatError";
    case HICU_ERR_CUDA: return "CudaError";
    case HICU_ERR_WORKSPACE: return "WorkspaceError";
    default: return "unknown";
  }
}

extern "C" int hicu_device_sm_count(int* out) {
  if (!out) return hicu_set_error(HICU_ERR_PARAMETER, "null out");
  *out = hicu_sm_count();
  return HICU_OK;
}

// Gram path: the shift-structured lag Gram (gram_lag.cu) wherever it applies,
// else the dense implicit-im2col Gram (tcgen05 3xTF32, or SIMT).
// Measured crossover: for the 5x5x8 kernels of C1/C2 (n = 200) the dense
// tcgen05 Gram is faster (0.17 vs 0.68 ms at C2's full 252^2 region: the lag
// Gram's fixed costs -- per-lag partials, reduction, n^2 assembly -- dominate
// at n = 200); from n ~ 500 on the lag Gram wins (C3 slice 3.9 -> 0.7 ms SIMT,
// C5 volume 186 -> 56 ms tcgen05).
static int gram_path(const hicu_geom* hg, const DevGeom& g) {
  const bool dense = (hg->flags & (HICU_GEOM_FORCE_DENSE_GRAM | HICU_GEOM_FORCE_SIMT_GRAM)) != 0;
  const bool tc = !(hg->flags & HICU_GEOM_FORCE_SIMT_GRAM) && hicu_gram_tc_supported(g);
  const bool want_lag = (hg->flags & HICU_GEOM_FORCE_LAG_GRAM) != 0;
  if (!dense && hicu_gram_lag_supported(g) && (want_lag || !(tc && g.n < 400))) return HICU_GRAM_PATH_LAG;
  if (!(hg->flags & HICU_GEOM_FORCE_SIMT_GRAM) && hicu_gram_tc_supported(g)) return HICU_GRAM_PATH_TCGEN05;
  return HICU_GRAM_PATH_SIMT;
}

extern "C" size_t hicu_gram_workspace(const hicu_geom* hg) {
  DevGeom g;
  if (hicu_make_devgeom(hg, &g)) return 0;
  switch (gram_path(hg, g)) {
    case HICU_GRAM_PATH_LAG: return hicu_gram_lag_workspace(g);
    case HICU_GRAM_PATH_TCGEN05: {
      const size_t a = hicu_gram_simt_workspace(g), b = hicu_gram_tc_workspace(g);
      return a > b ? a : b;
    }
    default: return hicu_gram_simt_workspace(g);
  }
}

extern "C" int hicu_gram_path(const hicu_geom* hg) {
  DevGeom g;
  if (hicu_make_devgeom(hg, &g)) return -1;
  return gram_path(hg, g);
}

extern "C" double hicu_gram_flops(const hicu_geom* hg) {
  DevGeom g;
  if (hicu_make_devgeom(hg, &g)) return -1.0;
  if (gram_path(hg, g) == HICU_GRAM_PATH_LAG) return hicu_gram_lag_flops(g);
  return 4.0 * (double)g.s * g.n * (g.n + 1);  // dense Hermitian H^H H
}

extern "C" int hicu_gram_lag_uses_tensor_cores(const hicu_geom* hg) {
  DevGeom g;
  if (hicu_make_devgeom(hg, &g)) return 0;
  return gram_path(hg, g) == HICU_GRAM_PATH_LAG && hicu_gram_lag_tc(g) ? 1 : 0;
}

extern "C" int hicu_gram_uses_tensor_cores(const hicu_geom* hg) {
  return hicu_gram_path(hg) == HICU_GRAM_PATH_TCGEN05 ? 1 : 0;
}

extern "C" int hicu_gram(const hicu_geom* hg, const void* x, void* G, void* ws, size_t ws_bytes, void* stream) {
  if (!x || !G || !ws) return hicu_set_error(HICU_ERR_PARAMETER, "gram: null pointer");
  DevGeom g;
  int s = hicu_make_devgeom(hg, &g);
  if (s) return s;
  switch (gram_path(hg, g)) {
    case HICU_GRAM_PATH_LAG:
      return hicu_gram_lag(g, (const float2*)x, (double2*)G, ws, ws_bytes, (cudaStream_t)stream);
    case HICU_GRAM_PATH_TCGEN05:
      return hicu_gram_tc(g, (const float2*)x, (double2*)G, ws, ws_bytes, (cudaStream_t)stream);
    default:
      return hicu_gram_simt(g, (const float2*)x, (double2*)G, ws, ws_bytes, (cudaStream_t)stream);
  }
}
