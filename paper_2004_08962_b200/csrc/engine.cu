// Native stage driver: the reference's outer/inner loop body
// (solver.py:322-393) as a sequence of asynchronous launches on one stream.
// One ABI call per stage; no host synchronisation inside, so a whole stage
// can be captured into a CUDA graph and replayed.
#include <vector>

#include "common.cuh"

size_t hicu_conv_images_prepare(const hicu_geom* hg, const void* qt_all, int p, int G, void* ws, size_t ws_bytes,
                                void* stream);
void hicu_conv_image_hint(const void* img, int early);
void hicu_conv_amax_hint(const float* in, float* out);
float* hicu_conv_amax_slots(void* stream);
int hicu_step_update_amax(int64_t N, void* y, const void* gdir, const double* obj_parts, int n_obj,
                          const double* dc_parts, int n_dc, const double* els_parts, int n_els, int dc_mode,
                          double lam, double* rec, float* amax_out, void* stream);
int hicu_householder_gated(int n, int r, const void* V, double tol, void* refl, void* tau, int* flags, int* status_dev,
                           const int* gate, void* stream);
int hicu_apply_reflectors_gated(int n, int r, const void* refl, const void* tau, const int* flags, int cols,
                                const void* Bin, void* B, void* out32, int p, const int* gate, void* stream);

// ---------------------------------------------------------------------------
// Native per-kernel-class profiler: a pool of CUDA events recorded around each
// launch group on the launching stream (created once, outside timed regions).
// ---------------------------------------------------------------------------
struct HicuProf {
  std::vector<cudaEvent_t> ev;  // 2 per record
  std::vector<int> kind;
  int used = 0;
};

extern "C" int hicu_prof_create(int capacity, void** out) {
  if (!out || capacity < 1) return hicu_set_error(HICU_ERR_PARAMETER, "prof_create: bad arguments");
  HicuProf* p = new HicuProf();
  p->ev.resize(2 * (size_t)capacity);
  p->kind.resize(capacity);
  for (auto& e : p->ev) {
    int s = hicu_check_cuda(cudaEventCreate(&e), "prof_create");
    if (s) return s;
  }
  *out = p;
  return HICU_OK;
}

extern "C" int hicu_prof_destroy(void* h) {
  HicuProf* p = (HicuProf*)h;
  if (!p) return HICU_OK;
  for (auto& e : p->ev) cudaEventDestroy(e);
  delete p;
  return HICU_OK;
}

extern "C" int hicu_prof_reset(void* h) {
  if (h) ((HicuProf*)h)->used = 0;
  return HICU_OK;
}

// ms and launch-group counts per kind (arrays of HICU_PROF_KINDS); syncs.
extern "C" int hicu_prof_summary(void* h, double* ms, int* count) {
  HicuProf* p = (HicuProf*)h;
  if (!p || !ms || !count) return hicu_set_error(HICU_ERR_PARAMETER, "prof_summary: bad arguments");
  for (int k = 0; k < HICU_PROF_KINDS; ++k) { ms[k] = 0.0; count[k] = 0; }
  if (p->used == 0) return HICU_OK;
  int s = hicu_check_cuda(cudaEventSynchronize(p->ev[2 * (size_t)(p->used - 1) + 1]), "prof_summary");
  if (s) return s;
  for (int i = 0; i < p->used; ++i) {
    float t = 0.f;
    s = hicu_check_cuda(cudaEventElapsedTime(&t, p->ev[2 * (size_t)i], p->ev[2 * (size_t)i + 1]), "prof elapsed");
    if (s) return s;
    ms[p->kind[i]] += t;
    count[p->kind[i]] += 1;
  }
  return HICU_OK;
}

namespace {
// B-image hint for the next conv_tc launch on this thread, cleared when the
// scope ends whether or not the call consumed it (error paths included)
struct ImageHint {
  explicit ImageHint(const void* img, int early) {
    if (img) hicu_conv_image_hint(img, early);
  }
  ~ImageHint() { hicu_conv_image_hint(nullptr, 0); }
};

// Operand-scale hint for the next tensor-core convolution on this thread:
// the A operand's max partials (written by its producer) and where the
// launch writes its own output's max partials; cleared when the scope ends.
struct AmaxHint {
  explicit AmaxHint(bool on, const float* in, float* out) {
    if (on) hicu_conv_amax_hint(in, out);
  }
  ~AmaxHint() { hicu_conv_amax_hint(nullptr, nullptr); }
};

struct ProfScope {
  HicuProf* p;
  cudaStream_t st;
  int idx = -1;
  ProfScope(void* h, int kind, cudaStream_t s) : p((HicuProf*)h), st(s) {
    if (p && p->used < (int)p->kind.size()) {
      idx = p->used++;
      p->kind[idx] = kind;
      cudaEventRecord(p->ev[2 * (size_t)idx], st);
    }
  }
  ~ProfScope() {
    if (idx >= 0) cudaEventRecord(p->ev[2 * (size_t)idx + 1], st);
  }
};
}  // namespace

// Householder complement of V and Q~_j = Q P_j for the cols = G p JL columns
// (subspace.py:158-229): the closed form (nsjl.cu) when it applies, the
// reference's reflector chain gated on its pivot check otherwise.  refl holds
// 2 n r complex (also the closed form's scratch), flags r + 1 ints.
extern "C" int hicu_complement_jl(int n, int r, int cols, int p, const void* V, const void* pbig, void* B, void* qt32,
                                  void* refl, void* tau, int* flags, double tol, int* status, void* stream) {
  const size_t refl_bytes = (size_t)2 * n * r * sizeof(double2);
  const bool use_jl = hicu_nullspace_jl_supported(n, r) && hicu_nullspace_jl_workspace(n, r) <= refl_bytes;
  const int* gate = nullptr;
  int s;
  if (use_jl) {
    if ((s = hicu_nullspace_jl_ws(n, r, V, cols, pbig, B, qt32, p, flags + r, refl, refl_bytes, stream))) return s;
    gate = flags + r;
  }
  if ((s = hicu_householder_gated(n, r, V, tol, refl, tau, flags, status, gate, stream))) return s;
  return hicu_apply_reflectors_gated(n, r, refl, tau, flags, cols, pbig, B, qt32, p, gate, stream);
}

extern "C" int hicu_run_stage(const hicu_stage_args* a, void* stream) {
  if (!a) return hicu_set_error(HICU_ERR_PARAMETER, "run_stage: null args");
  const hicu_geom* gm = &a->geom;
  const int n = gm->n, r = a->r, ell = a->ell, p = a->p, G = a->gsteps;
  if (!(1 <= r && r < n)) return hicu_set_error(HICU_ERR_CONFIG, "rank must be below the kernel support size");
  if (p < 1 || G < 1 || a->iters < 0) return hicu_set_error(HICU_ERR_CONFIG, "bad stage schedule");
  cudaStream_t st = (cudaStream_t)stream;
  const int ncp = hicu_conv_nparts(gm);
  const int nsp = hicu_scatter_nparts(gm);
  if (ncp < 0 || nsp < 0) return HICU_ERR_SHAPE;
  const size_t nomega = (size_t)n * ell, npbig = (size_t)n * G * p;
  int s;
  // producer max partials (tensor-core convolutions): y from the update, u
  // from the forward convolution, g from the scatter -- no amax pass per call
  const bool tcv = hicu_conv_uses_tensor_cores(gm, p) == 1;
  float* slots = tcv ? hicu_conv_amax_slots(stream) : nullptr;
  float* sY = slots;
  float* sU = slots ? slots + 512 : nullptr;
  float* sG = slots ? slots + 1024 : nullptr;
  bool y_valid = false;  // sY holds max |y| of the current y
  for (int it = 0; it < a->iters; ++it) {
    // ---- nullspace: Gram + Nystrom (== rSVD subspace), or injected V ----
    if (a->inject_v) {
      ProfScope ps(a->prof, HICU_PROF_NYSTROM, st);
      s = hicu_check_cuda(cudaMemcpyAsync(a->V, (const double2*)a->inject_v + (size_t)it * n * r,
                                          (size_t)n * r * sizeof(double2), cudaMemcpyDeviceToDevice, st),
                          "inject_v copy");
      if (s) return s;
    } else {
      {
        ProfScope ps(a->prof, HICU_PROF_GRAM, st);
        if ((s = hicu_gram(gm, a->y, a->G, a->gram_ws, a->gram_ws_bytes, stream))) return s;
      }
      ProfScope ps(a->prof, HICU_PROF_NYSTROM, st);
      if ((s = hicu_nystrom(n, ell, r, a->G, (const double2*)a->omega + (size_t)it * nomega, a->V, a->nys_ws,
                            a->nys_ws_bytes, a->status, stream)))
        return s;
    }
    // ---- Householder complement and Q~_j = Q P_j for all steps ----
    {
      ProfScope ps(a->prof, HICU_PROF_HOUSEHOLDER, st);
      const double2* pb = (const double2*)a->pbig + (size_t)it * npbig;
      if ((s = hicu_complement_jl(n, r, G * p, p, a->V, pb, a->B, a->qt32, a->refl, a->tau, a->flags,
                                  a->householder_tol, a->status, stream)))
        return s;
    }
    // ---- gradient steps ----
    // tcgen05 B images of every step's Q~, built once (the Gram workspace is
    // idle until the next iteration); each conv copies its image with one
    // bulk copy, before its grid-dependency wait when the image kernel is at
    // least two launches back (every conv but the first).
    size_t ib = 0;
    {
      ProfScope ps(a->prof, HICU_PROF_HOUSEHOLDER, st);
      ib = hicu_conv_images_prepare(gm, a->qt32, p, G, a->gram_ws, a->gram_ws_bytes, stream);
    }
    const uint8_t* imgs = (const uint8_t*)a->gram_ws;
    for (int j = 0; j < G; ++j) {
      const float2* qt = (const float2*)a->qt32 + (size_t)j * n * p;
      double* rec = a->rec + ((size_t)it * G + j) * HICU_REC_SLOTS;
      {
        ProfScope ps(a->prof, HICU_PROF_CONV_FWD, st);
        ImageHint hint(ib ? imgs + (size_t)(2 * j) * ib : nullptr, j > 0 ? 1 : 0);
        AmaxHint ah(slots != nullptr, y_valid ? sY : nullptr, sU);
        if ((s = hicu_conv_fwd(gm, a->y, qt, p, a->u, a->obj_parts, stream))) return s;
      }
      {
        ProfScope ps(a->prof, HICU_PROF_SCATTER, st);
        ImageHint hint(ib ? imgs + (size_t)(2 * j + 1) * ib : nullptr, 1);
        AmaxHint ah(slots != nullptr, sU, sG);
        if ((s = hicu_scatter_dc(gm, qt, p, a->u, a->mask, a->y, a->x0, a->dc_mode, a->lam, a->g, a->dc_parts,
                                 stream)))
          return s;
      }
      {
        ProfScope ps(a->prof, HICU_PROF_CONV_ELS, st);
        ImageHint hint(ib ? imgs + (size_t)(2 * j) * ib : nullptr, 1);
        AmaxHint ah(slots != nullptr, sG, nullptr);
        if ((s = hicu_conv_els(gm, a->g, qt, p, a->u, a->els_parts, stream))) return s;
      }
      {
        ProfScope ps(a->prof, HICU_PROF_UPDATE, st);
        if ((s = hicu_step_update_amax(a->N, a->y, a->g, a->obj_parts, ncp, a->dc_parts, nsp, a->els_parts, ncp,
                                       a->dc_mode, a->lam, rec, sY, stream)))
          return s;
        y_valid = sY != nullptr;
      }
      if (a->ref && a->ser_parts) {
        double* sp = a->ser_parts + ((size_t)it * G + j) * a->ser_stride;
        if ((s = hicu_ser_parts(a->N, a->ref, a->y, sp, nullptr, stream))) return s;
      }
    }
  }
  return HICU_OK;
}
