// Native stage driver: the reference's outer/inner loop body
// (solver.py:322-393) as a sequence of asynchronous launches on one stream.
// One ABI call per stage; no host synchronisation inside, so a whole stage
// can be captured into a CUDA graph and replayed.
#include "common.cuh"

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
  for (int it = 0; it < a->iters; ++it) {
    // ---- nullspace: Gram + Nystrom (== rSVD subspace), or injected V ----
    if (a->inject_v) {
      s = hicu_check_cuda(cudaMemcpyAsync(a->V, (const double2*)a->inject_v + (size_t)it * n * r,
                                          (size_t)n * r * sizeof(double2), cudaMemcpyDeviceToDevice, st),
                          "inject_v copy");
      if (s) return s;
    } else {
      if ((s = hicu_gram(gm, a->y, a->G, a->gram_ws, a->gram_ws_bytes, stream))) return s;
      if ((s = hicu_nystrom(n, ell, r, a->G, (const double2*)a->omega + (size_t)it * nomega, a->V, a->nys_ws,
                            a->nys_ws_bytes, a->status, stream)))
        return s;
    }
    // ---- Householder complement and Q~_j = Q P_j for all steps ----
    if ((s = hicu_householder(n, r, a->V, a->householder_tol, a->refl, a->tau, a->flags, a->status, stream)))
      return s;
    if ((s = hicu_apply_reflectors(n, r, a->refl, a->tau, a->flags, G * p,
                                   (const double2*)a->pbig + (size_t)it * npbig, a->B, a->qt32, p, stream)))
      return s;
    // ---- gradient steps ----
    for (int j = 0; j < G; ++j) {
      const float2* qt = (const float2*)a->qt32 + (size_t)j * n * p;
      double* rec = a->rec + ((size_t)it * G + j) * HICU_REC_SLOTS;
      if ((s = hicu_conv_fwd(gm, a->y, qt, p, a->u, a->obj_parts, stream))) return s;
      if ((s = hicu_scatter_dc(gm, qt, p, a->u, a->mask, a->y, a->x0, a->dc_mode, a->lam, a->g, a->dc_parts,
                               stream)))
        return s;
      if ((s = hicu_conv_els(gm, a->g, qt, p, a->u, a->els_parts, stream))) return s;
      if ((s = hicu_step_update(a->N, a->y, a->g, a->obj_parts, ncp, a->dc_parts, nsp, a->els_parts, ncp,
                                a->dc_mode, a->lam, rec, stream)))
        return s;
      if (a->ref && a->ser_parts) {
        double* sp = a->ser_parts + ((size_t)it * G + j) * a->ser_stride;
        if ((s = hicu_ser_parts(a->N, a->ref, a->y, sp, nullptr, stream))) return s;
      }
    }
  }
  return HICU_OK;
}
