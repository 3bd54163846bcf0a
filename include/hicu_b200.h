/*
 * hicu_b200.h — C ABI of the B200-native HICU reconstruction hot path.
 *
 * The reference (arXiv 2004.08962 package, /root/reference/pkg/src/hicu) is
 * pure Python; it has no FFI.  Each entry point below replaces one reference
 * function (or one fused group of them) on the path entered through
 * hicu_reconstruct (solver.py:258); the replaced interface is cited per
 * function.  INTEGRATION.md shows the ctypes binding a maintainer would add.
 *
 * Conventions (all functions):
 *   - k-space arrays are complex64 (interleaved float re/im, "c64"), C order,
 *     dims = [spatial..., (time), coil] as in reference arrays.py:1-10;
 *   - small dense matrices (Gram, sketches, bases) are complex128 ("c128"),
 *     row-major;
 *   - every pointer is a DEVICE pointer owned by the caller unless noted;
 *     the library never allocates or frees caller memory;
 *   - every call is asynchronous on `stream` (a cudaStream_t, passed as void*);
 *   - the return value is a status code (HICU_OK or one of the codes mapping
 *     1:1 to reference errors.py:4-29); nothing throws across the ABI;
 *   - deterministic: fixed-order reductions, no floating-point atomics.
 */
#ifndef HICU_B200_H
#define HICU_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HICU_MAX_NDIM 8

/* status codes: 1..7 mirror reference errors.py:4-29 */
enum {
  HICU_OK = 0,
  HICU_ERR_SHAPE = 1,                /* ShapeError            errors.py:4  */
  HICU_ERR_PARAMETER = 2,            /* ParameterError        errors.py:8  */
  HICU_ERR_DEGENERATE_INPUT = 3,     /* DegenerateInputError  errors.py:12 */
  HICU_ERR_DEGENERATE_DIRECTION = 4, /* DegenerateDirectionError errors.py:16 */
  HICU_ERR_SIZE = 5,                 /* SizeError             errors.py:20 */
  HICU_ERR_CONFIG = 6,               /* ConfigError           errors.py:24 */
  HICU_ERR_ARRAY_FORMAT = 7,         /* ArrayFormatError      errors.py:28 */
  HICU_ERR_CUDA = 100,               /* CUDA runtime error (message via hicu_last_error) */
  HICU_ERR_WORKSPACE = 101           /* workspace smaller than the *_workspace query */
};

/* Geometry of one lifted (block-Hankel) operator: the reference's KernelMask +
 * Region pair (hankel.py:52-145).  Row i of H enumerates the region block in
 * row-major order, column kappa the kernel support in row-major order
 * (hankel.py:81); H[i,kappa] = X[roff + i + pos[kappa]] with wrap-around on
 * circular axes. */
typedef struct hicu_geom {
  int32_t ndim;
  int32_t n;                      /* kernel support size                      */
  int64_t dims[HICU_MAX_NDIM];    /* k-space extents                          */
  int64_t roff[HICU_MAX_NDIM];    /* region offsets (0 on circular axes)      */
  int64_t rext[HICU_MAX_NDIM];    /* region extents                           */
  uint32_t circular;              /* bit d set: axis d is circular            */
  int32_t flags;                  /* HICU_GEOM_COIL_SEPARABLE: the support is  *
                                   * (spatial support) x (all dims[last] coils), *
                                   * kappa = sp*dims[last] + c                  */
  const int32_t* pos;             /* device: n x ndim support positions       */
  const int64_t* koff;            /* device: n flat offsets, non-circular axes */
  int64_t kext[HICU_MAX_NDIM];    /* kernel bounding-box extents (KernelMask.extents,
                                   * hankel.py:58); 0 = unknown (disables the
                                   * tensor-core conv/scatter, which size their
                                   * operand tiles from it)                     */
} hicu_geom;

#define HICU_GEOM_COIL_SEPARABLE 1
#define HICU_GEOM_FORCE_SIMT_GRAM 2   /* use the SIMT Gram even when tcgen05 applies */
#define HICU_GEOM_FORCE_SIMT_CONV 4   /* use the SIMT conv/scatter even when tcgen05 applies */
#define HICU_GEOM_FORCE_DENSE_GRAM 8  /* dense implicit-im2col Gram instead of the lag Gram */
#define HICU_GEOM_FORCE_LAG_GRAM 16   /* lag Gram wherever it applies (default: by size) */
#define HICU_GEOM_FORCE_FFMA_LAG 32   /* lag Gram core on the CUDA cores even where its tensor-core form applies */

/* hicu_gram_path() values */
#define HICU_GRAM_PATH_SIMT 0     /* dense implicit-im2col Gram, fp32 SIMT (gram_simt.cu) */
#define HICU_GRAM_PATH_TCGEN05 1  /* dense implicit-im2col Gram, tcgen05 3xTF32 (gram_tc.cu) */
#define HICU_GRAM_PATH_LAG 2      /* shift-structured lag Gram (gram_lag.cu) */

/* Per-step scalar record written by hicu_step_update (doubles). */
enum {
  HICU_REC_OBJ = 0,       /* objective before the step                        */
  HICU_REC_NUM = 1,       /* ELS numerator  sum Re<w,u> (+ soft term)         */
  HICU_REC_DEN = 2,       /* ELS curvature  sum |w|^2 (+ soft term)           */
  HICU_REC_ETA = 3,       /* step size (0 when degenerate)                    */
  HICU_REC_OBJ_AFTER = 4, /* obj - num^2/den                                  */
  HICU_REC_GNORM2 = 5,    /* ||g||^2 after data consistency                   */
  HICU_REC_DEGENERATE = 6,/* 1.0 when den <= 0 (step skipped)                 */
  HICU_REC_SLOTS = 8
};

/* ---- library info -------------------------------------------------------- */
int hicu_abi_version(void);
const char* hicu_last_error(void);
const char* hicu_status_string(int status);
int hicu_device_sm_count(int* out);

/* ---- gradient step (replaces solver.py:333-376 inner loop body) ----------- */

/* Number of fp64 partial-sum slots each fused reduction writes (per slot
 * group); callers size their partial buffers with these. */
int hicu_conv_nparts(const hicu_geom* g);     /* blocks of hicu_conv_fwd/els   */
int hicu_scatter_nparts(const hicu_geom* g);  /* blocks of hicu_scatter_dc     */

/* u = H(y) qt  (s x p, row-major, c64), obj_parts[b] = partial sum |u|^2.
 * Replaces hankel_apply (hankel.py:255-322) + np.vdot (solver.py:334-335). */
int hicu_conv_fwd(const hicu_geom* g, const void* y, const void* qt, int p,
                  void* u, double* obj_parts, void* stream);

/* w = H(gdir) qt is never stored; numden_parts[2b] = sum Re(conj(w) u),
 * numden_parts[2b+1] = sum |w|^2.  Replaces hankel_apply + the two vdots of
 * exact_line_search (hankel.py:512-558, solver.py:346-351). */
int hicu_conv_els(const hicu_geom* g, const void* gdir, const void* qt, int p,
                  const void* u, double* numden_parts, void* stream);

/* g = scatter(qt, u) (hankel.py:394-440) with data consistency fused:
 * dc_mode 0 (hard): g[mask==1] = 0 (solver.py:345);
 * dc_mode 1 (soft): g += lam * mask*(y - x0) (solver.py:342-343);
 * dc_mode 2 (none): plain kspace_adjoint_scatter (mask/y/x0 unused).
 * dc_parts[4b+0..3] = ||g||^2, ||res||^2, Re<Mg,res>, ||Mg||^2 partials. */
int hicu_scatter_dc(const hicu_geom* g, const void* qt, int p, const void* u,
                    const uint8_t* mask, const void* y, const void* x0,
                    int dc_mode, double lam, void* gout, double* dc_parts,
                    void* stream);

/* Reduce the partials (fixed order), form eta = num/den on the device, write
 * the HICU_REC_* record to rec[0..7], and apply y -= eta*g unless den <= 0
 * (solver.py:356-370).  No host synchronisation. */
int hicu_step_update(int64_t N, void* y, const void* gdir,
                     const double* obj_parts, int n_obj,
                     const double* dc_parts, int n_dc,
                     const double* els_parts, int n_els,
                     int dc_mode, double lam, double* rec, void* stream);

/* Soft-DC line-search terms (hankel.py:546-550): parts[3b+0..2] =
 * Re<Mg, res>, |Mg|^2, |res|^2 with res = M(y - x0); *nparts_out blocks. */
int hicu_soft_terms(int64_t N, const void* g, const void* y, const void* x0,
                    const uint8_t* mask, double* parts, int* nparts_out,
                    void* stream);

/* out[kappa, j] = sum_i conj(X[i+kappa]) u[i, j]: kernel-slot adjoint
 * (hankel_adjoint_apply hankel.py:325-391); u is s x k c64, out n x k c128. */
int hicu_conv_adj(const hicu_geom* g, const void* x, const void* u, int k,
                  void* out, void* stream);

/* Split step update for the halo-sharded volume path (several GPUs hold one
 * volume): hicu_step_reduce writes sums7 = [obj_conv, ||g||^2, ||res||^2,
 * Re<Mg,res>, ||Mg||^2, num_conv, den_conv] from the local partials; the
 * caller all-reduces sums7 over ranks; hicu_step_apply forms eta (identical on
 * every rank) and updates y (solver.py:356-370). */
int hicu_step_reduce(const double* obj_parts, int n_obj, const double* dc_parts,
                     int n_dc, const double* els_parts, int n_els,
                     double* sums7, void* stream);
int hicu_step_apply(int64_t N, void* y, const void* gdir, const double* sums7,
                    int dc_mode, double lam, double* rec, void* stream);
/* Data consistency on n contiguous samples of g (after the halo
 * accumulation of raw scatter partials); parts as hicu_scatter_dc's.  mask
 * bit 0: observed sample; bit 1: a halo copy of a plane another rank owns
 * (the data consistency is applied, but the sample is left out of parts). */
int hicu_dc_nparts(int64_t n);
int hicu_dc_apply(int64_t n, void* g, const uint8_t* mask, const void* y,
                  const void* x0, int dc_mode, double lam, double* parts,
                  void* stream);

/* ser_parts[2b] = sum |ref - y|^2, [2b+1] = sum |ref|^2 (solver.py:251-255).
 * Returns the number of blocks used in *nparts_out when not NULL. */
int hicu_ser_parts(int64_t N, const void* ref, const void* y, double* ser_parts,
                   int* nparts_out, void* stream);

/* ---- nullspace (replaces rsvd_right_vectors subspace.py:67-155) ----------- */

/* G = H(x)^H H(x), n x n c128 Hermitian (full storage).  No reference
 * function; equals hankel_adjoint_apply(x, hankel_apply(x, I)). */
size_t hicu_gram_workspace(const hicu_geom* g);
/* 1 when hicu_gram runs the tcgen05 3xTF32 kernel for this geometry (coil-
 * separable support with 8 coils, no circular axes, >= 8 spatial taps, and
 * the dense Gram selected: HICU_GEOM_FORCE_DENSE_GRAM or no lag path). */
int hicu_gram_uses_tensor_cores(const hicu_geom* g);
/* Which Gram hicu_gram runs for this geometry: HICU_GRAM_PATH_LAG (coil-
 * separable support, 1-3 spatial axes, spatial kernel extents <= 8, Nc in
 * 1..8, 10, 12, 16: G assembled from per-lag coil correlations over the
 * per-axis position classes of the shifted region boxes), else the dense
 * tcgen05 or SIMT implicit-im2col Gram; the dense tcgen05 Gram is kept for
 * n < 400 (measured faster at the 5x5x8 kernels of C1/C2) unless
 * HICU_GEOM_FORCE_LAG_GRAM; -1 on a bad geometry. */
int hicu_gram_path(const hicu_geom* g);
/* 1 when the lag Gram runs its core class on the tcgen05 kernels for this
 * geometry (8 coils, non-circular line axis of <= 256 positions, <= 5 taps
 * along it; fp16 hi/lo operands, HICU_GEOM_FORCE_FFMA_LAG not set). */
int hicu_gram_lag_uses_tensor_cores(const hicu_geom* g);
/* Real flops hicu_gram executes for this geometry on its path (lag: the
 * fp32 lag-correlation products; dense: 4 s n (n+1)); -1 on a bad geometry. */
double hicu_gram_flops(const hicu_geom* g);
/* 1 when hicu_conv_fwd / hicu_conv_els / hicu_scatter_dc with p columns run
 * on the tcgen05 kernels (conv_tc.cu) for this geometry. */
int hicu_conv_uses_tensor_cores(const hicu_geom* g, int p);
int hicu_gram(const hicu_geom* g, const void* x, void* G, void* ws,
              size_t ws_bytes, void* stream);

/* Top-r eigenpairs of a Hermitian n x n c128 matrix (row-major, full
 * storage): evals descending (r doubles), V n x r orthonormal (row-major).  The
 * dense Cadzow baseline's rank-r truncation (oracle.py:138-174). */
size_t hicu_eigh_top_workspace(int n, int r);
int hicu_eigh_top(int n, int r, const void* A, double* evals, void* V, void* ws,
                  size_t ws_bytes, void* stream);

/* C = op(A) op(B) for small row-major c128 matrices; op 'N' or 'C' (conj
 * transpose).  C is m x n; op(A) is m x k; op(B) is k x n. */
int hicu_zgemm(char opa, char opb, int m, int n, int k, const void* A, int lda,
               const void* B, int ldb, void* C, int ldc, void* stream);

/* Top-r right singular subspace of H from its Gram matrix with the host
 * sketch omega (n x ell c128): Nystrom form of the reference's single-pass
 * rSVD (same subspace for the same omega).  Writes V (n x r c128, orthonormal
 * columns ordered by decreasing singular value, each column's phase fixed so
 * its largest-magnitude entry, first on ties, is real positive) and
 * *status_dev (device int, HICU_OK or HICU_ERR_DEGENERATE_INPUT). */
size_t hicu_nystrom_workspace(int n, int ell);
int hicu_nystrom(int n, int ell, int r, const void* G, const void* omega,
                 void* V, void* ws, size_t ws_bytes, int* status_dev,
                 void* stream);

/* Householder reflectors of V (subspace.py:158-212, triangularisation part):
 * refl (r x n c128, row j holds w_j in entries j..n-1; the buffer must hold
 * 2*n*r elements, the second half is scratch), tau (r c128),
 * flags (r int: 0 identity reflector, 1 active).  *status_dev set to
 * HICU_ERR_DEGENERATE_INPUT when a column is dependent (beta < tol). */
int hicu_householder(int n, int r, const void* V, double tol, void* refl,
                     void* tau, int* flags, int* status_dev, void* stream);

/* B = H_0^H ... H_{r-1}^H Bin, reflectors applied in reverse order
 * (subspace.py:203-211).  With Bin = [0; I] this is the nullspace basis Q;
 * with Bin = [0; P_0 | ... | P_{G-1}] it yields Q~_j = Q P_j for every
 * gradient step at once (jl_compress subspace.py:215-229).  Bin and B are
 * n x cols c128 row-major (B may alias Bin).
 * If out32 != NULL it also receives B as c64 in step-major layout
 * out32[j][row][t] = B[row][j*p + t] for cols = G*p. */
int hicu_apply_reflectors(int n, int r, const void* refl, const void* tau,
                          const int* flags, int cols, const void* Bin, void* B,
                          void* out32, int p, void* stream);

/* Q~ = Q [P] in closed form, replacing hicu_householder + hicu_apply_reflectors
 * (subspace.py:158-229) for orthonormal V: with A = V - [I; 0] and
 * A_1 = V_1 - I (top r x r block), Q = [0; I] + A A_1^{-H} V_2^H, which is the
 * reference's reflector product exactly because its nonnegative-pivot
 * convention makes R = I.  B = Q Bin[r:, :] (n x cols c128 row-major; rows < r
 * of Bin are ignored), out32 as in hicu_apply_reflectors.  *gate_dev (device
 * int) is set to 1 when an LU pivot (the reference's u0) is below 1e-3 in
 * modulus; the caller must then recompute with the Householder kernels.
 * Supported for 1 <= r <= 160, r < n (hicu_nullspace_jl_supported). */
int hicu_nullspace_jl_supported(int n, int r);
int hicu_nullspace_jl(int n, int r, const void* V, int cols, const void* Bin,
                      void* B, void* out32, int p, int* gate_dev, void* stream);
/* Same with a caller workspace: ranks whose r x r LU does not fit one SM
 * (64 < r <= 160 for large n, e.g. C4/C5) factor A_1 in global memory.
 * hicu_nullspace_jl_workspace(n, r) bytes (0: none needed). */
size_t hicu_nullspace_jl_workspace(int n, int r);
/* The outer iteration's nullspace tail as the stage driver runs it: Q~ = Q P
 * for cols = G p JL columns from V (the closed form when it applies, the
 * reflector chain -- householder_nullspace, subspace.py:158-212 -- when its
 * pivot check gates it in).  pbig: n x cols c128 (rows < r ignored); B: n x
 * cols c128 out; qt32: [cols/p][n][p] c64 out; refl: 2 n r c128 scratch; tau:
 * r c128; flags: r + 1 ints; status: device int (DegenerateInputError). */
int hicu_complement_jl(int n, int r, int cols, int p, const void* V, const void* pbig, void* B, void* qt32,
                       void* refl, void* tau, int* flags, double tol, int* status, void* stream);
int hicu_nullspace_jl_ws(int n, int r, const void* V, int cols, const void* Bin,
                         void* B, void* out32, int p, int* gate_dev, void* ws,
                         size_t ws_bytes, void* stream);

/* ---- native stage driver (replaces the solver.py:322-393 loop body) ------- */
/* One call runs `iters` outer iterations of one stage: Gram -> Nystrom ->
 * Householder -> Q~ for all steps -> gsteps x (conv_fwd, scatter_dc,
 * conv_els, step_update [, ser]).  All buffers are caller-owned device
 * memory; nothing synchronises with the host, so the call can be captured
 * into a CUDA graph.  rec receives iters*gsteps records of HICU_REC_SLOTS
 * doubles; slot 7 holds the device globaltimer (ns) at the step's update. */
typedef struct hicu_stage_args {
  hicu_geom geom;          /* stage region geometry                           */
  int32_t r, ell, p, gsteps, iters;
  int32_t dc_mode;         /* 0 hard, 1 soft                                  */
  double lam;              /* soft-DC weight                                  */
  double householder_tol;  /* subspace.py:158 tol (1e-12)                     */
  int64_t N;               /* k-space size                                    */
  void* y;                 /* c64 N, iterate (in/out)                         */
  const uint8_t* mask;     /* N                                               */
  const void* x0;          /* c64 N masked data (soft mode), may be NULL      */
  const void* omega;       /* c128 iters x n x ell sketches                   */
  const void* pbig;        /* c128 iters x n x (gsteps*p), rows < r zero      */
  const void* inject_v;    /* optional c128 iters x n x r (lockstep parity)   */
  void* G; void* gram_ws; size_t gram_ws_bytes;
  void* nys_ws; size_t nys_ws_bytes;
  void* V;                 /* c128 n x r                                      */
  void* refl;              /* c128 2*n*r                                      */
  void* tau;               /* c128 r                                          */
  int32_t* flags;          /* r + 1 (the last int is the nullspace_jl gate)   */
  int32_t* status;         /* device int, sticky error                        */
  void* B;                 /* c128 n x (gsteps*p)                             */
  void* qt32;              /* c64 gsteps x n x p                              */
  void* u;                 /* c64 s x p                                       */
  void* g;                 /* c64 N                                           */
  double* obj_parts; double* dc_parts; double* els_parts;
  double* rec;             /* iters*gsteps*HICU_REC_SLOTS                     */
  const void* ref;         /* optional c64 N fully sampled reference          */
  double* ser_parts;       /* iters*gsteps*ser_stride doubles when ref        */
  int32_t ser_stride;
  void* prof;              /* optional hicu_prof handle (NULL: no events)     */
} hicu_stage_args;

/* ---- native profiler: CUDA events around each launch group --------------- */
enum {
  HICU_PROF_GRAM = 0, HICU_PROF_NYSTROM = 1, HICU_PROF_HOUSEHOLDER = 2,
  HICU_PROF_CONV_FWD = 3, HICU_PROF_SCATTER = 4, HICU_PROF_CONV_ELS = 5,
  HICU_PROF_UPDATE = 6, HICU_PROF_KINDS = 7
};
int hicu_prof_create(int capacity, void** out);
int hicu_prof_destroy(void* h);
int hicu_prof_reset(void* h);
/* per-kind total milliseconds and launch-group counts (synchronises) */
int hicu_prof_summary(void* h, double* ms, int* count);
/* number of kernels this library has launched in the process */
long long hicu_launch_count(void);

int hicu_ser_nparts(int64_t N);
int hicu_run_stage(const hicu_stage_args* a, void* stream);
/* writes the device globaltimer (ns, as double) to *out */
int hicu_timestamp(double* out, void* stream);

/* ---- SVD coil compression (no reference function) -------- */
/* cov = sum over sampled locations l (mask[l*nc] == 1) of x_l^H x_l
 * (nc x nc c128); x is nloc x nc c64. */
size_t hicu_coil_workspace(int64_t nloc, int nc);
int hicu_coil_cov(int64_t nloc, int nc, const void* x, const uint8_t* mask,
                  void* cov, void* ws, size_t ws_bytes, void* stream);
/* eigenvectors of cov by Jacobi, sorted by decreasing eigenvalue, phase fixed
 * (largest |entry| real positive, first on ties); basis nc x nv c128,
 * evals (nc doubles, descending, may be NULL). */
size_t hicu_coil_basis_workspace(int nc);
int hicu_coil_basis(int nc, int nv, const void* cov, void* basis, double* evals,
                    void* ws, size_t ws_bytes, void* stream);
/* y[l, j] = sum_c m[l, c] x[l, c] basis[c, j]  (nloc x nv c64), with
 * m = (mask == 1) when mask != NULL (the reference's mask_apply,
 * arrays.py:54-67, fused: x may be raw k-space) and m = 1 otherwise;
 * mask_out[l, j] = mask[l, 0] when mask_out != NULL. */
int hicu_coil_apply(int64_t nloc, int nc, int nv, const void* x,
                    const uint8_t* mask, const void* basis, void* y,
                    uint8_t* mask_out, void* stream);

/* ---- collectives of a sharded volume ----------------------
 * NCCL, resolved at run time from libnccl.so.2.  One communicator per
 * process/GPU; the 128-byte id comes from hicu_comm_unique_id on rank 0 and
 * is broadcast by the host.  All calls are asynchronous on `stream`. */
#define HICU_P2P_SEND 0
#define HICU_P2P_RECV 1
typedef struct {
  int32_t peer;   /* rank in the communicator */
  int32_t kind;   /* HICU_P2P_SEND / HICU_P2P_RECV */
  void* buf;      /* device buffer (send: read, recv: written) */
  int64_t bytes;
} hicu_p2p_op;
int hicu_comm_available(void);
int hicu_comm_unique_id(void* id128_out);
int hicu_comm_init(int nranks, int rank, const void* id128, void** comm_out);
int hicu_comm_destroy(void* comm);
/* in-place sum over ranks of count doubles (Gram partials as 2 n^2 doubles,
 * the step scalars) */
int hicu_allreduce(void* comm, double* buf, int64_t count, void* stream);
/* one grouped round of sends and receives (halo accumulate / refresh) */
int hicu_halo_exchange(void* comm, int nops, const hicu_p2p_op* ops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HICU_B200_H */
