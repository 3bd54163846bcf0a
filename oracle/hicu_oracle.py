"""HICU oracle: a CPU restatement of the reference's reconstruction hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and only as the
checker or the timed CPU baseline.

Every function restates the reference algorithm (``/root/reference/pkg/src/
hicu``) in numpy/scipy (complex128, LAPACK through scipy) and cites the
file:line it follows.  The restatement is pinned against golden vectors that
``tests/golden/make_golden.py`` produced by importing the reference itself
(``tests/test_oracle_golden.py``).

Geometry is passed as a small :class:`Geom` record instead of the
reference's ``KernelMask``/``Region`` objects:

* ``dims``        k-space extents, C order, coil axis last;
* ``positions``   kernel support positions (n x ndim), row-major argwhere
                  order (reference ``hankel.py:81``);
* ``offsets``/``extents``  the output block (reference ``Region``,
                  ``hankel.py:103-145``);
* ``circular``    axes that wrap modulo the extent (``hankel.py:210-221``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np
import scipy.linalg

__all__ = [
    "OracleError",
    "Geom",
    "support_positions",
    "full_geom",
    "stage_geom",
    "flat_index",
    "hankel_apply",
    "hankel_adjoint_apply",
    "kspace_adjoint_scatter",
    "gram",
    "objective_and_gradient",
    "exact_line_search",
    "rng_generator",
    "complex_normal",
    "rsvd_right_vectors",
    "nystrom_right_vectors",
    "householder_nullspace",
    "canonicalize_phases",
    "jl_compress",
    "mask_apply",
    "hicu_reconstruct",
    "ser_db",
    "coil_compress",
]


class OracleError(ValueError):
    """Raised where the reference raises one of its ValueError subclasses."""


# ---------------------------------------------------------------------------
# geometry (reference hankel.py:52-157, solver.py:104-158)
# ---------------------------------------------------------------------------


def support_positions(extents, support=None) -> np.ndarray:
    """Row-major positions of the ones of the kernel box (hankel.py:66-84)."""
    extents = tuple(int(e) for e in extents)
    if support is None:
        support = np.ones(extents, np.uint8)
    return np.argwhere(np.asarray(support) == 1)


@dataclass
class Geom:
    dims: tuple
    positions: np.ndarray
    offsets: tuple
    extents: tuple
    circular: frozenset = field(default_factory=frozenset)

    @property
    def n(self) -> int:
        return int(self.positions.shape[0])

    @property
    def s(self) -> int:
        return int(np.prod(self.extents))


def full_geom(dims, kext, circular=(), support=None) -> Geom:
    """All valid outputs, full extent on circular axes (hankel.py:148-157)."""
    dims = tuple(int(d) for d in dims)
    circ = frozenset(int(a) for a in circular)
    ext = tuple(n if d in circ else n - k + 1 for d, (n, k) in enumerate(zip(dims, kext)))
    if any(e < 1 for e in ext):
        raise OracleError("kernel larger than array")
    return Geom(dims, support_positions(kext, support), (0,) * len(dims), ext, circ)


def _window(entry, n_d, k_d):
    # solver.py:104-124 (Python round() is banker's rounding, kept on purpose)
    if entry == "full":
        return n_d
    if isinstance(entry, bool):
        raise OracleError("bad region entry")
    if isinstance(entry, int):
        w = entry
    elif isinstance(entry, (float, Fraction)):
        f = float(entry)
        if not (0.0 < f <= 1.0):
            raise OracleError("fraction out of range")
        w = int(round(f * n_d))
    else:
        raise OracleError("bad region entry")
    if w < k_d or w > n_d:
        raise OracleError("window out of range")
    return w


def stage_geom(dims, kext, fraction, circular=(), support=None) -> Geom:
    """Centered stage region (solver.py:127-158): offset (N-w)//2, extent w-K+1."""
    dims = tuple(int(d) for d in dims)
    nd = len(dims)
    circ = frozenset(int(a) % nd for a in circular)
    entries = ["full"] * nd if fraction == "full" else list(fraction) + ["full"] * (nd - len(fraction))
    offs, exts = [], []
    for d, (n_d, k_d) in enumerate(zip(dims, kext)):
        if k_d > n_d:
            raise OracleError("kernel exceeds array")
        if d in circ:
            offs.append(0)
            exts.append(n_d)
            continue
        w = _window("full" if d == nd - 1 else entries[d], n_d, k_d)
        offs.append((n_d - w) // 2)
        exts.append(w - k_d + 1)
    return Geom(dims, support_positions(kext, support), tuple(offs), tuple(exts), circ)


def _row_cache(geom: Geom):
    """Per-geometry cache: flat base offset of every region row over the
    non-circular axes, the region coordinates on circular axes, strides."""
    c = getattr(geom, "_cache", None)
    if c is None:
        dims = geom.dims
        nd = len(dims)
        strides = np.ones(nd, np.int64)
        for d in range(nd - 2, -1, -1):
            strides[d] = strides[d + 1] * dims[d + 1]
        grids = np.meshgrid(*[np.arange(e, dtype=np.int64) for e in geom.extents], indexing="ij")
        base = np.zeros(geom.s, np.int64)
        circ = {}
        for d in range(nd):
            a = grids[d].reshape(-1) + geom.offsets[d]
            if d in geom.circular:
                circ[d] = a
            else:
                base += a * strides[d]
        c = (base, circ, strides)
        geom._cache = c
    return c


def flat_index(geom: Geom, rows_of_positions: np.ndarray) -> np.ndarray:
    """Flat k-space index of H[i, kappa] for every region row i (row-major)
    and each given support position: ``(s, c)`` int64.

    Restates the window decomposition of hankel.py:210-252 (``_axis_pieces``,
    ``_window_pieces``, ``_gather_slab``) as modular index arithmetic.
    """
    base, circ, strides = _row_cache(geom)
    pos = np.asarray(rows_of_positions, np.int64)
    koff = np.zeros(pos.shape[0], np.int64)
    for d in range(len(geom.dims)):
        if d not in circ:
            koff += pos[:, d] * strides[d]
    idx = base[:, None] + koff[None, :]
    for d, a in circ.items():
        idx += ((a[:, None] + pos[None, :, d]) % geom.dims[d]) * strides[d]
    return idx


# ---------------------------------------------------------------------------
# operators (reference hankel.py:255-558)
# ---------------------------------------------------------------------------


def _as_mat(v):
    v = np.asarray(v, np.complex128)
    return (v[:, None], True) if v.ndim == 1 else (v, False)


def hankel_apply(x, v, geom: Geom, chunk: int = 16) -> np.ndarray:
    """out[i, j] = sum_kappa X[i + kappa] v[kappa, j]  (hankel.py:255-322).

    Explicit im2col of ``chunk`` taps at a time followed by one GEMM per
    chunk, as the reference's slab path does (hankel.py:297-313)."""
    x = np.asarray(x, np.complex128).reshape(-1)
    vm, sq = _as_mat(v)
    out = np.zeros((geom.s, vm.shape[1]), np.complex128)
    for st in range(0, geom.n, chunk):
        idx = flat_index(geom, geom.positions[st:st + chunk])
        out += x[idx] @ vm[st:st + idx.shape[1]]
    return out[:, 0] if sq else out


def hankel_adjoint_apply(x, u, geom: Geom, chunk: int = 16) -> np.ndarray:
    """out[kappa, j] = sum_i conj(X[i + kappa]) u[i, j]  (hankel.py:325-391)."""
    x = np.asarray(x, np.complex128).reshape(-1)
    um, sq = _as_mat(u)
    out = np.empty((geom.n, um.shape[1]), np.complex128)
    for st in range(0, geom.n, chunk):
        idx = flat_index(geom, geom.positions[st:st + chunk])
        out[st:st + idx.shape[1]] = x[idx].conj().T @ um
    return out[:, 0] if sq else out


def kspace_adjoint_scatter(q, u, geom: Geom) -> np.ndarray:
    """out[m] = sum_k sum_{i+kappa=m} conj(q[kappa,k]) u[i,k]  (hankel.py:394-440).

    One tap at a time: t = u conj(q[kappa]) then an indexed add.  For a
    fixed tap the map i -> i + kappa is injective, so plain fancy-index
    accumulation is exact (no duplicate targets)."""
    qm, _ = _as_mat(q)
    um, _ = _as_mat(u)
    out = np.zeros(int(np.prod(geom.dims)), np.complex128)
    for row in range(geom.n):
        idx = flat_index(geom, geom.positions[row:row + 1])[:, 0]
        out[idx] += um @ np.conj(qm[row, :])
    return out.reshape(geom.dims)


def gram(x, geom: Geom, chunk: int = 64) -> np.ndarray:
    """G = H^H H (n x n).  No reference function computes this; it equals
    ``hankel_adjoint_apply(x, hankel_apply(x, I))``."""
    x = np.asarray(x, np.complex128).reshape(-1)
    h = np.empty((geom.s, geom.n), np.complex128)
    for st in range(0, geom.n, chunk):
        idx = flat_index(geom, geom.positions[st:st + chunk])
        h[:, st:st + idx.shape[1]] = x[idx]
    return h.conj().T @ h


def mask_apply(x, mask):
    """arrays.py:54-67: copy where mask==1, zero elsewhere (bit-exact)."""
    x = np.asarray(x)
    out = np.zeros_like(x)
    on = np.asarray(mask) == 1
    out[on] = x[on]
    return out


def _soft_res(y, mask, x0):
    # hankel.py:467-470
    on = np.asarray(mask) == 1
    return np.where(on, y, 0) - np.where(on, x0, 0)


def objective_and_gradient(y, qt, geom: Geom, mask, mode="hard", x0=None, lam=0.0):
    """hankel.py:473-509.  Returns (g, obj, u)."""
    y = np.asarray(y, np.complex128)
    u = hankel_apply(y, qt, geom)
    um, _ = _as_mat(u)
    obj = float(np.vdot(um, um).real)
    g = kspace_adjoint_scatter(qt, um, geom)
    if mode == "soft":
        res = _soft_res(y, mask, x0)
        obj += lam * float(np.vdot(res, res).real)
        g += lam * res
    else:
        g[np.asarray(mask) == 1] = 0.0
    return g, obj, um


def exact_line_search(y, g, qt, geom: Geom, mask, u=None, mode="hard", x0=None, lam=0.0):
    """hankel.py:512-558.  Returns (eta, num, den); raises OracleError when
    the curvature is not positive (reference: DegenerateDirectionError)."""
    if u is None:
        u = hankel_apply(y, qt, geom)
    w = hankel_apply(g, qt, geom)
    num = float(np.vdot(w, u).real)
    den = float(np.vdot(w, w).real)
    if mode == "soft":
        on = np.asarray(mask) == 1
        mg = np.where(on, g, 0)
        res = _soft_res(y, mask, x0)
        num += lam * float(np.vdot(mg, res).real)
        den += lam * float(np.vdot(mg, mg).real)
    if den <= 0.0 or not math.isfinite(den):
        raise OracleError("degenerate direction")
    return num / den, num, den


# ---------------------------------------------------------------------------
# subspace (reference subspace.py)
# ---------------------------------------------------------------------------


def rng_generator(seed: int, ids=()) -> np.random.Generator:
    """subspace.py:29-46: SeedSequence(entropy=seed, spawn_key=ids) -> PCG64."""
    ss = np.random.SeedSequence(entropy=seed, spawn_key=tuple(int(i) for i in ids))
    return np.random.Generator(np.random.PCG64(ss))


def complex_normal(gen, shape, scale=1.0) -> np.ndarray:
    """subspace.py:49-52: (N(0,1) + i N(0,1)) * sqrt(scale / 2)."""
    b = gen.standard_normal(tuple(shape) + (2,))
    return (b[..., 0] + 1j * b[..., 1]) * math.sqrt(scale / 2.0)


def rsvd_right_vectors(x, geom: Geom, r: int, seed: int, ids=()) -> np.ndarray:
    """Single-pass randomized SVD (subspace.py:67-155).

    Z = H Omega with Omega (n x l) drawn in support order (the reference
    draws it in row blocks from one generator, which is the same stream,
    subspace.py:112-116), Householder QR of Z (zgeqrf/zungqr, :132-137),
    W = H^H U (:141-145), left singular vectors of W by zgesdd (:150)."""
    n, s = geom.n, geom.s
    if not (1 <= r < n):
        raise OracleError("rank out of range")
    ell = math.ceil(1.5 * r)
    if ell > s:
        raise OracleError("sketch wider than region")
    omega = complex_normal(rng_generator(seed, ids), (n, ell), 1.0)
    z = hankel_apply(x, omega, geom)
    qr, tau, _, info = scipy.linalg.lapack.zgeqrf(np.asfortranarray(z))
    u_range, _, info = scipy.linalg.lapack.zungqr(qr, tau)
    w = hankel_adjoint_apply(x, u_range, geom)
    left, _, _, info = scipy.linalg.lapack.zgesdd(w, compute_uv=1, full_matrices=0)
    return np.ascontiguousarray(left[:, :r])


def nystrom_right_vectors(g, omega, r: int, rel_floor: float = 1e-13) -> np.ndarray:
    """The B200 route to the same subspace from the Gram matrix (no reference
    function; SURVEY §0 parity fact 1): Y = G Omega, C = Omega^H Y,
    C = E D E^H, Z = Y E D^{-1/2} (eigenvalues below rel_floor*max dropped),
    M = Z^H Z = F L F^H, V = Z F_r L_r^{-1/2}.  span(V) equals span of the
    reference's rSVD output for the same Omega (W W^H = Y C^+ Y^H)."""
    y = g @ omega
    c = omega.conj().T @ y
    c = 0.5 * (c + c.conj().T)
    d, e = np.linalg.eigh(c)
    keep = d > rel_floor * d.max()
    z = (y @ e[:, keep]) / np.sqrt(d[keep])
    m = z.conj().T @ z
    lam, f = np.linalg.eigh(0.5 * (m + m.conj().T))
    order = np.argsort(lam)[::-1][:r]
    return (z @ f[:, order]) / np.sqrt(lam[order])


def canonicalize_phases(v) -> np.ndarray:
    """Rotate each column so its largest-|.| entry (first on ties) is real
    positive.  Not a reference function: the reference keeps LAPACK zgesdd's
    phases (subspace.py:150-154), an implementation detail that the
    Householder basis depends on.  Oracle and device both apply this
    convention when compared free-running (nullspace_phase="canonical")."""
    v = np.array(v, np.complex128, copy=True)
    for j in range(v.shape[1]):
        k = int(np.argmax(np.abs(v[:, j]) ** 2))
        e = v[k, j]
        if abs(e) > 0:
            v[:, j] *= np.conj(e) / abs(e)
    return v


def householder_nullspace(v, tol: float = 1e-12) -> np.ndarray:
    """Orthonormal complement of span(v) by r complex reflections
    (subspace.py:158-212); returns Q (n x (n-r))."""
    v = np.array(v, np.complex128, order="C", copy=True)
    n, r = v.shape
    if r > n:
        raise OracleError("too many columns")
    refl = []
    for col in range(r):
        xv = v[col:, col]
        x0 = complex(xv[0])
        tail = float(np.real(np.vdot(xv[1:], xv[1:])))
        beta = math.sqrt(tail + x0.real * x0.real + x0.imag * x0.imag)
        if beta < tol:
            raise OracleError("dependent column")
        if tail == 0.0 and x0.imag == 0.0 and x0.real >= 0.0:
            refl.append(None)
            continue
        if x0.real > 0.0:
            u0 = (-tail + 2j * beta * x0.imag) / (np.conj(x0) + beta)
        else:
            u0 = x0 - beta
        w = xv.copy()
        w[0] = u0
        w /= u0
        tau = (beta - np.conj(x0)) / beta
        if col + 1 < r:
            rest = v[col:, col + 1:]
            rest -= np.outer(tau * w, w.conj() @ rest)
        refl.append((w, tau))
    q = np.zeros((n, n - r), np.complex128)
    q[r:, :] = np.eye(n - r)
    for col in range(r - 1, -1, -1):
        if refl[col] is None:
            continue
        w, tau = refl[col]
        blk = q[col:, :]
        blk -= np.outer(np.conj(tau) * w, w.conj() @ blk)
    return q


def jl_compress(q, p: int, seed: int, ids=()) -> np.ndarray:
    """Q~ = Q P with P ~ CN(0, 1/p) drawn from stream ids (subspace.py:215-229)."""
    if p < 1:
        raise OracleError("p must be >= 1")
    proj = complex_normal(rng_generator(seed, ids), (q.shape[1], p), 1.0 / p)
    return np.asarray(q, np.complex128) @ proj


# ---------------------------------------------------------------------------
# solver (reference solver.py:258-398)
# ---------------------------------------------------------------------------


def ser_db(reference, est) -> float:
    """solver.py:251-255."""
    err = float(np.linalg.norm(np.asarray(est) - np.asarray(reference)))
    if err == 0.0:
        return float("inf")
    return 20.0 * math.log10(float(np.linalg.norm(reference)) / err)


def hicu_reconstruct(x0, mask, kext, stages, rank, circular=(), dc_mode="hard", dc_lambda=0.0,
                     seed=0, support=None, nullspace="rsvd", inject_v=None, trace=None, v_log=None,
                     canonical=False):
    """Algorithm 1 driver restated from solver.py:258-398.

    ``stages`` is a list of ``(region, p, gradient_steps, iterations)``.
    ``nullspace="rsvd"`` follows the reference (subspace.py:67); "nystrom"
    follows the B200 route (Gram + Nystrom) in fp64.  ``inject_v(si, it)``
    may return a V to use instead (lockstep parity); ``v_log`` (a dict) receives
    the V used at each (stage, iteration); ``canonical=True`` applies
    :func:`canonicalize_phases` to V (the device convention).  ``trace`` (a list) gets one dict
    per step with eta/objective values.  Returns (xhat, trace)."""
    x0 = np.ascontiguousarray(x0, dtype=np.complex128)
    mask = np.asarray(mask)
    if x0.shape != mask.shape:
        raise OracleError("mask shape mismatch")
    geoms = [stage_geom(x0.shape, kext, st[0], circular, support) for st in stages]
    n = geoms[0].n
    if rank < 1 or rank >= n:
        raise OracleError("rank out of range")
    for gm in geoms:
        if math.ceil(1.5 * rank) > gm.s:
            raise OracleError("sketch wider than region")
    x = mask_apply(x0, mask)
    observed = mask == 1
    xdc = x if dc_mode == "soft" else None
    for si, (_, p, gsteps, iters) in enumerate(stages):
        gm = geoms[si]
        for it in range(iters):
            if inject_v is not None:
                v = inject_v(si, it)
            elif nullspace == "rsvd":
                v = rsvd_right_vectors(x, gm, rank, seed, (1, si, it))
            else:
                ell = math.ceil(1.5 * rank)
                omega = complex_normal(rng_generator(seed, (1, si, it)), (n, ell), 1.0)
                v = nystrom_right_vectors(gram(x, gm), omega, rank)
            if canonical and inject_v is None:
                v = canonicalize_phases(v)
            if v_log is not None:
                v_log[(si, it)] = v
            q = householder_nullspace(v)
            y = x
            for j in range(gsteps):
                qt = jl_compress(q, p, seed, (2, si, it, j))
                u = hankel_apply(y, qt, gm)
                obj = float(np.vdot(u, u).real)
                if dc_mode == "soft":
                    res = np.where(observed, y - xdc, 0)
                    obj += dc_lambda * float(np.vdot(res, res).real)
                g = kspace_adjoint_scatter(qt, u, gm)
                if dc_mode == "soft":
                    g += dc_lambda * res
                else:
                    g[observed] = 0.0
                num = den = 0.0
                if np.any(g):
                    w = hankel_apply(g, qt, gm)
                    num = float(np.vdot(w, u).real)
                    den = float(np.vdot(w, w).real)
                    if dc_mode == "soft":
                        mg = np.where(observed, g, 0)
                        num += dc_lambda * float(np.vdot(mg, res).real)
                        den += dc_lambda * float(np.vdot(mg, mg).real)
                if den <= 0.0:
                    if trace is not None:
                        trace.append(dict(stage=si, iteration=it, step=j, eta=0.0,
                                          obj=obj, obj_after=obj, degenerate=True))
                    continue
                eta = num / den
                y = y - eta * g
                if trace is not None:
                    trace.append(dict(stage=si, iteration=it, step=j, eta=eta, obj=obj,
                                      obj_after=obj - num * num / den, degenerate=False))
            x = y
    return x, trace


# ---------------------------------------------------------------------------
# SVD coil compression (no reference implementation: SPEC.md:8 puts it out of
# the reference's scope; the paper applies it before recon)
# PARITY UNPINNED for this function.
# ---------------------------------------------------------------------------


def coil_compress(x, mask, nv: int):
    """Compress the coil axis (last) to ``nv`` virtual coils.

    Coil covariance over the sampled locations C = X_s^H X_s (X_s has one row
    per sampled spatial location, one column per coil), eigenvectors sorted by
    descending eigenvalue, each eigenvector's phase fixed so its
    largest-magnitude entry (first on ties) is real positive; returns
    (x @ V[:, :nv], mask[..., :nv], V)."""
    x = np.asarray(x, np.complex128)
    nc = x.shape[-1]
    m = np.asarray(mask).reshape(-1, nc)
    xs = x.reshape(-1, nc)
    sampled = m[:, 0] == 1
    c = xs[sampled].conj().T @ xs[sampled]
    lam, e = np.linalg.eigh(0.5 * (c + c.conj().T))
    order = np.argsort(lam)[::-1]
    e = e[:, order]
    for j in range(nc):
        k = int(np.argmax(np.abs(e[:, j])))
        ph = e[k, j] / abs(e[k, j])
        e[:, j] /= ph
    v = e[:, :nv]
    return (xs @ v).reshape(x.shape[:-1] + (nv,)), np.ascontiguousarray(np.asarray(mask)[..., :nv]), v
