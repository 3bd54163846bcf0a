"""Nullspace estimation on the B200: seeded streams, the rSVD subspace from
the Gram matrix, Householder complement and JL compression.

Mirrors the reference module ``hicu.subspace`` (subspace.py).  Random draws
stay on the host with the reference's exact streams (``RngStream``,
``complex_normal``), so the device sees the same sketch Omega and the same
JL matrices P as the reference for the same seed.

``rsvd_right_vectors`` keeps the reference signature but computes the
subspace as Gram + Nystrom on the device (include/hicu_b200.h:
hicu_gram, hicu_nystrom).  For the same Omega it spans the same subspace as
the reference's single-pass rSVD (subspace.py:67-155); the individual
singular-vector phases differ from LAPACK zgesdd's.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import DegenerateInputError, ParameterError
from .hankel import Counters, KernelMask, MemoryMeter, Region, device_geometry, to_dev

__all__ = [
    "nullspace_product",
    "RngStream",
    "complex_normal",
    "NullspaceBasis",
    "rsvd_right_vectors",
    "householder_nullspace",
    "jl_compress",
    "gram_matrix",
    "gram_uses_tensor_cores",
]


@dataclass(frozen=True)
class RngStream:
    """Deterministic stream addressed by a seed and integer ids
    (subspace.py:29-46): SeedSequence(entropy=seed, spawn_key=ids) -> PCG64."""

    seed: int
    ids: tuple = ()

    def child(self, *ids: int) -> "RngStream":
        return RngStream(self.seed, self.ids + tuple(int(i) for i in ids))

    def generator(self) -> np.random.Generator:
        ss = np.random.SeedSequence(entropy=self.seed, spawn_key=self.ids)
        return np.random.Generator(np.random.PCG64(ss))


def complex_normal(rng: np.random.Generator, shape, scale: float = 1.0) -> np.ndarray:
    """i.i.d. complex Gaussian, per-entry variance ``scale`` (subspace.py:49-52)."""
    block = rng.standard_normal(tuple(shape) + (2,))
    return (block[..., 0] + 1j * block[..., 1]) * math.sqrt(scale / 2.0)


@dataclass(eq=False)
class NullspaceBasis:
    """Orthonormal complement ``q`` (n x (n-r)) of the retained subspace."""

    q: np.ndarray
    r: int

    @property
    def n(self) -> int:
        return self.q.shape[0]


def gram_uses_tensor_cores(kernel: KernelMask, region: Region, dims) -> bool:
    """True when the dense Gram (``gram_matrix(..., path="tcgen05")``) runs the
    tcgen05 3xTF32 kernel for this geometry."""
    dg = device_geometry(kernel, region, tuple(dims))
    st = nat.HicuGeom.from_buffer_copy(dg.struct)
    st.flags |= nat.GEOM_FORCE_DENSE_GRAM
    import ctypes

    return bool(nat.lib().hicu_gram_uses_tensor_cores(ctypes.byref(st)))


def gram_path(kernel: KernelMask, region: Region, dims, force_lag: bool = False) -> str:
    """Which Gram kernel hicu_gram runs: "lag", "tcgen05" or "simt"."""
    import ctypes

    dg = device_geometry(kernel, region, tuple(dims))
    st = nat.HicuGeom.from_buffer_copy(dg.struct)
    if force_lag:
        st.flags |= nat.GEOM_FORCE_LAG_GRAM
    return nat.GRAM_PATHS[int(nat.lib().hicu_gram_path(ctypes.byref(st)))]


def gram_matrix(x, kernel: KernelMask, region: Region, force_simt: bool = False, path: str | None = None):
    """G = H(x)^H H(x) (n x n, complex128) on the device; returns a CUDA tensor.

    ``path`` forces an implementation for cross-checks: "simt" / "tcgen05"
    (the dense implicit-im2col Gram; "tcgen05" falls back to SIMT where the
    tensor-core kernel does not apply), "lag" (the lag Gram wherever it
    applies) or None (the library's choice, :func:`gram_path`).
    ``force_simt`` is ``path="simt"``."""
    if force_simt:
        path = "simt"
    torch = nat.require_cuda()
    x = np.asarray(x) if not isinstance(x, torch.Tensor) else x
    region.validate(kernel, tuple(x.shape))
    dg = device_geometry(kernel, region, tuple(x.shape))
    if path in ("simt", "tcgen05"):
        import copy

        dg = copy.copy(dg)
        dg.struct = nat.HicuGeom.from_buffer_copy(dg.struct)
        dg.struct.flags |= nat.GEOM_FORCE_DENSE_GRAM | (nat.GEOM_FORCE_SIMT_GRAM if path == "simt" else 0)
    elif path == "lag":
        import copy

        dg = copy.copy(dg)
        dg.struct = nat.HicuGeom.from_buffer_copy(dg.struct)
        dg.struct.flags |= nat.GEOM_FORCE_LAG_GRAM
    elif path is not None:
        raise ValueError(f"unknown Gram path {path!r}")
    L = nat.lib()
    ws_bytes = L.hicu_gram_workspace(dg.ref())
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device="cuda")
    G = torch.empty((kernel.n, kernel.n), dtype=torch.complex128, device="cuda")
    xd = to_dev(x)  # keep alive across the launch
    nat.check(L.hicu_gram(dg.ref(), xd.data_ptr(), G.data_ptr(), ws.data_ptr(), ws_bytes, nat.stream_handle()),
              "gram")
    return G


def _status(torch, st_t, what):
    v = int(st_t.item())
    if v != 0:
        raise DegenerateInputError(f"{what}: device reported {nat.lib().hicu_status_string(v).decode()}")


def rsvd_right_vectors(x, kernel: KernelMask, region: Region, r: int, rng: RngStream,
                       counters: Counters | None = None, meter: MemoryMeter | None = None) -> np.ndarray:
    """Principal r right singular vectors of the lifted matrix, sketched with
    the reference's Omega (width l = ceil(1.5 r), stream ``rng``)."""
    n = kernel.n
    s = region.s
    if not (1 <= r < n):
        raise ParameterError(f"rank must satisfy 1 <= r < n={n}, got {r}")
    ell = math.ceil(1.5 * r)
    if ell > s:
        raise ParameterError(f"sketch width {ell} exceeds region size {s}")
    torch = nat.require_cuda()
    omega = complex_normal(rng.generator(), (n, ell), 1.0)
    G = gram_matrix(x, kernel, region)
    if counters is not None:
        counters.gram += 1
    if meter is not None:
        held = meter.alloc(n * n + 3 * n * ell)
    L = nat.lib()
    ws_bytes = L.hicu_nystrom_workspace(n, ell)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    V = torch.empty((n, r), dtype=torch.complex128, device="cuda")
    st_t = torch.zeros(1, dtype=torch.int32, device="cuda")
    omd = to_dev(omega, np.complex128)
    nat.check(L.hicu_nystrom(n, ell, r, G.data_ptr(), omd.data_ptr(), V.data_ptr(),
                             ws.data_ptr(), ws_bytes, st_t.data_ptr(), nat.stream_handle()), "rsvd_right_vectors")
    _status(torch, st_t, "rsvd_right_vectors")
    if meter is not None:
        meter.free(held)
    return V.cpu().numpy()


def _reflectors(torch, vd, n, r, tol):
    L = nat.lib()
    refl = torch.empty(2 * n * r, dtype=torch.complex128, device="cuda")
    tau = torch.empty(r, dtype=torch.complex128, device="cuda")
    flags = torch.empty(r, dtype=torch.int32, device="cuda")
    st_t = torch.zeros(1, dtype=torch.int32, device="cuda")
    nat.check(L.hicu_householder(n, r, vd.data_ptr(), float(tol), refl.data_ptr(), tau.data_ptr(), flags.data_ptr(),
                                 st_t.data_ptr(), nat.stream_handle()), "householder_nullspace")
    return refl, tau, flags, st_t


def householder_nullspace(v, tol: float = 1e-12) -> NullspaceBasis:
    """Orthonormal complement of span(v) by r complex reflections
    (subspace.py:158-212), built on the device in fp64."""
    v = np.array(v, dtype=np.complex128, order="C", copy=True)
    if v.ndim != 2:
        raise DegenerateInputError("v must be a 2-D matrix")
    n, r = v.shape
    if r > n:
        raise DegenerateInputError(f"cannot have {r} orthonormal columns in dimension {n}")
    m = n - r
    if r == 0:
        return NullspaceBasis(q=np.eye(n, dtype=np.complex128), r=0)
    if m == 0:
        # every column is spanned: the complement is empty (still validate v)
        pass
    torch = nat.require_cuda()
    vd = to_dev(v, np.complex128)
    refl, tau, flags, st_t = _reflectors(torch, vd, n, r, tol)
    _status(torch, st_t, "householder_nullspace")
    if m == 0:
        return NullspaceBasis(q=np.zeros((n, 0), np.complex128), r=r)
    b = np.zeros((n, m), np.complex128)
    b[r:, :] = np.eye(m)
    bd = to_dev(b, np.complex128)
    nat.check(nat.lib().hicu_apply_reflectors(n, r, refl.data_ptr(), tau.data_ptr(), flags.data_ptr(), m,
                                              bd.data_ptr(), bd.data_ptr(), None, 0, nat.stream_handle()),
              "householder_nullspace")
    return NullspaceBasis(q=bd.cpu().numpy(), r=r)


def nullspace_product(v, proj):
    """Q P for Q = householder_nullspace(v).q and P (n - r) x m, through the
    stage driver's closed form (csrc/nsjl.cu: Q = [0; I] + A A_1^{-H} V_2^H,
    A = V - [I; 0]).  Returns (QP, closed) where ``closed`` is False when an
    LU pivot fell below the floor and the Householder kernels produced QP."""
    v = np.array(v, dtype=np.complex128, order="C", copy=True)
    proj = np.asarray(proj, dtype=np.complex128)
    n, r = v.shape
    m = proj.shape[1]
    if proj.shape[0] != n - r:
        raise ParameterError("proj must have n - r rows")
    L = nat.lib()
    if not L.hicu_nullspace_jl_supported(n, r):
        raise ParameterError(f"closed-form nullspace not supported for n={n}, r={r}")
    torch = nat.require_cuda()
    vd = to_dev(v, np.complex128)
    b = np.zeros((n, m), np.complex128)
    b[r:, :] = proj
    bd = to_dev(b, np.complex128)
    out = torch.empty((n, m), dtype=torch.complex128, device="cuda")
    flags = torch.zeros(r + 1, dtype=torch.int32, device="cuda")
    st_t = torch.zeros(1, dtype=torch.int32, device="cuda")
    wsb = int(L.hicu_nullspace_jl_workspace(n, r))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    nat.check(L.hicu_nullspace_jl_ws(n, r, vd.data_ptr(), m, bd.data_ptr(), out.data_ptr(), None, 0,
                                     flags[r:].data_ptr(), ws.data_ptr(), wsb, nat.stream_handle()),
              "nullspace_product")
    closed = int(flags[r].item()) == 0
    if not closed:
        refl, tau, fl, st_t = _reflectors(torch, vd, n, r, 1e-12)
        _status(torch, st_t, "nullspace_product")
        nat.check(L.hicu_apply_reflectors(n, r, refl.data_ptr(), tau.data_ptr(), fl.data_ptr(), m,
                                          bd.data_ptr(), out.data_ptr(), None, 0, nat.stream_handle()),
                  "nullspace_product")
    return out.cpu().numpy(), closed


def jl_compress(q, p: int, rng: RngStream) -> np.ndarray:
    """Q~ = Q P with P ~ CN(0, 1/p) from stream ``rng`` (subspace.py:215-229)."""
    if p < 1:
        raise ParameterError(f"compression dimension must be >= 1, got {p}")
    q = np.asarray(q, dtype=np.complex128)
    if q.ndim != 2 or q.shape[1] < 1:
        raise ParameterError("nullspace must have at least one column")
    torch = nat.require_cuda()
    proj = complex_normal(rng.generator(), (q.shape[1], p), 1.0 / p)
    n, m = q.shape
    out = torch.empty((n, p), dtype=torch.complex128, device="cuda")
    qd, pd = to_dev(q, np.complex128), to_dev(proj, np.complex128)
    nat.check(nat.lib().hicu_zgemm(b"N", b"N", n, p, m, qd.data_ptr(), m,
                                   pd.data_ptr(), p, out.data_ptr(), p,
                                   nat.stream_handle()), "jl_compress")
    return out.cpu().numpy()
