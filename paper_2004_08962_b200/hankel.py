"""Matrix-free multi-level Hankel operators on the B200.

Mirrors the reference module ``hicu.hankel`` (hankel.py) name for name:
``KernelMask``, ``Region``, ``full_region``, ``Counters``, ``MemoryMeter``,
``DataConsistency``, ``hankel_apply``, ``hankel_adjoint_apply``,
``kspace_adjoint_scatter``, ``objective_and_gradient`` and
``exact_line_search`` keep the reference's signatures, index conventions
(row i = region block in row-major order, row kappa = kernel support in
row-major order, no flip, no conjugation in the forward map, wrap-around on
circular axes) and error behaviour.  The arithmetic runs in
``libhicu_b200.so`` (complex64 data, fp32 FMA, fp64 reductions); inputs and
outputs are numpy complex128 like the reference.  There is no CPU fallback.
"""

from __future__ import annotations

import contextlib
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import DegenerateDirectionError, ShapeError

__all__ = [
    "KernelMask",
    "Region",
    "full_region",
    "Counters",
    "MemoryMeter",
    "DataConsistency",
    "hankel_apply",
    "hankel_adjoint_apply",
    "kspace_adjoint_scatter",
    "objective_and_gradient",
    "exact_line_search",
    "DeviceGeometry",
    "device_geometry",
    "kernel_paths",
    "conv_uses_tensor_cores",
]

_PCHUNK = 16  # columns per device call (kernels are compiled for p <= 16)


@dataclass(eq=False)
class KernelMask:
    """Binary support of an annihilating kernel inside a rectangular box
    (reference hankel.py:52-100).  ``positions`` is the row-major argwhere of
    the support and fixes the row order of every kernel-coefficient matrix."""

    extents: tuple
    support: np.ndarray | None = None

    def __post_init__(self):
        self.extents = tuple(int(e) for e in self.extents)
        if any(e < 1 for e in self.extents):
            raise ShapeError(f"kernel extents must be >= 1, got {self.extents}")
        if self.support is None:
            self.support = np.ones(self.extents, dtype=np.uint8)
        else:
            self.support = np.ascontiguousarray(self.support).astype(np.uint8)
            if self.support.shape != self.extents:
                raise ShapeError("support shape does not match kernel extents")
            if not np.all((self.support == 0) | (self.support == 1)):
                raise ShapeError("kernel support must be {0,1}-valued")
        self.positions = np.argwhere(self.support == 1)
        self.n = int(self.positions.shape[0])
        if self.n < 1:
            raise ShapeError("kernel support is empty")

    @classmethod
    def full(cls, extents) -> "KernelMask":
        return cls(tuple(extents))

    @classmethod
    def ellipsoid(cls, extents) -> "KernelMask":
        """Inscribed-ellipsoid support (hankel.py:87-100)."""
        extents = tuple(int(e) for e in extents)
        grids = np.meshgrid(*[np.arange(e) for e in extents], indexing="ij")
        rho = np.zeros(extents)
        for g, e in zip(grids, extents):
            c = (e - 1) / 2.0
            half = max(e / 2.0, 0.5)
            rho += ((g - c) / half) ** 2
        return cls(extents, (rho <= 1.0 + 1e-12).astype(np.uint8))


@dataclass(eq=False)
class Region:
    """Contiguous block of valid-convolution outputs (hankel.py:103-145)."""

    offsets: tuple
    extents: tuple
    circular_axes: frozenset = field(default_factory=frozenset)

    def __post_init__(self):
        self.offsets = tuple(int(o) for o in self.offsets)
        self.extents = tuple(int(e) for e in self.extents)
        self.circular_axes = frozenset(int(a) for a in self.circular_axes)
        if len(self.offsets) != len(self.extents):
            raise ShapeError("region offsets/extents rank mismatch")
        if any(e < 1 for e in self.extents) or any(o < 0 for o in self.offsets):
            raise ShapeError(f"invalid region block {self.offsets}/{self.extents}")

    @property
    def s(self) -> int:
        return int(np.prod(self.extents))

    def validate(self, kernel: KernelMask, dims) -> None:
        dims = tuple(int(d) for d in dims)
        if len(dims) != len(self.extents) or len(dims) != len(kernel.extents):
            raise ShapeError(f"rank mismatch: dims {dims}, kernel {kernel.extents}, region {self.extents}")
        for d, (n_d, k_d) in enumerate(zip(dims, kernel.extents)):
            if k_d > n_d:
                raise ShapeError(f"kernel extent {k_d} exceeds array extent {n_d} on axis {d}")
            if d in self.circular_axes:
                if self.offsets[d] != 0 or self.extents[d] != n_d:
                    raise ShapeError(f"circular axis {d} must span the full extent with offset 0")
            elif self.offsets[d] + self.extents[d] > n_d - k_d + 1:
                raise ShapeError(
                    f"region exceeds valid outputs on axis {d}: "
                    f"{self.offsets[d]}+{self.extents[d]} > {n_d - k_d + 1}"
                )


def full_region(dims, kernel: KernelMask, circular_axes=()) -> Region:
    """All valid outputs, full extent on circular axes (hankel.py:148-157)."""
    circ = frozenset(int(a) for a in circular_axes)
    extents = tuple(n_d if d in circ else n_d - k_d + 1 for d, (n_d, k_d) in enumerate(zip(dims, kernel.extents)))
    if any(e < 1 for e in extents):
        bad = next(d for d, e in enumerate(extents) if e < 1)
        raise ShapeError(f"kernel extent {kernel.extents[bad]} exceeds array extent {dims[bad]} on axis {bad}")
    region = Region((0,) * len(extents), extents, circ)
    region.validate(kernel, tuple(dims))
    return region


class Counters:
    """Operator applications, one per kernel column (hankel.py:160-179).

    ``gram`` counts Gram builds; the B200 nullspace step forms ``H^H H``
    instead of the reference's l forward + l adjoint sketch passes, so
    ``forward``/``kernel_adjoint`` do not include rSVD applications."""

    __slots__ = ("forward", "kernel_adjoint", "kspace_scatter", "gram")

    def __init__(self):
        self.forward = 0
        self.kernel_adjoint = 0
        self.kspace_scatter = 0
        self.gram = 0

    @property
    def adjoint_total(self) -> int:
        return self.kernel_adjoint + self.kspace_scatter

    def snapshot(self) -> dict:
        return {
            "forward": self.forward,
            "kernel_adjoint": self.kernel_adjoint,
            "kspace_scatter": self.kspace_scatter,
            "gram": self.gram,
        }


class MemoryMeter:
    """Live auxiliary buffer sizes in complex units (hankel.py:182-203)."""

    __slots__ = ("current", "peak")

    def __init__(self):
        self.current = 0
        self.peak = 0

    def alloc(self, n_complex: int) -> int:
        self.current += int(n_complex)
        if self.current > self.peak:
            self.peak = self.current
        return int(n_complex)

    def free(self, n_complex: int) -> None:
        self.current -= int(n_complex)


@dataclass
class DataConsistency:
    """Hard/soft data consistency (hankel.py:443-464)."""

    mode: str
    mask: np.ndarray
    x0: np.ndarray | None = None
    lam: float = 0.0

    def __post_init__(self):
        if self.mode not in ("hard", "soft"):
            raise ShapeError(f"unknown data-consistency mode {self.mode!r}")
        if self.mode == "soft":
            if self.x0 is None:
                raise ShapeError("soft data consistency requires x0")
            if self.lam <= 0:
                raise ShapeError("soft data consistency requires lam > 0")


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------


class DeviceGeometry:
    """Kernel support tables and the ``hicu_geom`` struct for one
    (kernel, region, dims) triple, resident on the current CUDA device."""

    def __init__(self, kernel: KernelMask, region: Region, dims):
        torch = nat.require_cuda()
        dims = tuple(int(d) for d in dims)
        nd = len(dims)
        if nd > nat.MAX_NDIM:
            raise ShapeError(f"at most {nat.MAX_NDIM} axes are supported")
        strides = np.ones(nd, np.int64)
        for d in range(nd - 2, -1, -1):
            strides[d] = strides[d + 1] * dims[d + 1]
        pos = np.ascontiguousarray(kernel.positions.astype(np.int32))
        koff = np.zeros(kernel.n, np.int64)
        for d in range(nd):
            if d not in region.circular_axes:
                koff += pos[:, d].astype(np.int64) * strides[d]
        self.dims = dims
        self.N = int(np.prod(dims))
        self.s = region.s
        self.n = kernel.n
        self.pos_t = torch.from_numpy(pos).cuda()
        self.koff_t = torch.from_numpy(koff).cuda()
        g = nat.HicuGeom()
        g.ndim = nd
        g.n = kernel.n
        for d in range(nd):
            g.dims[d] = dims[d]
            g.roff[d] = region.offsets[d]
            g.rext[d] = region.extents[d]
        g.circular = sum(1 << a for a in region.circular_axes)
        g.flags = (nat.GEOM_COIL_SEPARABLE if _coil_separable(kernel, dims) else 0) | _PATH_FLAGS
        g.pos = self.pos_t.data_ptr()
        g.koff = self.koff_t.data_ptr()
        for d in range(nd):
            g.kext[d] = int(kernel.extents[d])
        self.struct = g
        L = nat.lib()
        self.conv_nparts = L.hicu_conv_nparts(self.ref())
        self.scatter_nparts = L.hicu_scatter_nparts(self.ref())

    def ref(self):
        import ctypes

        return ctypes.byref(self.struct)


def _coil_separable(kernel: KernelMask, dims) -> bool:
    """True when the support is (spatial support) x (all coils): kappa =
    sp*Nc + c.  Enables the coil-vectorised device kernels."""
    nc = int(dims[-1])
    if len(dims) < 2 or kernel.extents[-1] != nc or kernel.n % nc != 0:
        return False
    pos = kernel.positions
    c = np.arange(kernel.n) % nc
    if not np.array_equal(pos[:, -1], c):
        return False
    sp = pos[::nc, :-1]
    return bool(np.array_equal(pos[:, :-1], np.repeat(sp, nc, axis=0)))


_GEOM_CACHE: dict = {}
_PATH_FLAGS = 0


@contextlib.contextmanager
def kernel_paths(simt_conv: bool = False, simt_gram: bool = False, dense_gram: bool = False,
                 ffma_lag: bool = False):
    """Select the SIMT conv/scatter and/or Gram kernels even where the
    tcgen05 kernels apply, the dense implicit-im2col Gram instead of the
    lag Gram, or the CUDA-core lag Gram core instead of its tensor-core form
    (cross-checks and A/B timing).  Geometries built inside the context
    carry the choice; the cache keys on it."""
    global _PATH_FLAGS
    old = _PATH_FLAGS
    _PATH_FLAGS = ((nat.GEOM_FORCE_SIMT_CONV if simt_conv else 0) | (nat.GEOM_FORCE_SIMT_GRAM if simt_gram else 0)
                   | (nat.GEOM_FORCE_DENSE_GRAM if (dense_gram or simt_gram) else 0)
                   | (nat.GEOM_FORCE_FFMA_LAG if ffma_lag else 0))
    try:
        yield
    finally:
        _PATH_FLAGS = old


def device_geometry(kernel: KernelMask, region: Region, dims) -> DeviceGeometry:
    torch = nat.require_cuda()

    key = (kernel.positions.tobytes(), kernel.positions.shape, region.offsets, region.extents,
           tuple(sorted(region.circular_axes)), tuple(int(d) for d in dims), torch.cuda.current_device(),
           _PATH_FLAGS)
    dg = _GEOM_CACHE.get(key)
    if dg is None:
        if len(_GEOM_CACHE) > 64:
            _GEOM_CACHE.clear()
        dg = DeviceGeometry(kernel, region, dims)
        _GEOM_CACHE[key] = dg
    return dg


def conv_uses_tensor_cores(kernel: KernelMask, region: Region, dims, p: int = 8) -> bool:
    """True when conv / ELS / scatter with ``p`` columns run on the tcgen05
    kernels (``csrc/conv_tc.cu``) for this geometry."""
    dg = device_geometry(kernel, region, dims)
    return bool(nat.lib().hicu_conv_uses_tensor_cores(dg.ref(), int(p)))


def to_dev(a, dtype_np=np.complex64):
    """numpy/torch array -> contiguous CUDA tensor of the matching torch dtype."""
    import torch

    tdt = {np.complex64: torch.complex64, np.complex128: torch.complex128, np.uint8: torch.uint8,
           np.float64: torch.float64}[dtype_np]
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=tdt).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype_np)).cuda()


def _sum_parts(t, stride: int, off: int) -> float:
    """Fixed-order fp64 sum of a partial-sum buffer on the host."""
    v = t.cpu().numpy().reshape(-1, stride)[:, off]
    return float(math.fsum(v.tolist()))


def _check_operands(x, kernel: KernelMask, region: Region):
    shape = tuple(x.shape)
    region.validate(kernel, shape)
    return shape


def _as_mat(v):
    v = np.asarray(v, dtype=np.complex128)
    return (v[:, None], True) if v.ndim == 1 else (v, False)


def _fwd_device(xd, vmat, dg: DeviceGeometry, want_obj=False):
    """u = H(x) v on the device in column chunks of 16; returns (u_dev, obj)."""
    torch = nat.require_cuda()
    L = nat.lib()
    st = nat.stream_handle()
    k = vmat.shape[1]
    out = torch.empty((dg.s, k), dtype=torch.complex64, device="cuda")
    parts = torch.empty(max(dg.conv_nparts, 1), dtype=torch.float64, device="cuda")
    obj = 0.0
    for c0 in range(0, k, _PCHUNK):
        kc = min(_PCHUNK, k - c0)
        vd = to_dev(vmat[:, c0:c0 + kc])
        ud = torch.empty((dg.s, kc), dtype=torch.complex64, device="cuda")
        nat.check(L.hicu_conv_fwd(dg.ref(), xd.data_ptr(), vd.data_ptr(), kc, ud.data_ptr(), parts.data_ptr(), st),
                  "hankel_apply")
        out[:, c0:c0 + kc] = ud
        if want_obj:
            obj += _sum_parts(parts, 1, 0)
    return out, obj


def hankel_apply(x, v, kernel: KernelMask, region: Region, pos_chunk: int = 16,
                 counters: Counters | None = None, meter: MemoryMeter | None = None) -> np.ndarray:
    """out[i, j] = sum_kappa X[i + kappa] v[kappa, j] (hankel.py:255-322).

    ``pos_chunk`` is accepted for signature compatibility; the device kernel
    is matrix-free (implicit im2col) for every value."""
    x = np.asarray(x)
    dims = _check_operands(x, kernel, region)
    vmat, squeeze = _as_mat(v)
    if vmat.shape[0] != kernel.n:
        raise ShapeError(f"kernel matrix has {vmat.shape[0]} rows, support size is {kernel.n}")
    k = vmat.shape[1]
    if counters is not None:
        counters.forward += k
    if meter is not None:
        held = meter.alloc(region.s * k)
    dg = device_geometry(kernel, region, dims)
    out, _ = _fwd_device(to_dev(x), vmat, dg)
    res = out.cpu().numpy().astype(np.complex128)
    if meter is not None:
        meter.free(held)
    return res[:, 0] if squeeze else res


def hankel_adjoint_apply(x, u, kernel: KernelMask, region: Region, pos_chunk: int = 16,
                         counters: Counters | None = None, meter: MemoryMeter | None = None) -> np.ndarray:
    """out[kappa, j] = sum_{i in S} conj(X[i + kappa]) u[i, j] (hankel.py:325-391)."""
    torch = nat.require_cuda()
    x = np.asarray(x)
    dims = _check_operands(x, kernel, region)
    umat, squeeze = _as_mat(u)
    if umat.shape[0] != region.s:
        raise ShapeError(f"u has {umat.shape[0]} rows, region size is {region.s}")
    k = umat.shape[1]
    if counters is not None:
        counters.kernel_adjoint += k
    dg = device_geometry(kernel, region, dims)
    out = torch.empty((kernel.n, k), dtype=torch.complex128, device="cuda")
    L = nat.lib()
    xd, ud = to_dev(x), to_dev(umat)  # keep the device copies alive across the launch
    nat.check(L.hicu_conv_adj(dg.ref(), xd.data_ptr(), ud.data_ptr(), k, out.data_ptr(),
                              nat.stream_handle()), "hankel_adjoint_apply")
    res = out.cpu().numpy()
    return res[:, 0] if squeeze else res


def _scatter_device(qmat, ud, dg: DeviceGeometry, dc_mode=2, maskd=None, yd=None, x0d=None, lam=0.0):
    """g = scatter(q, u) (+DC) on the device; returns (g_dev, parts_dev)."""
    torch = nat.require_cuda()
    L = nat.lib()
    st = nat.stream_handle()
    k = qmat.shape[1]
    g = torch.zeros(dg.N, dtype=torch.complex64, device="cuda")
    parts = torch.zeros(4 * max(dg.scatter_nparts, 1), dtype=torch.float64, device="cuda")
    if k <= _PCHUNK:
        qd = to_dev(qmat)
        nat.check(L.hicu_scatter_dc(dg.ref(), qd.data_ptr(), k, ud.contiguous().data_ptr(),
                                    maskd.data_ptr() if maskd is not None else None,
                                    yd.data_ptr() if yd is not None else None,
                                    x0d.data_ptr() if x0d is not None else None, dc_mode, float(lam), g.data_ptr(),
                                    parts.data_ptr(), st), "kspace_adjoint_scatter")
        return g, parts
    # wide q: scatter column chunks without DC, then apply DC with one more call at width 1
    acc = torch.zeros(dg.N, dtype=torch.complex64, device="cuda")
    for c0 in range(0, k, _PCHUNK):
        kc = min(_PCHUNK, k - c0)
        gc, _ = _scatter_device(qmat[:, c0:c0 + kc], ud[:, c0:c0 + kc].contiguous(), dg)
        acc += gc
    if dc_mode == 2:
        return acc, parts
    raise ShapeError("data consistency with more than 16 kernel columns is not supported")


def kspace_adjoint_scatter(q, u, kernel: KernelMask, region: Region, dims, counters: Counters | None = None,
                           meter: MemoryMeter | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """Adjoint of X -> hankel_apply(X, q) (hankel.py:394-440)."""
    dims = tuple(int(d) for d in dims)
    qmat, _ = _as_mat(q)
    umat, _ = _as_mat(u)
    if qmat.shape[0] != kernel.n:
        raise ShapeError(f"q has {qmat.shape[0]} rows, support size is {kernel.n}")
    if umat.shape[0] != region.s:
        raise ShapeError(f"u has {umat.shape[0]} rows, region size is {region.s}")
    if qmat.shape[1] != umat.shape[1]:
        raise ShapeError("q and u must have the same number of columns")
    region.validate(kernel, dims)
    if out is not None and tuple(out.shape) != dims:
        raise ShapeError("out has wrong shape")
    if counters is not None:
        counters.kspace_scatter += qmat.shape[1]
    dg = device_geometry(kernel, region, dims)
    g, _ = _scatter_device(qmat, to_dev(umat), dg)
    res = g.cpu().numpy().astype(np.complex128).reshape(dims)
    if out is not None:
        out += res
        return out
    return res


def objective_and_gradient(y, qt, kernel: KernelMask, region: Region, dc: DataConsistency,
                           counters: Counters | None = None, meter: MemoryMeter | None = None,
                           return_products: bool = False):
    """Objective sum_k ||H(y) qt_k||^2 (+ soft penalty) and its gradient
    (hankel.py:473-509); returns (g, obj[, u])."""
    y = np.asarray(y, dtype=np.complex128)
    if y.shape != np.asarray(dc.mask).shape:
        raise ShapeError("mask shape does not match iterate shape")
    dims = _check_operands(y, kernel, region)
    qmat, _ = _as_mat(qt)
    if qmat.shape[0] != kernel.n:
        raise ShapeError(f"kernel matrix has {qmat.shape[0]} rows, support size is {kernel.n}")
    if qmat.shape[1] > _PCHUNK:
        raise ShapeError("at most 16 kernel columns per gradient evaluation")
    k = qmat.shape[1]
    if counters is not None:
        counters.forward += k
        counters.kspace_scatter += k
    dg = device_geometry(kernel, region, dims)
    yd = to_dev(y)
    ud, obj = _fwd_device(yd, qmat, dg, want_obj=True)
    maskd = to_dev(dc.mask, np.uint8)
    soft = dc.mode == "soft"
    x0d = to_dev(dc.x0) if soft else None
    g, parts = _scatter_device(qmat, ud, dg, 1 if soft else 0, maskd, yd, x0d, dc.lam if soft else 0.0)
    if soft:
        obj += dc.lam * _sum_parts(parts, 4, 1)
    grad = g.cpu().numpy().astype(np.complex128).reshape(dims)
    if return_products:
        return grad, obj, ud.cpu().numpy().astype(np.complex128)
    return grad, obj


def exact_line_search(y, g, qt, kernel: KernelMask, region: Region, dc: DataConsistency, u=None,
                      counters: Counters | None = None, meter: MemoryMeter | None = None,
                      return_decrease: bool = False):
    """eta* = (sum Re<w,u> + soft) / (sum |w|^2 + soft) (hankel.py:512-558)."""
    torch = nat.require_cuda()
    y = np.asarray(y, dtype=np.complex128)
    g = np.asarray(g, dtype=np.complex128)
    dims = _check_operands(y, kernel, region)
    qmat, _ = _as_mat(qt)
    if qmat.shape[1] > _PCHUNK:
        raise ShapeError("at most 16 kernel columns per line search")
    k = qmat.shape[1]
    dg = device_geometry(kernel, region, dims)
    yd = to_dev(y)
    if u is None:
        if counters is not None:
            counters.forward += k
        ud, _ = _fwd_device(yd, qmat, dg)
    else:
        ud = to_dev(np.asarray(u, dtype=np.complex128).reshape(region.s, k))
    if counters is not None:
        counters.forward += k
    L = nat.lib()
    st = nat.stream_handle()
    gd = to_dev(g)
    parts = torch.empty(2 * max(dg.conv_nparts, 1), dtype=torch.float64, device="cuda")
    qd = to_dev(qmat)
    nat.check(L.hicu_conv_els(dg.ref(), gd.data_ptr(), qd.data_ptr(), k, ud.data_ptr(), parts.data_ptr(),
                              st), "exact_line_search")
    num = _sum_parts(parts, 2, 0)
    den = _sum_parts(parts, 2, 1)
    if dc.mode == "soft":
        import ctypes

        sp = torch.empty(3 * nat.lib().hicu_ser_nparts(dg.N), dtype=torch.float64, device="cuda")
        npt = ctypes.c_int(0)
        x0d, md = to_dev(dc.x0), to_dev(dc.mask, np.uint8)
        nat.check(L.hicu_soft_terms(dg.N, gd.data_ptr(), yd.data_ptr(), x0d.data_ptr(),
                                    md.data_ptr(), sp.data_ptr(), ctypes.byref(npt), st),
                  "exact_line_search")
        num += dc.lam * _sum_parts(sp, 3, 0)
        den += dc.lam * _sum_parts(sp, 3, 1)
    if den <= 0.0 or not math.isfinite(den):
        raise DegenerateDirectionError("line-search curvature is zero; direction is annihilated")
    eta = num / den
    if return_decrease:
        return eta, num * num / den
    return eta
