"""SVD coil compression on the B200 (the north star's coil-compression option).

No reference function exists (SPEC.md:8 puts coil compression outside the
reference package; the paper compresses before reconstruction,
PAPER.md:170,179,184), so parity is against the oracle restatement
``oracle.hicu_oracle.coil_compress`` only ("parity unpinned").

Algorithm: coil covariance C = sum over sampled locations of x_l^H x_l
(HBM-bound reduction, hicu_coil_cov), eigenvectors by the device Jacobi
kernel sorted by decreasing eigenvalue with the phase fixed so the
largest-magnitude entry is real positive (hicu_coil_basis), then
y_l = x_l V[:, :Nv] (hicu_coil_apply).  Sampling masks are per location and
replicated over coils (the first coil's mask entry decides).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .errors import ShapeError
from .hankel import to_dev

__all__ = ["coil_compress", "coil_compress_device"]


def coil_compress_device(xd, maskd, nc: int, nv: int, cov_from=None, cov_reduce=None):
    """Device tensors in/out: xd (nloc*nc c64), maskd (nloc*nc u8).
    Returns (y (nloc*nv c64), mask_out (nloc*nv u8), basis (nc x nv c128),
    evals (nc f64)).

    Sharded volumes: ``cov_from = (xd_owned, maskd_owned)`` restricts the
    covariance to this rank's owned samples and ``cov_reduce(cov)`` sums it
    over ranks in place, so every rank derives the same basis (the one the
    whole volume gives) and compresses its local slab, halo included."""
    torch = nat.require_cuda()
    L = nat.lib()
    st = nat.stream_handle()
    nloc = xd.numel() // nc
    ws_bytes = max(int(L.hicu_coil_workspace(nloc, nc)), int(L.hicu_coil_basis_workspace(nc)))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    cov = torch.empty((nc, nc), dtype=torch.complex128, device="cuda")
    cx, cm = cov_from if cov_from is not None else (xd, maskd)
    ncov = cx.numel() // nc
    if cov_from is not None:
        ws_bytes = max(ws_bytes, int(L.hicu_coil_workspace(ncov, nc)))
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    nat.check(L.hicu_coil_cov(ncov, nc, cx.data_ptr(), cm.data_ptr(), cov.data_ptr(), ws.data_ptr(), ws_bytes,
                              st), "coil_cov")
    if cov_reduce is not None:
        cov_reduce(cov)
    basis = torch.empty((nc, nv), dtype=torch.complex128, device="cuda")
    evals = torch.empty(nc, dtype=torch.float64, device="cuda")
    ws2 = torch.empty(int(L.hicu_coil_basis_workspace(nc)), dtype=torch.uint8, device="cuda")
    nat.check(L.hicu_coil_basis(nc, nv, cov.data_ptr(), basis.data_ptr(), evals.data_ptr(), ws2.data_ptr(),
                                ws2.numel(), st), "coil_basis")
    y = torch.empty(nloc * nv, dtype=torch.complex64, device="cuda")
    mout = torch.empty(nloc * nv, dtype=torch.uint8, device="cuda")
    nat.check(L.hicu_coil_apply(nloc, nc, nv, xd.data_ptr(), maskd.data_ptr(), basis.data_ptr(), y.data_ptr(),
                                mout.data_ptr(), st), "coil_apply")
    return y, mout, basis, evals


def coil_compress(x, mask, nv: int):
    """Compress the last (coil) axis of ``x`` to ``nv`` virtual coils.

    Returns ``(x_c (complex128, [..., nv]), mask_c (uint8, [..., nv]),
    basis (nc x nv complex128))``."""
    x = np.asarray(x)
    mask = np.asarray(mask)
    if x.shape != mask.shape:
        raise ShapeError("mask shape does not match k-space shape")
    nc = x.shape[-1]
    if not (1 <= nv <= nc):
        raise ShapeError(f"virtual coil count must be in [1, {nc}], got {nv}")
    if nc > 32:
        raise ShapeError("at most 32 physical coils are supported")
    y, mout, basis, _ = coil_compress_device(to_dev(x).reshape(-1), to_dev((mask == 1).astype(np.uint8), np.uint8)
                                             .reshape(-1), nc, nv)
    shp = x.shape[:-1] + (nv,)
    return (y.reshape(shp).cpu().numpy().astype(np.complex128), mout.reshape(shp).cpu().numpy(),
            basis.cpu().numpy())
