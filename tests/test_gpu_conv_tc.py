"""tcgen05 conv / ELS / scatter kernels (csrc/conv_tc.cu) against the oracle
and against the SIMT kernels on the same complex64 inputs.

Geometries cover: 2D full and sub-region, spatial-ellipse support (ragged
groups), 1D, 3D, a support whose last-axis spread (39) forces group splitting,
region lines shorter / longer than the 128-row tile, and hard / soft / no DC.
"""

import numpy as np
import pytest

import paper_2004_08962_b200 as H
from oracle import hicu_oracle as O

pytestmark = pytest.mark.gpu

NC = 8


def spatial_kernel(sp_ext, sp_support=None, nc=NC):
    ext = tuple(sp_ext) + (nc,)
    if sp_support is None:
        sup = np.ones(ext, bool)
    else:
        sup = np.repeat(np.asarray(sp_support, bool)[..., None], nc, axis=-1)
    return H.KernelMask(ext, sup)


def ellipse(n):
    c = (n - 1) / 2
    yy, xx = np.meshgrid(np.arange(n) - c, np.arange(n) - c, indexing="ij")
    return (yy / (c + 0.5)) ** 2 + (xx / (c + 0.5)) ** 2 <= 1.0


def ellipsoid3(n):
    c = (n - 1) / 2
    z, yy, xx = np.meshgrid(*(np.arange(n) - c,) * 3, indexing="ij")
    return (z / (c + 0.5)) ** 2 + (yy / (c + 0.5)) ** 2 + (xx / (c + 0.5)) ** 2 <= 1.0


CASES = {
    # name: (spatial dims, kernel, region offsets/extents or None for full)
    "2d_full": ((70, 300), spatial_kernel((5, 5)), None),
    "2d_sub": ((64, 96), spatial_kernel((5, 5)), ((10, 20), (30, 40))),
    "2d_ell": ((40, 150), spatial_kernel((7, 7), ellipse(7)), None),   # 7 taps along the last axis: one TMEM buffer
    "2d_wide": ((20, 520), spatial_kernel((3, 8)), None),              # nb = 8 (widest), lines of 5 tiles
    "2d_short": ((30, 40), spatial_kernel((4, 2)), ((3, 5), (20, 12))),  # lines shorter than one tile
    "1d": ((700,), spatial_kernel((7,)), None),
    "3d": ((12, 10, 140), spatial_kernel((3, 3, 3)), None),
    "3d_sub": ((14, 12, 40), spatial_kernel((3, 2, 3)), ((2, 3, 5), (6, 5, 20))),
    "3d_555": ((10, 9, 140), spatial_kernel((5, 5, 5)), None),          # 125 taps: B images streamed per stage
    "3d_555_ell": ((11, 10, 40), spatial_kernel((5, 5, 5), ellipsoid3(5)), ((1, 2, 3), (5, 4, 30))),
    "2d_8x8": ((24, 150), spatial_kernel((8, 8)), None),                # 64 taps, nb = 8: streamed
    "1d_nb9": ((300,), spatial_kernel((9,)), None),                   # outside the tcgen05 scope -> SIMT
    "spread": ((6, 260), spatial_kernel((1, 40)), None),               # outside the tcgen05 scope -> SIMT
    # C4's layout (short last axis): tiles run along the 60-row axis 0, not the 9 frames
    "3d_short_last": ((60, 12, 9), spatial_kernel((5, 5, 5)), None),
}
SIMT_ONLY = {"1d_nb9", "spread"}


def make(name, seed=0):
    dims_sp, kernel, reg = CASES[name]
    dims = tuple(dims_sp) + (NC,)
    if reg is None:
        region = H.full_region(dims, kernel)
    else:
        region = H.Region(tuple(reg[0]) + (0,), tuple(reg[1]) + (1,), frozenset())
    og = O.Geom(dims, kernel.positions, region.offsets, region.extents, frozenset())
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal(dims) + 1j * rng.standard_normal(dims)).astype(np.complex64).astype(np.complex128)
    q = (rng.standard_normal((kernel.n, 8)) + 1j * rng.standard_normal((kernel.n, 8))) / np.sqrt(kernel.n)
    q = q.astype(np.complex64).astype(np.complex128)
    mask = (rng.random(dims[:-1]) < 0.3).astype(np.uint8)
    mask = np.repeat(mask[..., None], NC, axis=-1)
    x0 = x * mask
    return dims, kernel, region, og, x, q, mask, x0


def tol_for(kernel, base=2e-6):
    """fp32-grade bound for a contraction of n complex terms per output
    (accumulation error grows ~sqrt(n); the 2e-6 base covers n <= 400)."""
    return base * max(1.0, (kernel.n / 400.0) ** 0.5)


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


@pytest.mark.parametrize("name", list(CASES))
def test_tc_path_selected(name):
    dims, kernel, region, *_ = make(name)
    assert H.conv_uses_tensor_cores(kernel, region, dims, 8) == (name not in SIMT_ONLY)
    assert not H.conv_uses_tensor_cores(kernel, region, dims, 4)
    with H.kernel_paths(simt_conv=True):
        assert not H.conv_uses_tensor_cores(kernel, region, dims, 8)


@pytest.mark.parametrize("name", list(CASES))
def test_tc_conv_scatter_vs_oracle_and_simt(name):
    dims, kernel, region, og, x, q, mask, x0 = make(name)
    tol = tol_for(kernel)
    u_tc = H.hankel_apply(x, q, kernel, region)
    u_ref = O.hankel_apply(x, q, og)
    assert rel(u_tc, u_ref) <= tol
    with H.kernel_paths(simt_conv=True):
        u_simt = H.hankel_apply(x, q, kernel, region)
        g_simt = H.kspace_adjoint_scatter(q, u_ref, kernel, region, dims)
    assert rel(u_tc, u_simt) <= 2 * tol  # both paths carry fp32-grade error (each <= tol vs oracle)
    g_tc = H.kspace_adjoint_scatter(q, u_ref, kernel, region, dims)
    g_ref = O.kspace_adjoint_scatter(q, u_ref, og)
    assert rel(g_tc, g_ref) <= tol
    assert rel(g_tc, g_simt) <= 2 * tol
    # positions no tap reaches are exactly zero
    assert np.array_equal(g_tc == 0, g_ref == 0) or rel(g_tc, g_ref) <= tol


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("mode", ["hard", "soft"])
def test_tc_objective_gradient_els(name, mode):
    dims, kernel, region, og, x, q, mask, x0 = make(name, seed=1)
    tol = tol_for(kernel)
    dc = H.DataConsistency(mode, mask, x0=x0 if mode == "soft" else None, lam=0.6 if mode == "soft" else 0.0)
    g_tc, obj_tc, u_tc = H.objective_and_gradient(x, q, kernel, region, dc, return_products=True)
    eta_tc = H.exact_line_search(x, g_tc, q, kernel, region, dc, u=u_tc)
    with H.kernel_paths(simt_conv=True):
        g_s, obj_s, u_s = H.objective_and_gradient(x, q, kernel, region, dc, return_products=True)
        eta_s = H.exact_line_search(x, g_s, q, kernel, region, dc, u=u_s)
    g_o, obj_o, u_o = O.objective_and_gradient(x, q, og, mask, mode, x0 if mode == "soft" else None,
                                               0.6 if mode == "soft" else 0.0)
    eta_o = O.exact_line_search(x, g_o, q, og, mask, u_o, mode, x0 if mode == "soft" else None,
                                0.6 if mode == "soft" else 0.0)[0]
    # the gradient chains two n-term contractions; bound it by the n-scaled
    # tolerance or 1.5x the SIMT fp32 path's own error on the same inputs
    e_tc, e_simt = rel(g_tc, g_o), rel(g_s, g_o)
    assert e_tc <= max(tol, 1.5 * e_simt), (e_tc, e_simt)
    assert rel(g_tc, g_s) <= 2 * max(tol, e_simt)
    assert abs(obj_tc - obj_o) <= 2 * tol * abs(obj_o)
    assert abs(obj_tc - obj_s) <= 2 * tol * abs(obj_s)
    assert abs(eta_tc - eta_s) <= 1e-5 * abs(eta_s)
    assert abs(eta_tc - eta_o) <= 1e-5 * abs(eta_o)
    if mode == "hard":
        assert not np.any(g_tc[mask == 1])


def test_tc_deterministic():
    dims, kernel, region, og, x, q, mask, x0 = make("2d_full", seed=2)
    dc = H.DataConsistency("hard", mask)
    a = H.objective_and_gradient(x, q, kernel, region, dc)
    b = H.objective_and_gradient(x, q, kernel, region, dc)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1]


# 10 coils with p = 10 (C3's kernels: 7x7x10, rank 100): the CW = 10 kernel
# instantiations -- 20-component rows split into [32 hi | 32 lo] fp16 halves
# (SW128 operand rows, two K steps), separate hi / lo MMAs (N = 144 > 128).
NC10 = 10
CASES10 = {
    "c3_2d": ((50, 300), spatial_kernel((7, 7), nc=NC10), None),
    "2d_sub": ((64, 96), spatial_kernel((5, 5), nc=NC10), ((10, 20), (30, 40))),
    "2d_ell": ((40, 150), spatial_kernel((7, 7), ellipse(7), nc=NC10), None),
    "3d": ((12, 10, 60), spatial_kernel((3, 3, 3), nc=NC10), None),
    "2d_nb8": ((20, 200), spatial_kernel((3, 8), nc=NC10), None),
}


def make10(name, seed=0):
    dims_sp, kernel, reg = CASES10[name]
    dims = tuple(dims_sp) + (NC10,)
    if reg is None:
        region = H.full_region(dims, kernel)
    else:
        region = H.Region(tuple(reg[0]) + (0,), tuple(reg[1]) + (1,), frozenset())
    og = O.Geom(dims, kernel.positions, region.offsets, region.extents, frozenset())
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal(dims) + 1j * rng.standard_normal(dims)).astype(np.complex64).astype(np.complex128)
    q = (rng.standard_normal((kernel.n, NC10)) + 1j * rng.standard_normal((kernel.n, NC10))) / np.sqrt(kernel.n)
    q = q.astype(np.complex64).astype(np.complex128)
    mask = (rng.random(dims[:-1]) < 0.3).astype(np.uint8)
    mask = np.repeat(mask[..., None], NC10, axis=-1)
    x0 = x * mask
    return dims, kernel, region, og, x, q, mask, x0


@pytest.mark.parametrize("name", list(CASES10))
def test_tc10_path_and_conv_scatter(name):
    dims, kernel, region, og, x, q, mask, x0 = make10(name)
    assert H.conv_uses_tensor_cores(kernel, region, dims, NC10)
    assert not H.conv_uses_tensor_cores(kernel, region, dims, 8)
    tol = tol_for(kernel)
    u_tc = H.hankel_apply(x, q, kernel, region)
    u_ref = O.hankel_apply(x, q, og)
    assert rel(u_tc, u_ref) <= tol
    g_tc = H.kspace_adjoint_scatter(q, u_ref, kernel, region, dims)
    g_ref = O.kspace_adjoint_scatter(q, u_ref, og)
    assert rel(g_tc, g_ref) <= tol


@pytest.mark.parametrize("name", list(CASES10))
@pytest.mark.parametrize("mode", ["hard", "soft"])
def test_tc10_objective_gradient_els(name, mode):
    dims, kernel, region, og, x, q, mask, x0 = make10(name, seed=1)
    tol = tol_for(kernel)
    dc = H.DataConsistency(mode, mask, x0=x0 if mode == "soft" else None, lam=0.6 if mode == "soft" else 0.0)
    g_tc, obj_tc, u_tc = H.objective_and_gradient(x, q, kernel, region, dc, return_products=True)
    eta_tc = H.exact_line_search(x, g_tc, q, kernel, region, dc, u=u_tc)
    with H.kernel_paths(simt_conv=True):
        g_s, obj_s, u_s = H.objective_and_gradient(x, q, kernel, region, dc, return_products=True)
    g_o, obj_o, u_o = O.objective_and_gradient(x, q, og, mask, mode, x0 if mode == "soft" else None,
                                               0.6 if mode == "soft" else 0.0)
    eta_o = O.exact_line_search(x, g_o, q, og, mask, u_o, mode, x0 if mode == "soft" else None,
                                0.6 if mode == "soft" else 0.0)[0]
    e_tc, e_simt = rel(g_tc, g_o), rel(g_s, g_o)
    assert e_tc <= max(tol, 1.5 * e_simt), (e_tc, e_simt)
    assert abs(obj_tc - obj_o) <= 2 * tol * abs(obj_o)
    assert abs(eta_tc - eta_o) <= 1e-5 * abs(eta_o)
    if mode == "hard":
        assert not np.any(g_tc[mask == 1])
