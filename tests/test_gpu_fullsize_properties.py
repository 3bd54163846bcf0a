"""Size-independent properties of the hot-path operators at BASELINE.json's
FULL sizes (C3 slice, C4 series, C5 volume), where the CPU oracle cannot run
in test time.  Each property ties independently written kernels together:

* adjointness  <H(x) q, u> = <x, scatter(q, u)>  (forward convolution against
  the k-space scatter; reference pkg/src/hicu/hankel.py:255-322 / :394-440),
* the Gram identity  ||H(x) q||_F^2 = Re tr(q^H G q)  (forward convolution
  against the Gram build, hankel.py:325-391 applied to the identity),
* linearity of the forward convolution in x,
* one full-size outer iteration of hicu_reconstruct: hard data consistency is
  bit-exact on the observed samples and the exact line search decreases the
  objective (solver.py:323-372).

The checker side is torch complex128 inner products over device buffers; the
operators under test run through the C ABI."""

import numpy as np
import pytest

import paper_2004_08962_b200 as H
from paper_2004_08962_b200 import hankel as HK
from paper_2004_08962_b200.subspace import gram_matrix, gram_path

pytestmark = pytest.mark.gpu

FULL = {
    # name: dims, kernel extents, p
    "C3": ((320, 320, 10), (7, 7, 10), 10),
    "C4": ((192, 144, 25, 8), (5, 5, 5, 8), 8),
    "C5": ((256, 160, 160, 8), (5, 5, 5, 8), 8),
}


def _rand_c64(torch, gen, shape):
    re = torch.randn(shape, generator=gen, device="cuda", dtype=torch.float32)
    im = torch.randn(shape, generator=gen, device="cuda", dtype=torch.float32)
    return torch.complex(re, im)


def _vdot(torch, a, b):
    """<a, b> = sum conj(a) b in complex128, chunked (the test's checker)."""
    a = a.reshape(-1)
    b = b.reshape(-1)
    acc = torch.zeros((), dtype=torch.complex128, device="cuda")
    step = 1 << 26
    for i in range(0, a.numel(), step):
        acc += torch.vdot(a[i:i + step].to(torch.complex128), b[i:i + step].to(torch.complex128))
    return complex(acc.item())


@pytest.mark.parametrize("name", list(FULL))
def test_fullsize_adjointness_gram_identity_linearity(name):
    import torch

    dims, kext, p = FULL[name]
    kernel = H.KernelMask.full(kext)
    region = H.full_region(dims, kernel)
    dg = HK.device_geometry(kernel, region, dims)
    assert H.conv_uses_tensor_cores(kernel, region, dims, p), "the full-size configs run the tcgen05 convolutions"
    gen = torch.Generator(device="cuda").manual_seed(17)
    rng = np.random.default_rng(5)
    x = _rand_c64(torch, gen, dims)
    q = (rng.standard_normal((kernel.n, p)) + 1j * rng.standard_normal((kernel.n, p))).astype(np.complex64)
    q = q.astype(np.complex128)
    u, obj = HK._fwd_device(x.reshape(-1), q, dg, want_obj=True)
    assert tuple(u.shape) == (region.s, p)

    # the fused objective is ||u||^2
    uu = _vdot(torch, u, u).real
    assert abs(obj - uu) <= 1e-6 * uu, (obj, uu)

    # adjointness against the scatter (no DC: dc_mode 2)
    w = _rand_c64(torch, gen, (region.s, p))
    g, _ = HK._scatter_device(q, w, dg)
    lhs = _vdot(torch, w, u)            # <w, H(x) q>
    rhs = _vdot(torch, g, x)            # <scatter(q, w), x>
    scale = (uu * _vdot(torch, w, w).real) ** 0.5
    assert abs(lhs - rhs) <= 1e-5 * scale, (lhs, rhs, scale)

    # Gram identity: the lag / dense Gram against the convolution
    G = gram_matrix(x, kernel, region)
    qd = torch.as_tensor(q, device="cuda")
    tr = float(torch.einsum("ij,ik,kj->", qd.conj(), G, qd).real.item())
    print(f"{name}: gram path {gram_path(kernel, region, dims)}, ||Hq||^2 {uu:.6e}, tr {tr:.6e}")
    assert abs(tr - uu) <= 1e-5 * uu, (tr, uu)
    assert torch.equal(G, G.conj().T)

    # linearity in x
    x2 = _rand_c64(torch, gen, dims)
    a, b = 0.75 - 0.5j, -1.25 + 0.25j
    u2, _ = HK._fwd_device(x2.reshape(-1), q, dg)
    u12, _ = HK._fwd_device((a * x + b * x2).reshape(-1), q, dg)
    err = float((u12 - (a * u + b * u2)).abs().max() / u12.abs().max())
    assert err <= 1e-5, err


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_fullsize_one_iteration_hard_dc_and_descent(name):
    from paper_2004_08962_b200.synthetic import make_config

    dims, kext, p = FULL[name]
    ksp, mask, x0 = make_config(name)
    if ksp.shape[-1] != dims[-1]:
        # C4: 12 physical coils compressed to 8 virtual coils with one basis
        # (from the acquired samples) for the input and the truth
        x0, mask, basis = H.coil_compress(x0, mask, dims[-1])
        x0 = x0.astype(np.complex64)
        ksp = (ksp.astype(np.complex128) @ basis).astype(np.complex64)
    assert tuple(ksp.shape) == dims and tuple(x0.shape) == dims
    kernel = H.KernelMask.full(kext)
    rank = {"C4": 150, "C5": 120}[name]
    sched = H.SolverSchedule(rank=rank, stages=[H.StageSpec("full", p, 3, 1)], seed=11)
    xg, rep = H.hicu_reconstruct(x0, mask, kernel, sched, tail_energy_threshold=0)
    obs = mask == 1
    assert np.array_equal(xg[obs], np.asarray(x0)[obs]), "hard data consistency is not bit-exact"
    assert len(rep.steps) == 3
    for s in rep.steps:
        assert s.eta > 0 and s.objective_after < s.objective_before
    # a recovered iterate is closer to the fully sampled k-space than the zero-filled input
    e0 = np.linalg.norm(np.asarray(x0) - ksp)
    e1 = np.linalg.norm(xg - ksp)
    print(f"{name}: ||x0 - truth|| {e0:.4e} -> {e1:.4e} after one outer iteration")
    assert e1 < e0
