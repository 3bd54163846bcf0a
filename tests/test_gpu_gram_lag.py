"""The shift-structured lag Gram (csrc/gram_lag.cu) against the fp64 oracle
Gram (hankel_adjoint_apply(x, hankel_apply(x, I)) restated in
oracle/hicu_oracle.py, pinned to the reference's golden Gram) on geometries
that exercise every class structure: center-out windows, windows narrower
than the kernel (no core class), circular axes (single class, wrapped lags),
ellipsoid supports, 1-3 spatial axes and the coil counts the lag kernels are
instantiated for."""

import numpy as np
import pytest

import paper_2004_08962_b200 as H
from oracle import hicu_oracle as O
from paper_2004_08962_b200.subspace import gram_matrix, gram_path

pytestmark = pytest.mark.gpu


def c64(a):
    return np.asarray(a).astype(np.complex64).astype(np.complex128)


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


CASES = [
    # dims, kernel extents, region (stage fraction or "full"), circular axes, support
    ((40, 36, 8), (5, 5, 8), "full", (), "full"),
    ((64, 64, 8), (5, 5, 8), [24, 24], (), "full"),
    ((30, 29, 10), (7, 7, 10), "full", (), "full"),              # C3 geometry (Nc = 10, CB = 5)
    ((20, 18, 9, 8), (5, 5, 5, 8), "full", (), "full"),           # C4/C5 kernel
    ((24, 20, 12, 8), (5, 5, 5, 8), [16, 12, "full"], (), "full"),  # C4 center-out stage
    ((16, 14, 10, 8), (5, 5, 5, 8), "full", (2,), "full"),       # circular time
    ((12, 11, 3), (3, 3, 3), "full", (0, 1), "full"),            # both spatial axes circular
    ((9, 9, 2), (5, 5, 2), "full", (), "ellipsoid"),
    ((10, 9, 6, 4), (3, 2, 2, 4), "full", (2,), "full"),
    ((33, 5), (6, 5), "full", (), "full"),                       # 1 spatial axis
    ((20, 20, 3), (5, 5, 3), [6, 7], (), "full"),                # windows narrower than 2K-1: no core class
    ((18, 16, 1), (4, 3, 1), "full", (), "full"),
    ((14, 13, 2), (3, 4, 2), "full", (), "full"),
    ((14, 13, 5), (3, 4, 5), "full", (), "full"),
    ((14, 13, 6), (3, 4, 6), "full", (), "full"),
    ((14, 13, 7), (3, 4, 7), "full", (), "full"),
    ((14, 13, 12), (3, 3, 12), "full", (), "full"),
    ((12, 12, 16), (3, 3, 16), "full", (), "full"),
    ((10, 10, 40, 8), (8, 3, 8, 8), "full", (), "full"),          # the largest kernel extent (8)
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_lag_gram_matches_oracle(case):
    dims, kext, frac, circ, sup = CASES[case]
    rng = np.random.default_rng(100 + case)
    x = c64(rng.standard_normal(dims) + 1j * rng.standard_normal(dims))
    k = H.KernelMask.ellipsoid(kext) if sup == "ellipsoid" else H.KernelMask.full(kext)
    reg = H.stage_region(dims, k, frac, circ)
    assert gram_path(k, reg, dims, force_lag=True) == "lag", (dims, kext)
    G = gram_matrix(x, k, reg, path="lag").cpu().numpy()
    gm = O.stage_geom(dims, kext, frac, circ, None if sup == "full" else k.support)
    Gr = O.gram(x, gm)
    err = rel(G, Gr)
    assert err <= 2e-6, err
    assert np.array_equal(G, G.conj().T)               # Hermitian by construction
    assert np.all(np.diag(G).imag == 0)
    assert np.array_equal(G, gram_matrix(x, k, reg, path="lag").cpu().numpy())  # deterministic


def test_lag_gram_c5_shard_accuracy():
    """A C5 shard (36x160x160x8 phantom k-space: the large dynamic range of a
    real acquisition) against an fp64 Gram of the same patches."""
    import torch

    from paper_2004_08962_b200.synthetic import make_config

    ksp, _, _ = make_config("C5", scale=0.25)
    x = torch.as_tensor(ksp[:20].astype(np.complex64)).cuda()
    dims, kext = tuple(x.shape), (5, 5, 5, 8)
    kernel = H.KernelMask.full(kext)
    region = H.full_region(dims, kernel)
    out = tuple(s - k + 1 for s, k in zip(dims[:-1], kext[:-1]))
    st = x.stride()
    v = x.as_strided(out + kext[:-1] + (dims[-1],), st[:-1] + st[:-1] + (st[-1],)).reshape(-1, kernel.n)
    G64 = torch.zeros((kernel.n, kernel.n), dtype=torch.complex128, device="cuda")
    for i in range(0, v.shape[0], 4096):
        P = v[i:i + 4096].to(torch.complex128)
        G64 += P.conj().T @ P
    assert gram_path(kernel, region, dims) == "lag"  # the library's choice at n = 1000
    G = gram_matrix(x, kernel, region)
    err = float((G - G64).abs().max() / G64.abs().max())
    print(f"lag Gram, C5 phantom shard {dims}: max rel err {err:.2e}")
    assert err <= 2e-6


TC_CASES = [0, 1, 3, 4, 5, 18]  # 8 coils, non-circular line axis <= 256 positions: the tensor-core core class
# (case 5: circular time as an OUTER axis -- the neighbour lines wrap)


@pytest.mark.parametrize("case", TC_CASES)
def test_lag_gram_tensor_core_matches_cuda_core(case):
    """The tcgen05 polyphase core class (lagtc_core_kernel, fp16 hi/lo
    operands) and the CUDA-core FFMA2 core class give the same Gram (both
    against the fp64 oracle)."""
    dims, kext, frac, circ, sup = CASES[case]
    rng = np.random.default_rng(300 + case)
    x = c64(rng.standard_normal(dims) + 1j * rng.standard_normal(dims))
    # a k-space-like dynamic range: one bright centre
    x[tuple(d // 2 for d in dims[:-1])] *= 300.0
    k = H.KernelMask.full(kext)
    reg = H.stage_region(dims, k, frac, circ)
    G_tc = gram_matrix(x, k, reg, path="lag").cpu().numpy()
    with H.kernel_paths(ffma_lag=True):
        G_ff = gram_matrix(x, k, reg, path="lag").cpu().numpy()
    gm = O.stage_geom(dims, kext, frac, circ, None)
    Gr = O.gram(x, gm)
    assert rel(G_ff, Gr) <= 2e-6
    assert rel(G_tc, Gr) <= 2e-6, rel(G_tc, Gr)
    assert np.array_equal(G_tc, G_tc.conj().T)
