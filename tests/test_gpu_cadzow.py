"""Dense Cadzow baseline on the device (cadzow.py) against the reference's
own ``cadzow_complete`` (oracle.py:144-174) on the recovery problem of the
goldens (24x24x3, 5x5x3 kernel, rank 49), non-circular and circular, 12
sweeps; plus the eigensolver ABI it relies on."""

import numpy as np
import pytest

import paper_2004_08962_b200 as H
from oracle import hicu_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden_cadzow():
    from pathlib import Path

    return dict(np.load(Path(__file__).resolve().parent / "golden" / "golden_cadzow.npz", allow_pickle=False))


@pytest.mark.parametrize("name,circ", [("cadzow", ()), ("cadzow_circ", (0, 1))])
def test_cadzow_matches_reference(golden_recon, golden_cadzow, name, circ):
    g = golden_recon
    x0, mask, ref = g["lp_x0"], g["lp_mask"], g["lp_ref"]
    kern = H.KernelMask.full(tuple(g["lp_kext"]))
    norms = []
    x = H.cadzow_complete(x0, mask, kern, 49, 12, circular_axes=circ,
                          callback=lambda it, xx: norms.append(np.linalg.norm(xx)))
    want = golden_cadzow[name + "_x"]
    err = np.linalg.norm(x - want) / np.linalg.norm(want)
    print(f"{name}: rel err vs reference {err:.2e}, SER {O.ser_db(ref, x):.3f} vs {O.ser_db(ref, want):.3f} dB")
    assert err <= 1e-5  # measured 6e-7 (non-circular) and 1e-6 (circular)
    assert abs(O.ser_db(ref, x) - O.ser_db(ref, want)) <= 0.01
    assert np.allclose(norms, golden_cadzow[name + "_norms"], rtol=2e-4)
    obs = mask == 1
    assert np.array_equal(x[obs], x0[obs])


def test_eigh_top_matches_numpy():
    import torch

    from paper_2004_08962_b200 import _native as nat

    rng = np.random.default_rng(4)
    n, r = 200, 40
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    A = a @ a.conj().T
    L = nat.lib()
    Ad = torch.as_tensor(A).cuda()
    ev = torch.empty(r, dtype=torch.float64, device="cuda")
    V = torch.empty((n, r), dtype=torch.complex128, device="cuda")
    ws = torch.empty(int(L.hicu_eigh_top_workspace(n, r)), dtype=torch.uint8, device="cuda")
    nat.check(L.hicu_eigh_top(n, r, Ad.data_ptr(), ev.data_ptr(), V.data_ptr(), ws.data_ptr(), ws.numel(),
                              nat.stream_handle()))
    lam, vec = np.linalg.eigh(A)
    assert np.allclose(ev.cpu().numpy(), lam[::-1][:r], rtol=1e-10)
    Vh = V.cpu().numpy()
    P1, P2 = Vh @ Vh.conj().T, vec[:, ::-1][:, :r] @ vec[:, ::-1][:, :r].conj().T
    assert np.linalg.norm(P1 - P2, 2) <= 1e-8


def test_eigh_top_block_diagonal_identity_reflector():
    """Two decoupled Hermitian blocks: at the block boundary the column below
    the diagonal is exactly zero, so the tridiagonalisation takes its
    H = I branch (tau = 0) in the middle of the reduction -- on the cluster
    kernel that branch re-arms the split barrier without an update phase."""
    import torch

    from paper_2004_08962_b200 import _native as nat

    rng = np.random.default_rng(9)
    n1, n2, r = 60, 90, 30
    n = n1 + n2
    a1 = rng.standard_normal((n1, n1)) + 1j * rng.standard_normal((n1, n1))
    a2 = rng.standard_normal((n2, n2)) + 1j * rng.standard_normal((n2, n2))
    A = np.zeros((n, n), np.complex128)
    A[:n1, :n1] = a1 @ a1.conj().T
    A[n1:, n1:] = a2 @ a2.conj().T
    L = nat.lib()
    Ad = torch.as_tensor(A).cuda()
    ev = torch.empty(r, dtype=torch.float64, device="cuda")
    V = torch.empty((n, r), dtype=torch.complex128, device="cuda")
    ws = torch.empty(int(L.hicu_eigh_top_workspace(n, r)), dtype=torch.uint8, device="cuda")
    nat.check(L.hicu_eigh_top(n, r, Ad.data_ptr(), ev.data_ptr(), V.data_ptr(), ws.data_ptr(), ws.numel(),
                              nat.stream_handle()))
    lam, vec = np.linalg.eigh(A)
    assert np.allclose(ev.cpu().numpy(), lam[::-1][:r], rtol=1e-10)
    Vh = V.cpu().numpy()
    P1, P2 = Vh @ Vh.conj().T, vec[:, ::-1][:, :r] @ vec[:, ::-1][:, :r].conj().T
    assert np.linalg.norm(P1 - P2, 2) <= 1e-8
