"""Gram accuracy against an fp64 torch reference at full config sizes
(the CPU oracle is too slow there).  G64 = sum over region rows of
conj(P)^T P with P the complex128 patch matrix, built in row chunks from an
as_strided view of the k-space (positions in KernelMask order: taps row-major,
coil fastest).  Prints one JSON line per case."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2004_08962_b200 as H


def g64(x, kext, chunk=4096):
    sp = x.shape[:-1]
    ks = kext[:-1]
    out = tuple(s - k + 1 for s, k in zip(sp, ks))
    st = x.stride()
    v = x.as_strided(out + tuple(ks) + (x.shape[-1],), st[:-1] + st[:-1] + (st[-1],))
    n = int(np.prod(kext))
    v = v.reshape(-1, n) if v.is_contiguous() else v.reshape(int(np.prod(out)), n)
    G = torch.zeros((n, n), dtype=torch.complex128, device=x.device)
    for i in range(0, v.shape[0], chunk):
        P = v[i:i + chunk].to(torch.complex128)
        G += P.conj().T @ P
    return G


def case(tag, dims, kext):
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(dims, dtype=torch.complex64, device="cuda", generator=g)
    kernel = H.KernelMask.full(kext)
    region = H.full_region(dims, kernel)
    Gt = H.gram_matrix(x, kernel, region)
    Gs = H.gram_matrix(x, kernel, region, force_simt=True)
    Gr = g64(x, kext)
    sc = float(Gr.abs().max())
    print(json.dumps({"case": tag, "n": kernel.n, "rows": region.s,
                      "tc_vs_fp64": float((Gt - Gr).abs().max()) / sc,
                      "simt_vs_fp64": float((Gs - Gr).abs().max()) / sc}), flush=True)


if __name__ == "__main__":
    case("C2_full", (256, 256, 8), (5, 5, 8))
    case("C5_shard_small", (12, 40, 40, 8), (5, 5, 5, 8))
    case("C5_shard", (36, 160, 160, 8), (5, 5, 5, 8))
