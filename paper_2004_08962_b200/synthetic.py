"""Seeded synthetic inputs for the BASELINE.json configurations C1..C5.

The reference measures on in-vivo datasets that are not available (PAPER.md:
159-166); BASELINE.json instead names seeded synthetic phantoms, written here
from its text (not from the reference's simdata.py, whose phantoms differ):

* C1  128x128, 10 random ellipses (intensity U(0.2,1)), smooth random phase,
      8 Gaussian-bump coils (sigma 0.4 FOV), SNR 30 dB, 2D variable-density
      random mask R=3 (exact count, no ACS); kernel 5x5x8, rank 40.
* C2  256x256 ellipse + texture phantom, 16 coils compressed to 8, 1D
      variable-density phase-encode mask R=4 (line density
      (1 + |dk|/sigma)^-2, sigma = n/8, as the reference's vd_1d); kernel 5x5x8, rank 60, stages
      64x64 -> 128x128 -> full (25/25/50 iterations).
* C3  64 slices of 320x320, 16 coils compressed to 10, per-slice 1D random
      mask R=4; kernel 7x7x10, rank 100.
* C4  192x144x25 cine, central ellipse dilating sinusoidally (period 25),
      12 coils compressed to 8, per-frame phase-encode mask R=6 (vd_1d
      density per frame, the reference's vd_t family); kernel
      5x5x5x8, rank 150, center-region then full stages.
* C5  256x160x160 smooth-boundary ellipsoids, 8 coils with 3D Gaussian
      sensitivities, readout fully sampled, 2D Poisson-disc on the
      phase/partition plane R=5, SNR 30 dB; kernel 5x5x5x8, rank 120.

Conventions follow the reference (arrays.py:1-10,121-132): dims =
[spatial..., (time), coil], centered unitary FFT with DC at floor(N/2);
noise is scaled so 20 log10(||x|| / ||noise||) equals the SNR exactly
(simdata.py:320-335 semantics).  Seeds: phantom 1000+c, coils 2000+c, mask
3000+c, noise 4000+c for config c.  Host-side numpy; not on the hot path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = ["ConfigSpec", "CONFIGS", "make_config", "fft_kspace"]


def fft_kspace(img: np.ndarray, axes) -> np.ndarray:
    return np.fft.fftshift(np.fft.fftn(np.fft.ifftshift(img, axes=axes), axes=axes, norm="ortho"), axes=axes)


def _grid(shape):
    return np.meshgrid(*[(np.arange(n) - n // 2) / n for n in shape], indexing="ij")


def _ellipses_2d(shape, rng, count, smooth=0.0, texture=0.0):
    yy, xx = _grid(shape)
    img = np.zeros(shape)
    for _ in range(count):
        cx, cy = rng.uniform(-0.3, 0.3, 2)
        ax, ay = rng.uniform(0.05, 0.35, 2)
        th = rng.uniform(0, np.pi)
        a = rng.uniform(0.2, 1.0)
        u = ((xx - cx) * np.cos(th) + (yy - cy) * np.sin(th)) / ax
        v = (-(xx - cx) * np.sin(th) + (yy - cy) * np.cos(th)) / ay
        rho = u * u + v * v
        img += a * (1.0 / (1.0 + np.exp((rho - 1.0) / smooth)) if smooth > 0 else (rho <= 1.0))
    if texture > 0:
        f = np.fft.fftn(rng.standard_normal(shape))
        ky, kx = np.meshgrid(*[np.fft.fftfreq(n) for n in shape], indexing="ij")
        f *= np.exp(-(kx ** 2 + ky ** 2) / (2 * 0.03 ** 2))
        tex = np.real(np.fft.ifftn(f))
        tex /= np.abs(tex).max() + 1e-12
        img = img * (1.0 + texture * tex)
    return img


def _smooth_phase(shape, rng, order=2, amp=np.pi / 2):
    grids = _grid(shape)
    ph = np.zeros(shape)
    for kk in np.ndindex(*([2 * order + 1] * len(shape))):
        k = np.array(kk) - order
        c = rng.standard_normal() / (1.0 + np.sum(k * k))
        ph += c * np.cos(2 * np.pi * sum(ki * g for ki, g in zip(k, grids)) + rng.uniform(0, 2 * np.pi))
    ph *= amp / (np.abs(ph).max() + 1e-12)
    return np.exp(1j * ph)


def _gaussian_coils(shape, ncoils, rng, sigma=0.4):
    grids = _grid(shape)
    out = np.empty(tuple(shape) + (ncoils,), np.complex128)
    for c in range(ncoils):
        ang = 2 * np.pi * c / ncoils + rng.uniform(-0.3, 0.3)
        center = [0.45 * np.cos(ang), 0.45 * np.sin(ang)] + list(rng.uniform(-0.3, 0.3, max(0, len(shape) - 2)))
        r2 = sum((g - ctr) ** 2 for g, ctr in zip(grids, center))
        out[..., c] = np.exp(-r2 / (2 * sigma ** 2)) * np.exp(1j * rng.uniform(0, 2 * np.pi))
    return out


def _add_noise(x, snr_db, rng):
    n = rng.standard_normal(x.shape) + 1j * rng.standard_normal(x.shape)
    n *= np.linalg.norm(x) / np.linalg.norm(n) / (10.0 ** (snr_db / 20.0))
    return x + n


def _vd_weights(shape, power=2.0, floor=0.05):
    grids = _grid(shape)
    r = np.sqrt(sum(g * g for g in grids)) / (0.5 * math.sqrt(len(shape)))
    return floor + (1.0 - np.clip(r, 0, 1)) ** power


def _vd_line_weights(n: int, sigma_frac: float = 0.125, decay: float = 2.0):
    """Phase-encode line density (1 + |k - n/2| / sigma)^-decay with
    sigma = n/8: the reference's ``vd_1d`` family (simdata.py:229-246 states
    this density; this is an independent generator, not its code)."""
    k = np.abs(np.arange(n) - n // 2)
    return (1.0 + k / max(sigma_frac * n, 1.0)) ** (-decay)


def _weighted_pick(weights, count, rng):
    w = weights.reshape(-1)
    idx = rng.choice(w.size, size=count, replace=False, p=w / w.sum())
    m = np.zeros(w.size, np.uint8)
    m[idx] = 1
    return m.reshape(weights.shape)


def _poisson_disc(shape, count, rng):
    """Variable-density Poisson-disc-like pattern: dart throwing with a
    radius that grows away from the center, then trimmed/topped up to the
    exact count."""
    ny, nz = shape
    w = _vd_weights(shape, power=1.0, floor=0.15)
    rmin = math.sqrt(ny * nz / (count * math.pi)) * 0.85
    taken = np.zeros(shape, bool)
    pts = []
    order = rng.permutation(ny * nz)
    for flat in order:
        y, z = divmod(int(flat), nz)
        rad = rmin * (0.6 + 0.8 * (1 - w[y, z]))
        y0, y1 = max(0, int(y - rad)), min(ny, int(y + rad) + 1)
        z0, z1 = max(0, int(z - rad)), min(nz, int(z + rad) + 1)
        if taken[y0:y1, z0:z1].any():
            # check true distances only when a neighbour is in the box
            ys, zs = np.nonzero(taken[y0:y1, z0:z1])
            if np.any((ys + y0 - y) ** 2 + (zs + z0 - z) ** 2 < rad * rad):
                continue
        taken[y, z] = True
        pts.append((y, z))
    m = taken.astype(np.uint8)
    have = int(m.sum())
    if have > count:
        on = np.flatnonzero(m)
        drop = rng.choice(on, size=have - count, replace=False)
        m.reshape(-1)[drop] = 0
    elif have < count:
        off = np.flatnonzero(m.reshape(-1) == 0)
        ww = w.reshape(-1)[off]
        add = rng.choice(off, size=count - have, replace=False, p=ww / ww.sum())
        m.reshape(-1)[add] = 1
    return m


@dataclass
class ConfigSpec:
    name: str
    kernel: tuple
    rank: int
    stages: list                  # [(region, p, gradient_steps, iterations)]
    coils_in: int
    coils_out: int
    circular_axes: tuple = ()
    slices: int = 1
    notes: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def iterations(self) -> int:
        return sum(s[3] for s in self.stages)


CONFIGS = {
    "C1": ConfigSpec("C1", (5, 5, 8), 40, [("full", 8, 5, 50)], 8, 8,
                     notes="128x128 2D, 8 coils, VD 2D random R=3, SNR 30 dB"),
    "C2": ConfigSpec("C2", (5, 5, 8), 60, [([64, 64], 8, 5, 25), ([128, 128], 8, 5, 25), ("full", 8, 5, 50)], 16, 8,
                     notes="256x256 2D, 16->8 coils, 1D VD PE R=4, 3-stage center-out"),
    "C3": ConfigSpec("C3", (7, 7, 10), 100, [("full", 10, 5, 20)], 16, 10, slices=64,
                     notes="64 x 320x320, 16->10 coils, per-slice 1D random R=4"),
    "C4": ConfigSpec("C4", (5, 5, 5, 8), 150, [([48, 36, "full"], 8, 5, 50), ("full", 8, 5, 10)], 12, 8,
                     notes="192x144x25 cine, 12->8 coils, per-frame PE R=6"),
    "C5": ConfigSpec("C5", (5, 5, 5, 8), 120, [("full", 8, 5, 40)], 8, 8,
                     notes="256x160x160 3D, 8 coils, Poisson-disc R=5, SNR 30 dB"),
}


def make_config(name: str, slice_index: int = 0, scale: float = 1.0):
    """Return (kspace_full, mask, x0) for one config (one slice for C3).

    ``scale`` < 1 shrinks every spatial extent (for CPU-sized parity runs);
    k-space is complex64 like the BASELINE inputs."""
    c = int(name[1])
    rng_ph = np.random.default_rng([1000 + c, slice_index])
    rng_co = np.random.default_rng([2000 + c, slice_index])
    rng_ma = np.random.default_rng([3000 + c, slice_index])
    rng_no = np.random.default_rng([4000 + c, slice_index])

    def sz(n):
        return max(8, int(round(n * scale)))

    if name == "C1":
        shape = (sz(128), sz(128))
        img = _ellipses_2d(shape, rng_ph, 10) * _smooth_phase(shape, rng_ph)
        coils = _gaussian_coils(shape, 8, rng_co)
        ksp = fft_kspace(img[..., None] * coils, (0, 1))
        ksp = _add_noise(ksp, 30.0, rng_no)
        m2 = _weighted_pick(_vd_weights(shape), shape[0] * shape[1] // 3, rng_ma)
        mask = np.repeat(m2[..., None], 8, axis=2)
    elif name in ("C2", "C3"):
        n = 256 if name == "C2" else 320
        nc = 16
        shape = (sz(n), sz(n))
        img = _ellipses_2d(shape, rng_ph, 12, texture=0.15 if name == "C2" else 0.0) * _smooth_phase(shape, rng_ph)
        coils = _gaussian_coils(shape, nc, rng_co)
        ksp = fft_kspace(img[..., None] * coils, (0, 1))
        ksp = _add_noise(ksp, 30.0, rng_no)
        w1 = _vd_line_weights(shape[1]) if name == "C2" else np.ones(shape[1])
        lines = _weighted_pick(w1, shape[1] // 4, rng_ma)
        mask = np.broadcast_to(lines[None, :, None], shape + (nc,)).astype(np.uint8)
    elif name == "C4":
        nx, ny, nt, nc = sz(192), sz(144), 25, 12
        base = _ellipses_2d((nx, ny), rng_ph, 8)
        phase = _smooth_phase((nx, ny), rng_ph)
        yy, xx = _grid((nx, ny))
        frames = []
        for t in range(nt):
            a = 0.18 * (1.0 + 0.25 * math.sin(2 * math.pi * t / nt))
            heart = ((xx / a) ** 2 + (yy / (0.8 * a)) ** 2 <= 1.0) * 0.9
            frames.append((base + heart) * phase)
        img = np.stack(frames, axis=2)
        coils = _gaussian_coils((nx, ny), nc, rng_co)
        ksp = fft_kspace(img[..., None] * coils[:, :, None, :], (0, 1))
        ksp = _add_noise(ksp, 30.0, rng_no)
        mask = np.zeros((nx, ny, nt, nc), np.uint8)
        w1 = _vd_line_weights(ny)
        for t in range(nt):
            lines = _weighted_pick(w1, ny // 6, np.random.default_rng([3000 + c, slice_index, t]))
            mask[:, lines == 1, t, :] = 1
    elif name == "C5":
        nx, ny, nz, nc = sz(256), sz(160), sz(160), 8
        shape = (nx, ny, nz)
        grids = _grid(shape)
        img = np.zeros(shape)
        for _ in range(10):
            ctr = rng_ph.uniform(-0.25, 0.25, 3)
            ax = rng_ph.uniform(0.08, 0.35, 3)
            rho = sum(((g - cc) / a) ** 2 for g, cc, a in zip(grids, ctr, ax))
            img += rng_ph.uniform(0.2, 1.0) / (1.0 + np.exp(np.clip((rho - 1.0) / 0.08, -60, 60)))
        img = img * _smooth_phase(shape, rng_ph, order=1)
        coils = _gaussian_coils(shape, nc, rng_co)
        ksp = fft_kspace(img[..., None] * coils, (0, 1, 2))
        ksp = _add_noise(ksp, 30.0, rng_no)
        m2 = _poisson_disc((ny, nz), ny * nz // 5, rng_ma)
        mask = np.broadcast_to(m2[None, :, :, None], shape + (nc,)).astype(np.uint8)
    else:
        raise KeyError(name)
    ksp = ksp.astype(np.complex64)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    x0 = np.where(mask == 1, ksp, 0).astype(np.complex64)
    return ksp, mask, x0
