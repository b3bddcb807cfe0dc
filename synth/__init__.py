"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NONE of the method's arithmetic (no multislice, no gradient, no
geometry of tiles): only the inputs the paper's problem statement takes
(§Math Formulation: measurements |y_i|, probe p_i, probe
locations, initial V) and the workload shapes of BASELINE.json's configs.

Recipe:
  * V_true = default_rng(seed).random((S, H, W), float32): uniform [0, 1) random
    potential ("random potential", BASELINE.json north_star).
  * probe: centred inverse DFT of an aperture disk |m| <= 0.1196 N (30 mrad at
    200 keV, 10 pm pixels) times a defocus phase exp(-i*1969.7*(df/25nm)*|m|^2/N^2)
    (25 nm defocus), normalised to sum |p|^2 = 1.  Beam axis at (N/2, N/2).
  * scan: full-coverage raster, centre_j = floor((2j+1) * extent / (2 n)), row-major
    (Fig. ptycho_setup b; reading #11 in DESIGN.md).
"""
from __future__ import annotations

import dataclasses
import numpy as np

__all__ = ["Config", "CONFIGS", "volume", "probe", "scan_centers", "random_amplitudes", "lattice_phantom"]


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int          # window / detector side N
    slices: int     # S
    height: int     # object H
    width: int      # object W
    scan_ny: int    # raster rows
    scan_nx: int    # raster columns
    grid: tuple     # (R, C) tile grid
    halo: int       # halo width (voxels)
    defocus_nm: float = 25.0
    sigma: float = 0.1          # t = exp(i sigma V)
    prop_c: float = 3.135       # c = lambda dz / dx^2 at 200 keV, 125 pm slices, 10 pm pixels

    @property
    def n_probes(self) -> int:
        return self.scan_ny * self.scan_nx


# BASELINE.json "configs", in order.
CONFIGS = {
    "tiny": Config("tiny", 64, 4, 128, 128, 4, 4, (1, 1), 32, defocus_nm=8.0),
    "small": Config("small", 256, 20, 512, 512, 32, 32, (1, 1), 128),
    "appp": Config("appp", 256, 20, 1024, 1024, 64, 64, (2, 2), 128),
    "lt_small": Config("lt_small", 1024, 100, 1536, 1536, 63, 66, (2, 4), 512),
    "lt_large": Config("lt_large", 1024, 100, 3072, 3072, 126, 132, (2, 4), 512),
}


def volume(seed: int, slices: int, height: int, width: int) -> np.ndarray:
    """Random potential V_true, float32 [S][H][W], uniform [0, 1)."""
    return np.random.default_rng(seed).random((slices, height, width), dtype=np.float32)


def probe(n: int, defocus_nm: float = 25.0, aperture_frac: float = 0.1196) -> np.ndarray:
    """Aperture-limited defocused probe, complex128 [N][N], axis at (N/2, N/2), sum|p|^2 = 1."""
    m = np.arange(n)
    m = np.where(m < n // 2, m, m - n).astype(np.float64)
    m2 = m[:, None] ** 2 + m[None, :] ** 2
    aperture = (np.sqrt(m2) <= aperture_frac * n).astype(np.float64)
    spectrum = aperture * np.exp(-1j * 1969.7 * (defocus_nm / 25.0) * m2 / float(n * n))
    p = np.fft.fftshift(np.fft.ifft2(spectrum))
    return p / np.sqrt(np.sum(np.abs(p) ** 2))


def scan_centers(height: int, width: int, ny: int, nx: int) -> np.ndarray:
    """Raster probe centres int32 [ny*nx][2] as (cy, cx), row-major time order."""
    cy = (2 * np.arange(ny) + 1) * height // (2 * ny)
    cx = (2 * np.arange(nx) + 1) * width // (2 * nx)
    yy, xx = np.meshgrid(cy, cx, indexing="ij")
    return np.stack([yy.ravel(), xx.ravel()], axis=1).astype(np.int32)


def random_amplitudes(seed: int, count: int, n: int, scale: float = 1.0) -> np.ndarray:
    """Non-negative float32 amplitudes [count][N][N] (DC at [0,0]) with the RMS of a unit probe."""
    rng = np.random.default_rng(seed)
    return (rng.random((count, n, n), dtype=np.float32) * (2.0 * scale / n)).astype(np.float32)


def lattice_phantom(seed: int, slices: int, height: int, width: int, period: float = 39.0, sigma_px: float = 6.0,
                    amplitude: float = 1.0, jitter: float = 1.5) -> np.ndarray:
    """Structured potential for the seam / quality studies only (SPEC make_phantom
    S:523-531): a PbTiO3-like square lattice of Gaussian atom columns, period ~3.9 A = 39 px at
    10 pm/px ("each circle ... a small group of atoms"), seeded positional jitter, values
    in [0, amplitude], float32 [S][H][W]."""
    rng = np.random.default_rng(seed)
    out = np.zeros((slices, height, width), np.float64)
    yy = np.arange(height)[:, None]
    xx = np.arange(width)[None, :]
    cys = np.arange(period / 2, height, period)
    cxs = np.arange(period / 2, width, period)
    for s in range(slices):
        acc = np.zeros((height, width))
        for cy in cys:
            for cx in cxs:
                jy, jx = rng.normal(0.0, jitter, 2)
                y0, x0 = cy + jy, cx + jx
                ys = slice(max(0, int(y0 - 4 * sigma_px)), min(height, int(y0 + 4 * sigma_px) + 1))
                xs = slice(max(0, int(x0 - 4 * sigma_px)), min(width, int(x0 + 4 * sigma_px) + 1))
                acc[ys, xs] += np.exp(-((yy[ys] - y0) ** 2 + (xx[:, xs] - x0) ** 2) / (2 * sigma_px ** 2))
        out[s] = acc
    out *= amplitude / max(out.max(), 1e-30)
    return out.astype(np.float32)
