"""BASELINE.json configs C1-C5 as seeded synthetic point clouds.

Recipe:
  * PRNG numpy Generator(PCG64(seed)); draw order x, y, z-or-field lattice,
    a-field lattice, a.
  * Aperture A = N_h * p, hologram-centred: x, y ~ U[-A/2, A/2).
  * a ~ 1 - U[0,1) in (0,1] unless the config says otherwise.
  * Points are float32 (x, y, z, a) in metres, AoS, exactly what the C-ABI takes.

The paper's 3D model (95,949 points) is not available; these
seeded scenes stand in for it with the paper's shapes.
Nothing here computes any part of the method.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n_h: int
    pitch: float
    wavelength: float
    n_points: int
    n_depth: int
    z_min: float
    z_max: float
    levels: int
    retention: float
    seed: int
    kind: str            # "levels" | "uniform" | "rgbd" | "heightfield"
    tile: int = 64
    bands: int = 1       # row bands for the multi-GPU split (PAPER.md:115-125 analogue)
    aligned: bool = False  # snap x, y to the 2^L pixel grid (C5 PSNR variant)
    ref: tuple = (0.0, 0.030, -0.400)   # spherical reference wave

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


MM = 1e-3
UM = 1e-6

CONFIGS = {
    # BASELINE.json configs[0]
    "C1": Config("C1", 512, 1 * UM, 633e-9, 1_000, 8, 0.1 * MM, 0.4 * MM, 3, 0.10, 1, "levels"),
    # configs[1] (r in {1,5,10}%; 10% is the default line)
    "C2": Config("C2", 2048, 1 * UM, 633e-9, 10_000, 32, 0.1 * MM, 1.0 * MM, 4, 0.10, 2, "uniform"),
    # configs[2]
    "C3": Config("C3", 8192, 1 * UM, 532e-9, 100_000, 64, 0.2 * MM, 0.8 * MM, 5, 0.05, 3, "rgbd"),
    # configs[3]: paper scale, 8 row bands
    "C4": Config("C4", 65536, 1 * UM, 633e-9, 2_000_000, 128, -2.0 * MM, 2.0 * MM, 6, 0.05, 4,
                 "heightfield", bands=8),
    # configs[4]: sweep base point; N and r are overridden per sweep cell
    "C5": Config("C5", 16384, 1 * UM, 633e-9, 1_000_000, 64, 0.1 * MM, 1.0 * MM, 5, 0.05, 5, "uniform"),
}


def value_noise(rng: np.random.Generator, lo: float, hi: float, lo_open: bool = False) -> np.ndarray:
    """17x17 lattice of i.i.d. values (16x16 cells spanning the aperture)."""
    if lo_open:
        return hi - (hi - lo) * rng.random((17, 17))     # (lo, hi]
    return lo + (hi - lo) * rng.random((17, 17))          # [lo, hi)


def _interp_noise(lat: np.ndarray, x: np.ndarray, y: np.ndarray, aperture: float) -> np.ndarray:
    """Smoothstep-bilinear interpolation of the lattice at (x, y) (hologram-centred metres)."""
    u = np.clip((x + aperture / 2) / aperture * 16.0, 0.0, 16.0 - 1e-12)
    v = np.clip((y + aperture / 2) / aperture * 16.0, 0.0, 16.0 - 1e-12)
    i = np.floor(u).astype(np.int64)
    j = np.floor(v).astype(np.int64)
    tu = u - i
    tv = v - j
    su = tu * tu * (3.0 - 2.0 * tu)
    sv = tv * tv * (3.0 - 2.0 * tv)
    l00 = lat[j, i]
    l01 = lat[j, i + 1]
    l10 = lat[j + 1, i]
    l11 = lat[j + 1, i + 1]
    return (l00 * (1 - su) + l01 * su) * (1 - sv) + (l10 * (1 - su) + l11 * su) * sv


def make_points(cfg: Config, n: Optional[int] = None, seed: Optional[int] = None) -> np.ndarray:
    """Return float32 array (n, 4) of (x, y, z, a) for the config."""
    n = cfg.n_points if n is None else int(n)
    seed = cfg.seed if seed is None else int(seed)
    rng = np.random.Generator(np.random.PCG64(seed))
    A = cfg.n_h * cfg.pitch
    x = -A / 2 + A * rng.random(n)
    y = -A / 2 + A * rng.random(n)
    if cfg.aligned:
        step = 1 << cfg.levels
        ix = np.floor((x / cfg.pitch + cfg.n_h / 2) / step).astype(np.int64) * step
        iy = np.floor((y / cfg.pitch + cfg.n_h / 2) / step).astype(np.int64) * step
        x = (ix - cfg.n_h // 2) * cfg.pitch
        y = (iy - cfg.n_h // 2) * cfg.pitch
    a_lat = None
    if cfg.kind == "levels":
        d = rng.integers(0, cfg.n_depth, n)
        dz = (cfg.z_max - cfg.z_min) / (cfg.n_depth - 1) if cfg.n_depth > 1 else 0.0
        z = cfg.z_min + d * dz
    elif cfg.kind == "uniform":
        z = cfg.z_min + (cfg.z_max - cfg.z_min) * rng.random(n)
    elif cfg.kind == "rgbd":
        # synthetic RGB-D surface of BASELINE.json configs[2]
        z = 0.5 * MM + 0.3 * MM * np.sin(2 * np.pi * x / (3 * MM)) * np.cos(2 * np.pi * y / (4 * MM))
        a_lat = value_noise(rng, 0.05, 1.0, lo_open=True)
    elif cfg.kind == "heightfield":
        h_lat = value_noise(rng, -1.0, 1.0)
        z = 2.0 * MM * _interp_noise(h_lat, x, y, A)
    else:
        raise ValueError(cfg.kind)
    if a_lat is not None:
        a = _interp_noise(a_lat, x, y, A)
    else:
        a = 1.0 - rng.random(n)
    pts = np.empty((n, 4), dtype=np.float32)
    pts[:, 0] = x
    pts[:, 1] = y
    pts[:, 2] = z
    pts[:, 3] = a
    return pts
