"""Pins for the oracle's WASABI superposition + inverse (Eq.(2)) and direct
sums (Eq.(1)): north_star validations V2, V3, V4 plus linearity, translation,
window additivity and the exact accumulation count.

Non-aligned points under the R-A8 shift rule are pinned in tests/test_oracle_shift.py (hand-worked
s_l(i), the L = 1 closed form, the per-level basis-function synthesis)."""
import math

import numpy as np
import pytest


def _P(orc, **kw):
    base = dict(wavelength=633e-9, pitch=1e-6, n_h=256, n_depth=6, levels=3, z_min=0.05e-3, z_max=0.3e-3,
                retention=1.0)
    base.update(kw)
    return orc.Params(**base)


def _aligned_points(orc, P, rng, n, margin=0):
    B = 1 << P.levels
    geo = orc.geometry(P)
    d = rng.integers(0, P.n_depth, n)
    ix = rng.integers(-margin // B, (P.n_h + margin) // B, n) * B
    iy = rng.integers(-margin // B, (P.n_h + margin) // B, n) * B
    pts = np.zeros((n, 4))
    pts[:, 0] = (ix - P.n_h // 2) * P.pitch
    pts[:, 1] = (iy - P.n_h // 2) * P.pitch
    pts[:, 2] = geo["z"][d]
    pts[:, 3] = 1.0 - rng.random(n)
    return pts


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("d", [0, 3, 5])
def test_v2_single_point_is_analytic_psf(orc, d):
    """V2: one aligned point, r = 100%: u = a exp(i k sqrt(rho^2 + z^2)) on the disc
    rho < |z| tan(asin(lambda/2p)), 0 elsewhere, <= 1e-12 abs."""
    P = _P(orc)
    geo = orc.geometry_one(P, d)
    z = geo["z"]
    pts = np.array([[8e-6, -16e-6, z, 0.75]])       # (136, 112): multiples of 8
    u, _, _ = orc.Lut(P).hologram_window(pts, 0, 0, 256, 256)
    Y, X = np.mgrid[0:256, 0:256]
    dx, dy = X - 136, Y - 112
    lam = P.wavelength
    tan = (lam / 2e-6) / math.sqrt(1 - (lam / 2e-6) ** 2)
    R = abs(z) * tan / 1e-6
    inside = (dx * dx + dy * dy < R * R) | ((dx == 0) & (dy == 0))
    r = np.sqrt((dx * 1e-6) ** 2 + (dy * 1e-6) ** 2 + z * z)
    exp = np.where(inside, 0.75 * np.exp(1j * 2 * np.pi / lam * r), 0)
    assert np.max(np.abs(u - exp)) <= 1e-12


@pytest.mark.parametrize("seed", [1, 2])
def test_v3_aligned_keep_all_equals_direct_sums(orc, seed):
    """V3: r = 100%, 2^L-aligned points on levels, several depths, overlapping PSFs, some clipped
    at the hologram edge: WASABI u = D2 = D1 to <= 1e-12 rel L2."""
    P = _P(orc)
    rng = np.random.default_rng(seed)
    pts = _aligned_points(orc, P, rng, 12, margin=64)
    lut = orc.Lut(P)
    u, _, _ = lut.hologram_window(pts, 0, 0, 256, 256)
    d2 = orc.direct_d2(P, pts, 0, 0, 256, 256)
    d1 = orc.direct_d1(P, pts, 0, 0, 256, 256)
    assert _rel(u, d2) <= 1e-12
    assert _rel(d1, d2) <= 1e-12
    assert np.linalg.norm(d2) > 0


@pytest.mark.parametrize("seed", [3, 4, 5])
def test_v4_tiny_brute_force(orc, seed):
    """V4: tiny holograms (32^2, 64^2), 1-50 random points: per-pixel D1 vs per-point D2 (written
    independently) agree <= 1e-13 for aligned points on levels; WASABI(r=1, aligned) equals both."""
    rng = np.random.default_rng(seed)
    n_h = [32, 64, 64][seed - 3]
    P = _P(orc, n_h=n_h, levels=2, z_min=0.02e-3, z_max=0.06e-3, n_depth=3)
    n = int(rng.integers(1, 51))
    pts = _aligned_points(orc, P, rng, n, margin=16)
    d1 = orc.direct_d1(P, pts, 0, 0, n_h, n_h)
    d2 = orc.direct_d2(P, pts, 0, 0, n_h, n_h)
    u, _, _ = orc.Lut(P).hologram_window(pts, 0, 0, n_h, n_h)
    scale = max(np.max(np.abs(d2)), 1e-300)
    assert np.max(np.abs(d1 - d2)) <= 1e-13 * scale * max(1, n)
    assert np.max(np.abs(u - d2)) <= 1e-12 * scale * max(1, n)


def test_d1_differs_from_d2_off_grid(orc):
    """D1 keeps continuous positions/depths; D2 snaps them (the approximation WASABI inherits)."""
    P = _P(orc)
    pts = np.array([[3.3e-6, 1.7e-6, 0.123e-3, 1.0]])
    d1 = orc.direct_d1(P, pts, 0, 0, 256, 256)
    d2 = orc.direct_d2(P, pts, 0, 0, 256, 256)
    assert _rel(d1, d2) > 1e-3


def test_linearity_and_translation(orc):
    """Eq.(2) is linear in a_j and additive over points; translating every point by a multiple
    of 2^L translates psi and u exactly (the alpha rule is exact on the decimated grid)."""
    P = _P(orc, retention=0.2, levels=3)
    rng = np.random.default_rng(9)
    pts = np.zeros((2, 4))
    pts[:, 0] = (rng.integers(-40, 40, 2) + 0.3) * 1e-6
    pts[:, 1] = (rng.integers(-40, 40, 2) - 0.2) * 1e-6
    pts[:, 2] = orc.geometry(P)["z"][[2, 4]]
    pts[:, 3] = [0.6, 0.9]
    lut = orc.Lut(P)
    both, _ = lut.wasabi_window(pts, 0, 0, 256, 256)
    one, _ = lut.wasabi_window(pts[:1], 0, 0, 256, 256)
    two, _ = lut.wasabi_window(pts[1:], 0, 0, 256, 256)
    assert np.max(np.abs(both - (one + two))) < 1e-13
    p2 = pts.copy(); p2[:, 3] *= 2.5
    scaled, _ = lut.wasabi_window(p2, 0, 0, 256, 256)
    assert np.max(np.abs(scaled - 2.5 * both)) < 1e-12
    sh = pts.copy(); sh[:, 0] += 16e-6; sh[:, 1] -= 8e-6
    moved, _ = lut.wasabi_window(sh, 0, 0, 256, 256)
    # compare away from the hologram edges (dropped coefficients differ there)
    assert np.max(np.abs(moved[64:-72, 80:-64] - both[72:-64, 64:-80])) < 1e-12
    assert np.max(np.abs(both[72:-64, 64:-80])) > 0.1


def test_windows_tile_the_hologram(orc):
    """Band/window additivity (R-A12): the inverse of psi on 2^L-aligned
    windows equals the full-field result exactly (no halo)."""
    P = _P(orc, retention=0.1)
    rng = np.random.default_rng(11)
    pts = np.zeros((20, 4))
    pts[:, 0] = (rng.random(20) - 0.5) * 300e-6
    pts[:, 1] = (rng.random(20) - 0.5) * 300e-6
    pts[:, 2] = 0.05e-3 + 0.25e-3 * rng.random(20)
    pts[:, 3] = 1 - rng.random(20)
    lut = orc.Lut(P)
    full, _, _ = lut.hologram_window(pts, 0, 0, 256, 256)
    parts = np.zeros_like(full)
    for y0 in (0, 64, 128, 192):
        for x0 in (0, 128):
            u, _, _ = lut.hologram_window(pts, x0, y0, 128, 64)
            parts[y0:y0 + 64, x0:x0 + 128] = u
    assert np.array_equal(parts, full)


def test_accumulation_count_is_sum_of_in_bounds_n_r(orc):
    """cost = sum_j N_r exactly when every coefficient lands in the hologram."""
    P = _P(orc, n_h=1024, retention=0.05)
    geo = orc.geometry(P)
    rng = np.random.default_rng(2)
    n = 30
    pts = np.zeros((n, 4))
    pts[:, 0] = (rng.random(n) - 0.5) * 400e-6
    pts[:, 1] = (rng.random(n) - 0.5) * 400e-6
    d = rng.integers(0, P.n_depth, n)
    pts[:, 2] = geo["z"][d]
    pts[:, 3] = 1.0
    _, cnt = orc.Lut(P).wasabi_window(pts, 0, 0, 1024, 1024)
    assert cnt == int(geo["n_r"][d].sum())


def test_parallel_window_harness_equals_one_window(orc):
    """helpers.oracle_window (row strips of 2^L rows in a process pool, harness-side point
    pre-filter) returns exactly the oracle's single-window u, psi and bits."""
    from helpers import CONFIGS, make_points, oracle_window, orc_params, REF
    cfg = CONFIGS["C2"]
    pts = make_points(cfg, n=3000).astype(np.float64)
    P = orc_params(orc, cfg)
    u1, psi1, _ = orc.Lut(P).hologram_window(pts, 256, 512, 768, 320)
    b1, I1 = orc.quantize(P, REF, u1, 256, 512)
    u2, psi2, b2, I2 = oracle_window(P, pts, 256, 512, 768, 320, procs=4)
    assert np.array_equal(u1, u2) and np.array_equal(psi1, psi2) and np.array_equal(b1, b2)
    assert np.array_equal(I1, I2)
