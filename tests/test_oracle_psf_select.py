"""Pins for the oracle's step 1: PSF, window, geometry, structural nnz, N_r and top-k selection
(readings R-A2, R-A4, R-A5, R-A13).

Independent references: the paper's printed parameters (tests/golden/paper_params.json), the
Nyquist property of the diffraction-limited window (the per-pixel phase step reaches pi exactly
at rho = R), Gauss-circle lattice counts, nonzero counts of the transformed table, a full
numpy sort as the definition of top-k, and the Parseval identity for shrinkage.
"""
import json
import math
import os

import numpy as np
import pytest

from inputs import CONFIGS

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_params.json")))


def _P(orc, **kw):
    base = dict(wavelength=633e-9, pitch=1e-6, n_h=512, n_depth=8, levels=3, z_min=0.1e-3, z_max=0.4e-3,
                retention=0.10)
    base.update(kw)
    return orc.Params(**base)


def test_paper_psf_radius_example(orc):
    """SPEC.md:183 with the paper's lambda/pitch/depth: footprint radius ~5004 px at 15 mm."""
    g = GOLD["psf_radius_example"]
    P = orc.Params(g["wavelength_m"], g["pitch_m"], 65536, 1, 6, g["z_m"], g["z_m"], 0.05)
    geo = orc.geometry_one(P, 0)
    assert abs(geo["R"] - g["footprint_radius_px_approx"]) <= g["tol_px"]
    assert geo["H"] % 64 == 0 and geo["H"] > geo["R"]


def test_paper_depth_grid_reading(orc):
    """PAPER.md:133 prints dz = 30 mm/29 for N_z=29; reading R-A3 uses inclusive endpoints
    ((z_max - z_min)/(N_z - 1)).  Both readings are recorded; the level grid is checked against
    an integer count of intervals: 28 intervals span the 30 mm exactly."""
    span = GOLD["depth_span_m"]["value"]
    nz = GOLD["depth_levels_Nz"]["value"]
    assert abs(span / nz - GOLD["paper_delta_z_m"]["value"]) < 1e-15
    P = orc.Params(632.8e-9, 1e-6, 8192, nz, 3, -span / 2, span / 2, 0.05)
    zs = [orc.geometry_one(P, d)["z"] for d in (0, 14, 28)]
    assert zs[0] == -span / 2 and abs(zs[1]) < 1e-15 and abs(zs[2] - span / 2) < 1e-15


@pytest.mark.parametrize("d", [0, 3, 7])
def test_psf_unit_modulus_on_support_zero_off(orc, d):
    """PAPER.md:90 circ window with unit amplitude: |f| = 1 on S, 0 off S; the
    support pixel count is the Gauss circle count of the open disc (plus the centre)."""
    P = _P(orc)
    geo = orc.geometry_one(P, d)
    f = orc.psf_table(P, d)
    H, R = geo["H"], geo["R"]
    on = np.abs(f) > 0.5
    np.testing.assert_allclose(np.abs(f[on]), 1.0, atol=1e-14)
    assert np.all(np.abs(f[~on]) == 0)
    r_int = int(math.floor(R))
    gauss = sum(2 * int(math.isqrt(max(0, math.ceil(R * R) - 1 - x * x))) + 1
                for x in range(-r_int, r_int + 1) if x * x < R * R)
    assert on.sum() == gauss
    assert abs(on.sum() - math.pi * R * R) < 8 * R   # boundary term O(R)
    assert on[H, H]


@pytest.mark.parametrize("z", [0.1e-3, 0.25e-3, 0.4e-3])
def test_centre_phase_closed_form(orc, z):
    """r_hj = |z| at the PSF centre: f(H, H) = exp(i 2 pi z / lambda)."""
    P = _P(orc, n_depth=1, z_min=z, z_max=z)
    f = orc.psf_table(P, 0)
    H = orc.geometry_one(P, 0)["H"]
    ph = (2 * math.pi * z / 633e-9) % (2 * math.pi)
    assert abs(f[H, H] - complex(math.cos(ph), math.sin(ph))) < 1e-9


@pytest.mark.parametrize("lam,pitch,z", [(633e-9, 1e-6, 0.4e-3), (532e-9, 1e-6, 0.8e-3), (633e-9, 2e-6, 1e-3)])
def test_window_is_nyquist_limited(orc, lam, pitch, z):
    """Diffraction-limited window asin(lambda/2p) (BASELINE configs[0]): along the x axis the
    per-pixel phase step k p x/r grows with x and reaches pi exactly at the window edge; inside S
    every step is < pi and the last step is within 1% of pi.  A radius from sin instead of tan
    (or any wrong radius) fails one of the two bounds."""
    P = _P(orc, wavelength=lam, pitch=pitch, n_depth=1, z_min=z, z_max=z)
    f = orc.psf_table(P, 0)
    H = orc.geometry_one(P, 0)["H"]
    row = f[H, H:]
    inside = np.abs(row) > 0.5
    n = int(inside.sum())
    steps = np.abs(np.angle(row[1:n] / row[: n - 1]))
    # local phase steps are smooth: unwrap is unambiguous below pi
    assert np.all(steps < math.pi)
    k = 2 * math.pi / lam
    xs = np.arange(n) * pitch
    r = np.sqrt(xs ** 2 + z * z)
    true_steps = np.diff(k * r)
    assert true_steps[-1] < math.pi and true_steps[-1] > 0.99 * math.pi
    np.testing.assert_allclose(steps, true_steps, atol=1e-8)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_structural_nnz_equals_nonzero_coefficients(orc, cfg):
    """nnz_d (blocks touching S) equals the count of nonzero coefficients of the transformed PSF
    (generic: no cancellation to exactly zero), and an independent numpy block count."""
    c = CONFIGS[cfg]
    P = orc.Params.from_config(c)
    for d in (0, c.n_depth // 2, c.n_depth - 1):
        g = orc.geometry_one(P, d)
        W = orc.table_coeffs(P, d, g["H"])
        assert int(np.count_nonzero(W)) == g["nnz"]
        m = np.abs(orc.psf_table(P, d)) > 0
        cnt = 0
        for l in range(1, c.levels + 1):
            b = 1 << l
            blocks = m.reshape(m.shape[0] // b, b, m.shape[1] // b, b).any(axis=(1, 3))
            cnt += blocks.sum() * (4 if l == c.levels else 3)
        assert cnt == g["nnz"]


def test_n_r_closed_form(orc):
    """R-A4: N_r = ceil(r nnz) in exact integer arithmetic, clamped to nnz."""
    for r in (0.01, 0.05, 0.10, 0.25, 1.0, 0.123457):
        P = _P(orc, retention=r)
        g = orc.geometry(P)
        for nnz, nr in zip(g["nnz"], g["n_r"]):
            rp = round(r * 1e6)
            assert nr == min(nnz, -(-rp * int(nnz) // 1_000_000))
    g = orc.geometry(_P(orc, retention=1.0))
    assert np.array_equal(g["nnz"], g["n_r"])


@pytest.mark.parametrize("cfg,d", [("C1", 0), ("C1", 7), ("C2", 10), ("C3", 63)])
def test_topk_is_full_sort_prefix(orc, cfg, d):
    """the kept set is the first N_r of a full sort by (kappa desc, linear index asc);
    min kept kappa >= max discarded kappa; values are the table's coefficients;
    output is sorted canonically by (level, Y, X)."""
    c = CONFIGS[cfg]
    P = orc.Params.from_config(c)
    g = orc.geometry_one(P, d)
    H, nr = g["H"], g["n_r"]
    lv, dx, dy, val = orc.select(P, d, nr)
    assert len(lv) == nr
    W = orc.table_coeffs(P, d, H)
    side = 2 * H
    kap = (W.real * W.real + W.imag * W.imag).astype(np.float32).ravel()
    order = np.lexsort((np.arange(side * side), -kap.astype(np.float64)))
    ref = set(order[:nr].tolist())
    lin = (dy.astype(np.int64) + H) * side + (dx.astype(np.int64) + H)
    assert set(lin.tolist()) == ref
    kept = np.zeros(side * side, bool)
    kept[lin] = True
    assert kap[kept].min() >= kap[~kept].max()
    thr = kap[kept].min()
    assert lin[kap[lin] == thr].max() < np.flatnonzero((~kept) & (kap == thr)).min(initial=side * side)
    np.testing.assert_array_equal(val, W.ravel()[lin])
    # canonical order and level classification (interleaved layout)
    X = dx + H
    Y = dy + H
    key = np.stack([lv, Y, X]).T
    assert all(tuple(key[i]) < tuple(key[i + 1]) for i in range(len(key) - 1))
    for x, y, l in zip(X[:200], Y[:200], lv[:200]):
        t = 0
        while t < c.levels and (x >> t) & 1 == 0 and (y >> t) & 1 == 0:
            t += 1
        assert l == min(t + 1, c.levels)


@pytest.mark.parametrize("r", [0.05, 0.25])
def test_shrinkage_parseval_single_aligned_point(orc, r):
    """Exact identity: for one 2^L-aligned point on a level, ||u_r||^2 = sum_kept |c|^2 and
    ||u_1 - u_r||^2 = sum_discarded |c|^2 (orthonormal Haar)."""
    P1 = _P(orc, retention=1.0, n_h=256)
    Pr = _P(orc, retention=r, n_h=256)
    z = orc.geometry_one(P1, 4)["z"]
    pts = np.array([[0.0, 0.0, z, 1.0]])
    u1, _, _ = orc.Lut(P1).hologram_window(pts, 0, 0, 256, 256)
    ur, _, _ = orc.Lut(Pr).hologram_window(pts, 0, 0, 256, 256)
    g = orc.geometry_one(Pr, 4)
    _, _, _, val = orc.select(Pr, 4, g["n_r"])
    W = orc.table_coeffs(Pr, 4, g["H"])
    e_kept = np.sum(np.abs(val) ** 2)
    e_all = np.sum(np.abs(W) ** 2)
    assert abs(np.sum(np.abs(ur) ** 2) - e_kept) <= 1e-10 * e_all
    assert abs(np.sum(np.abs(u1 - ur) ** 2) - (e_all - e_kept)) <= 1e-10 * e_all
