"""Pins for the oracle's coiflet mode (reading R-A21): "we used coiflets as
the wavelets at level 3", order unstated -> coif1 (6 taps) on the infinite grid with
zero extension, same interleaved layout and shift rule (R-A6, R-A8) as the Haar path.

Pins, each chosen so that a plausible mistake fails one of them:
  * the filter equations that define coif1 (sum sqrt2, orthonormality to all even shifts, QMF
    highpass, two vanishing wavelet moments, vanishing first moment of the scaling filter about its
    centre tap) -- a wrong coefficient, sign or order breaks several;
  * perfect reconstruction and Parseval of the 2-D L-level transform of random compact fields
    (catches a wrong offset, synthesis index or level order);
  * the generic filter bank run with Haar filters equals the pinned Haar transform (R-A6);
  * exact covariance with 2^L shifts (the property Eq.(2)'s shift weight relies on);
  * the structural nnz rule: with Haar filters it equals the block count, with coif1 every nonzero
    coefficient lies inside it;
  * V3 for coiflets: r = 100%, 2^L-aligned interior points -> WASABI u = D2 (1e-12), and the same
    with r < 100% is NOT (control)."""
import numpy as np
import pytest

S7 = np.sqrt(7.0)


def _P(orc, **kw):
    base = dict(wavelength=633e-9, pitch=1e-6, n_h=256, n_depth=4, levels=3, z_min=0.05e-3, z_max=0.2e-3,
                retention=1.0, wavelet=1)
    base.update(kw)
    return orc.Params(**base)


def test_coif1_filter_equations(orc):
    h0, h1, off = orc.filter_bank(1)
    k = np.arange(6)
    assert len(h0) == 6 and off == 2
    assert abs(h0.sum() - np.sqrt(2)) < 1e-15
    for j in range(3):                                    # orthonormal to its even shifts
        assert abs(np.dot(h0[2 * j:], h0[:6 - 2 * j]) - (1.0 if j == 0 else 0.0)) < 1e-15
    for j in range(-2, 3):                                # highpass orthogonal to all even shifts
        a = np.zeros(16); b = np.zeros(16)
        a[5:11] = h0; b[5 + 2 * j:11 + 2 * j] = h1
        assert abs(np.dot(a, b)) < 1e-15
    assert np.allclose(h1, (-1.0) ** k * h0[::-1], atol=0, rtol=0)
    assert abs(h1.sum()) < 1e-15 and abs((k * h1).sum()) < 1e-14     # two vanishing wavelet moments
    assert abs(((k - off) * h0).sum()) < 1e-14                        # coiflet: scaling moment 1 about tap 2
    # closed form (Daubechies K = 1 coiflet), independent of the oracle's arithmetic order
    ref = np.sqrt(2) / 32 * np.array([1 - S7, 5 + S7, 14 + 2 * S7, 14 - 2 * S7, 1 - S7, -3 + S7])
    assert np.allclose(h0, ref, atol=1e-16)


@pytest.mark.parametrize("L,seed", [(1, 1), (3, 2), (4, 3)])
def test_perfect_reconstruction_and_parseval(orc, L, seed):
    rng = np.random.default_rng(seed)
    n = 256                      # support + 3 (2^L - 1) growth stays inside the array (zero extension)
    f = np.zeros((n, n), complex)
    f[100:150, 90:160] = rng.standard_normal((50, 70)) + 1j * rng.standard_normal((50, 70))
    c = orc.fb_fwd(1, f, L)
    assert abs(np.linalg.norm(c) - np.linalg.norm(f)) <= 1e-13 * np.linalg.norm(f)
    g = orc.fb_inv(1, c, L)
    assert np.max(np.abs(g - f)) <= 1e-13


def test_haar_filters_reproduce_haar_transform(orc):
    rng = np.random.default_rng(4)
    f = rng.standard_normal((64, 64)) + 1j * rng.standard_normal((64, 64))
    a = orc.fb_fwd(0, f, 4)
    b = orc.haar_fwd(f, 4)
    assert np.max(np.abs(a - b)) <= 1e-14
    assert np.max(np.abs(orc.fb_inv(0, b, 4) - orc.haar_inv(b, 4))) <= 1e-14


def test_shift_covariance(orc):
    """Shifting the input by 2^L (= 8, L = 3) shifts every level-l coefficient by exactly 8 px in
    the interleaved layout (the property behind Eq.(2)'s shift weight alpha = 2^-l)."""
    rng = np.random.default_rng(5)
    f = np.zeros((128, 128), complex)
    f[40:70, 40:80] = rng.standard_normal((30, 40))
    g = np.roll(np.roll(f, 8, axis=0), 16, axis=1)
    cf = orc.fb_fwd(1, f, 3)
    cg = orc.fb_fwd(1, g, 3)
    assert np.max(np.abs(np.roll(np.roll(cf, 8, axis=0), 16, axis=1) - cg)) <= 1e-13


def test_structural_nnz_rule(orc):
    """Footprint rule with Haar filters == the block-touch count; with coif1 it covers every nonzero
    coefficient of the transformed table (and the padded table side keeps all of them inside)."""
    Ph = _P(orc, wavelet=0)
    for d in range(Ph.n_depth):
        assert orc.nnz_footprint(Ph, d) == orc.table_info(Ph, d)["nnz"]
    P = _P(orc)
    for d in range(P.n_depth):
        info = orc.table_info(P, d)
        c = orc.table_coeffs(P, d)
        assert info["nnz"] == orc.nnz_footprint(P, d)
        nz = int(np.sum(np.abs(c) > 1e-300))
        assert nz <= info["nnz"]
        assert np.all(np.abs(c[:4]) == 0) and np.all(np.abs(c[-4:]) == 0)   # padding holds the support


def _aligned_points(orc, P, rng, n, lo, hi):
    B = 1 << P.levels
    geo = orc.geometry(P)
    d = rng.integers(0, P.n_depth, n)
    ix = rng.integers(lo // B, hi // B, n) * B
    iy = rng.integers(lo // B, hi // B, n) * B
    pts = np.zeros((n, 4))
    pts[:, 0] = (ix - P.n_h // 2) * P.pitch
    pts[:, 1] = (iy - P.n_h // 2) * P.pitch
    pts[:, 2] = geo["z"][d]
    pts[:, 3] = 1.0 - rng.random(n)
    return pts


@pytest.mark.parametrize("seed", [1, 2])
def test_v3_coiflets_keep_all_equals_direct_sum(orc, seed):
    """r = 100%, 2^L-aligned points whose coefficients all fall inside the hologram: u = D2."""
    P = _P(orc)
    rng = np.random.default_rng(seed)
    pts = _aligned_points(orc, P, rng, 8, 96, 160)
    u, _, _ = orc.Lut(P).hologram_window(pts, 0, 0, 256, 256)
    d2 = orc.direct_d2(P, pts, 0, 0, 256, 256)
    assert np.linalg.norm(d2) > 0
    assert np.linalg.norm(u - d2) <= 1e-12 * np.linalg.norm(d2)
    # a window of the hologram gives the same u there (the 64-px psi halo covers the synthesis)
    uw, _, _ = orc.Lut(P).hologram_window(pts, 64, 128, 128, 64)
    assert np.max(np.abs(uw - u[128:192, 64:192])) <= 1e-13


def test_coiflets_shrunk_differs_and_beats_haar(orc):
    """Control and the reason for NEXT-2: at r = 5% the coiflet hologram is not the direct sum, and
    for aligned points it is closer to it than the Haar hologram at the same r (SURVEY.md §8(f):
    Haar keeps ~27% of the energy at r = 5%)."""
    rng = np.random.default_rng(3)
    P = _P(orc, retention=0.05)
    pts = _aligned_points(orc, P, rng, 8, 96, 160)
    d2 = orc.direct_d2(P, pts, 0, 0, 256, 256)
    uc, _, _ = orc.Lut(P).hologram_window(pts, 0, 0, 256, 256)
    uh, _, _ = orc.Lut(_P(orc, retention=0.05, wavelet=0)).hologram_window(pts, 0, 0, 256, 256)
    ec = np.linalg.norm(uc - d2) / np.linalg.norm(d2)
    eh = np.linalg.norm(uh - d2) / np.linalg.norm(d2)
    assert 1e-3 < ec < eh
