"""Pins for the oracle's Eq.(2) level shift on NON-aligned points (reading R-A8).

PAPER.md:110-113 (§1, Eq.(2)): psi(m, n) = sum_j a_j sum_k c_{z_j,k} delta(m - alpha x_j, n - alpha y_j),
"alpha_{z_j,k} is the shift weight according to the level l".  Reading R-A8: a level-l
coefficient (dX, dY) of a point at pixel (ix, iy) lands at (s_l(ix) + dX, s_l(iy) + dY) with
s_l(i) = 2^l floor((i + 2^(l-1)) / 2^l) (alpha_l = 2^-l, round half up, floor for negative i), the LL
band at l = L.  Every other WASABI pin uses 2^L-aligned points, where every rounding rule is the
identity; these tests fix the tie direction and the negative branch:

  (c) hand-written s_l(i) for i in {-9, -5, -2, -1, 0, 1, 3, 4, 7} at l = 1, 2, 3 (integer tables below,
      worked out by hand from the formula: a round-half-down rule fails s_1(1), s_2(1)... a truncating
      division fails s_1(-2), s_2(-5), s_3(-9));
  (a) closed form at L = 1, r = 100%: every coefficient carries level 1, so WASABI of one point at any
      integer (ix, iy) equals the analytic PSF centred at (2 floor((ix+1)/2),
      2 floor((iy+1)/2)) -- computed here from exp(ik r) directly, to 1e-12;
  (b) L > 1: psi equals each kept coefficient placed at its own level's shift, and u equals the sum of
      the textbook Haar basis functions (+-2^-l on the halves of a 2^l block; written as basis
      functions, not as the oracle's butterfly recursion) weighted by those coefficients.
"""
import math

import numpy as np
import pytest

# s_l(i) by hand: s_l(i) = 2^l floor((i + 2^(l-1)) / 2^l)
_I = [-9, -5, -2, -1, 0, 1, 3, 4, 7]
_S = {
    1: [-8, -4, -2, 0, 0, 2, 4, 4, 8],     # (i+1)/2 floored, times 2
    2: [-8, -4, 0, 0, 0, 0, 4, 4, 8],      # (i+2)/4 floored, times 4
    3: [-8, -8, 0, 0, 0, 0, 0, 8, 8],      # (i+4)/8 floored, times 8
}


def _P(orc, **kw):
    base = dict(wavelength=633e-9, pitch=1e-6, n_h=64, n_depth=3, levels=1, z_min=20e-6, z_max=40e-6,
                retention=1.0)
    base.update(kw)
    return orc.Params(**base)


@pytest.mark.parametrize("l", [1, 2, 3])
def test_hand_written_level_shifts(orc, l):
    """(c) s_l(i) for odd, even, negative and tie indices against the hand-worked table."""
    P = _P(orc, levels=3)
    got = [orc.level_shift(P, i, l) for i in _I]
    assert got == _S[l], (l, got)


def _point(P, ix, iy, z, a):
    """A point whose pixel (R-A9: ix = floor(x/p + 1/2) + N_h/2) is exactly (ix, iy)."""
    return [(ix - P.n_h // 2 + 0.25) * P.pitch, (iy - P.n_h // 2 - 0.25) * P.pitch, z, a]


def _analytic_psf(P, cx, cy, z, a, n):
    """a exp(i k sqrt((dx p)^2 + (dy p)^2 + z^2)) on rho < |z| tan(asin(lambda/2p)) (+ the centre)."""
    lam, p = P.wavelength, P.pitch
    s = lam / (2 * p)
    R = abs(z) * (s / math.sqrt(1 - s * s)) / p
    Y, X = np.mgrid[0:n, 0:n]
    dx, dy = X - cx, Y - cy
    inside = (dx * dx + dy * dy < R * R) | ((dx == 0) & (dy == 0))
    r = np.sqrt((dx * p) ** 2 + (dy * p) ** 2 + z * z)
    return np.where(inside, a * np.exp(1j * 2 * np.pi / lam * r), 0)


@pytest.mark.parametrize("ix,iy", [(31, 33), (32, 32), (5, -1), (-2, 7), (-3, -5), (66, 61), (0, 1), (63, 64)])
def test_l1_closed_form_any_integer_position(orc, ix, iy):
    """(a) L = 1, r = 100%: u = analytic PSF at (2 floor((ix+1)/2), 2 floor((iy+1)/2)), <= 1e-12 abs,
    for odd, even, negative and outside-the-hologram pixels (coefficients outside [0, N_h)^2 dropped,
    R-A12: with Haar blocks of 2 px this clips the PSF exactly at the hologram edge)."""
    P = _P(orc)
    z = orc.geometry(P)["z"][1]               # R = 10 px
    pts = np.array([_point(P, ix, iy, z, 0.8)])
    u, _, _ = orc.Lut(P).hologram_window(pts, 0, 0, P.n_h, P.n_h)
    sx, sy = 2 * ((ix + 1) // 2), 2 * ((iy + 1) // 2)
    exp = _analytic_psf(P, sx, sy, z, 0.8, P.n_h)
    assert np.max(np.abs(u - exp)) <= 1e-12
    assert np.max(np.abs(exp)) > 0.5
    if ix % 2:  # the rounding is visible: the unshifted PSF is a different field
        assert np.max(np.abs(u - _analytic_psf(P, ix, sy, z, 0.8, P.n_h))) > 0.1


def _level_of(X, Y, L):
    """(level, sub-band) of an interleaved position (R-A6): t = min(ctz X, ctz Y); t >= L -> LL_L."""
    t = 0
    while t < L and X % (1 << (t + 1)) == 0 and Y % (1 << (t + 1)) == 0:
        t += 1
    if t >= L:
        return L, "LL"
    bx, by = (X >> t) & 1, (Y >> t) & 1
    return t + 1, {(1, 0): "HL", (0, 1): "LH", (1, 1): "HH"}[(bx, by)]


def _basis(X, Y, L):
    """Textbook orthonormal Haar basis function of the coefficient at interleaved (X, Y): on the
    2^l block containing it, 2^-l times +1/-1 on the halves (HL: left/right, LH: top/bottom, HH:
    checkerboard of quadrants, LL: +1).  Returns (x0, y0, block)."""
    l, band = _level_of(X, Y, L)
    B = 1 << l
    x0, y0 = X & ~(B - 1), Y & ~(B - 1)
    h = B // 2
    sx = np.where(np.arange(B) < h, 1.0, -1.0)
    one = np.ones(B)
    fx, fy = {"LL": (one, one), "HL": (sx, one), "LH": (one, sx), "HH": (sx, sx)}[band]
    return x0, y0, np.outer(fy, fx) / B


@pytest.mark.parametrize("L,r,seed", [(2, 1.0, 1), (3, 1.0, 2), (3, 0.3, 3), (4, 0.5, 4)])
def test_per_level_shift_decomposition(orc, L, r, seed):
    """(b) Non-aligned points (odd, even, negative pixels), L > 1: psi[s_l(i) + dX] += a c for every
    kept coefficient (each level at its own shift, LL at l = L), and u = sum of a c times the Haar basis
    function at that position (independent synthesis), both <= 1e-12."""
    n = 64
    P = _P(orc, levels=L, retention=r, n_depth=3, z_min=15e-6, z_max=30e-6)
    geo = orc.geometry(P)
    rng = np.random.default_rng(seed)
    pix = rng.integers(-6, n + 6, size=(5, 2))
    pix[0] = (-3, 5)
    pix[1] = (7, -1)
    ds = rng.integers(0, P.n_depth, 5)
    amp = 1 - rng.random(5)
    pts = np.array([_point(P, int(ix), int(iy), geo["z"][d], a) for (ix, iy), d, a in zip(pix, ds, amp)])
    u_o, psi_o, _ = orc.Lut(P).hologram_window(pts, 0, 0, n, n)

    psi = np.zeros((n, n), np.complex128)
    u = np.zeros((n, n), np.complex128)
    for (ix, iy), d, a in zip(pix, ds, amp):
        lv, dx, dy, val = orc.select(P, int(d), int(geo["n_r"][d]) + 8)
        assert len(lv) == geo["n_r"][d]
        for l, ddx, ddy, c in zip(lv, dx, dy, val):
            l = int(l)
            s = 1 << l
            X = s * ((int(ix) + s // 2) // s) + int(ddx)
            Y = s * ((int(iy) + s // 2) // s) + int(ddy)
            if not (0 <= X < n and 0 <= Y < n):
                continue
            assert _level_of(X, Y, L)[0] == l      # the shift keeps a coefficient in its own level
            psi[Y, X] += a * c
            x0, y0, blk = _basis(X, Y, L)
            u[y0:y0 + blk.shape[0], x0:x0 + blk.shape[1]] += a * c * blk
    assert np.max(np.abs(psi_o - psi)) <= 1e-12
    assert np.max(np.abs(u_o - u)) <= 1e-12
    assert np.max(np.abs(u)) > 0.1
