"""Pins for the oracle's offset-class tables (reading R-A20).

R-A20: with exact shifts every depth has 4^L tables, one per sub-position class (cx, cy) =
(ix mod 2^L, iy mod 2^L): the PSF centred at (H + cx, H + cy) in a (2H + 2^L)^2 table, forward
transformed and shrunk on its own, and every coefficient of a point is shifted by the 2^L-aligned
(ix - cx, iy - cy).  Haar blocks are 2^L-local, so a 2^L shift commutes with the transform
exactly: the pins below hold for ANY integer point position, unlike R-A8 (aligned points only).

Pins: r = 100% WASABI equals the quantised direct sum D2 (and the continuous D1) for random
non-aligned points -- the defining property, which a wrong centre, class index, shift or table
side breaks; class (0, 0) reproduces the standard table's kept list; the structural nnz of a
shifted disc equals a numpy block count; the exact reach covers every target and is tight."""
import numpy as np
import pytest


def _P(orc, **kw):
    base = dict(wavelength=633e-9, pitch=1e-6, n_h=256, n_depth=5, levels=3, z_min=0.05e-3, z_max=0.3e-3,
                retention=1.0, exact=True)
    base.update(kw)
    return orc.Params(**base)


def _points(orc, P, rng, n, margin=0, levels_only=True):
    geo = orc.geometry(P)
    d = rng.integers(0, P.n_depth, n)
    ix = rng.integers(-margin, P.n_h + margin, n)
    iy = rng.integers(-margin, P.n_h + margin, n)
    pts = np.zeros((n, 4))
    pts[:, 0] = (ix - P.n_h // 2) * P.pitch
    pts[:, 1] = (iy - P.n_h // 2) * P.pitch
    pts[:, 2] = geo["z"][d]
    pts[:, 3] = 1.0 - rng.random(n)
    return pts


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("seed,levels", [(1, 3), (2, 2), (3, 1)])
def test_exact_keep_all_equals_direct_sum_anywhere(orc, seed, levels):
    """r = 100%, random integer (not 2^L-aligned) points, PSFs overlapping and clipped at the edge:
    WASABI with offset-class tables == D2 == D1 to <= 1e-12 rel L2."""
    P = _P(orc, levels=levels)
    rng = np.random.default_rng(seed)
    pts = _points(orc, P, rng, 10, margin=48)
    u, _, _ = orc.Lut(P).hologram_window(pts, 0, 0, 256, 256)
    d2 = orc.direct_d2(P, pts, 0, 0, 256, 256)
    d1 = orc.direct_d1(P, pts, 0, 0, 256, 256)
    assert np.linalg.norm(d2) > 0
    assert _rel(u, d2) <= 1e-12
    assert _rel(d1, d2) <= 1e-12


def test_standard_mode_is_not_exact_off_grid(orc):
    """Control: the same non-aligned points under R-A8 (one table per depth) do NOT reproduce the
    direct sum -- so the previous pin really exercises the offset classes."""
    P = _P(orc, exact=False)
    rng = np.random.default_rng(1)
    pts = _points(orc, P, rng, 10, margin=48)
    u, _, _ = orc.Lut(P).hologram_window(pts, 0, 0, 256, 256)
    d2 = orc.direct_d2(P, pts, 0, 0, 256, 256)
    assert _rel(u, d2) > 1e-3


@pytest.mark.parametrize("d", [0, 2, 4])
def test_class_zero_reproduces_standard_list(orc, d):
    """Class (0, 0) holds the standard table plus 2^L empty rows/columns: at r < 1 (only nonzero
    coefficients kept) its kept list (level, dx, dy, value) equals the standard one exactly."""
    Pe = _P(orc, retention=0.1)
    Ps = _P(orc, retention=0.1, exact=False)
    t = d << (2 * Pe.levels)
    cap = orc.table_info(Pe, t)["n_r"] + 8
    le, xe, ye, ve = orc.select(Pe, t, cap)
    ls, xs, ys, vs = orc.select(Ps, d, cap)
    assert orc.table_info(Pe, t)["side"] == orc.table_info(Ps, d)["side"] + (1 << Pe.levels)
    assert np.array_equal(le, ls) and np.array_equal(xe, xs) and np.array_equal(ye, ys)
    assert np.array_equal(ve, vs)


@pytest.mark.parametrize("t", [5, 3 * 64 + 27, 4 * 64 + 63])
def test_class_table_geometry_and_nnz(orc, t):
    """Table t = d 4^L + cy 2^L + cx: side 2H + 2^L; the PSF is centred at (H + cx, H + cy) (its
    modulus is 1 exactly on the shifted disc); structural nnz = numpy count of 2^l blocks touching
    the shifted disc (3 per block per level, 4 at level L)."""
    P = _P(orc)
    L = P.levels
    info = orc.table_info(P, t)
    d, cy, cx = t >> (2 * L), (t >> L) & 7, t & 7
    H, side = info["H"], info["side"]
    assert side == 2 * H + (1 << L)
    f = orc.psf_table(P, t)
    R = orc.geometry_one(P, d)["R"]
    Y, X = np.mgrid[0:side, 0:side]
    dx, dy = X - (H + cx), Y - (H + cy)
    disc = (dx * dx + dy * dy < R * R) | ((dx == 0) & (dy == 0))
    assert np.array_equal(np.abs(f) > 0.5, disc)
    assert np.allclose(np.abs(f[disc]), 1.0, atol=1e-14)
    nnz = 0
    for l in range(1, L + 1):
        b = 1 << l
        blk = disc.reshape(side // b, b, side // b, b).any(axis=(1, 3))
        nnz += int(blk.sum()) * (4 if l == L else 3)
    assert info["nnz"] == nnz


def test_exact_reach_covers_and_is_tight(orc):
    """Reach (R-A19 with R-A20's exact offsets): for a point of class (cx, cy), every kept entry
    lands at (ix - cx + dx, iy - cy + dy), within ek per axis and q in squared distance of the
    point, and both bounds are attained."""
    P = _P(orc, retention=0.2)
    L = P.levels
    ek, q = orc.reach(P)
    for t in (1, 2 * 64 + 9, 4 * 64 + 42):
        cx, cy = t & 7, (t >> L) & 7
        lv, dx, dy, _ = orc.select(P, t, orc.table_info(P, t)["n_r"] + 8)
        ox, oy = dx - cx, dy - cy
        assert max(np.abs(ox).max(), np.abs(oy).max()) == ek[t]
        assert (ox.astype(np.int64) ** 2 + oy.astype(np.int64) ** 2).max() == q[t]
