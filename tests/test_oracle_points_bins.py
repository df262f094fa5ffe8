"""Pins for the oracle's step 2a: point conversion and binning (R-A3, R-A9,
R-A11, R-A12, R-A17).  Independent references: SPEC.md's worked examples, the paper's
sub-hologram re-basing example, and a vectorised numpy box-overlap enumeration."""
import json
import os

import numpy as np
import pytest

from inputs import CONFIGS, make_points

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_params.json")))


def _P(orc, **kw):
    base = dict(wavelength=633e-9, pitch=1e-6, n_h=1024, n_depth=8, levels=3, z_min=0.1e-3, z_max=0.4e-3,
                retention=0.10)
    base.update(kw)
    return orc.Params(**base)


def test_to_pixel_examples(orc):
    """SPEC.md:64-70 to_pixel examples (hologram-centred origin, nearest pixel)."""
    P = _P(orc)
    pts = np.array([[0, 0, 0.2e-3, 1], [3e-6, -2e-6, 0.2e-3, 1], [0.4e-6, 0, 0.2e-3, 1],
                    [0.5e-6, -0.5e-6, 0.2e-3, 1]])
    ix, iy, iz, ok = orc.points(P, pts)
    assert ok.all()
    assert (ix[0], iy[0]) == (512, 512)
    assert (ix[1], iy[1]) == (515, 510)
    assert (ix[2], iy[2]) == (512, 512)
    assert (ix[3], iy[3]) == (513, 512)     # half-way rounds toward +inf (R-A9)


def test_depth_quantisation_rules(orc):
    """nearest level, ties to the lower index; half a level of slack at both ends;
    beyond that, a <= 0, or non-finite -> skipped (R-A17)."""
    P = _P(orc, n_depth=4, z_min=0.0, z_max=3e-3)   # levels at 0, 1, 2, 3 mm
    zs = [0.0, 0.49e-3, 0.5e-3, 0.51e-3, 1.6e-3, 2.5e-3, 3.0e-3, 3.5e-3, 3.51e-3, -0.5e-3, -0.51e-3]
    pts = np.array([[0, 0, z, 1.0] for z in zs])
    _, _, iz, ok = orc.points(P, pts)
    assert list(ok) == [True] * 8 + [False, True, False]
    assert list(iz[:8]) == [0, 0, 0, 1, 2, 2, 3, 3]
    assert iz[9] == 0
    bad = np.array([[0, 0, 1e-3, 0.0], [0, 0, 1e-3, -1.0], [np.nan, 0, 1e-3, 1], [0, np.inf, 1e-3, 1],
                    [0, 0, np.nan, 1]])
    assert not orc.points(P, bad)[3].any()


def test_paper_subhologram_rebasing_example(orc):
    """PAPER.md:121 x'_j = x_j - s N_h, worked in SPEC.md:257: pixel (20000, 5000) in
    sub-hologram (2, 0) of side 8192 is at (3616, 5000).  Row bands are the same re-basing on y."""
    g = GOLD["rebase_example"]
    (x, y), (s, t), nh = g["point_px"], g["subholo_st"], g["Nh"]
    assert (x - s * nh, y - t * nh) == tuple(g["expected"])
    # the oracle's band/tile bin of that point: tile containing (3616, 5000) in band row0 = 0 of an
    # 8192-wide sub-hologram holds the point when addressed with re-based coordinates
    P = _P(orc, n_h=8192)
    px = np.array([[(3616 - 4096) * 1e-6, (5000 - 4096) * 1e-6, 0.2e-3, 1.0]])
    ix, iy, _, ok = orc.points(P, px)
    assert ok[0] and (ix[0], iy[0]) == (3616, 5000)
    idx = orc.bin_tile(P, 64, px, 3584, 4992)
    assert list(idx) == [0]


def _numpy_bins(orc, P, T, pts, row0, row1):
    """Tile lists by the footprint definition (R-A12, R-A19), enumerated with numpy per point."""
    ix, iy, iz, ok = orc.points(P, pts)
    ek_d, q_d = orc.reach(P)
    tx_n = P.n_h // T
    ty_n = (row1 - row0) // T
    lists = [[] for _ in range(tx_n * ty_n)]
    X0 = np.arange(tx_n) * T
    Y0 = row0 + np.arange(ty_n) * T
    for j in np.flatnonzero(ok):
        ek, q = ek_d[iz[j]], q_d[iz[j]]
        ddx = np.maximum(np.maximum(X0 - ix[j], ix[j] - (X0 + T - 1)), 0)
        ddy = np.maximum(np.maximum(Y0 - iy[j], iy[j] - (Y0 + T - 1)), 0)
        mx = ddx <= ek
        my = ddy <= ek
        member = my[:, None] & mx[None, :] & (ddy[:, None] ** 2 + ddx[None, :] ** 2 <= q)
        for t in np.flatnonzero(member.reshape(-1)):
            lists[t].append(j)
    ptr = np.zeros(len(lists) + 1, np.int64)
    ptr[1:] = np.cumsum([len(l) for l in lists])
    idx = np.array([j for l in lists for j in l], np.int32)
    return ptr, idx


@pytest.mark.parametrize("row0,row1", [(0, 512), (128, 320)])
def test_bins_equal_numpy_footprint_enumeration(orc, row0, row1):
    """Every valid point appears, in ascending order, in exactly the tiles of its footprint
    (square +- ek_d and squared distance <= q_d, R-A19), restricted to the band."""
    c = CONFIGS["C1"]
    P = orc.Params.from_config(c)
    pts = make_points(c, n=300)
    pts[5, 3] = -1.0          # skipped
    pts[6, 0] = 0.9e-3        # far outside the aperture: partial/no overlap
    ptr, idx = orc.bins(P, 64, pts, row0, row1)
    ptr2, idx2 = _numpy_bins(orc, P, 64, pts, row0, row1)
    assert np.array_equal(ptr, ptr2) and np.array_equal(idx, idx2)
    assert 5 not in set(idx.tolist())
    for t in range(len(ptr) - 1):
        seg = idx[ptr[t]:ptr[t + 1]]
        assert np.all(np.diff(seg) > 0)
    # bin_tile gives the same lists
    tx_n = P.n_h // 64
    for t in (0, 3, len(ptr) - 2):
        X0 = (t % tx_n) * 64
        Y0 = row0 + (t // tx_n) * 64
        assert np.array_equal(orc.bin_tile(P, 64, pts, X0, Y0), idx[ptr[t]:ptr[t + 1]])


@pytest.mark.parametrize("retention", [0.05, 1.0])
def test_reach_covers_every_retained_coefficient(orc, retention):
    """R-A19: for every depth and every sub-position of the point on the 2^L grid, every retained
    coefficient of every level lands within ek_d (per axis) and within squared distance q_d of the
    point (R-A8 shift included); the bound is tight to one pixel; ek_d <= the structural E_d."""
    c = CONFIGS["C1"]
    P = orc.Params(**{**orc.Params.from_config(c).__dict__, "retention": retention})
    geo = orc.geometry(P)
    ek_d, q_d = orc.reach(P)
    for d in range(P.n_depth):
        lv, dx, dy, _ = orc.select(P, d, int(geo["n_r"][d]))
        worst_ax, worst_q = 0, 0
        for rho in range(1 << P.levels):
            i = 1000 + rho
            s = np.array([(1 << l) * ((i + (1 << (l - 1))) >> l) for l in lv])
            tx = np.abs(s + dx - i)
            ty = np.abs(s + dy - i)          # same sub-position on both axes
            worst_ax = max(worst_ax, int(tx.max()), int(ty.max()))
            worst_q = max(worst_q, int((tx * tx + ty * ty).max()))
            assert tx.max() <= ek_d[d] and ty.max() <= ek_d[d]
            assert (tx * tx + ty * ty).max() <= q_d[d]
        assert ek_d[d] - worst_ax <= 1
        assert ek_d[d] <= geo["E"][d]
        assert q_d[d] >= worst_q


def test_bins_contain_every_tile_a_point_writes(orc):
    """Brute force through Eq.(2) itself: for single points at assorted sub-pixel grid positions and
    depths, every tile holding a nonzero psi coefficient of that point (oracle WASABI window over the
    whole hologram) lists the point; and the footprint is much smaller than the old 3 2^(L-1) box."""
    c = CONFIGS["C1"]
    P = orc.Params.from_config(c)
    lut = orc.Lut(P)
    T = 64
    n_h = P.n_h
    rng = np.random.default_rng(7)
    for trial in range(6):
        ix, iy = int(rng.integers(0, n_h)), int(rng.integers(0, n_h))
        d = int(rng.integers(0, P.n_depth))
        dz = (P.z_max - P.z_min) / (P.n_depth - 1)
        pt = np.array([[(ix - n_h // 2) * P.pitch, (iy - n_h // 2) * P.pitch, P.z_min + d * dz, 1.0]])
        psi, cnt = lut.wasabi_window(pt, 0, 0, n_h, n_h)
        assert cnt > 0
        ys, xs = np.nonzero(psi)
        written = set(((ys // T) * (n_h // T) + xs // T).tolist())
        ptr, idx = orc.bins(P, T, pt, 0, n_h)
        listed = {t for t in range(len(ptr) - 1) if ptr[t + 1] > ptr[t]}
        assert written <= listed
        E = int(orc.geometry(P)["E"][d])
        bx = range(max(0, (ix - E) // T), min(n_h // T - 1, (ix + E) // T) + 1)
        by = range(max(0, (iy - E) // T), min(n_h // T - 1, (iy + E) // T) + 1)
        assert len(listed) <= len(bx) * len(by)
    lut.close()
