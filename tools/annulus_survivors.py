"""Design study (CPU only, oracle tables): how many (point, tile, warp) combinations of a C4 row band a
per-level radial (annulus) bound of the kept lists would reject, against the exact emptiness from
tools/analyze_ranges.py (/tmp/ranges_c4.npz) -- DESIGN.md §9."""
import sys, os, time
import numpy as np
sys.path.insert(0, '/root/repo')
from inputs import CONFIGS, make_points
from oracle import oracle as O
row0, rows = 32768, 256
cfg = CONFIGS["C4"]; P = O.Params.from_config(cfg); T = 64; L = P.levels
pts = make_points(cfg)
ptr, idx = O.bins(P, T, pts, row0, row0 + rows)
ix, iy, iz, ok = O.points(P, pts)
tiles_x = P.n_h // T
tile_of = np.repeat(np.arange(len(ptr) - 1), np.diff(ptr))
pp = idx.astype(np.int64)
tx0 = (tile_of % tiles_x) * T
ty0 = row0 + (tile_of // tiles_x) * T
g = O.geometry(P)
cls = {0: [1, 3, 6], 1: [2, 4, 5]}
surv = np.zeros((len(pp), 2, 2), bool)  # pair, class, half
for d in np.unique(iz[pp]):
    sel = np.nonzero(iz[pp] == d)[0]
    lv, dx, dy, v = O.select(P, int(d), int(g['n_r'][d]) + 8)
    r2 = dx.astype(np.int64)**2 + dy.astype(np.int64)**2
    for c, ls in cls.items():
        for l in ls:
            m = lv == l
            if not m.any(): continue
            rmin, rmax = r2[m].min(), r2[m].max()
            h = 1 << (l - 1)
            sx = ((ix[pp[sel]] + h) >> l) << l
            sy = ((iy[pp[sel]] + h) >> l) << l
            x0 = tx0[sel] - sx; x1 = x0 + T - 1
            for half in range(2):
                y0 = ty0[sel] + 32 * half - sy; y1 = y0 + 31
                gx = np.maximum(0, np.maximum(x0, -x1)); gy = np.maximum(0, np.maximum(y0, -y1))
                mind = gx**2 + gy**2
                fx = np.maximum(np.abs(x0), np.abs(x1)); fy = np.maximum(np.abs(y0), np.abs(y1))
                maxd = fx**2 + fy**2
                surv[sel, c, half] |= (mind <= rmax) & (maxd >= rmin)
print("pairs", len(pp), "annulus-test survivors per (pair, warp): %.3f" % surv.mean())
d = np.load('/tmp/ranges_c4.npz'); cnt = d['cnt']
exact = np.zeros_like(surv)
for c, ls in cls.items():
    for h in range(2): exact[:, c, h] = cnt[:, ls, h].sum(1) > 0
print("exact non-empty: %.3f" % exact.mean(), " missed (must be 0):", (exact & ~surv).sum())
