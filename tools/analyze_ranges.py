"""Design study (CPU only, oracle tables): per (point, tile, warp-class, row-half, level) kept-entry
counts on a C4 row band, to compare superpose work-distribution schemes."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import CONFIGS, make_points
from oracle import oracle as O

row0 = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 512
cfg = CONFIGS["C4"]; P = O.Params.from_config(cfg); T = 64; L = P.levels
pts = make_points(cfg)
t0 = time.time()
ptr, idx = O.bins(P, T, pts, row0, row0 + rows)
print("bins", len(idx), "pairs", time.time() - t0, "s")
ix, iy, iz, ok = O.points(P, pts)
tiles_x = P.n_h // T
tile_of = np.repeat(np.arange(len(ptr) - 1), np.diff(ptr))
pp = idx.astype(np.int64)
tx0 = (tile_of % tiles_x) * T
ty0 = row0 + (tile_of // tiles_x) * T
g = O.geometry(P)
cnt = np.zeros((len(pp), L + 1, 2), np.int64)   # [pair, level, half]
rows_rej = np.zeros((len(pp), L + 1, 2), np.int64)
for d in np.unique(iz[pp]):
    sel = np.nonzero(iz[pp] == d)[0]
    lv, dx, dy, v = O.select(P, int(d), int(g['n_r'][d]) + 8)
    H = int(g['H'][d]); side = 2 * H
    for l in range(1, L + 1):
        m = lv == l
        if not m.any():
            continue
        X = dx[m] + H; Y = dy[m] + H
        grid = np.zeros((side + 1, side + 1), np.int64)
        np.add.at(grid, (Y + 1, X + 1), 1)
        grid = grid.cumsum(0).cumsum(1)
        h = 1 << (l - 1)
        sx = ((ix[pp[sel]] + h) >> l) << l
        sy = ((iy[pp[sel]] + h) >> l) << l
        xa = np.clip(tx0[sel] - sx + H, 0, side); xb = np.clip(tx0[sel] - sx + H + T, 0, side)
        for half in range(2):
            ya = np.clip(ty0[sel] + 32 * half - sy + H, 0, side)
            yb = np.clip(ty0[sel] + 32 * half - sy + H + 32, 0, side)
            c = grid[yb, xb] - grid[ya, xb] - grid[yb, xa] + grid[ya, xa]
            cnt[sel, l, half] = c
print("useful entries", cnt.sum(), "per pair", cnt.sum() / len(pp))
print("per level", [int(cnt[:, l].sum()) for l in range(L + 1)])
cls = {0: [1, 4, 5, 6], 1: [2, 3]}
for name, cl in [("v14 classes", cls), ("l1 | rest", {0: [1], 1: [2, 3, 4, 5, 6]})]:
    ch_pt = 0; ch_mix = 0; units = 0; nz_ranges = 0; ch_rng = 0
    for c, ls in cl.items():
        for half in range(2):
            n = cnt[:, ls, half].sum(1)
            ch_pt += np.ceil(n / 32).sum(); ch_mix += n.sum() / 32; units += (n > 0).sum()
            for l in ls:
                nl = cnt[:, l, half]
                nz_ranges += (nl > 0).sum(); ch_rng += np.ceil(nl / 32).sum()
    print(f"{name}: chunks per-point-flattened {ch_pt:.3e}  per-range {ch_rng:.3e}  mixed {ch_mix:.3e}  "
          f"units {units:.3e} nonempty level-ranges {nz_ranges:.3e}")
np.savez_compressed("/tmp/ranges_c4.npz", cnt=cnt, ptr=ptr)
