"""Design study (CPU only, oracle tables): shared-memory bank wavefronts of the superpose RMW for a
Mallat (subband-planar) shared tile vs the interleaved + swizzle layout (v20..v28), on C4 depths.
A chunk = 32 consecutive entries of one (point, level, 32-row strip) range; model of an 8-byte shared
access: two phases of 16 lanes, a phase costs the largest number of distinct addresses sharing a
64-bit bank slot (slot = float2 index mod 16).  Entries inside a column group may be ordered freely
(one point: distinct targets)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import CONFIGS   # noqa: E402
from oracle import oracle as O   # noqa: E402

T, L = 64, 6
cfg = CONFIGS["C4"]
P = O.Params.from_config(cfg)
g = O.geometry(P)
rng = np.random.default_rng(0)


def phase_cost(addr):
    cost = 0
    for h in (addr[:16], addr[16:]):
        if len(h) == 0:
            continue
        u = np.unique(h)
        cost += np.bincount(u % 16, minlength=16).max()
    return cost


def interleaved_swz(l, b, i, j, strip):
    h = 1 << (l - 1)
    x = (i << l) + (h if b != 1 else 0)
    y = (j << l) + (h if b >= 1 else 0) - 32 * strip
    t = 8 + y * 72 + x
    return t ^ ((t >> 5) & 7)


def mallat(W, pad_sub):
    def f(l, b, i, j, strip):
        C = T >> l
        rows = max(1, 32 >> l)
        Wl = W(C)
        return b * (rows * Wl + pad_sub) + (j - strip * rows) * Wl + i + 4
    return f


layouts = {"interleaved+swz (v28)": interleaved_swz,
           "mallat W=C+8": mallat(lambda C: C + 8, 0),
           "mallat W=C+4": mallat(lambda C: C + 4, 0),
           "mallat W=C+12": mallat(lambda C: C + 12, 4),
           "mallat W=C+8 subpad8": mallat(lambda C: C + 8, 8)}
orders = ["grp,j,i", "grp,i,j", "grp,b,j,i", "grp,j,b,i"]
res, nch = {}, {}
for d in (10, 30, 60, 100, 120):
    lv, dx, dy, val = O.select(P, d, int(g['n_r'][d]))
    H = int(g['H'][d])
    for trial in range(150):
        ix, iy = (int(v) for v in rng.integers(0, 1 << 20, 2))
        for l in (1, 2, 3):
            h = 1 << (l - 1)
            sx = ((ix + h) >> l) << l
            sy = ((iy + h) >> l) << l
            m = lv == l
            X = sx + dx[m]
            Y = sy + dy[m]
            tx = (sx // T) * T + int(rng.integers(-H // T - 1, H // T + 1)) * T
            ty = (sy // 64) * 64 + int(rng.integers(-H // 64 - 1, H // 64 + 1)) * 64
            strip = int(rng.integers(0, 2))
            ty32 = ty + 32 * strip
            sel = (X >= tx) & (X < tx + T) & (Y >= ty32) & (Y < ty32 + 32)
            if not sel.any():
                continue
            lg = max(3, l)
            grp = (dx[m][sel] + H) >> lg
            xt, yt = X[sel] - tx, Y[sel] - ty
            b = ((yt >> (l - 1)) & 1) + (((xt >> (l - 1)) & 1) & ((yt >> (l - 1)) & 1))
            i, j = xt >> l, yt >> l
            for on in orders:
                keys = {"grp": grp, "i": i, "j": j, "b": b}
                order = np.lexsort(tuple(keys[k] for k in reversed(on.split(","))))
                for name, f in layouts.items():
                    a = np.array([f(l, int(b[o]), int(i[o]), int(j[o]), strip) for o in order])
                    c = sum(phase_cost(a[k:k + 32]) for k in range(0, len(a), 32))
                    res[(name, on, l)] = res.get((name, on, l), 0) + c
            nch[l] = nch.get(l, 0) + (int(sel.sum()) + 31) // 32
print("wavefronts per LDS.64 chunk (ideal 2 for a full chunk); chunks per level", nch)
for name in layouts:
    for on in orders:
        per = [res[(name, on, l)] / nch[l] for l in (1, 2, 3)]
        tot = sum(res[(name, on, l)] for l in (1, 2, 3)) / sum(nch.values())
        print(f"{name:24s} order {on:10s} l1 {per[0]:.2f} l2 {per[1]:.2f} l3 {per[2]:.2f} all {tot:.2f}")
