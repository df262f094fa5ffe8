"""Design study (CPU only, oracle tables): shared-memory bank wavefronts of the superpose
read-modify-write for one C4 depth, under candidate shared-tile layouts.

A chunk = 32 consecutive entries of one (point, level, strip) window-LUT range (column groups of
G_l = max(8, 2^l) columns, row-major inside a group).  Model of an 8-byte shared access: two
phases of 16 lanes; a phase costs the largest number of distinct addresses sharing a 64-bit bank
slot (slot = float2 index mod 16)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import CONFIGS   # noqa: E402
from oracle import oracle as O   # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 96
cfg = CONFIGS["C4"]
P = O.Params.from_config(cfg)
g = O.geometry(P)
lv, dx, dy, val = O.select(P, d, int(g['n_r'][d]) + 8)
H = int(g['H'][d])
T, L = 64, P.levels
rng = np.random.default_rng(0)


def layouts():
    yield "linear S=70 (v19)", lambda r, c: 6 + r * 70 + c
    yield "linear S=72", lambda r, c: 8 + r * 72 + c
    yield "linear S=80", lambda r, c: 16 + r * 80 + c
    # v20: cell t at t ^ ((t >> 5) & 7) (byte address bits 3..5 ^= bits 8..10, 2 KB-aligned base)
    yield "S=72 swizzle (v20)", lambda r, c: (lambda t: t ^ ((t >> 5) & 7))(8 + r * 72 + c)
    yield "S=80 t^(3(t>>6)&15)", lambda r, c: (lambda t: t ^ (((t >> 6) * 3) & 15))(16 + r * 80 + c)


def phase_cost(addr):
    cost = 0
    for h in (addr[:16], addr[16:]):
        if len(h) == 0:
            continue
        u = np.unique(h)
        cost += np.bincount(u % 16, minlength=16).max()
    return cost


res = {}
n_chunks = {}
for trial in range(400):
    ix, iy = rng.integers(0, 1 << 20, 2)
    tx0 = int(rng.integers(-H, H)) // T * T + ix // T * T * 0
    for l in range(1, L + 1):
        h = 1 << (l - 1)
        sx = ((ix + h) >> l) << l
        sy = ((iy + h) >> l) << l
        m = lv == l
        X = sx + dx[m]
        Y = sy + dy[m]
        tx = (sx // T) * T + int(rng.integers(-H // T - 1, H // T + 1)) * T
        ty = (sy // 32) * 32 + int(rng.integers(-H // 32 - 1, H // 32 + 1)) * 32
        sel = (X >= tx) & (X < tx + T) & (Y >= ty) & (Y < ty + 32)
        if not sel.any():
            continue
        lg = max(3, l)
        grp = (dx[m][sel] + H) >> lg
        r = Y[sel] - ty
        c = X[sel] - tx
        order = np.lexsort((c, r, grp))
        r, c = r[order], c[order]
        for name, f in layouts():
            a = f(r, c)
            for k in range(0, len(a), 32):
                res.setdefault((name, l), 0)
                res[(name, l)] += phase_cost(a[k:k + 32])
        n_chunks[l] = n_chunks.get(l, 0) + (len(r) + 31) // 32
names = [n for n, _ in layouts()]
print(f"depth {d} H {H}; wavefronts per LDS.64 chunk by level (ideal 2 for a full chunk)")
print("level chunks " + " | ".join(names))
tot = {n: 0 for n in names}
for l in range(1, L + 1):
    if l not in n_chunks:
        continue
    print(l, n_chunks[l], " ".join(f"{res[(n, l)] / n_chunks[l]:.2f}" for n in names))
    for n in names:
        tot[n] += res[(n, l)]
print("all", sum(n_chunks.values()), " ".join(f"{tot[n] / sum(n_chunks.values()):.2f}" for n in names))
