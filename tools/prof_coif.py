"""Profiling driver for the coiflet inverse (WASABI_FLAG_COIFLET, R-A21): C4 at level 3 on one row band;
superpose once, then time wasabi_inverse_wt fused (u in its own buffer) and as in-place line passes."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for i, arg in enumerate(sys.argv):          # --pkg DIR: import the package from a variant copy
    if arg == "--pkg":
        sys.path.insert(0, os.path.abspath(sys.argv[i + 1]))
import torch  # noqa: E402

import paper_1708_04233_b200 as W  # noqa: E402
from inputs import CONFIGS, make_points  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--row0", type=int, default=32768)
ap.add_argument("--rows", type=int, default=4096)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mode", default="both", choices=["both", "fused", "lines"])
ap.add_argument("--pkg", default=None)
a = ap.parse_args()
cfg = CONFIGS["C4"].replace(levels=3)
p = W.Params.from_config(cfg, wavelet=1)
pts = make_points(cfg)
pl = W.Pipeline(p, len(pts), a.row0, a.row0 + a.rows)
pl.build_tables()
pl.bin(torch.from_numpy(pts).cuda())
pl.superpose()
psi0 = pl.psi_band.clone()
pr = W.PrintParams()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
if a.mode in ("both", "fused"):
    W.inverse_wt(p, pl.psi_band, pl.field, pl.row0, pl.row1, pr, pl.bits)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(a.reps):
        W.inverse_wt(p, pl.psi_band, pl.field, pl.row0, pl.row1, pr, pl.bits)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"fused tiles: {ev[0].elapsed_time(ev[1]) / a.reps:.3f} ms for {a.rows} rows")
if a.mode in ("both", "lines"):
    ms = 0.0
    for _ in range(a.reps):
        pl.psi_band.copy_(psi0)
        u = pl.psi_band[pl.row0 - pl.e0:pl.row1 - pl.e0]
        ev[0].record()
        W.inverse_wt(p, pl.psi_band, u, pl.row0, pl.row1, pr, pl.bits)
        ev[1].record()
        torch.cuda.synchronize()
        ms += ev[0].elapsed_time(ev[1])
    print(f"line passes (halo band {pl.e1 - pl.e0} rows) + quantize: {ms / a.reps:.3f} ms for {a.rows} rows")
