"""Run one pipeline step of a config in a table mode (for launch lists / timing of the optional modes).
    python tools/run_mode.py --config C5 --levels 3 --wavelet 1 --points 100000 --retention 0.05"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_04233_b200 as W  # noqa: E402
from inputs import CONFIGS, make_points  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--levels", type=int, default=None)
ap.add_argument("--wavelet", type=int, default=0)
ap.add_argument("--exact", action="store_true")
ap.add_argument("--points", type=int, default=None)
ap.add_argument("--retention", type=float, default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
cfg = CONFIGS[a.config]
if a.levels:
    cfg = cfg.replace(levels=a.levels)
if a.retention:
    cfg = cfg.replace(retention=a.retention)
pts = make_points(cfg, n=a.points)
p = W.Params.from_config(cfg, wavelet=a.wavelet, exact=a.exact)
pl = W.Pipeline(p, len(pts), 0, p.n_h)
d = torch.from_numpy(pts).cuda()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for _ in range(a.reps):
    ev[0].record()
    pl.build_tables()
    ev[1].record()
    pl.bin(d)
    ev[2].record()
    if a.wavelet:
        pl.superpose()
        ev[3].record()
        pl.inverse()
    else:
        pl.superpose_inverse()
        ev[3].record()
    ev[4].record()
torch.cuda.synchronize()
print(f"{a.config} L={cfg.levels} wavelet={a.wavelet} exact={a.exact} N={len(pts)} r={cfg.retention}: tables "
      f"{ev[0].elapsed_time(ev[1]):.2f} bins {ev[1].elapsed_time(ev[2]):.2f} superpose {ev[2].elapsed_time(ev[3]):.2f} "
      f"inverse {ev[3].elapsed_time(ev[4]):.2f} ms")
