"""Profiling driver: C4-density workload restricted to one row band, runs each step once
(plus `--reps` superpose repeats) so ncu can capture single kernels quickly."""
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
ap.add_argument("--config", default="C4")
ap.add_argument("--row0", type=int, default=32768)
ap.add_argument("--rows", type=int, default=512)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--tile", type=int, default=None)
ap.add_argument("--fused", action="store_true", help="time superpose_inverse (fused path, as bench.py)")
ap.add_argument("--pkg", default=None)
ap.add_argument("--retention", type=float, default=None)
ap.add_argument("--n", type=int, default=None, help="point count (default: the config's)")
ap.add_argument("--path", default="auto", choices=["auto", "gather", "scatter"])
ap.add_argument("--wavelet", type=int, default=0, help="1: coif1 tables (superpose on the psi band, unfused)")
ap.add_argument("--levels", type=int, default=None)
ap.add_argument("--sort-depth", action="store_true", help="experiment: permute the points by depth (stable)")
ap.add_argument("--no-u", action="store_true", help="fused: bits only (no u write)")
ap.add_argument("--no-bits", action="store_true", help="fused: u only (no binarisation)")
ap.add_argument("--snap-y", type=int, default=0, help="experiment: snap every point's pixel row to a multiple of K")
ap.add_argument("--dump", default=None, help="np.save psi (after the timed superposes) to this path")
a = ap.parse_args()
cfg = CONFIGS[a.config]
if a.tile:
    cfg = cfg.replace(tile=a.tile)
if a.retention:
    cfg = cfg.replace(retention=a.retention)
if a.levels:
    cfg = cfg.replace(levels=a.levels)
p = W.Params.from_config(cfg, path=a.path, wavelet=a.wavelet)
pts = make_points(cfg, n=a.n)
if a.snap_y:
    import numpy as np
    iy = np.floor(pts[:, 1].astype(np.float64) / cfg.pitch + 0.5)
    pts[:, 1] = (np.round(iy / a.snap_y) * a.snap_y * cfg.pitch).astype(np.float32)
if a.sort_depth:
    import numpy as np
    pts = pts[np.argsort(pts[:, 2], kind="stable")]
pl = W.Pipeline(p, len(pts), a.row0, a.row0 + a.rows, want_u=not a.no_u, want_bits=not a.no_bits)
d = torch.from_numpy(pts).cuda()
pl.run(d)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import Clocks  # noqa: E402
clocks = Clocks(0, "/tmp/prof_superpose_clocks.csv")
clocks.start()
import time  # noqa: E402
time.sleep(0.3)
ev[0].record()
for _ in range(a.reps):
    if a.fused:
        pl.superpose_inverse()
    else:
        pl.superpose()
ev[1].record()
torch.cuda.synchronize()
ck = clocks.stop()
st = W.bins_stats(pl.bins)
print(f"[{a.pkg or 'tree'}] {W.__file__.split('/')[-3]} {('fused' + (' no-u' if a.no_u else '') + (' no-bits' if a.no_bits else '')) if a.fused else 'superpose'} {ev[0].elapsed_time(ev[1]) / a.reps:.3f} ms for {a.rows} rows; bin entries {st['entries']}; clocks {ck}")
if a.dump:
    import hashlib
    import numpy as np
    f = pl.field.cpu().numpy()
    np.save(a.dump, f)
    print(f"[{a.pkg or 'tree'}] psi sha1 {hashlib.sha1(f.tobytes()).hexdigest()} -> {a.dump}")
