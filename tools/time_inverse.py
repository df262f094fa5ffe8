"""Time the standalone inverse (+quantise) and quantise kernels on a band of a C4-sized field.
    python tools/time_inverse.py [--rows 8192]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_04233_b200 as W  # noqa: E402
from inputs import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=8192)
a = ap.parse_args()
p = W.Params.from_config(CONFIGS["C4"])
rows, n = a.rows, p.n_h
psi = torch.randn((rows, n, 2), device="cuda")
u = torch.empty_like(psi)
bits = torch.empty((rows, n // 8), dtype=torch.uint8, device="cuda")
pr = W.PrintParams()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


px = rows * n
for name, fn, bpp in [("inverse u only", lambda: W.inverse_wt(p, psi, u, 0, rows), 16.0),
                      ("inverse + bits", lambda: W.inverse_wt(p, psi, u, 0, rows, pr, bits), 16.125),
                      ("inverse bits only", lambda: W.inverse_wt(p, psi, None, 0, rows, pr, bits), 8.125),
                      ("quantize", lambda: W.quantize(p, pr, u, 0, rows, bits), 8.125)]:
    ms = t(fn)
    print(f"{name:20s} {ms:8.3f} ms  {bpp * px / ms / 1e6:8.1f} GB/s")
