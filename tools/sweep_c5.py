"""C5 sweep (BASELINE.json configs[4]): 16,384^2 hologram, N in {1e4..1e7} x r in {1,2,5,10,25,100}%.

For every cell: WASABI throughput (tables + bins + fused superpose/inverse/quantise, CUDA events)
and PSNR of u against the conventional method -- the quantised direct sum of Eq.(1) computed on the
GPU by PSF stamping (wasabi_direct_sum; reading R-A18: PSNR = 10 log10(max|u_ref|^2 / mean|u-u_ref|^2)).
The direct sum's own time gives the same-box WASABI-vs-conventional speed-up.
Uses only the product library.  Writes one JSON object per line.
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_04233_b200 as W  # noqa: E402
from inputs import CONFIGS, make_points  # noqa: E402


def timed(fn, reps=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="10000,100000,1000000,10000000")
    ap.add_argument("--rs", default="0.01,0.02,0.05,0.10,0.25,1.0")
    ap.add_argument("--aligned", action="store_true")
    ap.add_argument("--exact", action="store_true", help="offset-class tables (WASABI_FLAG_EXACT_SHIFT, R-A20)")
    ap.add_argument("--levels", type=int, default=None)
    ap.add_argument("--wavelet", type=int, default=0, help="1: coif1 tables (WASABI_FLAG_COIFLET, R-A21)")
    ap.add_argument("--depths", type=int, default=None)
    ap.add_argument("--out", default="gpurun_out/c5_sweep.jsonl")
    a = ap.parse_args()
    base = CONFIGS["C5"]
    if a.aligned:
        base = base.replace(aligned=True)
    if a.levels:
        base = base.replace(levels=a.levels)
    if a.depths:
        base = base.replace(n_depth=a.depths)
    f = open(a.out, "w")
    for n in [int(x) for x in a.ns.split(",")]:
        pts = make_points(base, n=n)
        d_pts = torch.from_numpy(pts).cuda()
        u_ref = None
        t_direct = None
        for r in [float(x) for x in a.rs.split(",")]:
            cfg = base.replace(retention=r)
            p = W.Params.from_config(cfg, exact=a.exact, wavelet=a.wavelet)
            pl = W.Pipeline(p, n, 0, p.n_h)
            t_w = timed(lambda: pl.run(d_pts), reps=3 if n < 10_000_000 else 1)
            if u_ref is None:
                # the reference stamps whole PSFs: bins of the standard mode at r = 1 (R-A19's reach of
                # a smaller r may not cover the PSF's edge)
                ps = W.Params.from_config(cfg.replace(retention=1.0))
                pls = W.Pipeline(ps, n, 0, ps.n_h, want_bits=False)
                pls.build_tables()
                pls.bin(d_pts)
                bins_ref = pls.bins
                dense = torch.empty(W.psf_dense_bytes(ps), dtype=torch.uint8, device="cuda")
                W.build_psf_dense(ps, dense)
                u_ref = torch.empty_like(pl.field)
                t_direct = timed(lambda: W.direct_sum(ps, dense, bins_ref, 0, ps.n_h, u_ref), reps=1)
                del dense, bins_ref, pls
            diff = (pl.field - u_ref).double()
            mse = float((diff * diff).sum(dim=-1).mean())
            peak = float((u_ref.double() ** 2).sum(dim=-1).max())
            psnr = 10 * math.log10(peak / mse) if mse > 0 else float("inf")
            st = W.bins_stats(pl.bins)
            rec = {"n_points": n, "retention": r, "aligned": a.aligned, "exact": a.exact, "wavelet": a.wavelet,
                   "levels": cfg.levels,
                   "n_depth": cfg.n_depth, "wasabi_ms": t_w,
                   "gpix_per_s": p.n_h ** 2 / (t_w * 1e-3) / 1e9, "points_per_s": n / (t_w * 1e-3),
                   "direct_sum_ms": t_direct, "speedup_vs_direct": t_direct / t_w, "psnr_db_vs_direct": psnr,
                   "bin_entries": st["entries"]}
            print(json.dumps(rec), flush=True)
            f.write(json.dumps(rec) + "\n")
            f.flush()
            del pl
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
