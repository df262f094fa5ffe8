"""C5 sweep (BASELINE.json configs[4]): 16,384^2 hologram, N in {1e4..1e7} x r in {1,2,5,10,25,100}%.

For every cell: the WASABI step (tables + bins + fused superpose/inverse/quantise, CUDA events; the
fused kernel timed on its own too), its exact Eq.(2) accumulation count (wasabi_count_accumulations)
and from it the FP32 and HBM roofline fractions of the fused kernel, and the PSNR of u (reading
R-A18: PSNR = 10 log10(max|u_ref|^2 / mean|u - u_ref|^2)) against both direct sums of Eq.(1) computed
on the GPU: D2 = the quantised direct sum by PSF stamping (wasabi_direct_sum, the conventional method
the paper compares against; its time gives the same-box speed-up) and D1 = the
exact Eq.(1) with continuous positions and depths (wasabi_direct_exact).  Uses only the product
library; nvidia-smi clocks are sampled during the sweep.  One JSON object per line.
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1708_04233_b200 as W  # noqa: E402
from bench import Clocks, _peaks  # noqa: E402
from inputs import CONFIGS, make_points  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


def psnr(u, ref):
    diff = (u - ref).double()
    mse = float((diff * diff).sum(dim=-1).mean())
    peak = float((ref.double() ** 2).sum(dim=-1).max())
    return 10 * math.log10(peak / mse) if mse > 0 else float("inf")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="10000,100000,1000000,10000000")
    ap.add_argument("--rs", default="0.01,0.02,0.05,0.10,0.25,1.0")
    ap.add_argument("--aligned", action="store_true")
    ap.add_argument("--exact", action="store_true", help="offset-class tables (WASABI_FLAG_EXACT_SHIFT, R-A20)")
    ap.add_argument("--levels", type=int, default=None)
    ap.add_argument("--wavelet", type=int, default=0, help="1: coif1 tables (WASABI_FLAG_COIFLET, R-A21)")
    ap.add_argument("--depths", type=int, default=None)
    ap.add_argument("--no-d1", action="store_true")
    ap.add_argument("--path", default="auto", choices=["auto", "gather", "scatter"],
                    help="superposition kernel (WASABI_FLAG_GATHER / _SCATTER; auto: gather iff r >= 0.25)")
    ap.add_argument("--out", default="gpurun_out/c5_sweep.jsonl")
    a = ap.parse_args()
    base = CONFIGS["C5"]
    if a.aligned:
        base = base.replace(aligned=True)
    if a.levels:
        base = base.replace(levels=a.levels)
    if a.depths:
        base = base.replace(n_depth=a.depths)
    (hbm, _), (fp32, _) = _peaks()
    clocks = Clocks(0, a.out.replace(".jsonl", "_clocks.csv"))
    clocks.start()
    f = open(a.out, "w")
    s8 = torch.zeros(8, dtype=torch.uint8, device="cuda")
    for n in [int(x) for x in a.ns.split(",")]:
        pts = make_points(base, n=n)
        d_pts = torch.from_numpy(pts).cuda()
        # references for this N: D2 (stamping, the conventional method) and D1 (exact Eq.(1)), bins by the
        # whole PSF disc, standard tables of the base r (only their descriptors are used)
        ps = W.Params.from_config(base)
        tb, sb = W.psf_tables_bytes(ps)
        tabs = torch.empty(tb, dtype=torch.uint8, device="cuda")
        scr = torch.empty(sb, dtype=torch.uint8, device="cuda")
        W.build_psf_tables(ps, tabs, scr)
        del scr
        bins_ref = torch.empty(W.bin_points_bytes(ps, n, 0, ps.n_h), dtype=torch.uint8, device="cuda")
        dense = torch.empty(W.psf_dense_bytes(ps), dtype=torch.uint8, device="cuda")
        u_d2 = torch.empty((ps.n_h, ps.n_h, 2), dtype=torch.float32, device="cuda")

        def direct():
            W.build_psf_dense(ps, dense)
            W.bin_points_psf(ps, tabs, d_pts, 0, ps.n_h, bins_ref)
            W.direct_sum(ps, dense, bins_ref, 0, ps.n_h, u_d2)
        t_direct = timed(direct, reps=1)
        u_d1, t_d1 = None, None
        if not a.no_d1:
            u_d1 = torch.empty_like(u_d2)
            t_d1 = timed(lambda: W.direct_exact(ps, d_pts, bins_ref, 0, ps.n_h, u_d1), reps=1)
        del dense, bins_ref, tabs
        for r in [float(x) for x in a.rs.split(",")]:
            cfg = base.replace(retention=r)
            p = W.Params.from_config(cfg, exact=a.exact, wavelet=a.wavelet, path=a.path)
            pl = W.Pipeline(p, n, 0, p.n_h)
            reps = 3 if n < 10_000_000 else 1
            t_w = timed(lambda: pl.run(d_pts), reps=reps)
            t_k = timed(pl.superpose_inverse, reps=reps) if a.wavelet == 0 else None
            acc = W.count_accumulations(p, pl.tables, d_pts, 0, p.n_h, s8)
            st = W.bins_stats(pl.bins)
            rec = {"n_points": n, "retention": r, "aligned": a.aligned, "exact": a.exact, "wavelet": a.wavelet,
                   "path": a.path if a.path != "auto" else ("gather" if r >= 0.25 and a.wavelet == 0 else "scatter"),
                   "levels": cfg.levels, "n_depth": cfg.n_depth, "wasabi_ms": t_w,
                   "gpix_per_s": p.n_h ** 2 / (t_w * 1e-3) / 1e9, "points_per_s": n / (t_w * 1e-3),
                   "fused_kernel_ms": t_k, "accumulations": acc,
                   "fp32_frac": 4.0 * acc / (t_k * 1e-3) / (fp32 * 1e12) if t_k else None,
                   "hbm_frac": (8.125 * p.n_h ** 2 + 16.0 * n) / (t_k * 1e-3) / (hbm * 1e9) if t_k else None,
                   "acc_per_s": acc / (t_k * 1e-3) if t_k else None,
                   "direct_sum_ms": t_direct, "speedup_vs_direct": t_direct / t_w,
                   "psnr_db_vs_d2": psnr(pl.field, u_d2),
                   "psnr_db_vs_d1": psnr(pl.field, u_d1) if u_d1 is not None else None,
                   "direct_exact_ms": t_d1, "bin_entries": st["entries"]}
            print(json.dumps(rec), flush=True)
            f.write(json.dumps(rec) + "\n")
            f.flush()
            del pl
            torch.cuda.empty_cache()
        if u_d1 is not None:
            rec = {"n_points": n, "d2_vs_d1_psnr_db": psnr(u_d2, u_d1)}
            f.write(json.dumps(rec) + "\n")
        del u_d2, u_d1
        torch.cuda.empty_cache()
    ck = clocks.stop()
    f.write(json.dumps({"clocks": ck}) + "\n")
    f.close()
    print(json.dumps({"clocks": ck}))


if __name__ == "__main__":
    main()
