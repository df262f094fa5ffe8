#!/usr/bin/env python
"""bench.py -- WASABI hot path (arXiv 1708.04233) on B200.

One step = one pass of the whole hot path over the workload: step 1 PSF tables (build), step 2a
bin, step 2b superpose (Eq.(2)), step 3 inverse Haar fused with step 4 print quantisation (u
written in place, bits written).  Default workload: BASELINE.json configs[3] (C4: 65,536^2,
2,000,000 points, 128 levels, L=6, r=5%) on one GPU -- it fits in one B200's HBM.
Under torchrun (N>1) each rank computes one 2^L-aligned row band (strong scaling: the hologram is
fixed) with no collective in the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]

`--impl reference` times the fp64 CPU oracle (the tier's reference arm) on a bounded sample of
the same workload, rank 0 only.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from inputs import CONFIGS, make_points  # noqa: E402

METRIC = "object points/s and hologram Gpixel/s (WASABI superpose+inverse WT), % of HBM roofline"
UNIT = "Gpixel/s"
FALLBACK_HBM_GBS = 6650.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def _workload(cfg):
    return (f"{cfg.name}: {cfg.n_h}x{cfg.n_h} hologram, {cfg.n_points:,} points ({cfg.kind}), "
            f"{cfg.n_depth} levels in [{cfg.z_min * 1e3:g},{cfg.z_max * 1e3:g}] mm, L={cfg.levels} Haar, "
            f"r={cfg.retention:g}, lambda={cfg.wavelength * 1e9:g} nm, pitch={cfg.pitch * 1e6:g} um")


# ----------------------------------------------------------------------------- CPU oracle sample
def oracle_sample(cfg, pts, window=None, table_depths=None, setup=None):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload and extrapolate to
    the whole hologram: t = t(sampled depth tables) x (all table area / sampled area) +
    t(window hot path: bins + Eq.(2) + inverse + quantise) x (N_h^2 / window area)."""
    from oracle import oracle as O
    P = O.Params.from_config(cfg)
    if setup is None:
        setup = {}
        geo = O.geometry(P)
        setup["area"] = [(2 * int(h)) ** 2 for h in geo["H"]]
        w = window or min(cfg.n_h, 6144)
        x0 = y0 = cfg.n_h // 2 - w // 2
        ix, iy, iz, ok = O.points(P, pts)
        E = geo["E"][iz]
        hit = ok & (ix + E >= x0) & (ix - E < x0 + w) & (iy + E >= y0) & (iy - E < y0 + w)
        lut = O.Lut(P)
        for d in sorted(set(iz[hit].tolist())):   # untimed: the window's tables are timed separately
            lut.build_depth(int(d))
        setup.update(lut=lut, w=w, x0=x0, y0=y0, geo=geo)
    lut, w, x0, y0 = setup["lut"], setup["w"], setup["x0"], setup["y0"]
    depths = table_depths if table_depths is not None else [cfg.n_depth // 2, cfg.n_depth - 1]
    t0 = time.perf_counter()
    tl = O.Lut(P)
    for d in depths:
        tl.build_depth(int(d))
    t_tab = time.perf_counter() - t0
    tl.close()
    t0 = time.perf_counter()
    u, _, _ = lut.hologram_window(pts, x0, y0, w, w)
    O.quantize(P, (0.0, 0.030, -0.400), u, x0, y0)
    t_win = time.perf_counter() - t0
    area = setup["area"]
    t_all = t_tab * sum(area) / sum(area[d] for d in depths) + t_win * (cfg.n_h ** 2) / (w * w)
    sample = (f"oracle (fp64 C, 1 thread): tables of depths {list(depths)} extrapolated by table area to "
              f"{cfg.n_depth} depths + a {w}x{w} window (bins+Eq.(2)+inverse+quantise) extrapolated to "
              f"{cfg.n_h}^2; measured {t_tab + t_win:.2f} s, full-hologram estimate {t_all:.1f} s")
    return dict(value=cfg.n_h ** 2 / t_all / 1e9, unit=UNIT, cores=1, kind="oracle", sample=sample,
                est_full_s=t_all), setup


# ----------------------------------------------------------------------------- clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, path: str):
        self.index, self.path, self.p = index, path, None

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.close()
        rows = []
        for line in open(self.path):
            c = [x.strip() for x in line.split(",")]
            if len(c) < 9 or not c[0].isdigit() or int(c[0]) != self.index:
                continue
            rows.append(c)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(rows[0][2]),
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pts = make_points(cfg)
    setup = None
    _, setup = oracle_sample(cfg, pts, table_depths=[cfg.n_depth - 1], setup=None)  # setup (untimed)
    vals, tot = [], 0.0
    sample_depths = [cfg.n_depth - 1, cfg.n_depth // 2, 3 * cfg.n_depth // 4, 0]
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        cb, _ = oracle_sample(cfg, pts, table_depths=[sample_depths[i % len(sample_depths)]], setup=setup)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(cb)
            tot += dt
    v = statistics.median([c["value"] for c in vals])
    cb = dict(vals[0])
    cb["value"] = v
    cb.pop("est_full_s", None)
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / max(1, args.steps),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded; paper's 3D model unavailable)",
           "config": {"workload": _workload(cfg), "sampled": True},
           "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    import paper_1708_04233_b200 as W

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus or "RANK" not in os.environ, "--gpus must match WORLD_SIZE"
    if args.same_device:        # test mode: every rank on cuda:0 (host logic check on a 1-GPU box)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    def barrier():
        if world > 1:
            dist.barrier()

    cdev = dev if args.dist_backend == "nccl" else torch.device("cpu")

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    p = W.Params.from_config(cfg)
    from paper_1708_04233_b200.distributed import band_of, checksums, gather_checksums
    row0, row1 = band_of(rank, world, cfg.n_h, p.tile)
    pts = make_points(cfg)
    n = len(pts)
    d_pts = torch.from_numpy(pts).to(dev)
    pl = W.Pipeline(p, n, row0, row1, device=dev)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        pl.run(d_pts, fused=not args.unfused)
    torch.cuda.synchronize(dev)
    st = W.bins_stats(pl.bins)

    stages = ["tables", "bin", "superpose", "inverse_quantize"] if args.unfused else \
        ["tables", "bin", "superpose_inverse_quantize"]
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)] for _ in range(args.steps)]
    clocks = Clocks(local, os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv")
                    if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else f"/tmp/clocks_rank{rank}.csv")
    barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.3)
    launches0 = W.kernel_launches()
    for k in range(args.steps):
        e = ev[k]
        e[0].record(stream)
        pl.build_tables()
        e[1].record(stream)
        pl.bin(d_pts)
        e[2].record(stream)
        if args.unfused:
            pl.superpose()
            e[3].record(stream)
            pl.inverse()
            e[4].record(stream)
        else:
            pl.superpose_inverse()
            e[3].record(stream)
    torch.cuda.synchronize(dev)
    launches = W.kernel_launches() - launches0
    barrier()
    ck = clocks.stop()
    total_ms = sum(ev[k][0].elapsed_time(ev[k][len(stages)]) for k in range(args.steps))
    stage_ms = {s: statistics.mean(ev[k][i].elapsed_time(ev[k][i + 1]) for k in range(args.steps))
                for i, s in enumerate(stages)}
    t_ms = max_over_ranks(total_ms)
    stage_ms = {s: max_over_ranks(v) for s, v in stage_ms.items()}
    ms_per_step = t_ms / args.steps
    px = cfg.n_h * cfg.n_h
    value = px / (ms_per_step * 1e-3) / 1e9
    points_per_s = n / (ms_per_step * 1e-3)

    # checksum assembly after the timed region (the only collective: NCCL all_gather)
    cs = checksums(pl.field, pl.bits)
    if world > 1:
        cs = gather_checksums(cs.to(cdev)).sum(dim=0)
    cs = cs.tolist()

    # roofline of the dominant kernel (algorithmic bytes per launch / event-timed duration)
    peak, peak_src = _peaks()
    rows = row1 - row0
    alg = {"superpose": 8.0 * rows * cfg.n_h + 16.0 * st["n_valid"],
           "inverse_quantize": 16.125 * rows * cfg.n_h,
           "superpose_inverse_quantize": 8.125 * rows * cfg.n_h + 16.0 * st["n_valid"],
           "bin": 16.0 * n + 16.0 * st["n_valid"] + 8.0 * st["entries"],
           "tables": 0.0}
    dom = max(stage_ms, key=stage_ms.get)
    # per-launch DRAM traffic and on-chip limiter of the dominant kernel, from one committed
    # `ncu --set full` capture of this same workload (tools/ncu_traffic.py -> profiles/ncu_traffic.json)
    traffic, onchip = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            rec = json.load(open(tpath)).get(dom)
            if isinstance(rec, dict):
                traffic = rec.get("traffic")
                onchip = rec.get("onchip")
                prof_rows = rec.get("rows")
                if traffic is not None and prof_rows and prof_rows != rows and cfg.name == "C4":
                    # the capture is of the full hologram; a band moves its share of it
                    traffic = traffic * rows / prof_rows
                    onchip = dict(onchip or {}, traffic_scaled_from_rows=prof_rows)
                elif cfg.name != "C4":
                    traffic, onchip = None, None   # the capture is of C4 only
            else:
                traffic = rec
        except Exception:
            traffic = None
    ach = alg[dom] / (stage_ms[dom] * 1e-3) / 1e9 if alg[dom] else 0.0
    step_bytes = (24.125 if args.unfused else 8.125) * rows * cfg.n_h + 32.0 * n
    roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": traffic, "peak_source": peak_src,
                "step_achieved": step_bytes / (ms_per_step * 1e-3) / 1e9,
                "step_frac": step_bytes / (ms_per_step * 1e-3) / 1e9 / peak}
    if onchip:
        roofline["onchip"] = onchip

    # end-to-end through the C ABI with host buffers (H2D points + whole path + D2H bits)
    e2e = None
    if not args.no_e2e:
        del pl
        torch.cuda.empty_cache()
        ws = torch.empty(W.hologram_workspace_bytes(p, n, row0, row1), dtype=torch.uint8, device=dev)
        h_pts = torch.from_numpy(pts).pin_memory()
        h_bits = torch.empty((rows, cfg.n_h // 8), dtype=torch.uint8).pin_memory()
        pr = W.PrintParams()
        for _ in range(max(1, args.warmup - 1)):
            W.hologram_host(p, pr, h_pts, row0, row1, ws, h_bits, None, stream)
        torch.cuda.synchronize(dev)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            W.hologram_host(p, pr, h_pts, row0, row1, ws, h_bits, None, stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        te = max_over_ranks(e0.elapsed_time(e1)) / args.steps
        e2e = {"value": px / (te * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": te,
               "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": rows * (cfg.n_h // 8)}
        del ws

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, _ = oracle_sample(cfg, pts)
        cpu.pop("est_full_s", None)

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (seeded generators, inputs/; the paper's 3D model is unavailable)",
               "config": {"workload": _workload(cfg), "path": "unfused" if args.unfused else "fused", "n_h": cfg.n_h, "n_points": n, "levels": cfg.levels,
                          "retention": cfg.retention, "n_depth": cfg.n_depth, "tile": p.tile,
                          "rows_per_gpu": rows, "parallelism": f"row bands x{world}",
                          "l2": f"inputs larger than L2 (psi/u {8 * rows * cfg.n_h / 1e9:.1f} GB per GPU per step)"},
               "points_per_s": points_per_s, "stage_ms": stage_ms, "bin_entries": st["entries"],
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
               "clocks": ck, "checksum": {"u_energy": cs[0], "u_re_sum": cs[1], "u_im_sum": cs[2], "bits_set": cs[3]},
               "paper_context": {"wasabi_s_65536sq_95949pts_cpu": 354, "nlut_s": 10533,
                                 "cite": "PAPER.md:166 (Xeon E5 v3; different point count and wavelet)"}}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--points", type=int, default=None, help="override the config's point count")
    ap.add_argument("--tile", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--unfused", action="store_true", help="time the 4-call path (psi through HBM)")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default) or gloo (test mode)")
    ap.add_argument("--same-device", action="store_true", help="test mode: all ranks on cuda:0")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.points:
        cfg = cfg.replace(n_points=args.points)
    if args.tile:
        cfg = cfg.replace(tile=args.tile)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
