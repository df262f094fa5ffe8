#!/usr/bin/env python
"""bench.py -- WASABI hot path (arXiv 1708.04233) on B200.

One step = one pass of the whole hot path over the workload: step 1 PSF tables (build), step 2a
bin, steps 2b-4 fused (Eq.(2) superposition, inverse Haar and print quantisation in one kernel; the
bits are written, u is not).  Default workload: BASELINE.json configs[3] (C4: 65,536^2, 2,000,000
points, 128 levels, L=6, r=5%) on one GPU -- it fits in one B200's HBM.  `--config C1|C2|C3|C5`
(+ `--retention`, `--points`) runs the other configs as their own bench lines.
Under torchrun (N>1) each rank computes one 2^L-aligned row band (strong scaling: the hologram is
fixed) with no collective in the timed region; bands are work-balanced by default (`--bands equal`
for equal heights), and the other partition is timed too and reported beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]

`--impl reference` times the fp64 CPU oracle (the tier's reference arm) on a bounded sample of
the same workload on all host cores, rank 0 only.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
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
NOMINAL_FP32_TFLOPS = 2 * 128 * 148 * 1.965e9 / 1e12     # FFMA lanes x SMs x max SM clock


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        hbm = (float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)")
    except Exception:
        hbm = (FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)")
    try:
        with open(os.path.join(ROOT, "profiles", "r2", "fp32_peak.json")) as f:
            fp = (float(json.load(f)["fp32_tflops"]), "measured (tools/fp32_peak.cu, profiles/r2/fp32_peak.json)")
    except Exception:
        fp = (NOMINAL_FP32_TFLOPS, "nominal (2 x 128 FFMA lanes x 148 SMs x 1.965 GHz)")
    return hbm, fp


def _workload(cfg, wavelet=0):
    return (f"{cfg.name}: {cfg.n_h}x{cfg.n_h} hologram, {cfg.n_points:,} points ({cfg.kind}), "
            f"{cfg.n_depth} levels in [{cfg.z_min * 1e3:g},{cfg.z_max * 1e3:g}] mm, L={cfg.levels} "
            f"{'coif1' if wavelet else 'Haar'}, "
            f"r={cfg.retention:g}, lambda={cfg.wavelength * 1e9:g} nm, pitch={cfg.pitch * 1e6:g} um")


# ----------------------------------------------------------------------------- CPU oracle sample
def _orc_worker(cfg, pts, strip, depths, barrier, q):
    """One host process of the oracle sample: builds its strip's LUT depths (untimed), then, between
    barriers, (A) the sampled depth tables and (B) its strip of the window (bins + Eq.(2) + inverse +
    quantise), reporting the wall-clock of each phase."""
    from oracle import oracle as O
    P = O.Params.from_config(cfg)
    x0, y0, w, h = strip
    lut = O.Lut(P)
    lut.hologram_window(pts, x0, y0, w, h)          # untimed: the strip's tables (timed in phase A)
    barrier.wait()
    t0 = time.perf_counter()
    tl = O.Lut(P)
    for d in depths:
        tl.build_depth(int(d))
    tl.close()
    t1 = time.perf_counter()
    barrier.wait()
    t2 = time.perf_counter()
    u, _, _ = lut.hologram_window(pts, x0, y0, w, h)
    O.quantize(P, (0.0, 0.030, -0.400), u, x0, y0)
    t3 = time.perf_counter()
    q.put((t0, t1, t2, t3))


def oracle_sample(cfg, pts, procs=1, window=None, table_depths=None):
    """Time the fp64 oracle (as it stands; the harness only splits the work) on `procs` host
    processes on a bounded sample of the workload and extrapolate to the whole hologram:
      t = wall(phase A: sampled depth tables, spread over the processes) x (all table area / sampled)
        + wall(phase B: a w x w window in row strips of 2^L multiples) x (N_h^2 / window area)."""
    from oracle import oracle as O
    P = O.Params.from_config(cfg)
    geo = O.geometry(P)
    area = [(2 * int(h)) ** 2 for h in geo["H"]]
    w = window or min(cfg.n_h, 6144)
    x0 = y0 = cfg.n_h // 2 - w // 2
    B = 1 << cfg.levels
    rows = max(B, (w // procs + B - 1) // B * B)
    strips = [(x0, y0 + r, w, min(rows, w - r)) for r in range(0, w, rows)]
    if table_depths is None:
        table_depths = [cfg.n_depth // 2, cfg.n_depth - 1] if procs == 1 else \
            [int(round(i * (cfg.n_depth - 1) / max(1, len(strips) - 1))) for i in range(len(strips))]
    per = [table_depths[i::len(strips)] for i in range(len(strips))]
    E = int(geo["E"].max()) + 2
    px = pts[:, 0] / cfg.pitch + cfg.n_h // 2
    py = pts[:, 1] / cfg.pitch + cfg.n_h // 2
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(len(strips))
    q = ctx.Queue()
    ps = []
    for s, dep in zip(strips, per):
        m = (px + E >= s[0]) & (px - E < s[0] + s[2]) & (py + E >= s[1]) & (py - E < s[1] + s[3])
        ps.append(ctx.Process(target=_orc_worker, args=(cfg, pts[m], s, dep, barrier, q)))
    for p in ps:
        p.start()
    res = [q.get(timeout=900) for _ in ps]
    for p in ps:
        p.join()
    t_tab = max(r[1] for r in res) - min(r[0] for r in res)
    t_win = max(r[3] for r in res) - min(r[2] for r in res)
    t_all = t_tab * sum(area) / sum(area[d] for d in table_depths) + t_win * (cfg.n_h ** 2) / (w * w)
    sample = (f"oracle (fp64 C, unchanged) on {len(strips)} host process(es): depth tables {table_depths} "
              f"extrapolated by table area to {cfg.n_depth} depths + a {w}x{w} window (bins+Eq.(2)+inverse+"
              f"quantise, row strips of {rows}) extrapolated to {cfg.n_h}^2; measured {t_tab + t_win:.2f} s wall, "
              f"full-hologram estimate {t_all:.1f} s")
    return dict(value=cfg.n_h ** 2 / t_all / 1e9, unit=UNIT, cores=len(strips), kind="oracle", sample=sample,
                est_full_s=t_all)


def cpu_baseline(cfg, pts):
    """The oracle on all host cores (the reported value) and on one thread (context)."""
    cores = os.cpu_count() or 1
    allc = oracle_sample(cfg, pts, procs=cores)
    one = oracle_sample(cfg, pts, procs=1)
    for d in (allc, one):
        d.pop("est_full_s", None)
    allc["single_thread"] = one
    allc["host"] = _host()
    return allc


def _host():
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        model = "?"
    return f"{model}, {os.cpu_count()} logical CPUs"


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
    cores = os.cpu_count() or 1
    # each step: the all-core oracle sample on another set of sampled depth tables
    vals, tot = [], 0.0
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        depths = [int((i * 7 + 13 * k) % cfg.n_depth) for k in range(cores)]
        cb = oracle_sample(cfg, pts, procs=cores, table_depths=depths)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(cb)
            tot += dt
    v = statistics.median([c["value"] for c in vals])
    cb = dict(vals[0])
    cb["value"] = v
    cb.pop("est_full_s", None)
    cb["host"] = _host()
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
    from paper_1708_04233_b200.distributed import (assemble_bits, balanced_bands, band_of, band_work, checksums,
                                                   gather_checksums)

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

    def gather(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=cdev)
        if world == 1:
            return [vals]
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [p.tolist() for p in parts]

    p = W.Params.from_config(cfg, wavelet=args.wavelet)
    if args.wavelet:
        args.unfused = True     # coiflets (R-A21): the synthesis is not tile-local -> superpose + inverse_wt
    pts = make_points(cfg)
    n = len(pts)
    d_pts = torch.from_numpy(pts).to(dev)
    stream = torch.cuda.current_stream(dev)
    scratch8 = torch.zeros(8, dtype=torch.uint8, device=dev)

    # row-work estimate (wasabi_row_work) -> equal and work-balanced bands (host logic, untimed)
    tb, sb = W.psf_tables_bytes(p)
    t_tab = torch.empty(tb, dtype=torch.uint8, device=dev)
    t_scr = torch.empty(sb, dtype=torch.uint8, device=dev)
    W.build_psf_tables(p, t_tab, t_scr)
    rw = torch.empty(cfg.n_h + 1, dtype=torch.float64, device=dev)
    W.row_work(p, t_tab, d_pts, rw, scratch8)
    row_work = rw[:cfg.n_h].cpu().numpy()
    eq = [band_of(r, world, cfg.n_h, p.tile) for r in range(world)]
    bal = balanced_bands(row_work, world, p.tile)
    mode = args.bands if args.bands else ("balanced" if world > 1 else "equal")
    parts = {"equal": eq, "balanced": bal}
    del t_scr, rw

    hbm, fp32 = _peaks()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if cfg.n_h < 65536 else None

    def timed_run(bands, steps, warmup, want_clocks):
        row0, row1 = bands[rank]
        pl = W.Pipeline(p, n, row0, row1, device=dev)
        for _ in range(warmup):
            pl.run(d_pts, fused=not args.unfused)
        torch.cuda.synchronize(dev)
        stages = ["tables", "bin", "superpose", "inverse_quantize"] if args.unfused else \
            ["tables", "bin", "superpose_inverse_quantize"]
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)] for _ in range(steps)]
        clocks = None
        if want_clocks:
            clocks = Clocks(local, os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv")
                            if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else f"/tmp/clocks_rank{rank}.csv")
        barrier()
        torch.cuda.synchronize(dev)
        if clocks:
            clocks.start()
            time.sleep(0.3)
        launches0 = W.kernel_launches()
        for k in range(steps):
            if flush is not None:
                flush.zero_()          # L2 flush between timed steps (outside the events)
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
        ck = clocks.stop() if clocks else None
        own_ms = sum(ev[k][0].elapsed_time(ev[k][len(stages)]) for k in range(steps))
        stage_ms = {s: statistics.mean(ev[k][i].elapsed_time(ev[k][i + 1]) for k in range(steps))
                    for i, s in enumerate(stages)}
        return pl, own_ms, stage_ms, launches, ck

    bands = parts[mode]
    row0, row1 = bands[rank]
    pl, own_ms, stage_ms, launches, ck = timed_run(bands, args.steps, args.warmup, True)
    graph = None
    if world == 1 and not args.unfused and cfg.n_h < 65536:
        # the same step as one CUDA graph (Pipeline.capture / replay): what the launch overhead costs
        # the small configs; reported beside the eager line, not instead of it
        pl.capture(d_pts)
        for _ in range(args.warmup):
            pl.replay()
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        torch.cuda.synchronize(dev)
        for e0, e1 in gev:
            if flush is not None:
                flush.zero_()
            e0.record(stream)
            pl.replay()
            e1.record(stream)
        torch.cuda.synchronize(dev)
        g_ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in gev)
        graph = {"ms_per_step": g_ms, "value": cfg.n_h * cfg.n_h / (g_ms * 1e-3) / 1e9, "unit": "Gpixel/s",
                 "note": "one CUDA graph per step (tables + bins + fused kernel), L2 flushed between replays"}
    t_ms = max_over_ranks(own_ms)
    stage_ms = {s: max_over_ranks(v) for s, v in stage_ms.items()}
    ms_per_step = t_ms / args.steps
    px = cfg.n_h * cfg.n_h
    value = px / (ms_per_step * 1e-3) / 1e9
    points_per_s = n / (ms_per_step * 1e-3)
    st = W.bins_stats(pl.bins)
    acc = W.count_accumulations(p, pl.tables, d_pts, row0, row1, scratch8)     # exact Eq.(2) work, untimed
    per_rank = [dict(rank=i, rows=[int(v[0]), int(v[1])], acc=int(v[2]), ms_per_step=v[3] / args.steps,
                     est_work=v[4])
                for i, v in enumerate(gather([row0, row1, acc, own_ms, band_work(row_work, [(row0, row1)])[0]]))]

    # checksums and assembly of the print bits after the timed region (the only collectives)
    cs = checksums(None, pl.bits).to(cdev)
    assembled = None
    if world > 1:
        cs_all = gather_checksums(cs)
        full = assemble_bits(pl.bits.to(cdev), cfg.n_h, p.tile, bands=bands)
        table = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.float64, device=full.device)
        assembled = {"rows": int(full.shape[0]), "bits_set": float(table[full.reshape(-1).long()].sum()),
                     "band_bits_set_sum": float(cs_all[:, 3].sum())}
        cs = cs_all.sum(dim=0)
        del full
    cs = cs.tolist()

    # roofline of the dominant kernel: HBM (algorithmic bytes per launch / event-timed duration) and
    # FP32 (4 flops per Eq.(2) accumulation, exact count) against the measured peaks
    rows = row1 - row0
    alg = {"superpose": 8.0 * rows * cfg.n_h + 16.0 * st["n_valid"],
           "inverse_quantize": 16.125 * rows * cfg.n_h,
           "superpose_inverse_quantize": 8.125 * rows * cfg.n_h + 16.0 * st["n_valid"],
           "bin": 16.0 * n + 16.0 * st["n_valid"] + 8.0 * st["entries"],
           "tables": float(tb)}      # the table buffer the build writes (canonical + window LUT)
    dom = max(stage_ms, key=stage_ms.get)
    traffic, onchip = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath) and cfg.name == "C4" and args.retention is None and args.points is None:
        try:
            rec = json.load(open(tpath)).get(dom)
            if isinstance(rec, dict):
                traffic, onchip = rec.get("traffic"), rec.get("onchip")
                prof_rows = rec.get("rows")
                if traffic is not None and prof_rows and prof_rows != rows:
                    traffic = traffic * rows / prof_rows      # the capture is of the full hologram
                    onchip = dict(onchip or {}, traffic_scaled_from_rows=prof_rows)
        except Exception:
            traffic = None
    ach = alg[dom] / (stage_ms[dom] * 1e-3) / 1e9 if alg[dom] else 0.0
    step_bytes = (24.125 if args.unfused else 8.125) * rows * cfg.n_h + 32.0 * n
    roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm[0], "unit": "GB/s",
                "frac": ach / hbm[0], "traffic": traffic, "peak_source": hbm[1],
                "alg_bytes_per_launch": alg[dom],
                "step_achieved": step_bytes / (ms_per_step * 1e-3) / 1e9,
                "step_frac": step_bytes / (ms_per_step * 1e-3) / 1e9 / hbm[0]}
    sup = "superpose" if args.unfused else "superpose_inverse_quantize"
    fl = 4.0 * acc / (stage_ms[sup] * 1e-3) / 1e12
    roofline["fp32"] = {"kernel": sup, "accumulations": acc, "flops_per_accumulation": 4,
                        "achieved": fl, "peak": fp32[0], "unit": "TFLOP/s", "frac": fl / fp32[0],
                        "peak_source": fp32[1],
                        "acc_per_s": acc / (stage_ms[sup] * 1e-3)}
    # on-chip ceiling of the scatter: one 64-bit shared read-modify-write per
    # accumulation, 32 lanes x 8 B = two 128-B wavefronts per LDS.64 and per STS.64, one wavefront per
    # clock per SM -> 8 accumulations / clock / SM at zero bank conflicts
    f_sm = (ck or {}).get("sm_max_mhz") or 1965.0
    ceil_acc = 148 * f_sm * 1e6 * 8
    roofline["onchip_acc"] = {"kernel": sup, "achieved": acc / (stage_ms[sup] * 1e-3), "peak": ceil_acc,
                              "unit": "accumulations/s", "frac": acc / (stage_ms[sup] * 1e-3) / ceil_acc,
                              "peak_source": "148 SMs x f_SM x 8 acc/clk (shared-memory RMW, conflict-free)"}
    if onchip:
        roofline["onchip"] = onchip
    # every timed stage against the HBM peak (algorithmic bytes of the stage / its event time)
    roofline["stages"] = {k: {"alg_bytes": alg[k], "achieved": alg[k] / (stage_ms[k] * 1e-3) / 1e9,
                              "frac": alg[k] / (stage_ms[k] * 1e-3) / 1e9 / hbm[0]}
                          for k in stage_ms if k in alg and stage_ms[k] > 0}

    # the other band partition, timed the same way (N > 1 only)
    alt = None
    if world > 1 and not args.no_alt_bands:
        other = "equal" if mode == "balanced" else "balanced"
        del pl
        torch.cuda.empty_cache()
        pl2, own2, _, _, _ = timed_run(parts[other], args.steps, 1, False)
        acc2 = W.count_accumulations(p, pl2.tables, d_pts, *parts[other][rank], scratch8)
        g2 = gather([own2, acc2])
        t2 = max(v[0] for v in g2) / args.steps
        alt = {"bands": other, "ms_per_step": t2, "value": px / (t2 * 1e-3) / 1e9,
               "per_rank": [dict(rank=i, rows=list(parts[other][i]), acc=int(v[1]), ms_per_step=v[0] / args.steps)
                            for i, v in enumerate(g2)]}
        del pl2
    else:
        del pl
    torch.cuda.empty_cache()

    # end-to-end through the C ABI with host buffers (H2D points + whole path + D2H bits)
    e2e = None
    if not args.no_e2e:
        ws = torch.empty(W.hologram_workspace_bytes(p, n, row0, row1), dtype=torch.uint8, device=dev)
        h_pts = torch.from_numpy(pts).pin_memory()
        h_bits = torch.empty((rows, cfg.n_h // 8), dtype=torch.uint8).pin_memory()
        pr = W.PrintParams()
        for _ in range(max(1, args.warmup - 1)):
            W.hologram_host(p, pr, h_pts, row0, row1, ws, h_bits, None, stream)
        torch.cuda.synchronize(dev)
        barrier()
        te_sum = 0.0
        for _ in range(args.steps):
            if flush is not None:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            W.hologram_host(p, pr, h_pts, row0, row1, ws, h_bits, None, stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            te_sum += e0.elapsed_time(e1)
        te = max_over_ranks(te_sum) / args.steps
        e2e = {"value": px / (te * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": te,
               "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": rows * (cfg.n_h // 8)}
        del ws

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, pts)

    if rank == 0:
        l2 = ("inputs larger than L2 (bits 0.5 GB, bins 0.6 GB, tables 0.45 GB per step)" if flush is None else
              "L2 flushed between timed steps (256 MB write outside the events)")
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (seeded generators, inputs/; the paper's 3D model is unavailable)",
               "config": {"workload": _workload(cfg, args.wavelet),
                          "path": ("superpose on the coif1 halo band, then fused coif1 tile synthesis + quantise (u written)" if args.wavelet else "unfused")
                          if args.unfused else "fused",
                          "n_h": cfg.n_h, "n_points": n, "levels": cfg.levels, "retention": cfg.retention,
                          "n_depth": cfg.n_depth, "tile": p.tile, "rows_per_gpu": rows,
                          "parallelism": f"row bands x{world} ({mode})", "l2": l2},
               "points_per_s": points_per_s, "stage_ms": stage_ms, "bin_entries": st["entries"],
               "accumulations": sum(r["acc"] for r in per_rank),
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
               "clocks": ck, "graph": graph, "per_rank": per_rank, "bands_alt": alt, "assembled": assembled,
               "checksum": {"bits_set": cs[3]},
               "paper_context": {"wasabi_s_65536sq_95949pts_cpu": 354, "nlut_s": 10533,
                                 "cite": "PAPER.md:166 (Xeon E5 v3; different point count and wavelet)"}}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- conventional method
def run_direct(args, cfg):
    """The paper's comparison (WASABI ~30x faster than the conventional method on
    a CPU) on this GPU: per step the conventional method -- dense PSF tables, bins by the whole PSF disc,
    the quantised direct sum of Eq.(1) by PSF stamping (wasabi_direct_sum) and the same print
    quantisation -- timed against the WASABI step on the same points, CUDA events, one GPU."""
    import torch
    import paper_1708_04233_b200 as W
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    p = W.Params.from_config(cfg)
    pts = make_points(cfg)
    n = len(pts)
    d_pts = torch.from_numpy(pts).to(dev)
    stream = torch.cuda.current_stream(dev)

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize(dev)
        tot = 0.0
        for _ in range(steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            tot += e0.elapsed_time(e1)
        return tot / steps

    pl = W.Pipeline(p, n, 0, p.n_h, device=dev, want_u=False)
    t_w = timed(lambda: pl.run(d_pts), args.steps, args.warmup)
    del pl
    torch.cuda.empty_cache()
    tb, sb = W.psf_tables_bytes(p)
    tables = torch.empty(tb, dtype=torch.uint8, device=dev)
    scr = torch.empty(sb, dtype=torch.uint8, device=dev)
    W.build_psf_tables(p, tables, scr)                 # descriptors only (untimed): geometry of every depth
    del scr
    dense = torch.empty(W.psf_dense_bytes(p), dtype=torch.uint8, device=dev)
    bins = torch.empty(W.bin_points_bytes(p, n, 0, p.n_h), dtype=torch.uint8, device=dev)
    u = torch.empty((p.n_h, p.n_h, 2), dtype=torch.float32, device=dev)
    bits = torch.empty((p.n_h, p.n_h // 8), dtype=torch.uint8, device=dev)
    pr = W.PrintParams()
    stage = {}

    def direct_step():
        W.build_psf_dense(p, dense)
        W.bin_points_psf(p, tables, d_pts, 0, p.n_h, bins)
        W.direct_sum(p, dense, bins, 0, p.n_h, u)
        W.quantize(p, pr, u, 0, p.n_h, bits)

    clocks = Clocks(0, os.path.join(ROOT, "gpurun_out", "clocks_direct.csv")
                    if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else "/tmp/clocks_direct.csv")
    clocks.start()
    t_d = timed(direct_step, max(1, args.steps // 2), 1)
    ck = clocks.stop()
    st = W.bins_stats(bins)
    px = cfg.n_h * cfg.n_h
    out = {"metric": METRIC, "value": px / (t_d * 1e-3) / 1e9, "unit": UNIT, "n_gpus": 1, "impl": "direct_sum",
           "steps": max(1, args.steps // 2), "warmup": 1, "ms_per_step": t_d, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (seeded generators, inputs/)",
           "config": {"workload": _workload(cfg), "path": "conventional: dense PSF + disc bins + stamping "
                      "(quantised direct sum of Eq.(1)) + quantise", "n_h": cfg.n_h, "n_points": n},
           "wasabi_ms_per_step": t_w, "wasabi_speedup_vs_direct": t_d / t_w, "direct_bin_entries": st["entries"],
           "clocks": ck,
           "paper_context": {"wasabi_vs_conventional_cpu": "~30x (PAPER.md:164-167; 354 s vs 10,533 s N-LUT)"}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--points", type=int, default=None, help="override the config's point count")
    ap.add_argument("--retention", type=float, default=None, help="override the config's r")
    ap.add_argument("--tile", type=int, default=None)
    ap.add_argument("--bands", default=None, choices=["equal", "balanced"],
                    help="row-band partition (default: balanced for N > 1)")
    ap.add_argument("--no-alt-bands", action="store_true", help="N > 1: skip timing the other partition")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--unfused", action="store_true", help="time the 4-call path (psi through HBM)")
    ap.add_argument("--levels", type=int, default=None, help="override the config's wavelet levels L")
    ap.add_argument("--wavelet", type=int, default=0, choices=[0, 1],
                    help="1: coif1 tables (WASABI_FLAG_COIFLET, R-A21; implies --unfused)")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default) or gloo (test mode)")
    ap.add_argument("--same-device", action="store_true", help="test mode: all ranks on cuda:0")
    ap.add_argument("--direct", action="store_true",
                    help="time the conventional method (GPU direct sum) against WASABI on one GPU")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.points:
        cfg = cfg.replace(n_points=args.points)
    if args.retention:
        cfg = cfg.replace(retention=args.retention)
    if args.tile:
        cfg = cfg.replace(tile=args.tile)
    if args.levels:
        cfg = cfg.replace(levels=args.levels)
    elif args.wavelet:
        cfg = cfg.replace(levels=min(cfg.levels, 3))    # "coiflets as the wavelets at level 3"
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.direct:
        run_direct(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
