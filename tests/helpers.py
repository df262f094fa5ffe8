"""Shared test helpers: run the CUDA path through the C ABI and compare with the oracle."""
from __future__ import annotations

import numpy as np

from inputs import CONFIGS, make_points

REF = (0.0, 0.030, -0.400)


def gpu_params(cfg, **kw):
    import paper_1708_04233_b200 as W
    return W.Params.from_config(cfg, **kw)


def orc_params(orc, cfg, **kw):
    P = orc.Params.from_config(cfg)
    if kw:
        d = dict(P.__dict__)
        d.update({k: v for k, v in kw.items() if k in d})
        P = orc.Params(**d)
    return P


def run_gpu(cfg, pts, row0=0, row1=None, want_bits=True, **kw):
    """Full GPU path for one band; returns (pipeline, u complex64 numpy, bits numpy)."""
    import torch
    import paper_1708_04233_b200 as W
    p = gpu_params(cfg, **kw)
    row1 = p.n_h if row1 is None else row1
    pl = W.Pipeline(p, max(1, len(pts)), row0, row1, want_bits=want_bits)
    d_pts = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float32)).cuda()
    pl.run(d_pts)
    torch.cuda.synchronize()
    return pl, d_pts


def field_np(t):
    a = t.cpu().numpy()
    return a[..., 0].astype(np.float64) + 1j * a[..., 1].astype(np.float64)


def rel_l2(g, o):
    n = np.linalg.norm(o)
    return np.linalg.norm(g - o) / (n if n > 0 else 1.0)


def bits_mismatch_outside_band(bits_g, bits_o, I_o, du_abs, u_abs):
    """Count print-bit differences that are NOT explained by the threshold band (DESIGN.md R-A16):
    a flip at pixel p is legitimate iff |I_oracle(p)| <= |u_gpu(p) - u_oracle(p)| + 1e-6 (rms(I) + |u(p)|)."""
    g = np.unpackbits(bits_g, axis=1, bitorder="big").astype(bool)
    o = np.unpackbits(bits_o, axis=1, bitorder="big").astype(bool)
    diff = g != o
    rms = float(np.sqrt(np.mean(I_o ** 2))) if I_o.size else 0.0
    band = np.abs(I_o) <= du_abs + 1e-6 * (rms + u_abs)
    return int(np.sum(diff & ~band)), int(np.sum(diff)), int(np.sum(np.abs(I_o) <= 1e-6 * rms))


def field_check(g, o, tol=1e-5):
    """Element-wise and rel-L2 comparison of a GPU field with the oracle's: returns (rel_l2,
    max|g - o| / max|o|); the parity bar is both <= tol (north_star 1e-5)."""
    m = float(np.max(np.abs(o))) if o.size else 0.0
    e_max = float(np.max(np.abs(g - o))) / m if m > 0 else float(np.max(np.abs(g))) if g.size else 0.0
    return rel_l2(g, o), e_max


def bits_check(bits_g, bits_o, I_o, u_g, u_o):
    """Print-bit comparison (R-A16) with a FIXED band, not a per-pixel one: a flip is allowed only
    where |I_oracle| <= eps + 1e-6 rms(I), eps = max|u_gpu - u_oracle| over the compared region (one
    scalar: the measured field error, itself asserted <= 1e-5 max|u_oracle| by the caller).
    Returns dict(bad=flips outside that band, flips=all flips, strict=flips outside the strict
    1e-6 rms(I) band of the quantise-alone criterion, band_px=pixels inside the fixed band)."""
    g = np.unpackbits(bits_g, axis=1, bitorder="big").astype(bool)
    o = np.unpackbits(bits_o, axis=1, bitorder="big").astype(bool)
    diff = g != o
    rms = float(np.sqrt(np.mean(I_o ** 2))) if I_o.size else 0.0
    eps = float(np.max(np.abs(u_g - u_o))) if u_o.size else 0.0
    band = np.abs(I_o) <= eps + 1e-6 * rms
    strict = np.abs(I_o) <= 1e-6 * rms
    return dict(bad=int(np.sum(diff & ~band)), flips=int(np.sum(diff)), strict=int(np.sum(diff & ~strict)),
                band_px=int(np.sum(band)), eps=eps, rms_I=rms)


def parity_log(record: dict):
    """Append one JSON record to $WASABI_PARITY_LOG (if set): the per-case numbers of the parity
    tests (errors, flip counts) for profiles/."""
    import json
    import os
    path = os.environ.get("WASABI_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(record) + "\n")


def _oracle_strip(args):
    from oracle import oracle as O
    P, pts, x0, y0, w, h, ref = args
    lut = O.Lut(P)
    u, psi, _ = lut.hologram_window(pts, x0, y0, w, h)
    bits, I = O.quantize(P, ref, u, x0, y0)
    lut.close()
    return u, psi, bits, I


def oracle_window(P, pts, x0, y0, w, h, ref=REF, procs=None):
    """The oracle's (u, psi, bits, I) on window [x0, x0+w) x [y0, y0+h), computed in row strips
    (multiples of 2^L: Haar windows are independent, R-A12) by a pool of host processes -- the
    harness parallelises, the oracle's arithmetic is unchanged."""
    import os
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    from oracle import oracle as O
    B = 1 << P.levels
    procs = procs or min(16, os.cpu_count() or 1)
    rows = max(B, (h // max(1, procs) + B - 1) // B * B)
    pts = np.asarray(pts, np.float64)
    # harness-side pre-filter (order preserved): points whose footprint box cannot reach a strip
    # are skipped by the oracle anyway (its own test uses E_d <= max E)
    E = int(O.geometry(P)["E"].max()) + 2
    px = pts[:, 0] / P.pitch + P.n_h // 2
    py = pts[:, 1] / P.pitch + P.n_h // 2
    okx = ~((px + E < x0) | (px - E >= x0 + w))
    jobs = []
    for r in range(0, h, rows):
        hh = min(rows, h - r)
        m = okx & ~((py + E < y0 + r) | (py - E >= y0 + r + hh)) | ~np.isfinite(px) | ~np.isfinite(py)
        jobs.append((P, pts[m], x0, y0 + r, w, hh, ref))
    if len(jobs) == 1 or procs == 1:
        out = [_oracle_strip(j) for j in jobs]
    else:
        with ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("fork")) as ex:
            out = list(ex.map(_oracle_strip, jobs))
    return tuple(np.concatenate([o[i] for o in out]) for i in range(4))


__all__ = ["CONFIGS", "make_points", "REF", "gpu_params", "orc_params", "run_gpu", "field_np", "rel_l2",
           "bits_mismatch_outside_band", "field_check", "bits_check", "parity_log", "oracle_window"]
