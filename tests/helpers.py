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


__all__ = ["CONFIGS", "make_points", "REF", "gpu_params", "orc_params", "run_gpu", "field_np", "rel_l2",
           "bits_mismatch_outside_band"]
