"""Dense gather superposition (wasabi.h WASABI_FLAG_GATHER, the r -> 100% regime of SURVEY.md §8(f)).

Eq.(2) is the same sum whichever side loops: the gather kernel reads, per pixel,
every binned point's dense wavelet table (kept value or an exact 0) in bin order, so psi must be
BIT-IDENTICAL to the window-LUT scatter kernel's on the same tables and bins, fused or not; and both
within 1e-5 of the fp64 oracle (checked for gather here, for scatter in test_gpu_parity)."""
import numpy as np
import pytest

from helpers import CONFIGS, REF, bits_check, field_check, field_np, make_points, orc_params, parity_log
from test_gpu_parity import W  # noqa: F401

pytestmark = pytest.mark.gpu


def _run(W, p, pts, row0, row1):
    """psi (unfused) and fused (u, bits) of band [row0, row1) for params p."""
    import torch
    pl = W.Pipeline(p, max(1, len(pts)), row0, row1)
    d = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float32)).cuda()
    pl.build_tables()
    pl.bin(d[:len(pts)])
    pl.superpose()
    psi = pl.field.clone()
    u = torch.zeros_like(pl.field)
    bits = torch.zeros_like(pl.bits)
    W.superpose_inverse(p, pl.tables, pl.bins, row0, row1, pl.print_params, u, bits)
    torch.cuda.synchronize()
    return psi, u, bits


CASES = [
    ("C1", dict(retention=1.0), {}, 0, None),
    ("C1", dict(retention=0.3), {}, 0, None),                  # sparse tables through the gather
    ("C1", dict(retention=1.0, levels=2), {}, 0, None),        # fewest levels the gather takes
    ("C1", dict(retention=1.0, levels=6), {}, 0, None),        # corner cells of levels 3..6 and LL
    ("C1", dict(retention=0.7), dict(exact=True), 0, None),    # offset-class tables (R-A20)
    ("C2", dict(retention=1.0, n_depth=8), {}, 0, 2048),
    # 36 tile rows: one full group of 28 and a partial group of 8 (the tile order of both kernels)
    ("C2", dict(retention=0.6, n_depth=8), {}, 0, 36 * 64),
    ("C5", dict(retention=1.0, levels=5), {}, 8192 - 256, 8192 + 256),
]


@pytest.mark.parametrize("name,ckw,pkw,row0,row1", CASES)
def test_gather_equals_scatter_bitwise(W, name, ckw, pkw, row0, row1):
    import torch
    cfg = CONFIGS[name].replace(**ckw)
    n = {"C1": 600, "C2": 3000, "C5": 20000}[name]
    pts = make_points(cfg, n=n)
    row1 = cfg.n_h if row1 is None else row1
    if row1 > cfg.n_h:
        row1 = cfg.n_h
    pg = W.Params.from_config(cfg, path="gather", **pkw)
    ps = W.Params.from_config(cfg, path="scatter", **pkw)
    psi_g, u_g, b_g = _run(W, pg, pts, row0, row1)
    psi_s, u_s, b_s = _run(W, ps, pts, row0, row1)
    assert torch.any(psi_s != 0)
    assert torch.equal(psi_g, psi_s), float((psi_g - psi_s).abs().max())
    assert torch.equal(u_g, u_s) and torch.equal(b_g, b_s)


def test_gather_oracle_parity_c2_keep_all(W, orc):
    """Gather path (auto at r = 100%) against the fp64 oracle on a C2 field."""
    cfg = CONFIGS["C2"].replace(retention=1.0, n_depth=8)
    pts = make_points(cfg, n=2000)
    p = W.Params.from_config(cfg, path="gather")
    psi_g, u_g, b_g = _run(W, p, pts, 0, 1024)
    P = orc_params(orc, cfg)
    u_o, psi_o, _ = orc.Lut(P).hologram_window(pts.astype(np.float64), 0, 0, cfg.n_h, 1024)
    e_psi, m_psi = field_check(field_np(psi_g), psi_o)
    e_u, m_u = field_check(field_np(u_g), u_o)
    bits_o, I_o = orc.quantize(P, REF, u_o, 0, 0)
    bc = bits_check(b_g.cpu().numpy(), bits_o, I_o, field_np(u_g), u_o)
    parity_log(dict(case="gather C2 r=1 rows 0..1024", rel_psi=e_psi, max_psi=m_psi, rel_u=e_u, max_u=m_u, **bc))
    assert max(e_psi, m_psi, e_u, m_u) <= 1e-5
    assert bc["bad"] == 0, bc
