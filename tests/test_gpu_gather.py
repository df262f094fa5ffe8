"""Dense gather superposition (wasabi.h WASABI_FLAG_GATHER, the r -> 100% regime of SURVEY.md §8(f)).

Eq.(2) is the same sum whichever side loops: the gather kernel reads, per pixel,
every binned point's dense wavelet table (kept value or an exact 0) in depth-major order (reading
R-A22: chunks of the bin sorted by depth level), so psi equals the window-LUT scatter kernel's up to
the fp32 rounding of a reordered sum (element-wise 1e-6 of max|psi|), and both are within 1e-5 of
the fp64 oracle (checked for gather here, for scatter in test_gpu_parity); the gather's own result is
bitwise independent of the band split."""
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
def test_gather_matches_scatter(W, name, ckw, pkw, row0, row1):
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
    for g, r in ((psi_g, psi_s), (u_g, u_s)):
        e_rel, e_max = field_check(field_np(g), field_np(r), tol=1e-6)
        assert e_max <= 1e-6 and e_rel <= 1e-6, (e_rel, e_max)
    # print bits: a reordered fp32 sum can only move pixels sitting on the threshold
    flips = int(np.unpackbits((b_g ^ b_s).cpu().numpy()).sum())
    assert flips <= max(2, b_s.numel() * 8 // 1_000_000), flips


def test_gather_band_split_is_bitwise_identical(W):
    """The depth-major order depends only on each tile's bin: row bands concatenate bit for bit."""
    import torch
    cfg = CONFIGS["C2"].replace(retention=1.0, n_depth=8)
    pts = make_points(cfg, n=3000)
    p = W.Params.from_config(cfg, path="gather")
    _, u_full, b_full = _run(W, p, pts, 0, 1024)
    parts = [_run(W, p, pts, r0, r0 + 256) for r0 in range(0, 1024, 256)]
    assert torch.equal(torch.cat([q[1] for q in parts]), u_full)
    assert torch.equal(torch.cat([q[2] for q in parts]), b_full)


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


def test_gather_multi_chunk_bins(W, orc):
    """Bins of several depth-sorted chunks (> 1024 points per tile): C2 geometry with 60,000 points at
    r = 100% on a 256-row band -- gather within 1e-6 of the scatter kernel, and within 1e-5 of the
    fp64 oracle on a 256^2 window (element-wise and rel L2)."""
    import torch
    cfg = CONFIGS["C2"].replace(retention=1.0, n_depth=8)
    pts = make_points(cfg, n=60000)
    row0, row1 = 896, 1152
    pg = W.Params.from_config(cfg, path="gather")
    ps = W.Params.from_config(cfg, path="scatter")
    psi_g, u_g, b_g = _run(W, pg, pts, row0, row1)
    psi_s, u_s, b_s = _run(W, ps, pts, row0, row1)
    pl = W.Pipeline(pg, len(pts), row0, row1)
    pl.build_tables()
    pl.bin(torch.from_numpy(pts).cuda())
    torch.cuda.synchronize()
    ptr, _ = W.export_bins(pg, pl.bins)
    assert int(np.max(np.diff(ptr))) > 2048, "bins must span several chunks"
    for g, r in ((psi_g, psi_s), (u_g, u_s)):   # ~8,000 terms per pixel: fp32 reordering, 5x inside the bar
        e_rel, e_max = field_check(field_np(g), field_np(r), tol=2e-6)
        assert e_max <= 2e-6 and e_rel <= 2e-6, (e_rel, e_max)
    P = orc_params(orc, cfg)
    x0 = 896
    u_o, psi_o, _ = orc.Lut(P).hologram_window(pts.astype(np.float64), x0, row0, 256, 256)
    e_psi = field_check(field_np(psi_g)[:, x0:x0 + 256], psi_o)
    e_u = field_check(field_np(u_g)[:, x0:x0 + 256], u_o)
    parity_log(dict(case="gather multi-chunk C2 r=1 60k points", rel_psi=e_psi[0], max_psi=e_psi[1],
                    rel_u=e_u[0], max_u=e_u[1]))
    assert max(e_psi + e_u) <= 1e-5, (e_psi, e_u)
