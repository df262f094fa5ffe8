"""GPU parity of the offset-class (exact-shift) mode, WASABI_FLAG_EXACT_SHIFT (SURVEY.md §8(f)
NEXT-4, reading R-A20), through the C ABI against the fp64 oracle: class tables' kept index lists
bit-exact, bins bit-exact, psi/u within 1e-5 rel L2, bits identical outside the threshold band;
and the mode's defining property between the two GPU paths: at r = 100% WASABI equals the
quantised direct sum for random (not 2^L-aligned) points."""
import numpy as np
import pytest

from helpers import field_check, CONFIGS, field_np, gpu_params, make_points, orc_params, rel_l2
from test_gpu_parity import W, _check_fields, _direct_gpu, _gpu_run, _tables  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,kw", [("C1", {}), ("C1", dict(retention=1.0)), ("C2", dict(retention=0.05, n_depth=4)),
                                     ("C1", dict(levels=1))])
def test_exact_tables_bitexact(W, orc, name, kw):
    cfg = CONFIGS[name].replace(**kw)
    p = gpu_params(cfg, exact=True)
    P = orc_params(orc, cfg, exact=True)
    assert W.table_count(p) == P.n_tables == cfg.n_depth << (2 * cfg.levels)
    t = _tables(W, p)
    L = cfg.levels
    n = P.n_tables
    sample = sorted({0, 1, (1 << L) + 1, n // 3 + 5, n // 2, n - 2, n - 1})
    for k in sample:
        lv, dx, dy, val = W.export_table(p, t, k)
        n_r = W.depth_geometry(p, k)["n_r"]
        assert n_r == orc.table_info(P, k)["n_r"]
        olv, odx, ody, oval = orc.select(P, k, n_r)
        assert np.array_equal(lv, olv) and np.array_equal(dx, odx) and np.array_equal(dy, ody), f"table {k}"
        assert np.max(np.abs(val - oval)) <= 1e-6 * np.max(np.abs(oval)) + 1e-7, f"table {k} values"
        assert W.export_reach(p, t, k) == orc.reach_one(P, k), f"table {k} reach"


@pytest.mark.parametrize("name,n,row0,row1", [("C1", None, 0, 512), ("C2", 3000, 512, 1024)])
def test_exact_bins_bitexact(W, orc, name, n, row0, row1):
    import torch
    cfg = CONFIGS[name].replace(n_depth=min(CONFIGS[name].n_depth, 8), retention=0.05)
    pts = make_points(cfg, n=n)
    p = gpu_params(cfg, exact=True)
    P = orc_params(orc, cfg, exact=True)
    t = _tables(W, p)
    bins = torch.empty(W.bin_points_bytes(p, len(pts), row0, row1), dtype=torch.uint8, device="cuda")
    W.bin_points(p, t, torch.from_numpy(pts).cuda(), row0, row1, bins)
    torch.cuda.synchronize()
    assert W.bins_stats(bins)["status"] == 0
    ptr_g, idx_g = W.export_bins(p, bins)
    ptr_o, idx_o = orc.bins(P, p.tile, pts, row0, row1)
    assert np.array_equal(ptr_g, ptr_o) and np.array_equal(idx_g, idx_o)


@pytest.mark.parametrize("name,n,row0,row1,kw", [("C1", None, 0, 512, {}), ("C1", None, 128, 384, dict(tile=128)),
                                                 ("C2", 3000, 0, 1024, dict(retention=0.05, n_depth=4))])
def test_exact_field_parity(W, orc, name, n, row0, row1, kw):
    cfg = CONFIGS[name].replace(**kw)
    pts = make_points(cfg, n=n)
    pl, psi_g, u_g, bits_g = _gpu_run(W, cfg, pts, row0, row1, exact=True)
    _check_fields(orc, cfg, pts, row0, row1, pl, psi_g, u_g, bits_g, exact=True)


def test_exact_keep_all_equals_gpu_direct_sum_anywhere(W):
    """r = 100%, random (non-aligned) points on depth levels: exact-mode WASABI u == the GPU direct
    sum (fp32 both) -- R-A20's claim, which the standard mode (R-A8) fails for such points."""
    cfg = CONFIGS["C2"].replace(n_h=1024, retention=1.0, kind="levels", n_depth=4, levels=3, z_max=0.4e-3)
    pts = make_points(cfg, n=300)
    _, _, u_w, _ = _gpu_run(W, cfg, pts, 0, 1024, exact=True)
    _, u_d = _direct_gpu(W, cfg, pts, 0, 1024)
    assert max(field_check(u_w, u_d)) <= 1e-5
    _, _, u_s, _ = _gpu_run(W, cfg, pts, 0, 1024)
    assert rel_l2(u_s, u_d) > 1e-2          # control: R-A8 shifts are not exact off-grid


def test_exact_fused_equals_unfused(W):
    import torch
    cfg = CONFIGS["C1"]
    pts = make_points(cfg)
    p = gpu_params(cfg, exact=True)
    pl = W.Pipeline(p, len(pts), 0, p.n_h)
    d = torch.from_numpy(pts).cuda()
    pl.run(d, fused=False)
    u1 = pl.field.clone(); b1 = pl.bits.clone()
    pl.run(d, fused=True)
    torch.cuda.synchronize()
    assert torch.equal(u1, pl.field) and torch.equal(b1, pl.bits)


def test_exact_rejects_deep_levels(W):
    cfg = CONFIGS["C3"]
    p = gpu_params(cfg, exact=True)           # L = 5: 4^5 tables per depth -> refused
    with pytest.raises(W.WasabiError, match="EXACT_SHIFT"):
        W.psf_tables_bytes(p)


def test_exact_hologram_host_equals_device_path(W):
    """The whole path from host buffers (chunked superposition, side-stream copies) in the
    offset-class mode equals the device pipeline bit for bit."""
    import torch
    cfg = CONFIGS["C1"]
    pts = make_points(cfg)
    p = gpu_params(cfg, exact=True)
    _, _, u_g, bits_g = _gpu_run(W, cfg, pts, 128, 384, exact=True)
    ws = torch.empty(W.hologram_workspace_bytes(p, len(pts), 128, 384), dtype=torch.uint8, device="cuda")
    h_bits = torch.empty((256, p.n_h // 8), dtype=torch.uint8)
    h_u = torch.empty((256, p.n_h, 2), dtype=torch.float32)
    W.hologram_host(p, W.PrintParams(), torch.from_numpy(pts), 128, 384, ws, h_bits, h_u)
    torch.cuda.synchronize()
    assert np.array_equal(h_bits.numpy(), bits_g)
    hu = h_u.numpy()
    assert np.array_equal(hu[..., 0] + 1j * hu[..., 1], u_g.astype(np.complex64).astype(np.complex128))
