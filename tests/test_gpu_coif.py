"""GPU parity of the coiflet mode, WASABI_FLAG_COIFLET (reading R-A21:
coif1, the paper's "coiflets at level 3"), through the C ABI against the fp64 oracle:
kept index lists bit-exact (the fp64 coif1 analysis uses the specification's IEEE sequence, so the
fp32 rank keys match bit for bit), bins bit-exact on the halo band, psi/u within 1e-5 rel L2, bits
identical outside the threshold band, a band equals the same rows of the full hologram, and the
chain's closed form: r = 100%, aligned points -> u equals the GPU direct sum."""
import numpy as np
import pytest

from helpers import field_check, field_np, CONFIGS, gpu_params, make_points, orc_params, rel_l2
from test_gpu_parity import W, _check_fields, _direct_gpu, _gpu_run, _tables  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,kw", [("C1", {}), ("C1", dict(retention=1.0)), ("C2", dict(levels=3)),
                                     ("C1", dict(levels=1)), ("C1", dict(levels=4))])
def test_coif_tables_bitexact(W, orc, name, kw):
    cfg = CONFIGS[name].replace(**kw)
    p = gpu_params(cfg, wavelet=1)
    P = orc_params(orc, cfg, wavelet=1)
    t = _tables(W, p)
    depths = range(cfg.n_depth) if cfg.n_depth <= 8 else (0, cfg.n_depth // 2, cfg.n_depth - 1)
    for d in depths:
        lv, dx, dy, val = W.export_table(p, t, d)
        n_r = W.depth_geometry(p, d)["n_r"]
        olv, odx, ody, oval = orc.select(P, d, n_r)
        assert np.array_equal(lv, olv) and np.array_equal(dx, odx) and np.array_equal(dy, ody), f"depth {d}"
        assert np.max(np.abs(val - oval)) <= 1e-6 * np.max(np.abs(oval)) + 1e-7, f"depth {d} values"
        assert W.export_reach(p, t, d) == orc.reach_one(P, d), f"depth {d} reach"


def test_coif_bins_bitexact_on_halo_band(W, orc):
    import torch
    cfg = CONFIGS["C2"].replace(levels=3)
    pts = make_points(cfg, n=3000)
    p = gpu_params(cfg, wavelet=1)
    P = orc_params(orc, cfg, wavelet=1)
    t = _tables(W, p)
    e0, e1 = 512 - p.halo_rows(), 1024 + p.halo_rows()
    bins = torch.empty(W.bin_points_bytes(p, len(pts), e0, e1), dtype=torch.uint8, device="cuda")
    W.bin_points(p, t, torch.from_numpy(pts).cuda(), e0, e1, bins)
    torch.cuda.synchronize()
    ptr_g, idx_g = W.export_bins(p, bins)
    ptr_o, idx_o = orc.bins(P, p.tile, pts, e0, e1)
    assert np.array_equal(ptr_g, ptr_o) and np.array_equal(idx_g, idx_o)


@pytest.mark.parametrize("name,n,row0,row1,kw", [("C1", None, 0, 512, {}), ("C1", None, 192, 384, {}),
                                                 ("C2", 4000, 0, 2048, dict(levels=3)),
                                                 ("C2", 3000, 1024, 1536, dict(levels=3, retention=0.05)),
                                                 ("C1", None, 128, 384, dict(tile=128))])
def test_coif_field_parity(W, orc, name, n, row0, row1, kw):
    cfg = CONFIGS[name].replace(**kw)
    pts = make_points(cfg, n=n)
    pl, psi_g, u_g, bits_g = _gpu_run(W, cfg, pts, row0, row1, wavelet=1)
    _check_fields(orc, cfg, pts, row0, row1, pl, psi_g, u_g, bits_g, wavelet=1)


def test_coif_band_equals_full_hologram_rows(W):
    import torch
    cfg = CONFIGS["C2"].replace(levels=3)
    pts = make_points(cfg, n=3000)
    pl_f, _, u_f, _ = _gpu_run(W, cfg, pts, 0, 2048, wavelet=1)
    pl_b, _, u_b, _ = _gpu_run(W, cfg, pts, 704, 1216, wavelet=1)
    assert rel_l2(u_b, u_f[704:1216]) <= 1e-6


def test_coif_keep_all_aligned_equals_gpu_direct_sum(W):
    """r = 100%, 2^L-aligned points on levels, away from the hologram edge: coiflet WASABI u ==
    the direct sum (the coif1 chain is exact for such points, as the oracle's V3 pin shows)."""
    cfg = CONFIGS["C2"].replace(n_h=1024, retention=1.0, aligned=True, kind="levels", n_depth=4, levels=3,
                                z_max=0.4e-3)
    pts = make_points(cfg, n=300)
    pts = pts[(np.abs(pts[:, 0]) < 300e-6) & (np.abs(pts[:, 1]) < 300e-6)]
    _, _, u_w, _ = _gpu_run(W, cfg, pts, 0, 1024, wavelet=1)
    _, u_d = _direct_gpu(W, cfg, pts, 0, 1024)
    assert max(field_check(u_w, u_d)) <= 1e-5


def test_coif_hologram_host_equals_device_path(W):
    import torch
    cfg = CONFIGS["C1"]
    pts = make_points(cfg)
    p = gpu_params(cfg, wavelet=1)
    pl, _, u_g, bits_g = _gpu_run(W, cfg, pts, 128, 384, wavelet=1)
    ws = torch.empty(W.hologram_workspace_bytes(p, len(pts), 128, 384), dtype=torch.uint8, device="cuda")
    h_bits = torch.empty((256, p.n_h // 8), dtype=torch.uint8)
    h_u = torch.empty((256, p.n_h, 2), dtype=torch.float32)
    W.hologram_host(p, W.PrintParams(), torch.from_numpy(pts), 128, 384, ws, h_bits, h_u)
    torch.cuda.synchronize()
    assert np.array_equal(h_bits.numpy(), bits_g)
    hu = h_u.numpy()
    assert np.array_equal(hu[..., 0] + 1j * hu[..., 1], u_g.astype(np.complex64).astype(np.complex128))


@pytest.mark.parametrize("name,row0,row1,kw", [("C1", 0, 512, {}), ("C1", 192, 384, dict(levels=4)),
                                             ("C1", 128, 448, dict(levels=1)), ("C1", 64, 320, dict(levels=2)),
                                             ("C2", 1024, 1536, dict(levels=3, retention=0.05)),
                                             ("C1", 128, 384, dict(tile=128))])
def test_coif_fused_tiles_equal_line_passes(W, name, row0, row1, kw):
    """wasabi_inverse_wt in coiflet mode: the fused tile synthesis + quantise (u in its own buffer,
    psi only read) is bit-identical to the in-place line passes + quantize_kernel (u = psi's band
    rows), for L = 1..4, bands inside and at the hologram edges, and tile 128 bins."""
    import torch
    cfg = CONFIGS[name].replace(**kw)
    pts = make_points(cfg, n=3000 if name == "C2" else None)
    p = gpu_params(cfg, wavelet=1)
    pl = W.Pipeline(p, len(pts), row0, row1)
    pl.build_tables()
    pl.bin(torch.from_numpy(pts).cuda())
    pl.superpose()
    psi = pl.psi_band.clone()
    rows = row1 - row0
    u_f = torch.empty((rows, p.n_h, 2), dtype=torch.float32, device="cuda")
    b_f = torch.empty((rows, p.n_h // 8), dtype=torch.uint8, device="cuda")
    W.inverse_wt(p, pl.psi_band, u_f, row0, row1, W.PrintParams(), b_f)          # fused
    b_p = torch.empty_like(b_f)
    W.inverse_wt(p, pl.psi_band, None, row0, row1, W.PrintParams(), b_p)         # fused, print only
    torch.cuda.synchronize()
    assert torch.equal(pl.psi_band, psi), "the fused path must not write psi"
    b_l = torch.empty_like(b_f)
    u_l = pl.psi_band[row0 - pl.e0:row1 - pl.e0]
    W.inverse_wt(p, pl.psi_band, u_l, row0, row1, W.PrintParams(), b_l)          # line passes in place
    torch.cuda.synchronize()
    assert torch.equal(u_f, u_l), float((u_f - u_l).abs().max())
    assert torch.equal(b_f, b_l) and torch.equal(b_p, b_l)
    assert float(u_f.abs().max()) > 0


def test_coif_hologram_host_print_only_uses_fused_tiles(W):
    """wasabi_hologram_host without u (print only) takes the fused tile synthesis; its bits equal the
    device path's (which writes u to its own buffer) bit for bit."""
    import torch
    cfg = CONFIGS["C2"].replace(levels=3)
    pts = make_points(cfg, n=2000)
    p = gpu_params(cfg, wavelet=1)
    pl, _, u_g, bits_g = _gpu_run(W, cfg, pts, 512, 1024, wavelet=1)
    ws = torch.empty(W.hologram_workspace_bytes(p, len(pts), 512, 1024), dtype=torch.uint8, device="cuda")
    h_bits = torch.empty((512, p.n_h // 8), dtype=torch.uint8)
    W.hologram_host(p, W.PrintParams(), torch.from_numpy(pts), 512, 1024, ws, h_bits)
    torch.cuda.synchronize()
    assert np.array_equal(h_bits.numpy(), bits_g)


def test_coif_fused_entry_refuses(W):
    import torch
    cfg = CONFIGS["C1"]
    p = gpu_params(cfg, wavelet=1)
    pl = W.Pipeline(p, 10, 0, p.n_h)
    with pytest.raises(W.WasabiError, match="COIFLET"):
        W.superpose_inverse(p, pl.tables, pl.bins, 0, p.n_h, W.PrintParams(), pl.field, pl.bits)


@pytest.mark.parametrize("row0,x0", [(32768, 32768), (0, 65536 - 1024)])
def test_coif_c4_band_paper_scale(W, orc, row0, x0):
    """Coiflets at the paper's scale (PAPER.md:106 "coiflets as the wavelets at level 3", :128 a
    65,536^2 hologram): C4 with L = 3 on a 1024-row band (psi on its halo band, then the coif1 line
    synthesis), u and psi element-wise and in rel L2 within 1e-5 of the oracle on a 1024^2 window of it,
    bits identical outside the fixed threshold band (a central window, and a hologram corner where
    the zero boundary of R-A21 applies)."""
    import torch
    from helpers import REF, bits_check, oracle_window, parity_log
    cfg = CONFIGS["C4"].replace(levels=3)
    pts = make_points(cfg)
    p = gpu_params(cfg, wavelet=1)
    row1, w = row0 + 1024, 1024
    pl = W.Pipeline(p, len(pts), row0, row1)
    d = torch.from_numpy(pts).cuda()
    pl.build_tables()
    pl.bin(d)
    pl.superpose()
    torch.cuda.synchronize()
    psi_g = field_np(pl.psi_band[row0 - pl.e0:row1 - pl.e0, x0:x0 + w])
    pl.inverse()
    torch.cuda.synchronize()
    u_g = field_np(pl.field[:, x0:x0 + w])
    bits_g = pl.bits[:, x0 // 8:(x0 + w) // 8].cpu().numpy()
    P = orc_params(orc, cfg, wavelet=1)
    u_o, psi_o, bits_o, I_o = oracle_window(P, pts, x0, row0, w, 1024)
    e_psi, m_psi = field_check(psi_g, psi_o)
    e_u, m_u = field_check(u_g, u_o)
    bc = bits_check(bits_g, bits_o, I_o, u_g, u_o)
    parity_log(dict(case=f"C4 coif1 L=3 [{x0},{x0 + w}) x [{row0},{row1})", rel_psi=e_psi, max_psi=m_psi,
                    rel_u=e_u, max_u=m_u, **bc))
    assert np.linalg.norm(u_o) > 0
    assert max(e_psi, m_psi, e_u, m_u) <= 1e-5, (e_psi, m_psi, e_u, m_u)
    assert bc["bad"] == 0, bc
