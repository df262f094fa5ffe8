"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same seeded inputs.

Bars (north_star): top-k index lists and bins bit-exact; psi and u within 1e-5
relative L2 (fp32 GPU vs fp64 oracle); print bits identical except on pixels inside the threshold
band (R-A16, helpers.bits_check: a fixed band, |I_oracle| <= max|u_gpu - u_oracle| + 1e-6 rms(I));
fields also element-wise, max|g - o| <= 1e-5 max|o|."""
import numpy as np
import pytest

from helpers import (CONFIGS, REF, bits_check, bits_mismatch_outside_band, field_check, field_np, gpu_params,
                     make_points, oracle_window, orc_params, parity_log, rel_l2)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import __graft_entry__
    __graft_entry__.build()
    import paper_1708_04233_b200 as W
    return W


def _tables(W, p):
    import torch
    tb, sb = W.psf_tables_bytes(p)
    t = torch.empty(tb, dtype=torch.uint8, device="cuda")
    s = torch.empty(sb, dtype=torch.uint8, device="cuda")
    W.build_psf_tables(p, t, s)
    torch.cuda.synchronize()
    W.tables_check(p, t)
    return t


def _compare_depth(W, orc, p, P, t, d):
    lv, dx, dy, val = W.export_table(p, t, d)
    n_r = W.depth_geometry(p, d)["n_r"]
    olv, odx, ody, oval = orc.select(P, d, n_r)
    assert len(lv) == n_r
    assert np.array_equal(lv, olv) and np.array_equal(dx, odx) and np.array_equal(dy, ody), f"depth {d}"
    scale = np.max(np.abs(oval))
    assert np.max(np.abs(val - oval)) <= 1e-6 * scale + 1e-7, f"depth {d} values"
    assert W.export_reach(p, t, d) == orc.reach_one(P, d), f"depth {d} reach (R-A19)"


# ---------------------------------------------------------------- step 1: tables (bit-exact indices)
@pytest.mark.parametrize("name,kw", [("C1", {}), ("C2", dict(retention=0.01)), ("C2", dict(retention=0.05)),
                                     ("C2", {}), ("C3", {}), ("C5", dict(retention=1.0)),
                                     ("C1", dict(levels=1)), ("C1", dict(levels=6, tile=128))])
def test_tables_bitexact(W, orc, name, kw):
    cfg = CONFIGS[name].replace(**{k: v for k, v in kw.items() if k in ("retention", "levels", "tile")})
    p = gpu_params(cfg)
    P = orc_params(orc, cfg)
    t = _tables(W, p)
    depths = range(cfg.n_depth) if cfg.n_depth <= 16 else sorted({0, 1, cfg.n_depth // 3, cfg.n_depth // 2,
                                                                   cfg.n_depth - 2, cfg.n_depth - 1})
    for d in depths:
        _compare_depth(W, orc, p, P, t, d)


def test_tables_bitexact_c4_sample(W, orc):
    cfg = CONFIGS["C4"]
    p = gpu_params(cfg)
    P = orc_params(orc, cfg)
    t = _tables(W, p)
    for d in (0, 31, 63, 64, 100, 127):   # |z| = 2 mm (largest table, 1408^2) ... 0.016 mm
        _compare_depth(W, orc, p, P, t, d)


# ---------------------------------------------------------------- step 2a: bins (bit-exact)
@pytest.mark.parametrize("name,n,row0,row1", [("C1", None, 0, 512), ("C1", None, 128, 320), ("C2", None, 0, 2048),
                                              ("C2", 3000, 1024, 1536), ("C3", 20000, 0, 8192)])
def test_bins_bitexact(W, orc, name, n, row0, row1):
    import torch
    cfg = CONFIGS[name]
    pts = make_points(cfg, n=n)
    pts[::97, 3] = -1.0           # skipped points
    p = gpu_params(cfg)
    P = orc_params(orc, cfg)
    t = _tables(W, p)
    bins = torch.empty(W.bin_points_bytes(p, len(pts), row0, row1), dtype=torch.uint8, device="cuda")
    W.bin_points(p, t, torch.from_numpy(pts).cuda(), row0, row1, bins)
    torch.cuda.synchronize()
    st = W.bins_stats(bins)
    assert st["status"] == 0 and st["n_skipped"] == len(pts[::97])
    ptr_g, idx_g = W.export_bins(p, bins)
    ptr_o, idx_o = orc.bins(P, p.tile, pts, row0, row1)
    assert np.array_equal(ptr_g, ptr_o)
    assert np.array_equal(idx_g, idx_o)


# ---------------------------------------------------------------- steps 2b-4: fields and bits
def _gpu_run(W, cfg, pts, row0, row1, **kw):
    import torch
    p = gpu_params(cfg, **kw)
    pl = W.Pipeline(p, max(1, len(pts)), row0, row1)
    d_pts = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
    pl.build_tables()
    pl.bin(d_pts)
    pl.superpose()
    psi = field_np(pl.psi_band[row0 - pl.e0:row1 - pl.e0])   # == pl.field unless coiflets (halo band)
    pl.inverse()
    torch.cuda.synchronize()
    return pl, psi, field_np(pl.field), pl.bits.cpu().numpy()


def _check_fields(orc, cfg, pts, row0, row1, pl, psi_g, u_g, bits_g, x0=0, w=None, case=None, **kw):
    """psi and u: rel L2 AND element-wise max|g - o| <= 1e-5 max|o|; bits identical outside the fixed
    threshold band of helpers.bits_check; the numbers go to $WASABI_PARITY_LOG."""
    P = orc_params(orc, cfg, **kw)
    w = cfg.n_h if w is None else w
    lut = orc.Lut(P)
    u_o, psi_o, _ = lut.hologram_window(pts, x0, row0, w, row1 - row0)
    psi_gw = psi_g[:, x0:x0 + w]
    u_gw = u_g[:, x0:x0 + w]
    e_psi, m_psi = field_check(psi_gw, psi_o)
    e_u, m_u = field_check(u_gw, u_o)
    bits_o, I_o = orc.quantize(P, REF, u_o, x0, row0)
    bc = bits_check(bits_g[:, x0 // 8:(x0 + w) // 8], bits_o, I_o, u_gw, u_o)
    parity_log(dict(case=case or f"{cfg.name} rows [{row0},{row1}) x [{x0},{x0 + w})", rel_psi=e_psi,
                    max_psi=m_psi, rel_u=e_u, max_u=m_u, **bc))
    assert e_psi <= 1e-5 and m_psi <= 1e-5, (e_psi, m_psi)
    assert e_u <= 1e-5 and m_u <= 1e-5, (e_u, m_u)
    assert bc["bad"] == 0, f"print bits differ outside the threshold band: {bc}"
    return e_psi, e_u


@pytest.mark.parametrize("name,n,row0,row1", [("C1", None, 0, 512), ("C1", None, 192, 448),
                                              ("C2", None, 0, 2048), ("C2", 4000, 640, 1152)])
def test_field_parity(W, orc, name, n, row0, row1):
    cfg = CONFIGS[name]
    pts = make_points(cfg, n=n)
    pl, psi_g, u_g, bits_g = _gpu_run(W, cfg, pts, row0, row1)
    _check_fields(orc, cfg, pts, row0, row1, pl, psi_g, u_g, bits_g)


@pytest.mark.parametrize("r", [0.01, 0.05])
def test_field_parity_c2_retentions(W, orc, r):
    cfg = CONFIGS["C2"].replace(retention=r)
    pts = make_points(cfg, n=5000)
    pl, psi_g, u_g, bits_g = _gpu_run(W, cfg, pts, 0, 2048)
    _check_fields(orc, cfg, pts, 0, 2048, pl, psi_g, u_g, bits_g)


def test_field_parity_c3_band(W, orc):
    """C3 (8192^2, 532 nm, RGB-D surface, L=5, r=5%): full GPU band of 512 rows vs oracle."""
    cfg = CONFIGS["C3"]
    pts = make_points(cfg)
    pl, psi_g, u_g, bits_g = _gpu_run(W, cfg, pts, 4096, 4608)
    _check_fields(orc, cfg, pts, 4096, 4608, pl, psi_g, u_g, bits_g, x0=2048, w=2048)


@pytest.mark.parametrize("kw", [dict(tile=128), dict(levels=1), dict(levels=6, tile=128),
                                dict(retention=1.0)])
def test_field_parity_variants(W, orc, kw):
    cfg = CONFIGS["C1"].replace(**kw)
    pts = make_points(cfg, n=600)
    pl, psi_g, u_g, bits_g = _gpu_run(W, cfg, pts, 0, cfg.n_h)
    _check_fields(orc, cfg, pts, 0, cfg.n_h, pl, psi_g, u_g, bits_g)


def test_aligned_keep_all_equals_direct_sum(W, orc):
    """V3 on the GPU: r=100%, 2^L-aligned points on levels -> u equals the D2 direct sum."""
    cfg = CONFIGS["C1"].replace(retention=1.0, aligned=True, kind="levels")
    pts = make_points(cfg, n=200)
    pl, psi_g, u_g, bits_g = _gpu_run(W, cfg, pts, 0, cfg.n_h)
    P = orc_params(orc, cfg)
    d2 = orc.direct_d2(P, pts.astype(np.float64), 0, 0, cfg.n_h, cfg.n_h)
    assert max(field_check(u_g, d2)) <= 1e-5


# ---------------------------------------------------------------- edge cases
def test_empty_and_invalid_points(W, orc):
    cfg = CONFIGS["C1"]
    for pts in (np.zeros((0, 4), np.float32),
                np.array([[0, 0, 0.2e-3, 0.0], [np.nan, 0, 0.2e-3, 1], [0, 0, 5e-3, 1]], np.float32),
                np.array([[0.9e-3, 0.9e-3, 0.2e-3, 1.0]], np.float32)):     # PSF far outside
        pl, psi_g, u_g, bits_g = _gpu_run(W, cfg, pts, 0, cfg.n_h)
        assert np.all(psi_g == 0) and np.all(u_g == 0)


def test_points_outside_aperture_contribute(W, orc):
    """A point outside the hologram whose PSF overlaps it contributes (R-A12: partial bins)."""
    cfg = CONFIGS["C1"]
    pts = np.array([[-0.27e-3, 0.1e-3, 0.4e-3, 1.0], [0.26e-3, -0.3e-3, 0.35e-3, 0.5]], np.float32)
    pl, psi_g, u_g, bits_g = _gpu_run(W, cfg, pts, 0, cfg.n_h)
    assert np.any(u_g != 0)
    _check_fields(orc, cfg, pts, 0, cfg.n_h, pl, psi_g, u_g, bits_g)


def test_band_split_is_bitwise_identical(W):
    """Row bands (the multi-GPU split) concatenate to the single-band result
    bit for bit: no halo, fixed per-pixel accumulation order."""
    cfg = CONFIGS["C2"]
    pts = make_points(cfg, n=4000)
    _, _, u_full, b_full = _gpu_run(W, cfg, pts, 0, 2048)
    parts_u, parts_b = [], []
    for b in range(4):
        _, _, u, bb = _gpu_run(W, cfg, pts, b * 512, (b + 1) * 512)
        parts_u.append(u)
        parts_b.append(bb)
    assert np.array_equal(np.concatenate(parts_u), u_full)
    assert np.array_equal(np.concatenate(parts_b), b_full)


def test_deterministic_repeat(W):
    cfg = CONFIGS["C2"]
    pts = make_points(cfg, n=3000)
    _, p1, u1, b1 = _gpu_run(W, cfg, pts, 0, 2048)
    _, p2, u2, b2 = _gpu_run(W, cfg, pts, 0, 2048)
    assert np.array_equal(p1, p2) and np.array_equal(u1, u2) and np.array_equal(b1, b2)


# ---------------------------------------------------------------- steps 3 and 4 standalone
@pytest.mark.parametrize("L", [1, 3, 6])
def test_inverse_standalone(W, orc, L):
    import torch
    cfg = CONFIGS["C1"].replace(levels=L, tile=64)
    p = gpu_params(cfg)
    rng = np.random.default_rng(L)
    psi = (rng.standard_normal((128, 512)) + 1j * rng.standard_normal((128, 512))).astype(np.complex64)
    d = torch.from_numpy(np.stack([psi.real, psi.imag], -1).astype(np.float32)).cuda()
    u = torch.empty_like(d)
    W.inverse_wt(p, d, u, 64, 192)
    torch.cuda.synchronize()
    u_o = orc.haar_inv(psi.astype(np.complex128), L)
    assert rel_l2(field_np(u), u_o) <= 1e-6


@pytest.mark.parametrize("ref", [REF, (0.0002, -0.0001, -0.002), (0.0, 0.0, -0.05)])
def test_quantize_standalone_same_input(W, orc, ref):
    """Step 4 alone on the same u: bits identical except |I| <= 1e-6 rms(I) (the decision is taken
    on identical inputs; only the fp64 phase reduction / fp32 (cos, sin) differ).  The references:
    the paper's (series path of print_byte), one 2 mm from the hologram (every pixel takes its own
    square root) and one between."""
    import torch
    REF = ref
    cfg = CONFIGS["C2"]
    p = gpu_params(cfg)
    rng = np.random.default_rng(5)
    u = (rng.standard_normal((256, 2048)) + 1j * rng.standard_normal((256, 2048))).astype(np.complex64)
    d = torch.from_numpy(np.stack([u.real, u.imag], -1)).cuda()
    bits = torch.empty((256, 256), dtype=torch.uint8, device="cuda")
    W.quantize(p, W.PrintParams(*REF), d, 512, 768, bits)
    torch.cuda.synchronize()
    P = orc_params(orc, cfg)
    bits_o, I_o = orc.quantize(P, REF, u.astype(np.complex128), 0, 512)
    g = np.unpackbits(bits.cpu().numpy(), axis=1, bitorder="big").astype(bool)
    o = np.unpackbits(bits_o, axis=1, bitorder="big").astype(bool)
    rms = np.sqrt(np.mean(I_o ** 2))
    assert np.sum((g != o) & (np.abs(I_o) > 1e-6 * rms)) == 0


def test_fused_equals_standalone_quantize(W):
    import torch
    cfg = CONFIGS["C1"]
    pts = make_points(cfg)
    pl, _, u_g, bits_fused = _gpu_run(W, cfg, pts, 0, 512)
    bits = torch.empty_like(pl.bits)
    W.quantize(pl.p, pl.print_params, pl.field, 0, 512, bits)
    torch.cuda.synchronize()
    assert np.array_equal(bits.cpu().numpy(), bits_fused)


@pytest.mark.parametrize("name,kw", [("C1", {}), ("C2", {}), ("C1", dict(levels=1)), ("C1", dict(tile=128, levels=6))])
def test_fused_superpose_inverse_bitwise(W, name, kw):
    """NEXT-1 fused kernel == superpose + inverse_wt (+ fused quantise), bit for bit; print-only too."""
    import torch
    cfg = CONFIGS[name].replace(**kw)
    pts = make_points(cfg, n=3000)
    p = gpu_params(cfg)
    pl = W.Pipeline(p, len(pts), 0, p.n_h)
    d = torch.from_numpy(pts).cuda()
    pl.run(d, fused=False)
    u_ref, b_ref = pl.field.clone(), pl.bits.clone()
    pl.field.zero_()
    pl.bits.zero_()
    pl.run(d, fused=True)
    torch.cuda.synchronize()
    assert torch.equal(pl.field, u_ref) and torch.equal(pl.bits, b_ref)
    pl.bits.zero_()
    W.superpose_inverse(p, pl.tables, pl.bins, 0, p.n_h, pl.print_params, None, pl.bits)
    torch.cuda.synchronize()
    assert torch.equal(pl.bits, b_ref)


# ---------------------------------------------------------------- whole path from host buffers
def test_hologram_host_equals_device_path(W):
    import torch
    cfg = CONFIGS["C2"]
    pts = make_points(cfg, n=5000)
    p = gpu_params(cfg)
    ws = torch.empty(W.hologram_workspace_bytes(p, len(pts), 512, 1024), dtype=torch.uint8, device="cuda")
    h_pts = torch.from_numpy(pts).pin_memory()
    h_bits = torch.empty((512, 256), dtype=torch.uint8).pin_memory()
    h_u = torch.empty((512, 2048, 2), dtype=torch.float32).pin_memory()
    W.hologram_host(p, W.PrintParams(*REF), h_pts, 512, 1024, ws, h_bits, h_u)
    torch.cuda.synchronize()
    _, _, u_d, b_d = _gpu_run(W, cfg, pts, 512, 1024)
    assert np.array_equal(h_bits.numpy(), b_d)
    assert np.array_equal(field_np(h_u), u_d)


# ---------------------------------------------------------------- full-size C4
@pytest.fixture(scope="module")
def c4_run(W):
    """BASELINE configs[3] at full size (65,536^2, 2e6 points, 128 levels, L=6, r=5%) in the bench's
    launch configuration (one GPU, all rows, fused superpose/inverse/quantise), here also writing u."""
    import torch
    cfg = CONFIGS["C4"]
    pts = make_points(cfg)
    p = gpu_params(cfg)
    pl = W.Pipeline(p, len(pts), 0, p.n_h)
    pl.run(torch.from_numpy(pts).cuda())
    torch.cuda.synchronize()
    return cfg, p, pts, pl


def _c4_windows(cfg, pts):
    """(name, x0, y0, w): the bench's central 6144^2 window (bench.py oracle_sample), 1024^2 windows at
    two hologram corners (the last, partial, 28-row tile group included), and 1024^2 windows where
    the points' mean |z| is largest (|z| -> 2 mm: 1408^2 tables) and smallest (z ~ 0: the plane
    crossing, tiny PSFs)."""
    n = cfg.n_h
    wins = [("bench6144", n // 2 - 3072, n // 2 - 3072, 6144), ("corner00", 0, 0, 1024),
            ("cornerNN", n - 1024, n - 1024, 1024)]
    cx = np.clip((pts[:, 0] / cfg.pitch + n // 2) // 1024, 0, n // 1024 - 1).astype(np.int64)
    cy = np.clip((pts[:, 1] / cfg.pitch + n // 2) // 1024, 0, n // 1024 - 1).astype(np.int64)
    cell = cy * (n // 1024) + cx
    cnt = np.bincount(cell, minlength=(n // 1024) ** 2)
    mz = np.bincount(cell, weights=np.abs(pts[:, 2]), minlength=cnt.size) / np.maximum(cnt, 1)
    mz_lo = np.where(cnt > 0, mz, np.inf)
    for name, c in (("zmax", int(np.argmax(mz))), ("zmin", int(np.argmin(mz_lo)))):
        wins.append((name, (c % (n // 1024)) * 1024, (c // (n // 1024)) * 1024, 1024))
    return wins


@pytest.mark.parametrize("win", ["bench6144", "corner00", "cornerNN", "zmax", "zmin"])
def test_c4_windows_vs_oracle(W, orc, c4_run, win):
    """C4 parity on oracle-computed windows of the full-size run ("at C4, on
    oracle-computed bands"): u element-wise and in rel L2 within 1e-5, bits identical outside the
    fixed threshold band; flip counts logged."""
    cfg, p, pts, pl = c4_run
    name, x0, y0, w = [x for x in _c4_windows(cfg, pts) if x[0] == win][0]
    P = orc_params(orc, cfg)
    u_o, psi_o, bits_o, I_o = oracle_window(P, pts, x0, y0, w, w)
    u_g = field_np(pl.field[y0:y0 + w, x0:x0 + w])
    e_u, m_u = field_check(u_g, u_o)
    bc = bits_check(pl.bits[y0:y0 + w, x0 // 8:(x0 + w) // 8].cpu().numpy(), bits_o, I_o, u_g, u_o)
    parity_log(dict(case=f"C4 {name} [{x0},{x0 + w}) x [{y0},{y0 + w})", rel_u=e_u, max_u=m_u, **bc))
    assert np.linalg.norm(u_o) > 0
    assert e_u <= 1e-5 and m_u <= 1e-5, (e_u, m_u)
    assert bc["bad"] == 0, bc


def test_c4_full_size_bins_sampled(W, orc, c4_run):
    """C4 bins at full size: point counts, and 8 sampled tiles bit-exact against the oracle's
    definition (orc_bin_tile)."""
    cfg, p, pts, pl = c4_run
    st = W.bins_stats(pl.bins)
    assert st["status"] == 0 and st["n_valid"] == len(pts)
    P = orc_params(orc, cfg)
    ptr_g, idx_g = W.export_bins(p, pl.bins)
    T = p.tile
    tiles_x = p.n_h // T
    rng = np.random.default_rng(44)
    for t in rng.integers(0, len(ptr_g) - 1, 8):
        X0, Y0 = int(t % tiles_x) * T, int(t // tiles_x) * T
        assert np.array_equal(idx_g[ptr_g[t]:ptr_g[t + 1]], orc.bin_tile(P, T, pts, X0, Y0))


def test_c4_band_fused_equals_unfused(W):
    """A full-width 2048-row C4 band (32 tile rows: one full 28-row tile group of the fused kernel's
    CTA order and a partial one): the fused kernel equals superpose + inverse_wt bit for bit (u and
    bits), and print-only fused bits equal them too."""
    import torch
    cfg = CONFIGS["C4"]
    pts = make_points(cfg)
    p = gpu_params(cfg)
    row0, row1 = 8192, 10240
    pl = W.Pipeline(p, len(pts), row0, row1)
    d = torch.from_numpy(pts).cuda()
    pl.run(d, fused=False)
    u_ref, b_ref = pl.field.clone(), pl.bits.clone()
    pl.field.zero_()
    pl.bits.zero_()
    pl.run(d, build_tables=False, fused=True)
    torch.cuda.synchronize()
    assert torch.equal(pl.field, u_ref) and torch.equal(pl.bits, b_ref)
    pl.bits.zero_()
    W.superpose_inverse(p, pl.tables, pl.bins, row0, row1, pl.print_params, None, pl.bits)
    torch.cuda.synchronize()
    assert torch.equal(pl.bits, b_ref)


# ---------------------------------------------------------------- C5 (BASELINE configs[4])
@pytest.mark.parametrize("r", [0.01, 0.25, 1.0])
def test_c5_band_parity(W, orc, r):
    """C5 (16,384^2, z ~ U[0.1,1] mm, 64 levels, L=5) at N=1e4 on a 256-row band; oracle on a
    2048-wide window of it."""
    cfg = CONFIGS["C5"].replace(retention=r)
    pts = make_points(cfg, n=10_000)
    pl, psi_g, u_g, bits_g = _gpu_run(W, cfg, pts, 8192, 8448)
    _check_fields(orc, cfg, pts, 8192, 8448, pl, psi_g, u_g, bits_g, x0=7168, w=2048)


def test_c5_aligned_keep_all_equals_direct_sum(W, orc):
    """r=100%, 2^L-aligned points on levels at C5 scale: u equals the quantised direct sum (D2)."""
    cfg = CONFIGS["C5"].replace(retention=1.0, aligned=True, kind="levels")
    pts = make_points(cfg, n=2000)
    pl, psi_g, u_g, bits_g = _gpu_run(W, cfg, pts, 4096, 4352)
    P = orc_params(orc, cfg)
    d2 = orc.direct_d2(P, pts.astype(np.float64), 6144, 4096, 1024, 256)
    assert max(field_check(u_g[:, 6144:7168], d2)) <= 1e-5


def test_c5_full_size_sampled(W, orc):
    """C5 at N=1e6, r=5% on the full 16,384^2 hologram; sampled 32x32 blocks recomputed by the oracle."""
    import torch
    cfg = CONFIGS["C5"]
    pts = make_points(cfg, n=1_000_000)
    p = gpu_params(cfg)
    pl = W.Pipeline(p, len(pts), 0, p.n_h)
    pl.run(torch.from_numpy(pts).cuda())
    torch.cuda.synchronize()
    assert W.bins_stats(pl.bins)["status"] == 0
    P = orc_params(orc, cfg)
    lut = orc.Lut(P)
    rng = np.random.default_rng(55)
    B = 32
    for _ in range(4):
        X0 = int(rng.integers(0, p.n_h // B)) * B
        Y0 = int(rng.integers(0, p.n_h // B)) * B
        u_o, _, _ = lut.hologram_window(pts, X0, Y0, B, B)
        u_g = field_np(pl.field[Y0:Y0 + B, X0:X0 + B])
        assert max(field_check(u_g, u_o)) <= 1e-5


# ---------------------------------------------------------------- conventional baseline (direct sum)
def _direct_gpu(W, cfg, pts, row0, row1):
    import torch
    p = gpu_params(cfg)
    pl = W.Pipeline(p, max(1, len(pts)), row0, row1)
    d = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
    pl.build_tables()
    W.bin_points_psf(p, pl.tables, d, row0, row1, pl.bins)      # the whole PSF disc (conventional method)
    dense = torch.empty(W.psf_dense_bytes(p), dtype=torch.uint8, device="cuda")
    W.build_psf_dense(p, dense)
    u = torch.empty((row1 - row0, p.n_h, 2), dtype=torch.float32, device="cuda")
    W.direct_sum(p, dense, pl.bins, row0, row1, u)
    torch.cuda.synchronize()
    return pl, field_np(u)


@pytest.mark.parametrize("name,n,row0,row1,kw", [("C1", None, 0, 512, {}), ("C2", 3000, 512, 1024, {}),
                                                 ("C1", 500, 128, 384, dict(tile=128, levels=6))])
def test_direct_sum_equals_oracle_d2(W, orc, name, n, row0, row1, kw):
    """GPU PSF stamping == the oracle's quantised direct sum D2 (Eq.(1) with snapped points/levels)."""
    cfg = CONFIGS[name].replace(**kw)
    pts = make_points(cfg, n=n)
    _, u_g = _direct_gpu(W, cfg, pts, row0, row1)
    P = orc_params(orc, cfg)
    d2 = orc.direct_d2(P, pts.astype(np.float64), 0, row0, cfg.n_h, row1 - row0)
    assert max(field_check(u_g, d2)) <= 1e-5


def test_wasabi_keep_all_aligned_equals_gpu_direct_sum(W):
    """V3 between the two GPU paths: r=100%, aligned points -> WASABI u == direct sum (fp32)."""
    cfg = CONFIGS["C2"].replace(retention=1.0, aligned=True, kind="levels", n_depth=8)
    pts = make_points(cfg, n=400)
    _, _, u_w, _ = _gpu_run(W, cfg, pts, 0, 2048)
    _, u_d = _direct_gpu(W, cfg, pts, 0, 2048)
    assert max(field_check(u_w, u_d)) <= 1e-5


def test_hologram_stream_equals_full(W):
    """Band-by-band streaming (PAPER.md:115-116 sub-holograms; buffers for one band only) gives the
    full hologram's print bits bit for bit."""
    import torch
    cfg = CONFIGS["C2"]
    pts = make_points(cfg, n=4000)
    _, _, _, bits_full = _gpu_run(W, cfg, pts, 0, 2048)
    p = gpu_params(cfg)
    hs = W.pipeline.HologramStream(p, len(pts), 384)
    d = torch.from_numpy(pts).cuda()
    parts = list(hs.run(d))
    assert [r for r, _ in parts] == list(range(0, 2048, 384))
    assert np.array_equal(np.concatenate([b for _, b in parts]), bits_full)


@pytest.mark.parametrize("kw", [{}, dict(exact=True)])
def test_cuda_graph_replay_equals_eager(W, kw):
    """A whole step (tables, bins, fused superpose/inverse/quantise) captured in a CUDA graph: the
    replay reads the points in place and reproduces the eager step bit for bit, also after new
    point data is copied into the captured tensor.  exact=True: C1 has 512 offset-class tables, so
    the table build's descriptor upload (40 KB) takes the capture-safe by-value path."""
    import torch
    cfg = CONFIGS["C1"]
    p = gpu_params(cfg, **kw)
    pts_a = make_points(cfg)
    pts_b = make_points(cfg, seed=cfg.seed + 1)
    d = torch.from_numpy(pts_a).cuda()
    pl = W.Pipeline(p, len(pts_a), 0, p.n_h)
    pl.capture(d)
    eager = W.Pipeline(p, len(pts_a), 0, p.n_h)
    for pts in (pts_a, pts_b):
        d.copy_(torch.from_numpy(np.ascontiguousarray(pts)))
        pl.field.zero_()
        pl.bits.zero_()
        pl.replay()
        eager.run(torch.from_numpy(np.ascontiguousarray(pts)).cuda())
        torch.cuda.synchronize()
        assert torch.equal(pl.bits, eager.bits)
        assert torch.equal(pl.field, eager.field)


# ---------------------------------------------------------------- work accounting
@pytest.mark.parametrize("name,n,row0,row1,kw", [("C2", 3000, 512, 1024, {}), ("C1", None, 0, 512, {}),
                                                 ("C1", 500, 128, 320, dict(exact=True)),
                                                 ("C3", 20000, 4096, 4608, {})])
def test_count_accumulations_equals_oracle(W, orc, name, n, row0, row1, kw):
    """wasabi_count_accumulations == the number of in-window accumulations the oracle's Eq.(2)
    performs on the full-width band (orc_wasabi_window's count), exactly; the row-work estimate sums
    to the full-hologram count."""
    import torch
    cfg = CONFIGS[name]
    pts = make_points(cfg, n=n)
    p = gpu_params(cfg, **kw)
    t = _tables(W, p)
    d = torch.from_numpy(pts).cuda()
    s8 = torch.zeros(8, dtype=torch.uint8, device="cuda")
    got = W.count_accumulations(p, t, d, row0, row1, s8)
    P = orc_params(orc, cfg, **kw)
    _, cnt = orc.Lut(P).wasabi_window(pts, 0, row0, cfg.n_h, row1 - row0)
    assert got == cnt
    rw = torch.empty(cfg.n_h + 1, dtype=torch.float64, device="cuda")
    W.row_work(p, t, d, rw, s8)
    full = W.count_accumulations(p, t, d, 0, cfg.n_h, s8)
    assert abs(float(rw[:cfg.n_h].sum()) - full) <= 1e-6 * full


def test_psf_bins_contain_reach_bins(W):
    """Bins by the PSF disc (wasabi_bin_points_psf) list, per tile, a superset of the reach bins
    (R-A19: the kept coefficients of a depth lie inside its PSF's Haar blocks), in ascending order."""
    import torch
    cfg = CONFIGS["C2"]
    pts = make_points(cfg, n=3000)
    p = gpu_params(cfg)
    t = _tables(W, p)
    d = torch.from_numpy(pts).cuda()
    b1 = torch.empty(W.bin_points_bytes(p, len(pts), 0, 2048), dtype=torch.uint8, device="cuda")
    b2 = torch.empty_like(b1)
    W.bin_points(p, t, d, 0, 2048, b1)
    W.bin_points_psf(p, t, d, 0, 2048, b2)
    torch.cuda.synchronize()
    p1, i1 = W.export_bins(p, b1)
    p2, i2 = W.export_bins(p, b2)
    for k in range(len(p1) - 1):
        a, b = i1[p1[k]:p1[k + 1]], i2[p2[k]:p2[k + 1]]
        assert np.all(np.diff(b) > 0)
        assert np.all(np.isin(a, b))


# ---------------------------------------------------------------- exact Eq.(1) (D1) on the GPU
@pytest.mark.parametrize("name,n,row0,row1,x0,w", [("C1", None, 0, 512, 0, 512), ("C2", 1500, 512, 768, 0, 2048),
                                                  ("C5", 10_000, 8192, 8256, 7680, 512),
                                                  ("C4", 200_000, 32768, 32832, 32768, 256)])
def test_direct_exact_equals_oracle_d1(W, orc, name, n, row0, row1, x0, w):
    """wasabi_direct_exact (continuous x, y, z) == the oracle's D1 on the same points,
    element-wise within 1e-5 of max|u| and in rel L2 (fp64 window test and distance, fp32 phase split)."""
    import torch
    cfg = CONFIGS[name]
    pts = make_points(cfg, n=n)
    p = gpu_params(cfg)
    t = _tables(W, p)
    d = torch.from_numpy(pts).cuda()
    bins = torch.empty(W.bin_points_bytes(p, len(pts), row0, row1), dtype=torch.uint8, device="cuda")
    W.bin_points_psf(p, t, d, row0, row1, bins)
    u = torch.empty((row1 - row0, p.n_h, 2), dtype=torch.float32, device="cuda")
    W.direct_exact(p, d, bins, row0, row1, u)
    torch.cuda.synchronize()
    P = orc_params(orc, cfg)
    sel = np.abs(pts[:, 1] / cfg.pitch + cfg.n_h // 2 - (row0 + row1) / 2) < (row1 - row0) / 2 + 800
    d1 = orc.direct_d1(P, pts[sel].astype(np.float64), x0, row0, w, row1 - row0)
    e, m = field_check(field_np(u)[:, x0:x0 + w], d1)
    parity_log(dict(case=f"D1 {name} rows [{row0},{row1}) x [{x0},{x0 + w})", rel_u=e, max_u=m))
    assert np.linalg.norm(d1) > 0
    assert e <= 1e-5 and m <= 1e-5, (e, m)
