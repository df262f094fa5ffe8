"""Randomised GPU parity sweep: seeded random small problems (wavelength, pitch, N_h, depth range
and count, L, r, tile, point count and placement including points off the aperture, on the
hologram edge, on depth-level boundaries, with a <= 0 or non-finite coordinates), each in all three
table modes where valid (Haar R-A8, exact shifts R-A20, coif1 R-A21), through the C ABI against
the fp64 oracle: bins bit-exact, psi and u within 1e-5 rel L2, print bits identical outside the
threshold band (R-A16).  The window LUT (variants, bands, column groups) and the shared-tile
margins see table sides that are not multiples of 32 or 64, odd level counts and both tile sizes."""
import os

import numpy as np
import pytest

from helpers import REF, bits_check, field_check, field_np, parity_log, rel_l2
from test_gpu_parity import W  # noqa: F401

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    L = int(rng.integers(1, 5))
    tile = int(rng.choice([64, 128]))
    n_h = tile * int(rng.integers(2, 7))
    lam = float(rng.uniform(450e-9, 700e-9))
    pitch = float(rng.choice([0.8e-6, 1e-6, 1.6e-6]))
    n_depth = int(rng.integers(1, 7))
    z0 = float(rng.uniform(0.03e-3, 0.15e-3)) * rng.choice([-1, 1])
    z1 = z0 + float(rng.uniform(0.02e-3, 0.2e-3)) if n_depth > 1 else z0
    r = float(rng.choice([0.01, 0.05, 0.3, 1.0]))
    n = int(rng.integers(0, 60))
    A = n_h * pitch
    pts = np.zeros((n, 4), np.float32)
    pts[:, 0] = rng.uniform(-0.6 * A, 0.6 * A, n)
    pts[:, 1] = rng.uniform(-0.6 * A, 0.6 * A, n)
    dz = (z1 - z0) / (n_depth - 1) if n_depth > 1 else 0.0
    k = rng.integers(0, n_depth, n)
    pts[:, 2] = z0 + k * dz + (rng.choice([-0.5, 0.0, 0.25, 0.5], n) * dz if n_depth > 1 else 0.0)
    pts[:, 3] = rng.uniform(-0.2, 1.0, n)
    if n >= 4:
        pts[0, 0] = -A / 2                       # hologram edge
        pts[1, 1] = (A / 2) - pitch / 2
        pts[2, 0] = np.nan                       # skipped
        pts[3, 3] = 0.0                          # skipped
    P = dict(wavelength=lam, pitch=pitch, n_h=n_h, n_depth=n_depth, levels=L, z_min=min(z0, z1),
             z_max=max(z0, z1), retention=r)
    return P, tile, pts, rng


# WASABI_RANDOM_SEEDS=<n> widens the sweep (the default run keeps 12 seeds per mode)
@pytest.mark.parametrize("seed", range(int(os.environ.get("WASABI_RANDOM_SEEDS", "12"))))
@pytest.mark.parametrize("mode", ["haar", "exact", "coif", "gather"])
def test_random_problem_parity(W, orc, seed, mode):
    import torch
    P, tile, pts, rng = _case(seed)
    kw = dict(exact=(mode == "exact"), wavelet=1 if mode == "coif" else 0)
    gkw = {}
    if mode == "gather":   # the dense gather superposition (WASABI_FLAG_GATHER: tile 64, L >= 2, Haar)
        tile, P["levels"] = 64, max(2, P["levels"])
        gkw = dict(path="gather")
    p = W.Params(P["wavelength"], P["pitch"], P["n_h"], P["n_depth"], P["levels"], P["z_min"], P["z_max"],
                 P["retention"], tile, **kw, **gkw)
    Po = orc.Params(**P, **kw)
    nb = P["n_h"] // tile
    t0 = int(rng.integers(0, nb))
    t1 = int(rng.integers(t0 + 1, nb + 1))
    row0, row1 = t0 * tile, t1 * tile
    pl = W.Pipeline(p, max(1, len(pts)), row0, row1)
    d = torch.from_numpy(np.ascontiguousarray(pts)).cuda() if len(pts) else torch.zeros((1, 4), device="cuda")
    pl.build_tables()
    pl.bin(d[:len(pts)])
    pl.superpose()
    psi_g = field_np(pl.psi_band[row0 - pl.e0:row1 - pl.e0])   # == pl.field unless coiflets (halo band)
    pl.inverse()
    torch.cuda.synchronize()
    u_g = field_np(pl.field)
    bits_g = pl.bits.cpu().numpy()
    # bins of the psi band (the band itself, or its coiflet halo band)
    ptr_g, idx_g = W.export_bins(p, pl.bins)
    ptr_o, idx_o = orc.bins(Po, tile, pts.astype(np.float64), pl.e0, pl.e1)
    assert np.array_equal(ptr_g, ptr_o) and np.array_equal(idx_g, idx_o)
    u_o, psi_o, _ = orc.Lut(Po).hologram_window(pts.astype(np.float64), 0, row0, P["n_h"], row1 - row0)
    if np.linalg.norm(psi_o) == 0:
        assert np.linalg.norm(psi_g) == 0 and np.linalg.norm(u_g) == 0
        return
    assert rel_l2(psi_g, psi_o) <= 1e-5
    assert rel_l2(u_g, u_o) <= 1e-5
    e_u, m_u = field_check(u_g, u_o)
    assert m_u <= 1e-5 and field_check(psi_g, psi_o)[1] <= 1e-5
    bits_o, I_o = orc.quantize(Po, REF, u_o, 0, row0)
    bc = bits_check(bits_g, bits_o, I_o, u_g, u_o)
    parity_log(dict(case=f"random {mode} seed {seed}", rel_u=e_u, max_u=m_u, **bc))
    assert bc["bad"] == 0, bc
    if mode != "coif":
        # the fused entry point (wasabi_superpose_inverse) equals the unfused path bit for bit
        u_f = torch.zeros_like(pl.field)
        b_f = torch.zeros_like(pl.bits)
        W.superpose_inverse(p, pl.tables, pl.bins, row0, row1, pl.print_params, u_f, b_f)
        torch.cuda.synchronize()
        assert torch.equal(u_f, pl.field) and torch.equal(b_f, pl.bits)
