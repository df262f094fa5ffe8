"""CPU tests of libwasabi: the library loads, exports every symbol include/wasabi.h declares, its
host-side geometry (L0) equals the oracle's independent computation exactly, and parameter
validation rejects what the header says it rejects.  No compute calls (no GPU here)."""
import os
import re

import numpy as np
import pytest

from inputs import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def W():
    import __graft_entry__
    __graft_entry__.build_library()
    import paper_1708_04233_b200 as W
    return W


def test_exports_every_declared_symbol(W):
    import ctypes
    hdr = open(os.path.join(ROOT, "include", "wasabi.h")).read()
    names = sorted(set(re.findall(r"\b(wasabi_[a-z_0-9]+)\s*\(", hdr)))
    assert len(names) >= 16
    lib = ctypes.CDLL(W.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert "sm_100a" in W.version()


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_host_geometry_equals_oracle(W, orc, name):
    cfg = CONFIGS[name]
    p = W.Params.from_config(cfg)
    P = orc.Params.from_config(cfg)
    g = orc.geometry(P)
    for d in range(cfg.n_depth):
        h = W.depth_geometry(p, d)
        assert h["z"] == g["z"][d] and h["R"] == g["R"][d]
        assert (h["H"], h["E"], h["nnz"], h["n_r"]) == (g["H"][d], g["E"][d], g["nnz"][d], g["n_r"][d])


def test_host_geometry_equals_oracle_c4_sample(W, orc):
    cfg = CONFIGS["C4"]
    p = W.Params.from_config(cfg)
    P = orc.Params.from_config(cfg)
    for d in (0, 1, 40, 63, 64, 90, 127):
        h = W.depth_geometry(p, d)
        o = orc.geometry_one(P, d)
        assert h["z"] == o["z"] and h["R"] == o["R"]
        assert (h["H"], h["E"], h["nnz"], h["n_r"]) == (o["H"], o["E"], o["nnz"], o["n_r"])


@pytest.mark.parametrize("r", [0.01, 0.05, 0.1, 0.25, 1.0])
def test_host_n_r_all_retentions(W, orc, r):
    cfg = CONFIGS["C2"]
    p = W.Params.from_config(cfg, retention=r)
    P = orc.Params.from_config(cfg.replace(retention=r))
    g = orc.geometry(P)
    for d in (0, 11, 31):
        assert W.depth_geometry(p, d)["n_r"] == g["n_r"][d]


def test_sizes_are_host_only(W):
    p = W.Params.from_config(CONFIGS["C4"])
    tb, sb = W.psf_tables_bytes(p)
    assert 30e6 < tb < 1.5e9 and sb > 0   # canonical LUT + window LUT (capacity 16 N_r)
    bb = W.bin_points_bytes(p, 2_000_000, 0, p.n_h)
    assert bb > 2_000_000 * 16
    wb = W.hologram_workspace_bytes(p, 2_000_000, 0, 8192)
    assert wb > 8192 * 65536 * 8


@pytest.mark.parametrize("kw,msg", [
    (dict(wavelength=2.1e-6), "Nyquist"),
    (dict(tile=96), "tile"),
    (dict(tile=256), "tile"),
    (dict(n_h=1000), "multiple of tile"),
    (dict(retention=0.0), "retention"),
    (dict(retention=1.5), "retention"),
    (dict(levels=7), "levels"),
    (dict(levels=0), "levels"),
    (dict(n_depth=0), "n_depth"),
    (dict(z_min=1e-3, z_max=0.5e-3), "z_min"),
    (dict(z_min=-0.03, z_max=0.03), "exceeds"),
])
def test_validation_rejects(W, kw, msg):
    p = W.Params.from_config(CONFIGS["C1"], **kw)
    with pytest.raises(W.WasabiError) as e:
        W.psf_tables_bytes(p)
    assert e.value.status == W.WASABI_EINVAL
    assert msg in str(e.value)


def test_band_validation(W):
    p = W.Params.from_config(CONFIGS["C1"])
    for r0, r1 in [(0, 100), (32, 128), (-64, 64), (0, 1024), (128, 64)]:
        with pytest.raises(W.WasabiError):
            W.bin_points_bytes(p, 10, r0, r1)
    assert W.bin_points_bytes(p, 0, 64, 64) > 0   # empty band is legal


def test_no_cpu_fallback_without_gpu(W):
    """The product path must fail loudly without a GPU (no silent CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = W.Params.from_config(CONFIGS["C1"])
    tb, sb = W.psf_tables_bytes(p)
    t = np.zeros(tb, np.uint8)
    s = np.zeros(sb, np.uint8)
    with pytest.raises(Exception):
        W.build_psf_tables(p, t, s, stream=0)


@pytest.mark.parametrize("name,kw", [("C1", {}), ("C2", dict(levels=3)), ("C1", dict(levels=1))])
def test_coif_host_geometry_equals_oracle(W, orc, name, kw):
    """WASABI_FLAG_COIFLET (R-A21): the library's padded table half side, structural nnz (footprint
    rule, written independently in C++) and N_r equal the oracle's for every depth."""
    cfg = CONFIGS[name].replace(**kw)
    p = W.Params.from_config(cfg, wavelet=1)
    P = orc.Params.from_config(cfg, wavelet=1)
    for d in range(cfg.n_depth):
        g, o = W.depth_geometry(p, d), orc.table_info(P, d)
        assert (g["H"], g["nnz"], g["n_r"]) == (o["H"], o["nnz"], o["n_r"]), d
    assert p.halo_rows() == max(64, p.tile)


@pytest.mark.parametrize("kw,msg", [(dict(levels=5), "levels <= 4"), (dict(exact=True), "EXACT_SHIFT")])
def test_coif_mode_validation(W, kw, msg):
    p = W.Params.from_config(CONFIGS["C3"].replace(levels=3), wavelet=1, **kw)
    with pytest.raises(W.WasabiError, match=msg):
        W.psf_tables_bytes(p)


@pytest.mark.parametrize("kw,msg", [(dict(path="gather", tile=128), "tile 64"),
                                    (dict(path="gather", levels=1), "levels >= 2"),
                                    (dict(path="gather", wavelet=1, levels=3), "Haar")])
def test_gather_mode_validation(W, kw, msg):
    p = W.Params.from_config(CONFIGS["C1"].replace(retention=1.0), **kw)
    with pytest.raises(W.WasabiError, match=msg):
        W.psf_tables_bytes(p)


def test_gather_tables_replace_window_lut(W):
    """WASABI_FLAG_GATHER: the table buffer holds the dense wavelet tables (sum of side^2 complex64)
    instead of the window LUT; auto selects the gather at r >= 0.25 only."""
    cfg = CONFIGS["C5"].replace(retention=1.0, levels=5)
    tg, _ = W.psf_tables_bytes(W.Params.from_config(cfg, path="gather"))
    ts, _ = W.psf_tables_bytes(W.Params.from_config(cfg, path="scatter"))
    ta, _ = W.psf_tables_bytes(W.Params.from_config(cfg))
    side2 = sum((2 * W.depth_geometry(W.Params.from_config(cfg), d)["H"]) ** 2 for d in range(cfg.n_depth))
    assert ta == tg and tg != ts
    assert tg >= 8 * side2
    t5, _ = W.psf_tables_bytes(W.Params.from_config(cfg.replace(retention=0.2)))
    t5s, _ = W.psf_tables_bytes(W.Params.from_config(cfg.replace(retention=0.2), path="scatter"))
    assert t5 == t5s


def test_coif_paper_scale_accepted(W):
    """The coiflet mode at the paper's scale (PAPER.md:106 level 3, :128 65,536^2): the line synthesis
    streams rolling windows along rows and columns, so N_h is not capped."""
    p = W.Params.from_config(CONFIGS["C4"].replace(levels=3), wavelet=1)
    tb, sb = W.psf_tables_bytes(p)
    assert tb > 0 and sb > 0 and p.halo_rows() == 64
