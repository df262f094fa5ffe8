"""World-size-2 CPU test (gloo) of the row-band sharding host logic: band partition, assembly of the
print bits and checksums.  The band compute here is the fp64 oracle (test infrastructure) so the
test runs without a GPU; on GPUs bench.py uses the same helpers with NCCL after the timed region."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1708_04233_b200.distributed import (assemble_bits, balanced_bands, band_of, band_work, checksums,
                                               gather_checksums)


def test_band_partition_properties():
    for n_h, align in [(512, 64), (65536, 64), (2048, 128), (8192, 64)]:
        for world in (1, 2, 3, 4, 8):
            if n_h // align < world:
                continue
            bands = [band_of(r, world, n_h, align) for r in range(world)]
            assert bands[0][0] == 0 and bands[-1][1] == n_h
            for (a0, a1), (b0, b1) in zip(bands, bands[1:]):
                assert a1 == b0
            for b0, b1 in bands:
                assert b0 % align == 0 and b1 % align == 0 and b1 > b0
            sizes = [b1 - b0 for b0, b1 in bands]
            assert max(sizes) - min(sizes) <= align
    assert band_of(3, 8, 65536, 64) == (3 * 8192, 4 * 8192)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_row_work(orc, P, pts):
    """Host-side stand-in for wasabi_row_work (test only): each valid point's kept-list size spread
    uniformly over its reach rows [iy - ek, iy + ek] (R-A19), from the oracle's points and reach."""
    ix, iy, iz, ok = orc.points(P, pts)
    ek, _ = orc.reach(P)
    nr = orc.geometry(P)["n_r"]
    diff = np.zeros(P.n_h + 1)
    for y, d, v in zip(iy, iz, ok):
        if not v:
            continue
        y0, y1 = max(0, y - ek[d]), min(P.n_h - 1, y + ek[d])
        if y1 >= y0:
            diff[y0] += nr[d] / (y1 - y0 + 1)
            diff[y1 + 1] -= nr[d] / (y1 - y0 + 1)
    return np.cumsum(diff)[:P.n_h]


def test_balanced_bands_properties():
    """Balanced bands tile [0, N_h) with aligned, strictly increasing edges, and even out a skewed
    work profile far better than equal bands."""
    rng = np.random.default_rng(3)
    for n_h, align, world in [(512, 64, 2), (512, 64, 4), (65536, 64, 8), (2048, 128, 3), (8192, 64, 8)]:
        w = rng.random(n_h) ** 4 * 10
        w[: n_h // 8] *= 20                      # a dense top strip
        bands = balanced_bands(w, world, align)
        assert bands[0][0] == 0 and bands[-1][1] == n_h
        for (a0, a1), (b0, b1) in zip(bands, bands[1:]):
            assert a1 == b0
        for b0, b1 in bands:
            assert b0 % align == 0 and b1 % align == 0 and b1 > b0
        if n_h // align >= 8 * world:
            bw, ew = band_work(w, bands), band_work(w, [band_of(r, world, n_h, align) for r in range(world)])
            assert max(bw) / np.mean(bw) < max(ew) / np.mean(ew)
    assert balanced_bands(np.zeros(512), 2, 64) == [(0, 256), (256, 512)]
    assert balanced_bands(np.ones(512), 8, 64) == [(64 * r, 64 * (r + 1)) for r in range(8)]


def _worker(rank, world, port, bands, out_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from inputs import CONFIGS, make_points
    from oracle import oracle as O
    cfg = CONFIGS["C1"]
    P = O.Params.from_config(cfg)
    pts = make_points(cfg, n=400)
    r0, r1 = bands[rank]
    u, _, _ = O.Lut(P).hologram_window(pts, 0, r0, cfg.n_h, r1 - r0)     # band compute (oracle)
    bits, _ = O.quantize(P, (0.0, 0.030, -0.400), u, 0, r0)
    tb = torch.from_numpy(bits)
    tu = torch.from_numpy(np.stack([u.real, u.imag], -1))
    full = assemble_bits(tb, cfg.n_h, cfg.tile, bands=bands)
    cs = gather_checksums(checksums(tu, tb))
    if rank == 0:
        out_q.put((full.numpy(), cs.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "equal"), (2, "balanced"), (4, "balanced")])
def test_rank_assembly_equals_single_band(world, kind, orc):
    """world-2/4 gloo: every rank computes its band (equal, or work-balanced from the row-work
    estimate); the assembled print bits equal the single-band hologram bit for bit, and the band
    checksums add up to the single band's."""
    from inputs import CONFIGS, make_points
    cfg = CONFIGS["C1"]
    P = orc.Params.from_config(cfg)
    pts = make_points(cfg, n=400)
    if kind == "equal":
        bands = [band_of(r, world, cfg.n_h, cfg.tile) for r in range(world)]
    else:
        bands = balanced_bands(_oracle_row_work(orc, P, pts), world, cfg.tile)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, bands, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, cs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    u, _, _ = orc.Lut(P).hologram_window(pts, 0, 0, cfg.n_h, cfg.n_h)
    bits, _ = orc.quantize(P, (0.0, 0.030, -0.400), u, 0, 0)
    assert np.array_equal(full, bits)
    ref = checksums(torch.from_numpy(np.stack([u.real, u.imag], -1)), torch.from_numpy(bits)).numpy()
    np.testing.assert_allclose(cs.sum(axis=0), ref, rtol=1e-12, atol=1e-9)
