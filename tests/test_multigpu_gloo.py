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

from paper_1708_04233_b200.distributed import assemble_bits, band_of, checksums, gather_checksums


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


def _worker(rank, world, port, out_q):
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
    r0, r1 = band_of(rank, world, cfg.n_h, cfg.tile)
    u, _, _ = O.Lut(P).hologram_window(pts, 0, r0, cfg.n_h, r1 - r0)     # band compute (oracle)
    bits, _ = O.quantize(P, (0.0, 0.030, -0.400), u, 0, r0)
    tb = torch.from_numpy(bits)
    tu = torch.from_numpy(np.stack([u.real, u.imag], -1))
    full = assemble_bits(tb, cfg.n_h, cfg.tile)
    cs = gather_checksums(checksums(tu, tb))
    if rank == 0:
        out_q.put((full.numpy(), cs.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_assembly_equals_single_band(world, orc):
    from inputs import CONFIGS, make_points
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, cs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    cfg = CONFIGS["C1"]
    P = orc.Params.from_config(cfg)
    pts = make_points(cfg, n=400)
    u, _, _ = orc.Lut(P).hologram_window(pts, 0, 0, cfg.n_h, cfg.n_h)
    bits, _ = orc.quantize(P, (0.0, 0.030, -0.400), u, 0, 0)
    assert np.array_equal(full, bits)
    ref = checksums(torch.from_numpy(np.stack([u.real, u.imag], -1)), torch.from_numpy(bits)).numpy()
    np.testing.assert_allclose(cs.sum(axis=0), ref, rtol=1e-12, atol=1e-9)
