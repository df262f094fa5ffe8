"""Row-band sharding across ranks (PAPER.md:115-125's sub-holograms, reduced to 2^L-aligned row bands).

Host logic only: which rows a rank computes, and the post-timing assembly of the print bits and of
per-band checksums with torch.distributed (NCCL over NVLink on GPUs; gloo in the CPU tests).  There
is no collective in the data path: bands are independent.
"""
from __future__ import annotations

from typing import List, Optional, Tuple


def band_of(rank: int, world: int, n_h: int, align: int) -> Tuple[int, int]:
    """Rows [row0, row1) of `rank`: equal bands whose edges are multiples of `align` (tile, 2^L).
    The remainder of rows (if n_h/align is not divisible by world) goes to the last ranks, one
    aligned block each, so every band stays aligned."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if n_h % align:
        raise ValueError("n_h must be a multiple of align")
    blocks = n_h // align
    base, extra = divmod(blocks, world)
    first_big = world - extra
    start = rank * base + max(0, rank - first_big)
    count = base + (1 if rank >= first_big else 0)
    return start * align, (start + count) * align


def balanced_bands(row_work, world: int, align: int) -> List[Tuple[int, int]]:
    """Work-balanced row bands (SURVEY.md §8(e) load balance; PAPER.md:115-125 sub-holograms): edges
    are multiples of `align` (tile, 2^L) chosen so each band's share of sum(row_work) is as close as
    possible to total/world.  `row_work` is the per-row work estimate of wasabi_row_work (length
    n_h).  Edge k is the aligned row nearest to the row where the work prefix reaches k/world of the
    total, kept strictly increasing (every band at least one aligned block).  Host logic only."""
    import numpy as np
    w = np.asarray(row_work, dtype=np.float64)
    n_h = w.shape[0]
    if world < 1 or n_h % align or n_h // align < world:
        raise ValueError("bad world / align for balanced bands")
    blocks = n_h // align
    cum = np.concatenate([[0.0], np.cumsum(w.reshape(blocks, align).sum(axis=1))])   # work before block b
    tot = cum[-1]
    edges = [0]
    for k in range(1, world):
        if tot > 0:
            b = int(np.searchsorted(cum, tot * k / world))
            b = b if b == 0 or abs(cum[b] - tot * k / world) <= abs(cum[b - 1] - tot * k / world) else b - 1
        else:
            b = round(blocks * k / world)
        b = min(max(b, edges[-1] + 1), blocks - (world - k))
        edges.append(b)
    edges.append(blocks)
    return [(edges[r] * align, edges[r + 1] * align) for r in range(world)]


def band_work(row_work, bands) -> List[float]:
    """Sum of the per-row work estimate over each band."""
    import numpy as np
    w = np.asarray(row_work, dtype=np.float64)
    return [float(w[b0:b1].sum()) for b0, b1 in bands]


def checksums(u, bits):
    """Per-band checksum vector: [sum |u|^2, sum Re u, sum Im u, set bits] (float64, same device)."""
    import torch
    dev = bits.device if bits is not None else u.device
    out = torch.zeros(4, dtype=torch.float64, device=dev)
    step = 1 << 24    # chunked: never materialise a float64 copy of a whole band
    if u is not None:
        uf = u.reshape(-1, 2)
        for i in range(0, uf.shape[0], step):
            uu = uf[i:i + step].double()
            out[0] += (uu * uu).sum()
            out[1] += uu[:, 0].sum()
            out[2] += uu[:, 1].sum()
    if bits is not None:
        table = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.float64, device=dev)
        bf = bits.reshape(-1)
        for i in range(0, bf.shape[0], step):
            out[3] += table[bf[i:i + step].long()].sum()
    return out


def gather_checksums(local, group=None):
    """all_gather of the per-band checksum vectors -> (world, 4)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [torch.zeros_like(local) for _ in range(world)]
    dist.all_gather(parts, local, group=group)
    return torch.stack(parts)


def assemble_bits(local_bits, n_h: int, align: int, group=None, bands: Optional[List[Tuple[int, int]]] = None):
    """Gather every rank's band of print bits into the full (n_h, n_h/8) pattern (all ranks get it).
    `bands` (default: the equal bands of band_of) lists every rank's [row0, row1); bands may differ
    in height, so each is padded to the largest band for the collective."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if bands is None:
        bands = [band_of(r, world, n_h, align) for r in range(world)]
    hmax = max(b1 - b0 for b0, b1 in bands)
    pad = torch.zeros((hmax, n_h // 8), dtype=torch.uint8, device=local_bits.device)
    pad[: local_bits.shape[0]] = local_bits
    parts = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[: b1 - b0] for p, (b0, b1) in zip(parts, bands)])
