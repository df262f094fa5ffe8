"""Pipeline: owns the device buffers of one band and runs steps 1-4 on one CUDA stream.

Marshalling and buffer management only (torch allocates; the C ABI computes).
"""
from __future__ import annotations

from typing import Optional

from . import (Params, PrintParams, bin_points, bin_points_bytes, build_psf_tables, inverse_wt,
               psf_tables_bytes, quantize, superpose, superpose_inverse)


class Pipeline:
    """Device buffers for band [row0, row1) of a hologram with params `p` and up to n_max points.

    run(points) executes: build tables (step 1) -> bin (2a) -> fused superpose + inverse + quantise
    (2b-4, psi never leaves shared memory); run(points, fused=False) runs the unfused four-call path
    (superpose writes psi, the inverse overwrites it in place with u).
    """

    def __init__(self, p: Params, n_max: int, row0: int = 0, row1: Optional[int] = None, device=None,
                 want_u: bool = True, want_bits: bool = True, print_params: Optional[PrintParams] = None,
                 stream=None):
        import torch
        self.torch = torch
        self.p = p
        self.row0 = row0
        self.row1 = p.n_h if row1 is None else row1
        self.device = torch.device(device if device is not None else "cuda")
        self.n_max = n_max
        self.print_params = print_params if print_params is not None else PrintParams()
        tb, sb = psf_tables_bytes(p)
        self.tables = torch.empty(tb, dtype=torch.uint8, device=self.device)
        self.scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
        # psi band: the band itself, or (coiflets, R-A21) the band grown by the inverse's halo rows
        h = p.halo_rows()
        self.e0, self.e1 = max(0, self.row0 - h), min(p.n_h, self.row1 + h)
        self.bins = torch.empty(bin_points_bytes(p, n_max, self.e0, self.e1), dtype=torch.uint8,
                                device=self.device)
        rows = self.row1 - self.row0
        if p.wavelet == 0:
            self.psi_band = self.field = torch.empty((rows, p.n_h, 2), dtype=torch.float32, device=self.device)
        else:
            # coiflets: psi on the halo band; u in its own buffer, so wasabi_inverse_wt runs the fused tile
            # synthesis (psi only read).  Print only (want_u False): field is a view of psi's band rows.
            self.psi_band = torch.empty((self.e1 - self.e0, p.n_h, 2), dtype=torch.float32, device=self.device)
            self.field = (torch.empty((rows, p.n_h, 2), dtype=torch.float32, device=self.device) if want_u
                          else self.psi_band[self.row0 - self.e0:self.row1 - self.e0])
        self.bits = torch.empty((rows, p.n_h // 8), dtype=torch.uint8, device=self.device) if want_bits else None
        self.want_u = want_u
        self.stream = stream
        self.tables_built = False

    def nbytes(self) -> int:
        t = self.tables.numel() + self.scratch.numel() + self.bins.numel() + self.field.numel() * 4
        return t + (self.bits.numel() if self.bits is not None else 0)

    # individual steps (all asynchronous on the stream)
    def build_tables(self):
        build_psf_tables(self.p, self.tables, self.scratch, self.stream)
        self.tables_built = True

    def bin(self, points):
        bin_points(self.p, self.tables, points, self.e0, self.e1, self.bins, self.stream)

    def superpose(self):
        """psi on the psi band (self.psi_band; == self.field unless coiflets)."""
        superpose(self.p, self.tables, self.bins, self.e0, self.e1, self.psi_band, self.stream)

    def inverse(self, fuse_bits: bool = True):
        bits = self.bits if (fuse_bits and self.bits is not None) else None
        u = self.field if self.want_u else None
        inverse_wt(self.p, self.psi_band, u, self.row0, self.row1, self.print_params, bits, self.stream)

    def quantize(self):
        quantize(self.p, self.print_params, self.field, self.row0, self.row1, self.bits, self.stream)

    def superpose_inverse(self):
        u = self.field if self.want_u else None
        superpose_inverse(self.p, self.tables, self.bins, self.row0, self.row1, self.print_params, u, self.bits,
                          self.stream)

    def run(self, points, build_tables: bool = True, fused: bool = True):
        if build_tables or not self.tables_built:
            self.build_tables()
        self.bin(points)
        if fused and self.p.wavelet == 0:
            self.superpose_inverse()
        else:
            self.superpose()
            self.inverse()
        return self.field, self.bits

    def capture(self, points, build_tables: bool = True, fused: bool = True):
        """Record one step (run(points, ...)) into a CUDA graph; replay() then re-launches the whole
        step with one call (no per-kernel launch overhead: ~0.08 ms per step at C1-C3).  The graph
        reads `points` in place, so new point data copied into the same tensor (same n) is picked up
        by the next replay.  Every C-ABI call is capturable (no host synchronisation inside); one
        eager step first settles the host-side geometry cache and the kernels' attributes."""
        torch = self.torch
        stream = self.stream if self.stream is not None else torch.cuda.Stream(self.device)
        saved = self.stream
        self.stream = stream
        try:
            stream.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(stream):
                self.run(points, build_tables=build_tables, fused=fused)
            stream.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                self.run(points, build_tables=build_tables, fused=fused)
        finally:
            self.stream = saved
        self._graph = graph
        return graph

    def replay(self):
        """Re-run the captured step (capture() first); ordered after the current stream's work."""
        self._graph.replay()
        return self.field, self.bits


class HologramStream:
    """Band-by-band generation of a print pattern with buffers for one band only -- the paper's
    sub-hologram division "to reduce the memory usage", so the hologram may be
    far larger than device memory: the tables are built once, then each 2^L-aligned band of
    `band_rows` rows is binned and run through the fused superpose/inverse/quantise kernel in
    print-only mode, and its bits are copied to the host.  `run(points)` yields (row0, bits) with
    bits a (rows, n_h // 8) uint8 numpy array; concatenated they equal the full hologram's bits
    bit for bit (R-A11: bands are independent).  Haar mode only (coiflets need psi halos)."""

    def __init__(self, p: Params, n_max: int, band_rows: int, device=None,
                 print_params: Optional[PrintParams] = None, stream=None):
        import torch
        if p.wavelet != 0:
            raise ValueError("HologramStream: the coiflet inverse needs psi halos; use Pipeline per band")
        if band_rows % p.tile or band_rows <= 0:
            raise ValueError("band_rows must be a positive multiple of the tile")
        self.torch, self.p, self.band_rows, self.stream = torch, p, band_rows, stream
        self.device = torch.device(device if device is not None else "cuda")
        self.print_params = print_params if print_params is not None else PrintParams()
        tb, sb = psf_tables_bytes(p)
        self.tables = torch.empty(tb, dtype=torch.uint8, device=self.device)
        self.scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
        self.bins = torch.empty(bin_points_bytes(p, n_max, 0, band_rows), dtype=torch.uint8, device=self.device)
        self.bits = torch.empty((band_rows, p.n_h // 8), dtype=torch.uint8, device=self.device)
        self.h_bits = torch.empty((band_rows, p.n_h // 8), dtype=torch.uint8).pin_memory()

    def run(self, points):
        torch = self.torch
        build_psf_tables(self.p, self.tables, self.scratch, self.stream)
        for row0 in range(0, self.p.n_h, self.band_rows):
            row1 = min(self.p.n_h, row0 + self.band_rows)
            rows = row1 - row0
            bin_points(self.p, self.tables, points, row0, row1, self.bins, self.stream)
            superpose_inverse(self.p, self.tables, self.bins, row0, row1, self.print_params, None,
                              self.bits[:rows], self.stream)
            # the D2H copy runs on the stream that ran the kernel (ordered after it), and that stream
            # is synchronised before the host reads h_bits and before the next band reuses self.bits
            s = self.stream if self.stream is not None else torch.cuda.current_stream(self.device)
            with torch.cuda.stream(s):
                self.h_bits[:rows].copy_(self.bits[:rows], non_blocking=True)
            s.synchronize()
            yield row0, self.h_bits[:rows].numpy().copy()
