"""B200-native WASABI hot path (arXiv 1708.04233) -- thin Python binding of libwasabi.so.

Argument marshalling only: every step of the path runs in the sm_100a kernels behind the C ABI
declared in include/wasabi.h.  PyTorch supplies device memory and streams.  There is no CPU
fallback: if libwasabi.so is missing or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwasabi.so")

WASABI_OK, WASABI_EINVAL, WASABI_ENOSPC, WASABI_ECUDA, WASABI_ESTATE = 0, -1, -2, -3, -4


FLAG_EXACT_SHIFT = 1   # include/wasabi.h WASABI_FLAG_EXACT_SHIFT
FLAG_COIFLET = 2       # include/wasabi.h WASABI_FLAG_COIFLET
FLAG_GATHER = 4        # include/wasabi.h WASABI_FLAG_GATHER (dense gather superposition)
FLAG_SCATTER = 8       # include/wasabi.h WASABI_FLAG_SCATTER (window-LUT scatter superposition)


class WasabiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"wasabi status {status}: {msg}")
        self.status = status


class _CParams(C.Structure):
    _fields_ = [("wavelength_m", C.c_double), ("pitch_m", C.c_double), ("n_h", C.c_int64),
                ("n_depth", C.c_int32), ("levels", C.c_int32), ("z_min_m", C.c_double),
                ("z_max_m", C.c_double), ("retention", C.c_double), ("tile", C.c_int32),
                ("flags", C.c_uint32)]


class _CPrint(C.Structure):
    _fields_ = [("x_r_m", C.c_double), ("y_r_m", C.c_double), ("z_r_m", C.c_double)]


class _CDepthInfo(C.Structure):
    _fields_ = [("z_m", C.c_double), ("radius_px", C.c_double), ("half", C.c_int64),
                ("footprint", C.c_int64), ("nnz", C.c_int64), ("n_r", C.c_int64)]


@dataclasses.dataclass(frozen=True)
class Params:
    """wasabi_params: the paper's problem statement + GPU tile."""
    wavelength: float
    pitch: float
    n_h: int
    n_depth: int
    levels: int
    z_min: float
    z_max: float
    retention: float
    tile: int = 64
    exact: bool = False   # WASABI_FLAG_EXACT_SHIFT: offset-class tables (R-A20)
    wavelet: int = 0      # 0 Haar; 1 WASABI_FLAG_COIFLET: coif1, the paper's coiflets (R-A21, NEXT-2)
    path: str = "auto"    # superposition: "auto" (gather iff r >= 0.25), "gather" or "scatter" (wasabi.h)

    @staticmethod
    def from_config(cfg, **kw) -> "Params":
        p = Params(cfg.wavelength, cfg.pitch, cfg.n_h, cfg.n_depth, cfg.levels, cfg.z_min, cfg.z_max,
                   cfg.retention, cfg.tile)
        return dataclasses.replace(p, **kw) if kw else p

    def c(self) -> _CParams:
        return _CParams(self.wavelength, self.pitch, self.n_h, self.n_depth, self.levels, self.z_min,
                        self.z_max, self.retention, self.tile,
                        (FLAG_EXACT_SHIFT if self.exact else 0) | (FLAG_COIFLET if self.wavelet == 1 else 0)
                        | {"auto": 0, "gather": FLAG_GATHER, "scatter": FLAG_SCATTER}[self.path])

    def halo_rows(self) -> int:
        """psi rows the inverse needs beyond a band on each side (wasabi_coif_halo_rows)."""
        return int(lib().wasabi_coif_halo_rows(C.byref(self.c())))


@dataclasses.dataclass(frozen=True)
class PrintParams:
    """Spherical reference wave point."""
    x_r: float = 0.0
    y_r: float = 0.030
    z_r: float = -0.400

    def c(self) -> _CPrint:
        return _CPrint(self.x_r, self.y_r, self.z_r)


_lib = None
_vp = C.c_void_p
_sz = C.c_size_t
_i64 = C.c_int64
_PP = C.POINTER(_CParams)
_PR = C.POINTER(_CPrint)


def lib() -> C.CDLL:
    """Load libwasabi.so (fails loudly if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not found: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.wasabi_last_error.restype = C.c_char_p
        L.wasabi_version.restype = C.c_char_p
        L.wasabi_kernel_launches.restype = C.c_ulonglong
        L.wasabi_kernel_launches.argtypes = []
        L.wasabi_coif_halo_rows.restype = C.c_int64
        L.wasabi_coif_halo_rows.argtypes = [_PP]
        sig = {
            "wasabi_psf_tables_bytes": [_PP, C.POINTER(_sz), C.POINTER(_sz)],
            "wasabi_build_psf_tables": [_PP, _vp, _sz, _vp, _sz, _vp],
            "wasabi_depth_geometry": [_PP, C.c_int32, C.POINTER(_CDepthInfo)],
            "wasabi_table_count": [_PP, C.POINTER(_i64)],
            "wasabi_bin_points_bytes": [_PP, _i64, _i64, _i64, C.POINTER(_sz)],
            "wasabi_bin_points": [_PP, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp],
            "wasabi_bin_points_psf": [_PP, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp],
            "wasabi_superpose": [_PP, _vp, _vp, _i64, _i64, _vp, _vp],
            "wasabi_superpose_inverse": [_PP, _vp, _vp, _i64, _i64, _PR, _vp, _vp, _vp],
            "wasabi_inverse_wt": [_PP, _vp, _vp, _i64, _i64, _PR, _vp, _vp],
            "wasabi_quantize": [_PP, _PR, _vp, _i64, _i64, _vp, _vp],
            "wasabi_hologram_workspace_bytes": [_PP, _i64, _i64, _i64, C.POINTER(_sz)],
            "wasabi_hologram_host": [_PP, _PR, _vp, _i64, _i64, _i64, _vp, _sz, _vp, _vp, _vp],
            "wasabi_psf_dense_bytes": [_PP, C.POINTER(_sz)],
            "wasabi_build_psf_dense": [_PP, _vp, _sz, _vp],
            "wasabi_direct_sum": [_PP, _vp, _vp, _i64, _i64, _vp, _vp],
            "wasabi_direct_exact": [_PP, _vp, _i64, _vp, _i64, _i64, _vp, _vp],
            "wasabi_tables_check": [_PP, _vp],
            "wasabi_export_table": [_PP, _vp, C.c_int32, _vp, _vp, _vp, _vp, _i64, C.POINTER(_i64)],
            "wasabi_export_bins": [_PP, _vp, _vp, _vp, _i64, C.POINTER(_i64)],
            "wasabi_export_reach": [_PP, _vp, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)],
            "wasabi_bins_stats": [_vp, C.POINTER(_i64 * 8)],
            "wasabi_count_accumulations": [_PP, _vp, _vp, _i64, _i64, _i64, _vp, C.POINTER(_i64), _vp],
            "wasabi_row_work": [_PP, _vp, _vp, _i64, _vp, _vp, _vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        _lib = L
    return _lib


def _check(status: int):
    if status != WASABI_OK:
        raise WasabiError(status, lib().wasabi_last_error().decode())


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data  # numpy


def _nbytes(t) -> int:
    if hasattr(t, "element_size"):
        return t.numel() * t.element_size()
    return int(t.nbytes)


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def version() -> str:
    return lib().wasabi_version().decode()


def kernel_launches() -> int:
    """Number of kernels libwasabi has launched in this process."""
    return int(lib().wasabi_kernel_launches())


# ----------------------------------------------------------------------------- step 1
def psf_tables_bytes(p: Params):
    tb, sb = _sz(), _sz()
    _check(lib().wasabi_psf_tables_bytes(C.byref(p.c()), C.byref(tb), C.byref(sb)))
    return tb.value, sb.value


def build_psf_tables(p: Params, tables, scratch, stream=None):
    _check(lib().wasabi_build_psf_tables(C.byref(p.c()), _ptr(tables), _nbytes(tables), _ptr(scratch),
                                         _nbytes(scratch), _stream(stream)))


def depth_geometry(p: Params, depth: int) -> dict:
    o = _CDepthInfo()
    _check(lib().wasabi_depth_geometry(C.byref(p.c()), depth, C.byref(o)))
    return dict(z=o.z_m, R=o.radius_px, H=o.half, E=o.footprint, nnz=o.nnz, n_r=o.n_r)


def table_count(p: Params) -> int:
    n = _i64()
    _check(lib().wasabi_table_count(C.byref(p.c()), C.byref(n)))
    return int(n.value)


# ----------------------------------------------------------------------------- step 2a
def bin_points_bytes(p: Params, n: int, row0: int, row1: int) -> int:
    b = _sz()
    _check(lib().wasabi_bin_points_bytes(C.byref(p.c()), n, row0, row1, C.byref(b)))
    return b.value


def bin_points(p: Params, tables, points, row0: int, row1: int, bins, stream=None):
    n = points.shape[0] if points is not None else 0
    _check(lib().wasabi_bin_points(C.byref(p.c()), _ptr(tables), _ptr(points), n, row0, row1, _ptr(bins),
                                   _nbytes(bins), _stream(stream)))


# ----------------------------------------------------------------------------- step 2b
def superpose(p: Params, tables, bins, row0: int, row1: int, psi, stream=None):
    _check(lib().wasabi_superpose(C.byref(p.c()), _ptr(tables), _ptr(bins), row0, row1, _ptr(psi),
                                  _stream(stream)))


def superpose_inverse(p: Params, tables, bins, row0: int, row1: int, print_params: Optional[PrintParams], u,
                      bits=None, stream=None):
    """Steps 2b-4 fused: psi stays in shared memory; writes u (may be None) and bits (may be None)."""
    pr = C.byref(print_params.c()) if print_params is not None else None
    _check(lib().wasabi_superpose_inverse(C.byref(p.c()), _ptr(tables), _ptr(bins), row0, row1, pr, _ptr(u),
                                          _ptr(bits), _stream(stream)))


# ----------------------------------------------------------------------------- steps 3, 4
def inverse_wt(p: Params, psi, u, row0: int, row1: int, print_params: Optional[PrintParams] = None, bits=None,
               stream=None):
    pr = C.byref(print_params.c()) if print_params is not None else None
    _check(lib().wasabi_inverse_wt(C.byref(p.c()), _ptr(psi), _ptr(u), row0, row1, pr, _ptr(bits),
                                   _stream(stream)))


def quantize(p: Params, print_params: PrintParams, u, row0: int, row1: int, bits, stream=None):
    _check(lib().wasabi_quantize(C.byref(p.c()), C.byref(print_params.c()), _ptr(u), row0, row1, _ptr(bits),
                                 _stream(stream)))


# ----------------------------------------------------------------------------- conventional baseline
def psf_dense_bytes(p: Params) -> int:
    b = _sz()
    _check(lib().wasabi_psf_dense_bytes(C.byref(p.c()), C.byref(b)))
    return b.value


def build_psf_dense(p: Params, dense, stream=None):
    _check(lib().wasabi_build_psf_dense(C.byref(p.c()), _ptr(dense), _nbytes(dense), _stream(stream)))


def bin_points_psf(p: Params, tables, points, row0: int, row1: int, bins, stream=None):
    """Bins by the whole PSF disc (the direct sum's footprint)."""
    _check(lib().wasabi_bin_points_psf(C.byref(p.c()), _ptr(tables), _ptr(points), points.shape[0], row0, row1,
                                       _ptr(bins), _nbytes(bins), _stream(stream)))


def direct_sum(p: Params, dense, bins, row0: int, row1: int, u, stream=None):
    """Quantised direct sum of Eq.(1) (PSF stamping; the paper's conventional method) for a band."""
    _check(lib().wasabi_direct_sum(C.byref(p.c()), _ptr(dense), _ptr(bins), row0, row1, _ptr(u), _stream(stream)))


# ----------------------------------------------------------------------------- work accounting
def count_accumulations(p: Params, tables, points, row0: int, row1: int, scratch, stream=None) -> int:
    """Exact Eq.(2) accumulation count of rows [row0, row1) (synchronous; scratch >= 8 device bytes)."""
    n = _i64()
    _check(lib().wasabi_count_accumulations(C.byref(p.c()), _ptr(tables), _ptr(points), points.shape[0], row0,
                                            row1, _ptr(scratch), C.byref(n), _stream(stream)))
    return n.value


def row_work(p: Params, tables, points, out, scratch, stream=None):
    """Per-row work estimate into `out` (n_h + 1 float64 device tensor; out[:n_h] meaningful)."""
    _check(lib().wasabi_row_work(C.byref(p.c()), _ptr(tables), _ptr(points), points.shape[0], _ptr(out),
                                 _ptr(scratch), _stream(stream)))


def direct_exact(p: Params, points, bins, row0: int, row1: int, u, stream=None):
    """Exact Eq.(1) (D1: continuous positions and depths) for a band; bins from bin_points_psf."""
    _check(lib().wasabi_direct_exact(C.byref(p.c()), _ptr(points), points.shape[0], _ptr(bins), row0, row1,
                                     _ptr(u), _stream(stream)))


# ----------------------------------------------------------------------------- whole path
def hologram_workspace_bytes(p: Params, n: int, row0: int, row1: int) -> int:
    b = _sz()
    _check(lib().wasabi_hologram_workspace_bytes(C.byref(p.c()), n, row0, row1, C.byref(b)))
    return b.value


def hologram_host(p: Params, print_params: PrintParams, h_points, row0: int, row1: int, workspace, h_bits,
                  h_u=None, stream=None):
    n = h_points.shape[0]
    _check(lib().wasabi_hologram_host(C.byref(p.c()), C.byref(print_params.c()), _ptr(h_points), n, row0, row1,
                                      _ptr(workspace), _nbytes(workspace), _ptr(h_bits), _ptr(h_u),
                                      _stream(stream)))


# ----------------------------------------------------------------------------- diagnostics
def tables_check(p: Params, tables):
    _check(lib().wasabi_tables_check(C.byref(p.c()), _ptr(tables)))


def export_table(p: Params, tables, depth: int):
    import numpy as np
    cap = depth_geometry(p, depth)["n_r"]
    lv = np.zeros(cap, np.int32); dx = np.zeros(cap, np.int32); dy = np.zeros(cap, np.int32)
    val = np.zeros((cap, 2), np.float32)
    n = _i64()
    _check(lib().wasabi_export_table(C.byref(p.c()), _ptr(tables), depth, lv.ctypes.data, dx.ctypes.data,
                                     dy.ctypes.data, val.ctypes.data, cap, C.byref(n)))
    return lv[:n.value], dx[:n.value], dy[:n.value], val[:n.value, 0] + 1j * val[:n.value, 1].astype(np.complex64)


def export_reach(p: Params, tables, depth: int):
    """(ek, q) footprint reach of one depth as computed by the table build (R-A19)."""
    ek = C.c_int32()
    q = C.c_int32()
    _check(lib().wasabi_export_reach(C.byref(p.c()), _ptr(tables), depth, C.byref(ek), C.byref(q)))
    return ek.value, q.value


def bins_stats(bins) -> dict:
    out = (_i64 * 8)()
    _check(lib().wasabi_bins_stats(_ptr(bins), C.byref(out)))
    keys = ["n_valid", "n_skipped", "entries", "capacity", "row0", "row1", "n_tiles", "status"]
    return dict(zip(keys, list(out)))


def export_bins(p: Params, bins):
    import numpy as np
    st = bins_stats(bins)
    ptr = np.zeros(st["n_tiles"] + 1, np.int64)
    cap = max(1, st["entries"])
    idx = np.zeros(cap, np.int32)
    n = _i64()
    _check(lib().wasabi_export_bins(C.byref(p.c()), _ptr(bins), ptr.ctypes.data, idx.ctypes.data, cap, C.byref(n)))
    return ptr, idx[:n.value]


from .pipeline import Pipeline  # noqa: E402,F401
